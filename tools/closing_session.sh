#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): the GPU suite, smoke(),
# the default bench line, the reference arm, the ncu launch list of a short
# bench and one --set full capture of the dominant kernel.
#   bash tools/closing_session.sh TAG
TAG=${1:-final}; O=gpurun_out/${TAG}
mkdir -p gpurun_out
nvidia-smi > ${O}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > ${O}_pytest.log 2>&1
echo "EXIT $?" >> ${O}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1
echo "EXIT $?" >> ${O}_smoke.log
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err
timeout 900 python bench.py --impl reference > ${O}_reference.json 2> ${O}_reference.err
for w in C3 C4a C4b; do
  timeout 600 python bench.py --workload $w --no-e2e --cpu-seconds 2 > ${O}_bench_$w.json 2> ${O}_bench_$w.err
done
# launch list (cold-cache, serialised: shares, not absolutes)
python bench.py --steps 2 --warmup 3 --no-e2e --no-backward --no-cpu-baseline --no-clocks > ${O}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-backward --no-cpu-baseline --no-clocks > ${O}_ncu_launch.log 2>&1
python tools/prof_step.py --workload C2 > ${O}_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_layout|k_reverse_k|k_gate" -s 5 -c 4 \
    -o ${O}_full python tools/prof_step.py --workload C2 > ${O}_ncu_full.log 2>&1
echo done > ${O}_done.txt
