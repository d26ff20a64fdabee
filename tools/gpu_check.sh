#!/bin/bash
# One GPU-box round trip: parity suite, bench line, ncu launch list and a full
# ncu capture of the three hot kernels.  Usage (from the repo root, under
# gpurun): bash tools/gpu_check.sh TAG [bench args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
S=gpurun_out/status_$TAG.txt
timeout 600 python -m pytest tests -m gpu -q --maxfail=15 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? >> $S
timeout 400 python bench.py --steps 20 --warmup 5 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$? >> $S
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-backward $*"
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_list_$TAG.log 2>&1; echo ncu_list=$? >> $S
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(gate|layout|reverse)" -c 6 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$? >> $S
timeout 300 python tools/bench_bwd.py --workload C2 --iters 10 > gpurun_out/bwd_$TAG.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(combine_bwd|gate_bwd|reverse)" -s 3 -c 3 -o gpurun_out/prof_bwd_$TAG python tools/bench_bwd.py --workload C2 --iters 1 > gpurun_out/ncu_bwd_$TAG.log 2>&1; echo ncu_bwd=$? >> $S
