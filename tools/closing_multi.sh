#!/bin/bash
# Round-end evidence on a multi-GPU box (run under gpurun --gpus N): the GPU
# suite (multi-GPU tests included) and the default bench line at N=2..NMAX.
#   bash tools/closing_multi.sh TAG NMAX
TAG=${1:-final}; NMAX=${2:-4}; O=gpurun_out/${TAG}
mkdir -p gpurun_out
nvidia-smi topo -m > ${O}_topo.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > ${O}_pytest.log 2>&1
echo "EXIT $?" >> ${O}_pytest.log
for N in 2 4; do
  [ $N -le $NMAX ] || continue
  timeout 900 python bench.py --gpus $N > ${O}_bench_N$N.json 2> ${O}_bench_N$N.err
  echo "N=$N rc=$?" >> ${O}_rc.txt
done
# back-to-back repeats of the short form (start-up robustness, spread)
for R in 1 2 3; do
  timeout 600 python bench.py --gpus 2 --no-e2e --no-backward --cpu-seconds 1 \
    > ${O}_rep_N2_$R.json 2> ${O}_rep_N2_$R.err
  echo "rep N=2 $R rc=$?" >> ${O}_rc.txt
done
echo done > ${O}_done.txt
