#!/bin/bash
# DRAM traffic of the dominant N=1 kernels for the non-default workloads
# (ncu --set full, one launch each of k_layout / k_reverse*), plus a plain
# bench line per workload first (the program must exit 0 without ncu).
# Usage (under gpurun): bash tools/gpu_traffic.sh TAG
TAG=${1:-traffic}
mkdir -p gpurun_out
S=gpurun_out/status_$TAG.txt
for W in C3 C4a C4b; do
  B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-backward --workload $W"
  timeout 400 python bench.py --steps 20 --warmup 5 --workload $W > gpurun_out/bench1_${TAG}_$W.json 2> gpurun_out/bench1_${TAG}_$W.err; echo bench1_$W=$? >> $S
  timeout 300 $B > gpurun_out/plain_${TAG}_$W.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(gate|layout|reverse)" -c 6 -o gpurun_out/prof_${TAG}_$W $B > gpurun_out/ncu_full_${TAG}_$W.log 2>&1; echo ncu_full_$W=$? >> $S
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$W.csv $B > gpurun_out/ncu_list_${TAG}_$W.log 2>&1; echo ncu_list_$W=$? >> $S
done
