#!/bin/bash
# N-GPU A/B of the one-sided path's receive buffers: two used in turn (the
# default; the combine skips its exit barrier) vs one (--single-buffer).
N=${N:-2}
B="timeout 600 python bench.py --gpus $N --no-e2e --no-backward --cpu-seconds 1"
for R in 1 2; do
for w in ${WORKLOADS:-C2 C3 C4a C4b}; do
  $B --workload $w > gpurun_out/db_${TAG:-x}_${w}_N${N}_double_$R.json 2> gpurun_out/db_${TAG:-x}_${w}_N${N}_double_$R.err
  $B --workload $w --single-buffer > gpurun_out/db_${TAG:-x}_${w}_N${N}_single_$R.json 2> gpurun_out/db_${TAG:-x}_${w}_N${N}_single_$R.err
done; done
