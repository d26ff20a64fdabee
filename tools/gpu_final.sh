#!/bin/bash
# Round-end evidence on N GPUs (run under gpurun --gpus 2): the N=1 check
# (pytest -m gpu, bench line, ncu launch list of the step, ncu --set full of
# the forward and backward kernels) and bench lines at N=2 for C2/C3.
TAG=${1:-fin}
bash tools/gpu_check.sh $TAG
S=gpurun_out/status_$TAG.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in C2 C3; do
  timeout 300 $RUN --master-port 29690 bench.py --gpus 2 --steps 20 --warmup 5 --workload $W > gpurun_out/bench2_${TAG}_$W.json 2> gpurun_out/bench2_${TAG}_$W.err; echo bench2_$W=$? >> $S
done
for W in C3 C4a C4b; do
  timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --no-e2e > gpurun_out/bench1_${TAG}_$W.json 2> gpurun_out/bench1_${TAG}_$W.err; echo bench1_$W=$? >> $S
done
# the combine in sequence with a warm L2 (no cache flush between kernels):
# how much of the dispatch the reversed walk finds in L2
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-backward"
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:"k_(layout|reverse)" --csv --log-file gpurun_out/l2warm_$TAG.csv $B > gpurun_out/ncu_l2warm_$TAG.log 2>&1; echo ncu_l2warm=$? >> $S
