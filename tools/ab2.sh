#!/bin/bash
# Multi-GPU A/B of tuning knobs (run under gpurun --gpus N): bench.py at N
# ranks per setting and workload.  Usage: WL="C2 C3" bash tools/ab2.sh TAG "ENV=a" "ENV=b" ...
TAG=$1; shift
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
N=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
for setting in "$@"; do
  for W in ${WL:-C2}; do
    env $setting timeout 400 $RUN --master-port $((29800 + i)) bench.py --gpus $N --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline ${EXTRA:---no-backward} > gpurun_out/ab2_${TAG}_${W}_$i.json 2> gpurun_out/ab2_${TAG}_${W}_$i.err
    echo "ab2_${W}_$i [$setting]=$?" >> $S
  done
  i=$((i+1))
done
