#!/bin/bash
# Bench lines for BASELINE.md §5 (run under gpurun --gpus N): every workload
# at N=1 and at N (p2p, plus NCCL flat for C2), back to back on one box.
# Usage: bash tools/gpu_numbers.sh TAG
TAG=${1:-num}
mkdir -p gpurun_out/num_$TAG; O=gpurun_out/num_$TAG; S=$O/status.txt
N=$(nvidia-smi -L | wc -l)
if [ "${SKIP_N1:-0}" != 1 ]; then
  timeout 400 python bench.py > $O/n1_C2.json 2> $O/n1_C2.err; echo n1_C2=$? >> $S
  for W in C3 C4a C4b; do
    timeout 300 python bench.py --workload $W --no-cpu-baseline > $O/n1_$W.json 2> $O/n1_$W.err; echo n1_$W=$? >> $S
  done
  timeout 300 python bench.py --workload C4b --dropless --no-cpu-baseline --no-e2e > $O/n1_C4b_dropless.json 2> $O/n1_C4b_dropless.err; echo n1_C4b_dropless=$? >> $S
fi
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
for W in C2 C3 C4a C4b; do
  timeout 400 $RUN --master-port $((29660 + i)) bench.py --gpus $N --workload $W > $O/n${N}_$W.json 2> $O/n${N}_$W.err; echo n${N}_$W=$? >> $S
  i=$((i+1))
done
timeout 400 $RUN --master-port 29670 bench.py --gpus $N --workload C4b --dropless --no-e2e > $O/n${N}_C4b_dropless.json 2> $O/n${N}_C4b_dropless.err; echo n${N}_C4b_dropless=$? >> $S
timeout 400 $RUN --master-port 29671 bench.py --gpus $N --workload C2 --algo flat --no-e2e > $O/n${N}_C2_flat.json 2> $O/n${N}_C2_flat.err; echo n${N}_C2_flat=$? >> $S
