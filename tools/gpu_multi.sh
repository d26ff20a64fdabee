#!/bin/bash
# Multi-GPU round trip (run under gpurun --gpus N): multi-GPU parity tests,
# bench at N, and the C5 flat-vs-hierarchical sweep.
TAG=${1:-m}; N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
nvidia-smi topo -m > gpurun_out/topo_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? >> $S
for W in ${WORKLOADS:-C2 C3}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 20 --warmup 5 --workload $W > gpurun_out/bench_${TAG}_${W}.json 2> gpurun_out/bench_${TAG}_${W}.err; echo bench_$W=$? >> $S
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/bench_a2a.py --max-mib ${MAXMIB:-1024} --out gpurun_out/c5_${TAG}.json > gpurun_out/c5_${TAG}.log 2>&1; echo c5=$? >> $S
