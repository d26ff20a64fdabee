#!/bin/bash
# Multi-GPU round trip (run under gpurun --gpus N): the whole -m gpu suite
# (single- and multi-GPU parity), bench at N for each AllToAll algorithm, and
# the C5 flat / hierarchical / one-sided sweep.
TAG=${1:-m}; N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
nvidia-smi topo -m > gpurun_out/topo_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? >> $S
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in ${WORKLOADS:-C2 C3}; do for A in ${ALGOS:-p2p flat}; do
timeout 300 $RUN --master-port 29511 bench.py --gpus $N --steps 20 --warmup 5 --workload $W --algo $A --verbose > gpurun_out/bench_${TAG}_${W}_${A}.json 2> gpurun_out/bench_${TAG}_${W}_${A}.err; echo bench_${W}_${A}=$? >> $S
done; done
timeout 900 $RUN --master-port 29512 tools/bench_a2a.py --p2p --max-mib ${MAXMIB:-1024} --out gpurun_out/c5_${TAG}.json > gpurun_out/c5_${TAG}.log 2>&1; echo c5=$? >> $S
NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=64 timeout 600 $RUN --master-port 29513 tools/bench_a2a.py --min-mib 16 --max-mib 256 --out gpurun_out/c5nccl_${TAG}.json > gpurun_out/c5nccl_${TAG}.log 2>&1; echo c5nccl=$? >> $S
