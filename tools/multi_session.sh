#!/bin/bash
# One multi-GPU measurement session (run under `gpurun --gpus N`):
#   bash tools/multi_session.sh N TAG [quick]
# Writes gpurun_out/TAG_*: the GPU test suite, bench.py lines for every
# workload and AllToAll algorithm, the C5 AllToAll sweep with the NCCL
# variants, and C5's end-to-end points (B = 16 / 128 / 1024 MiB per rank).
N=${1:-2}; TAG=${2:-multi}; QUICK=${3:-}
O=gpurun_out/${TAG}
mkdir -p gpurun_out
nvidia-smi topo -m > ${O}_topo.txt 2>&1
if [ -z "$QUICK" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > ${O}_pytest.log 2>&1
  echo "EXIT $?" >> ${O}_pytest.log
fi
B="timeout 600 python bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --cpu-seconds 1"
for w in C2 C3 C4a C4b; do
  $B --workload $w > ${O}_bench_${w}.json 2> ${O}_bench_${w}.err
done
for algo in flat hier hier2d; do
  $B --workload C2 --algo $algo --no-backward > ${O}_bench_C2_${algo}.json 2> ${O}_bench_C2_${algo}.err
done
for w in C2 C3 C4b; do
  $B --workload $w --fuse off --no-backward > ${O}_bench_${w}_nofuse.json 2> ${O}_bench_${w}_nofuse.err
done
for S in 4096 32768 262144; do
  for algo in p2p flat; do
    $B --workload C5 --tokens $S --algo $algo --no-backward > ${O}_c5e2e_${S}_${algo}.json 2> ${O}_c5e2e_${S}_${algo}.err
  done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29511 tools/bench_a2a.py --algos flat,flat_reg,a2a,a2a_reg,hier,hier2d,p2p \
  --max-mib 1024 --out ${O}_c5_sweep.json > ${O}_c5_sweep.log 2>&1
echo done > ${O}_done.txt
