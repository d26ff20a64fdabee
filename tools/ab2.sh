# A/B of the TMA-staged combine: 1 GPU (local) and 2 GPUs (NVLink), C2 and C3
mkdir -p gpurun_out; S=gpurun_out/status_ab4.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "layout_and_reverse" > gpurun_out/pytest_ab4.log 2>&1; echo pytest=$? >> $S
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in C2 C3; do
 for T in 0 1; do
  MOE_P2P_REVERSE_TMA=$T timeout 300 $RUN --master-port 2962$T bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/ab4_${W}_p2p$T.json 2>gpurun_out/ab4_${W}_p2p$T.err; echo ${W}_p2p$T=$? >> $S
  MOE_REVERSE_TMA=$T timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/ab4_${W}_loc$T.json 2>gpurun_out/ab4_${W}_loc$T.err; echo ${W}_loc$T=$? >> $S
 done
done
MOE_P2P_REVERSE_TMA=1 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_ab4m.log 2>&1; echo pytest_multi=$? >> $S
