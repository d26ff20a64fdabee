mkdir -p gpurun_out; S=gpurun_out/status_t4.txt
N=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_t4.log 2>&1; echo pytest=$? >> $S
for T in 1 0; do
 for W in C2 C3; do
  MOE_P2P_LAYOUT_TMA=$T timeout 400 $RUN --master-port $((29750 + T)) bench.py --gpus $N --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/t4_${W}_$T.json 2> gpurun_out/t4_${W}_$T.err; echo ${W}_$T=$? >> $S
 done
done
timeout 400 $RUN --master-port 29752 bench.py --gpus $N --steps 20 --warmup 5 --workload C4b > gpurun_out/t4_C4b.json 2> gpurun_out/t4_C4b.err; echo C4b=$? >> $S
