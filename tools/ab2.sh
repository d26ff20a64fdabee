mkdir -p gpurun_out; S=gpurun_out/status_lpb.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_lpb.log 2>&1; echo pytest=$? >> $S
for L in 0 1; do
  MOE_P2P_LOCAL_PAD=$L timeout 300 $RUN --master-port $((29760 + L)) bench.py --gpus 2 --steps 20 --warmup 5 --workload C4b --no-e2e --no-cpu-baseline > gpurun_out/lpb_$L.json 2>gpurun_out/lpb_$L.err; echo C4b_$L=$? >> $S
done
