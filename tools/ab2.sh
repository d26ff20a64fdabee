mkdir -p gpurun_out; S=gpurun_out/status_pu.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k backward > gpurun_out/pytest_pu.log 2>&1; echo pytest=$? >> $S
for B in 0 1; do
 for W in C2 C3; do
  MOE_BWD_PUSH=$B timeout 300 $RUN --master-port $((29700 + B)) bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline > gpurun_out/pu_${W}_$B.json 2>gpurun_out/pu_${W}_$B.err; echo ${W}_$B=$? >> $S
 done
done
