mkdir -p gpurun_out; S=gpurun_out/status_lp.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_lp.log 2>&1; echo pytest=$? >> $S
for L in 0 1; do
 for W in C4b C2; do
  MOE_P2P_LOCAL_PAD=$L timeout 300 $RUN --master-port $((29740 + L)) bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/lp_${W}_$L.json 2>gpurun_out/lp_${W}_$L.err; echo ${W}_$L=$? >> $S
 done
done
