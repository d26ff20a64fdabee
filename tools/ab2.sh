mkdir -p gpurun_out; S=gpurun_out/status_fu.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_equals or run_host or pipeline_full" > gpurun_out/pytest_fu.log 2>&1; echo pytest=$? >> $S
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for F in 0 1; do
 for W in C2 C3 C4a; do
  MOE_FUSE_GATE_LAYOUT=$F timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/fu_${W}_$F.json 2>gpurun_out/fu_${W}_$F.err; echo ${W}_$F=$? >> $S
 done
 MOE_FUSE_GATE_LAYOUT=$F timeout 300 $RUN --master-port $((29680 + F)) bench.py --gpus 2 --steps 20 --warmup 5 --workload C2 --no-e2e --no-cpu-baseline --no-backward > gpurun_out/fu_C2p2_$F.json 2>gpurun_out/fu_C2p2_$F.err; echo C2p2_$F=$? >> $S
done
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_fum.log 2>&1; echo pytest_multi=$? >> $S
