mkdir -p gpurun_out; S=gpurun_out/status_pkb2.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "dropless or backward" > gpurun_out/pytest_pkb2.log 2>&1; echo pytest=$? >> $S
timeout 300 $RUN --master-port 29710 bench.py --gpus 2 --steps 20 --warmup 5 --workload C4b --dropless --no-e2e --no-cpu-baseline > gpurun_out/pkb2_C4b.json 2>gpurun_out/pkb2_C4b.err; echo C4b=$? >> $S
timeout 300 python bench.py --steps 20 --warmup 5 --workload C4b --dropless --no-e2e --no-cpu-baseline > gpurun_out/pkb1_C4b.json 2>gpurun_out/pkb1_C4b.err; echo C4b1=$? >> $S
