mkdir -p gpurun_out; S=gpurun_out/status_v3.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_v3.log 2>&1; echo pytest=$? >> $S
for W in C2 C3 C4a C4b; do
  timeout 300 python bench.py --steps 20 --warmup 5 --workload $W > gpurun_out/v3_1_$W.json 2> gpurun_out/v3_1_$W.err; echo b1_$W=$? >> $S
done
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in C2 C3; do
  timeout 300 $RUN --master-port 29720 bench.py --gpus 2 --steps 20 --warmup 5 --workload $W > gpurun_out/v3_2_$W.json 2> gpurun_out/v3_2_$W.err; echo b2_$W=$? >> $S
done
