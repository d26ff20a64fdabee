mkdir -p gpurun_out; S=gpurun_out/status_c4.txt
N=$(nvidia-smi -L | wc -l)
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for W in C4a C4b C2 C3; do
  timeout 400 $RUN --master-port 29730 bench.py --gpus $N --steps 20 --warmup 5 --workload $W > gpurun_out/c4_${N}_$W.json 2> gpurun_out/c4_${N}_$W.err; echo ${W}=$? >> $S
done
timeout 400 $RUN --master-port 29731 bench.py --gpus $N --steps 20 --warmup 5 --workload C4b --dropless > gpurun_out/c4_${N}_C4b_dropless.json 2> gpurun_out/c4_${N}_C4b_dropless.err; echo C4b_dl=$? >> $S
