mkdir -p gpurun_out; S=gpurun_out/status_bar.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for M in 0 1 2; do
 for B in 0 1; do
  MOE_BARRIER_MODE=$M MOE_BARRIER_PDL=$B timeout 300 $RUN --master-port $((29660 + M * 2 + B)) tools/bench_barrier.py > gpurun_out/bar_$M$B.json 2>gpurun_out/bar_$M$B.err; echo bar_$M$B=$? >> $S
 done
done
