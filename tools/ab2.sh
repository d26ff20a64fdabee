# smoke + dropless bench at P=1 and P=2 + backward timing
mkdir -p gpurun_out; S=gpurun_out/status_dl.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_dl.log 2>&1; echo smoke=$? >> $S
python tools/bench_bwd.py --workload C2 --iters 10 > gpurun_out/dl_bwd.json 2>&1; echo bwd=$? >> $S
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for W in C4b C3; do
 timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --dropless --no-e2e > gpurun_out/dl_${W}_1.json 2>gpurun_out/dl_${W}_1.err; echo ${W}_1=$? >> $S
 timeout 300 $RUN --master-port 29631 bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --dropless --no-e2e > gpurun_out/dl_${W}_2.json 2>gpurun_out/dl_${W}_2.err; echo ${W}_2=$? >> $S
 timeout 300 $RUN --master-port 29632 bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-e2e --no-backward > gpurun_out/dl_${W}_2pad.json 2>gpurun_out/dl_${W}_2pad.err; echo ${W}_2pad=$? >> $S
done
