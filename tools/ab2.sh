mkdir -p gpurun_out; S=gpurun_out/status_v16.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for setting in "MOE_REVERSE_V16=0" "MOE_REVERSE_V16=1" "MOE_COMBINE_CTAS_PER_SM=8" "MOE_REVERSE_KU=4"; do
  env $setting timeout 300 $RUN --master-port $((29770 + i)) bench.py --gpus 2 --steps 20 --warmup 5 --workload C2 --no-e2e --no-cpu-baseline --no-backward > gpurun_out/v16_$i.json 2>gpurun_out/v16_$i.err; echo "$i [$setting]=$?" >> $S
  i=$((i+1))
done
