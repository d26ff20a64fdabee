# 2-GPU A/B of combine (peer reverse) settings, C2 and C3, p2p
mkdir -p gpurun_out; S=gpurun_out/status_ab3.txt
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for setting in "MOE_REVERSE_KU=4" "MOE_REVERSE_KU=8 MOE_REVERSE_TPW=1" "MOE_COMBINE_CTAS_PER_SM=2" "MOE_COMBINE_CTAS_PER_SM=8"; do
 for W in C2 C3; do
  env $setting timeout 300 $RUN --master-port 2961$i bench.py --gpus 2 --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/ab3_${W}_$i.json 2>gpurun_out/ab3_${W}_$i.err; echo "${W}_$i [$setting]=$?" >> $S
 done
 i=$((i+1))
done
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/pytest_ab3.log 2>&1; echo pytest=$? >> $S
