#!/bin/bash
# A/B a tuning knob on one GPU: pytest -m gpu once, then bench.py per setting.
# Usage: bash tools/ab.sh TAG "ENV1=a ENV2=b" "ENV1=c" ... (workload via WL=C2)
TAG=$1; shift
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? >> $S
i=0
for setting in "$@"; do
  for W in ${WL:-C2}; do
    env $setting timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline > gpurun_out/ab_${TAG}_${W}_$i.json 2> gpurun_out/ab_${TAG}_${W}_$i.err
    echo "ab_${W}_$i [$setting]=$?" >> $S
  done
  i=$((i+1))
done
