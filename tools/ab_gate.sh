#!/bin/bash
# Gate knob sweep (no pytest): bench.py stage times per setting and workload.
# Usage: WL="C2 C3" bash tools/ab_gate.sh TAG "ENV=a" "ENV=b" ...
TAG=$1; shift
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
i=0
for setting in "$@"; do
  for W in ${WL:-C2}; do
    env $setting timeout 300 python bench.py --steps 30 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/ab_${TAG}_${W}_$i.json 2> gpurun_out/ab_${TAG}_${W}_$i.err
    echo "ab_${W}_$i [$setting]=$?" >> $S
  done
  i=$((i+1))
done
