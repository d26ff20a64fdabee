# A/B with repetitions (alternating settings to spread box drift): WL, REPS env
TAG=$1; shift
mkdir -p gpurun_out; S=gpurun_out/status_$TAG.txt
for r in $(seq 1 ${REPS:-3}); do
  i=0
  for setting in "$@"; do
    for W in ${WL:-C2}; do
      env $setting timeout 300 python bench.py --steps 20 --warmup 5 --workload $W --no-e2e --no-cpu-baseline --no-backward > gpurun_out/ab_${TAG}_${W}_${i}_$r.json 2>/dev/null
      echo "ab_${W}_${i}_$r [$setting]=$?" >> $S
    done
    i=$((i+1))
  done
done
