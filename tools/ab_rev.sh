#!/bin/bash
# N=1 A/B of the local combine's grid: reverse_tokens_per_warp (0 = persistent, strided).
mkdir -p gpurun_out
OUT=gpurun_out/ab_rev_${1:-x}.txt; : > $OUT
for R in $(seq 1 ${REPS:-2}); do
for W in ${WORKLOADS:-C2 C3 C4a C4b}; do
for T in ${TPWS:-0 2 4 8}; do
  r=$(MOE_REVERSE_TOKENS_PER_WARP=$T \
      timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-clocks --no-backward 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('%.2f gate=%.2f layout=%.2f reverse=%.2f' % (d['ms_per_step']*1e3, s['gate']*1e3, s['layout']*1e3, s['reverse']*1e3))")
  echo "$R $W RTPW=$T $r" | tee -a $OUT
done; done; done
