#!/bin/bash
# N=1 A/B of the local layout's grid: layout_tokens_per_warp (0 = persistent).
mkdir -p gpurun_out
OUT=gpurun_out/ab_tpw_${1:-x}.txt; : > $OUT
for R in $(seq 1 ${REPS:-2}); do
for W in ${WORKLOADS:-C2 C3 C4a C4b}; do
for T in ${TPWS:-0 1 2 3 4}; do
  r=$(MOE_LAYOUT_TOKENS_PER_WARP=$T \
      timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('%.2f gate=%.2f layout=%.2f reverse=%.2f' % (d['ms_per_step']*1e3, s['gate']*1e3, s['layout']*1e3, s['reverse']*1e3))")
  echo "$R $W TPW=$T $r" | tee -a $OUT
done; done; done
