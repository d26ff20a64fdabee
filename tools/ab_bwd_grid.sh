#!/bin/bash
# N=1 A/B of layout_tokens_per_warp on the forward step and the backward
# (the combine adjoint shares the layout's grid rule).
mkdir -p gpurun_out
OUT=gpurun_out/ab_bwd_grid_${1:-x}.txt; : > $OUT
for R in $(seq 1 ${REPS:-2}); do
for W in ${WORKLOADS:-C2 C3 C4a C4b}; do
for T in ${TPWS:-0 2}; do
  r=$(MOE_LAYOUT_TOKENS_PER_WARP=$T \
      timeout 180 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fwd %.2f bwd %.2f' % (d['ms_per_step']*1e3, d['backward']['ms_per_step']*1e3))")
  echo "$R $W TPW=$T $r" | tee -a $OUT
done; done; done
