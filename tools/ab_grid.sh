#!/bin/bash
# N=1 A/B of the row kernels' grid size (persistent at the occupancy limit vs
# oversubscribed grids the block scheduler balances): bench.py step and stage
# times per (layout CTAs/SM, reverse CTAs/SM), interleaved over REPS rounds.
mkdir -p gpurun_out
OUT=gpurun_out/ab_grid_${1:-x}.txt; : > $OUT
for R in $(seq 1 ${REPS:-2}); do
for W in ${WORKLOADS:-C2 C3 C4a C4b}; do
for LO in ${LOS:-0 8 16 32}; do for RO in ${ROS:-0 16}; do
  r=$(MOE_ROW_CTAS_PER_SM=$LO MOE_REVERSE_CTAS_PER_SM=$RO \
      timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('%.2f gate=%.2f layout=%.2f reverse=%.2f' % (d['ms_per_step']*1e3, s['gate']*1e3, s['layout']*1e3, s['reverse']*1e3))")
  echo "$R $W LO=$LO RO=$RO $r" | tee -a $OUT
done; done; done; done
