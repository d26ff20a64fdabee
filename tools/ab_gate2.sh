#!/bin/bash
# N=1 A/B of the gate's second pass: select -> slots2 (every CTA reduces the
# tile table) vs select -> scan -> slots, via gate_two_maxw, and tile sizes.
mkdir -p gpurun_out
OUT=gpurun_out/ab_gate2_${1:-x}.txt; : > $OUT
for R in $(seq 1 ${REPS:-2}); do
for W in ${WORKLOADS:-C3 C4a C4b}; do
for CFG in ${CFGS:-"4096 0" "1048576 0" "1048576 64" "1048576 256"}; do
  set -- $CFG
  r=$(MOE_GATE_TWO_MAXW=$1 MOE_GATE_MAX_TILE=$2 \
      timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']; print('%.2f gate=%.2f layout=%.2f reverse=%.2f' % (d['ms_per_step']*1e3, s['gate']*1e3, s['layout']*1e3, s['reverse']*1e3))")
  echo "$R $W two_maxw=$1 max_tile=$2 $r" | tee -a $OUT
done; done; done
