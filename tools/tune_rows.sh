#!/bin/bash
# Sweep the row-kernel tuning knobs on one GPU (bench.py stage times).
mkdir -p gpurun_out
OUT=gpurun_out/tune_${1:-x}.txt; : > $OUT
for W in ${WORKLOADS:-C2 C3}; do
for LU in 2 4; do for RU in 2 4; do for LO in 0 2 3; do for RO in 0 3 4; do
  r=$(MOE_LAYOUT_U=$LU MOE_REVERSE_KU=$RU MOE_ROW_CTAS_PER_SM=$LO MOE_REVERSE_CTAS_PER_SM=$RO \
      timeout 120 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | \
      python -c "import json,sys; d=json.load(sys.stdin); s=d['stages_ms']; print('%.2f gate=%.2f layout=%.2f reverse=%.2f' % (d['ms_per_step']*1e3, s['gate']*1e3, s['layout']*1e3, s['reverse']*1e3))")
  echo "$W LU=$LU RU=$RU LO=$LO RO=$RO $r" | tee -a $OUT
done; done; done; done; done
