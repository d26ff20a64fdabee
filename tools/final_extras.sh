#!/bin/bash
# End-of-round extras on a 4-GPU box: fused gate + dispatch A/B at N=2/4 and
# the C5 end-to-end points (top-2, E=64, B = 16 / 128 / 1024 MiB) with the
# one-sided path at N=2 and N=4.
O=gpurun_out/fx2
B="timeout 900 python bench.py --no-e2e --no-backward --cpu-seconds 1"
for N in 2 4; do
  for F in on off; do
    $B --gpus $N --fuse $F > ${O}_fuse_${F}_N$N.json 2> ${O}_fuse_${F}_N$N.err
  done
  for S in 4096 32768 262144; do
    $B --gpus $N --workload C5 --tokens $S > ${O}_c5_N${N}_S$S.json 2> ${O}_c5_N${N}_S$S.err
  done
done
echo done > ${O}_done.txt
