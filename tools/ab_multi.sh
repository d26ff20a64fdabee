B="timeout 600 python bench.py --gpus 4 --no-e2e --no-backward --cpu-seconds 1"
for w in C2 C3 C4a C4b; do
  $B --workload $w --fuse off > gpurun_out/r2u_${w}_off.json 2> gpurun_out/r2u_${w}_off.err
  $B --workload $w --fuse on > gpurun_out/r2u_${w}_on.json 2> gpurun_out/r2u_${w}_on.err
  MOE_BARRIER_PDL=1 $B --workload $w --fuse off > gpurun_out/r2u_${w}_bpdl.json 2> gpurun_out/r2u_${w}_bpdl.err
done
$B --workload C2 --algo flat > gpurun_out/r2u_C2_flat.json 2> gpurun_out/r2u_C2_flat.err
