mkdir -p gpurun_out; S=gpurun_out/status_g2.txt
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_g2.log 2>&1; echo pytest=$? >> $S
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_g2.log 2>&1; echo smoke=$? >> $S
WL="C4a C4b C2 C3" bash tools/ab_gate.sh g2 "X=0" "MOE_GATE_MAX_TILE=256" "X=1" "MOE_GATE_MAX_TILE=256"
