#!/bin/bash
# Round-end check on 2 GPUs: pytest -m gpu (multi-GPU cases included), smoke,
# default bench lines at N=1 and N=2, the reference arm at N=1, C4a at N=1.
mkdir -p gpurun_out; S=gpurun_out/status_f2.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_f2.log 2>&1; echo pytest=$? >> $S
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f2.log 2>&1; echo smoke=$? >> $S
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/n1_C2.json 2> gpurun_out/n1_C2.err; echo n1=$? >> $S
timeout 400 python bench.py --steps 20 --warmup 5 --workload C4a > gpurun_out/n1_C4a.json 2> gpurun_out/n1_C4a.err; echo n1_C4a=$? >> $S
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/n2_C2.json 2> gpurun_out/n2_C2.err; echo n2=$? >> $S
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/n1_C2_reference.json 2> gpurun_out/n1_ref.err; echo ref=$? >> $S
