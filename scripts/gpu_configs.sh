#!/bin/bash
# Smoke of every bench configuration and launch mode (1 GPU): C1, C4 (sample / data), C5,
# torchrun N=1 (NCCL communicator path), the reference (oracle) arm. Summaries on stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1 || exit 1
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d.get('impl','ours'), d.get('ms_per_step'), d.get('value'), d.get('config',{}).get('workload'), d.get('config',{}).get('parallelism'), d.get('unavailable',''))" $1 || tail -3 $1; }
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg_C1.log 2>&1; summ gpurun_out/cfg_C1.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_C4.log 2>&1; summ gpurun_out/cfg_C4.log
timeout 600 python bench.py --config C4 --mode data --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_C4d.log 2>&1; summ gpurun_out/cfg_C4d.log
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_C5.log 2>&1; summ gpurun_out/cfg_C5.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_trun.log 2>&1; summ gpurun_out/cfg_trun.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cfg_ref.log 2>&1; summ gpurun_out/cfg_ref.log
