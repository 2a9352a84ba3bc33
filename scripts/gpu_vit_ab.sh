cd /root/repo
mkdir -p gpurun_out/r02
for v in 0 1 0 1; do BNN_WS_CHUNKS=$v timeout 300 python bench.py --config C7 --precision bf16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/b7_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02/b7_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if k in ('fwd','dgrad','wgrad')})"; done
