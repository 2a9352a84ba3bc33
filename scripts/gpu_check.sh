#!/bin/bash
# One gpurun call: smoke, GPU parity tests, short benches. Logs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 600 ${PYTEST_ARGS:--k "not slow"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${BENCH_CONFIGS:-C2}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_$c.log 2>&1
  echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
done
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench_*.log
