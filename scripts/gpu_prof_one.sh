#!/bin/bash
# One --set full capture of one kernel of a bench config, exported to CSV on the box.
#   KREGEX=wgrad_tc_kernel CFG=C2 SKIP=1 TAG=x bash scripts/gpu_prof_one.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2604_04736_b200.build > gpurun_out/build.log 2>&1
TAG=${TAG:-prof}
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:${KREGEX}" -s ${SKIP:-0} -c 1 -o gpurun_out/$TAG \
  python bench.py --config ${CFG:-C2} --steps 1 --warmup 3 --no-cpu-baseline ${EXTRA} > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>&1
