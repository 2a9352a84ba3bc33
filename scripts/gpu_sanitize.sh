#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on one small step of every
# path (scripts/sanitize_step.py). Summaries under gpurun_out/r02/sanitize_*.txt.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for w in mlp cnn; do
    timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_step.py $w \
        > $O/sanitize_${tool}_${w}.txt 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $O/sanitize_${tool}_${w}.txt | tail -1)"
  done
done
