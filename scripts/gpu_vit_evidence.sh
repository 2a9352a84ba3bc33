#!/bin/bash
# ViT (C7) evidence: bench lines (BF16, FP32), a launch list of the BF16 step, and --set full
# captures of the attention kernels and the QKV projection (W-stationary GEMM).
cd "$(dirname "$0")/.."
O=gpurun_out/vit; mkdir -p $O
python -m paper_2604_04736_b200.build > $O/build.log 2>&1
timeout 600 python bench.py --config C7 --precision bf16 --steps 30 --warmup 5 > $O/bench_C7_bf16.json 2> $O/bench_C7_bf16.err
timeout 900 python bench.py --config C7 --precision fp32 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C7_fp32.json 2> $O/bench_C7_fp32.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C7_bf16.csv \
  python bench.py --config C7 --precision bf16 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for spec in "attf:vit_attn_fwd_tc" "attb:vit_attn_bwd_tc" "qkv:ws_kernel<.int.0, .int.256" "lnb:vit_ln_bwd_fused"; do
  tag=${spec%%:*}; re=${spec#*:}
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$re" -s 2 -c 1 -o $O/full_$tag \
    python bench.py --config C7 --precision bf16 --steps 1 --warmup 3 --no-cpu-baseline > $O/full_$tag.log 2>&1
  ncu -i $O/full_$tag.ncu-rep --page raw --csv > $O/full_${tag}_raw.csv 2>&1
  ncu -i $O/full_$tag.ncu-rep --page source --csv --print-source sass > $O/full_${tag}_src.csv 2>&1
  rm -f $O/full_$tag.ncu-rep
done
ls -la $O
