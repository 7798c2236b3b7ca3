#!/bin/bash
# Encoder kernels under ncu (run on a B200 via gpurun from the repo root).
# The plain command must exit 0 before each ncu pass. One forward of 64
# segments (spec large: 12 layers, d=512, vocab 5000) after 2 warm-ups.
set -e
mkdir -p gpurun_out
CMD="python scripts/enc_bench.py --spec large --n 64 --chunk 64 --no-table --reps 1"
$CMD > gpurun_out/enc_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/enc_launches.csv $CMD > gpurun_out/enc_ncu_launches.log 2>&1
# third forward (after 2 warm-ups): conv1, then GEMMs conv2, out, qkv, oproj, ffn1, ffn2
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 102 -c 6 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/enc_ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attention_tc|conv1" -s 26 -c 2 \
    -o gpurun_out/prof_attn $CMD > gpurun_out/enc_ncu_attn.log 2>&1
echo ncu-done
