#!/bin/bash
# Encoder kernels under ncu (run on a B200 via gpurun from the repo root).
# The plain command must exit 0 before each ncu pass.
set -e
mkdir -p gpurun_out
CMD="python scripts/enc_bench.py --spec large --n 16 --chunk 16"
$CMD > gpurun_out/enc_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/enc_launches.csv $CMD > gpurun_out/enc_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 3 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/enc_ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attention_tc -s 2 -c 1 \
    -o gpurun_out/prof_attn $CMD > gpurun_out/enc_ncu_attn.log 2>&1
echo ncu-done
