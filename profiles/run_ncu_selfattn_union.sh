#!/bin/bash
# One late-step pair (l ~ 200) of the staged attention kernels under
# ncu --set full: dec_attn_staged_kernel<false> (union self-attention) and
# <true> (source attention) of the same layer. Run via gpurun from the repo
# root; plain run first.
set -e
mkdir -p gpurun_out
CMD="python scripts/bench_attn.py --n 512 --steps 1"
$CMD > gpurun_out/sa_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dec_attn_staged -s 1200 -c 2 \
    -o gpurun_out/prof_staged_attn $CMD > gpurun_out/sa_ncu.log 2>&1
echo done
