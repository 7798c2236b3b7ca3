#!/bin/bash
# ncu --set full of the opt-in mma.sync tf32 bulk (BL_MMA=1) on the C3 shape,
# 148 segments (one wave); the plain run goes first.
set -e
mkdir -p gpurun_out
BL_MMA=1 python scripts/c3_leg.py 148 > gpurun_out/mma_plain.log 2>&1
BL_MMA=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_mma python scripts/c3_leg.py 148 > gpurun_out/mma_ncu.log 2>&1
echo done
