#!/bin/bash
# One late-step launch (l ~ 200) of the union self-attention kernel under
# ncu --set full (run via gpurun from the repo root; plain run first).
set -e
mkdir -p gpurun_out
CMD="python scripts/bench_attn.py --n 512 --steps 1"
$CMD > gpurun_out/sa_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dec_self_attn_union -s 600 -c 1 \
    -o gpurun_out/prof_selfattn_union $CMD > gpurun_out/sa_ncu.log 2>&1
echo done
