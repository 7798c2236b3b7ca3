#!/bin/bash
# One --set full capture of the TMA decode kernel on the C3 shape (vocab 5000,
# ${NUTT:-296} segments, scripts/c3_leg.py); the plain run goes first.
set -e
mkdir -p gpurun_out
python scripts/c3_leg.py ${NUTT:-296} > gpurun_out/c3_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_c3 python scripts/c3_leg.py ${NUTT:-296} > gpurun_out/c3_ncu.log 2>&1
echo done
