#!/bin/bash
# one --set full capture of the decode kernel on the U=64 phase-profile workload
set -e
mkdir -p gpurun_out
CMD="python scripts/bench_small.py ${NUTT:-64}"
$CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_small_${NUTT:-64} $CMD > gpurun_out/ncu_small.log 2>&1
echo ncu-done
