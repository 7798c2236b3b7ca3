#!/bin/bash
# Run on a B200 via gpurun from the repo root. Each ncu command is preceded
# by the identical command without ncu (must exit 0 first).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-pipeline"
$CMD > gpurun_out/plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD2="python bench.py --segments 296 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-pipeline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/prof_decode $CMD2 > gpurun_out/ncu_full.log 2>&1
echo ncu-done
