#!/bin/bash
# Round-2 final evidence for the headline kernel decode_kernel<10,2> in slab
# mode (per-warp TMA rings, 16-row jobs, per-column early-out), C4 at N=1.
# Each ncu command is preceded by the same command without ncu.
set -e
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-legs --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/r02f_plain.json 2> gpurun_out/r02f_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py $ARGS > gpurun_out/r02f_ncu_launches.log 2>&1
python scripts/c3_leg.py 2880 > gpurun_out/r02f_c4_plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 \
    -o gpurun_out/r02f_prof_c4 python scripts/c3_leg.py 2880 > gpurun_out/r02f_ncu_full.log 2>&1
python scripts/prof_phases.py 5000 10 -1 296 > gpurun_out/r02f_phases.log 2>&1
echo done
