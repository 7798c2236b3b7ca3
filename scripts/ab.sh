#!/bin/bash
# Same-box A/B of two builds of the library: libbl_b200_base.so (baseline)
# against libbl_b200.so (current), alternating, C2 decode leg (and C3 with AB_C3=1).
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in base cur; do
    lib=$PWD/paper_2101_05600_b200/libbl_b200.so
    [ $v = base ] && lib=$PWD/paper_2101_05600_b200/libbl_b200_base.so
    BL_LIB=$lib python bench.py --no-e2e --no-cpu-baseline --no-pipeline ${AB_ARGS:---steps 5} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2), (d.get('prefix_score_c3') or {}).get('value'))"
  done
done
