#!/bin/bash
# Same-box A/B of library builds: paper_2101_05600_b200/libbl_b200_<v>.so for
# each v in $AB_VARIANTS (default "base cur"; "cur" = libbl_b200.so),
# alternating, C2 decode leg; prints ms/step and kernel ms.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in ${AB_VARIANTS:-base cur}; do
    lib=$PWD/paper_2101_05600_b200/libbl_b200_$v.so
    [ $v = cur ] && lib=$PWD/paper_2101_05600_b200/libbl_b200.so
    BL_LIB=$lib python bench.py --no-e2e --no-cpu-baseline --no-pipeline ${AB_ARGS:---steps 5} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"
  done
done
if [ -n "$AB_C3" ]; then
  for rep in 1 2; do
    for v in ${AB_VARIANTS:-base cur}; do
      lib=$PWD/paper_2101_05600_b200/libbl_b200_$v.so
      [ $v = cur ] && lib=$PWD/paper_2101_05600_b200/libbl_b200.so
      echo -n "$v "; BL_LIB=$lib python scripts/c3_leg.py 2>/dev/null | tail -1
    done
  done
fi
