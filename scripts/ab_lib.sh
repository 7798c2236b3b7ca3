#!/bin/bash
# Same-box A/B of build_probe/libbl_<v>.so variants on the C3/C4 decode
# shape: AB_VARIANTS="base x y" AB_N=2880 bash scripts/ab_lib.sh
for rep in 1 2; do for v in ${AB_VARIANTS:-base}; do
  echo -n "$v "; BL_LIB=$PWD/build_probe/libbl_$v.so python scripts/c3_leg.py ${AB_N:-2880} 2>/dev/null | tail -1
done; done
