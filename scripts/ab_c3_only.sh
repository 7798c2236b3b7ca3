#!/bin/bash
# Same-box A/B of the C3 prefix-score leg across library builds
# (paper_2101_05600_b200/libbl_b200_<v>.so for v in $AB_VARIANTS).
for rep in 1 2; do for v in ${AB_VARIANTS:-base cur}; do
  lib=$PWD/paper_2101_05600_b200/libbl_b200_$v.so
  [ $v = cur ] && lib=$PWD/paper_2101_05600_b200/libbl_b200.so
  echo -n "$v "; BL_LIB=$lib python scripts/c3_leg.py 2>/dev/null | tail -1
done; done
