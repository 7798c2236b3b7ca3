#!/bin/bash
# Rebuild with different source-attention launch shapes (keys per warp
# chunk, warps per CTA, min CTAs per SM; the self-attention shape fixed) and
# time the full-model decode. run via gpurun from the repo root.
# SWEEP="keys:warps:minb,..."
mkdir -p gpurun_out
for cfg in $(echo "${SWEEP:-16:2:11,32:2:8}" | tr , " "); do
  set -- $(echo "$cfg" | tr : " ")
  rm -f paper_2101_05600_b200/csrc/build/decoder_net.o
  make -s -C paper_2101_05600_b200/csrc EXTRA="-DBL_XS_KEYS=$1 -DBL_XS_WARPS=$2 -DBL_XS_MINB=$3" > gpurun_out/xs_build.log 2>&1
  python scripts/bench_attn.py --n 2880 --profile > gpurun_out/xs_$1_$2_$3.log 2>&1
  ms=$(grep -A2 dec_attn_staged gpurun_out/xs_$1_$2_$3.log | grep -v staged | tr -d ' \n')
  dec=$(grep decode_ms gpurun_out/xs_$1_$2_$3.log)
  echo "src keys=$1 warps=$2 minb=$3 staged_attn=$ms $dec"
done
