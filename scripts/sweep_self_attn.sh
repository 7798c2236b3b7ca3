#!/bin/bash
# Rebuild the staged attention kernel (union self-attention + source attention) with different (keys per warp
# chunk, warps per CTA, min CTAs per SM) and time it in the full pipeline.
# run via gpurun from the repo root
mkdir -p gpurun_out
# SWEEP="keys:warps:minb[:stages],..."
for cfg in $(echo "${SWEEP:-16:4:6,16:2:12,16:2:8}" | tr , " "); do
  set -- $(echo "$cfg" | tr : " ")
  rm -f paper_2101_05600_b200/csrc/build/decoder_net.o
  make -s -C paper_2101_05600_b200/csrc EXTRA="-DBL_SU_KEYS=$1 -DBL_SU_WARPS=$2 -DBL_SU_MINB=$3 -DBL_SU_STAGES=${4:-1}" > gpurun_out/sw_build.log 2>&1
  regs=$(grep -A3 attn_staged paper_2101_05600_b200/csrc/build/decoder_net.ptxas.log | grep -o "Used [0-9]* registers" | tr "\n" " ")
  spill=$(grep -A3 attn_staged paper_2101_05600_b200/csrc/build/decoder_net.ptxas.log | grep -o "[0-9]* bytes spill stores" | tr "\n" " ")
  python scripts/bench_attn.py --n 2880 --profile > gpurun_out/sw_$1_$2_$3_${4:-1}.log 2>&1
  ms=$(grep -A2 dec_attn_staged gpurun_out/sw_$1_$2_$3_${4:-1}.log | tail -1)
  dec=$(grep decode_ms gpurun_out/sw_$1_$2_$3_${4:-1}.log)
  echo "keys=$1 warps=$2 minb=$3 stages=${4:-1} $regs $spill staged_attn_ms=$ms $dec"
done
