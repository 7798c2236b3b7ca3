for cfg in "exp3 66" "exp4 50" "exp4 56" "exp3 66" "exp4 50"; do
  set -- $cfg
  BL_LIB=$PWD/paper_2101_05600_b200/libbl_b200_$1.so BL_SMEM_KB=$2 BL_DEBUG=1 python bench.py --no-e2e --no-cpu-baseline --no-pipeline --steps 5 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))"
  grep -m1 "CTA/SM" gpurun_out/ab.err
done
