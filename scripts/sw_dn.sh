for rep in 1 2; do for v in base $VARS; do
  if [ $v = base ]; then L=$PWD/paper_2101_05600_b200/libbl_b200.so; else L=$PWD/build_probe/libbl_$v.so; fi
  echo -n "$v "; BL_LIB=$L python scripts/bench_attn.py --spec large --n 2880 --m2 -1 --steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['decode_ms'])"
done; done
