set -e
timeout 300 python -m pytest tests/test_stream_in.py -q -x 2>&1 | tail -1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_stream_in.py -q -x 2>&1 | tail -1
python bench.py --no-pipeline --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['e2e']['value'])"
