timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "panel" 2>&1 | tail -2
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'])"
