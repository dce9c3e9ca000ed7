timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for k in auto merge stream vector; do timeout 600 python bench.py --config c3 --kernel $k --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['config']['kernel'], d['value'], d['ms_per_step'], d['permuted_vs_unpermuted'])"; done
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['config']['kernel'], d['value'], d['ms_per_step'])"
