timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
CONFIG=c2 KERNEL=seg bash tools/gpu_multi.sh
CONFIG=c3 KERNEL=auto bash tools/gpu_multi.sh
for cfg in c3 c5; do timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/auto_$cfg.json 2>gpurun_out/auto_$cfg.log; python -c "import json; d=json.load(open('gpurun_out/auto_$cfg.json')); print('$cfg', d['config']['kernel'], d['value'], d['permuted_vs_unpermuted'])"; done
