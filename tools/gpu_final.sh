# end-of-round refresh: GPU suite, smoke, bench lines for every config, the reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in c4 c2 c3; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/final_$cfg.json 2> gpurun_out/final_$cfg.log
  python -c "import json; d=json.load(open('gpurun_out/final_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 900 python bench.py --config c5 --iterative --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.log
python -c "import json; d=json.load(open('gpurun_out/final_c5.json')); print('c5', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.log
python -c "import json; d=json.load(open('gpurun_out/final_ref.json')); print('ref', d['value'], d['cpu_baseline']['cores'])"
