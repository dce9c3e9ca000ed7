# round check: GPU tests, smoke, C4 + C2 bench lines (with the PCIe e2e floor)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for cfg in ${CONFIGS:-c4 c2}; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.log
  tail -3 gpurun_out/bench_$cfg.log
  python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e'].get('pcie'), d['host_perm_gen_s'], d['clocks'])"
done
