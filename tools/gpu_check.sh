# GPU check: parity tests, smoke, bench on C2 and C4 (outputs in gpurun_out/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; cat gpurun_out/smoke.txt
for cfg in ${CONFIGS:-c2 c4}; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.log
  tail -4 gpurun_out/bench_$cfg.log; cat gpurun_out/bench_$cfg.json
done
