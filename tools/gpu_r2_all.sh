# round 2 refresh: GPU suite, smoke, every config's bench line, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "c4 rc=$?"
for c in c2 c3 c5 c4w; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log; echo "$c rc=$?"
done
timeout 900 python bench.py --config c5 --iterative > gpurun_out/bench_c5_iter.json 2> gpurun_out/bench_c5_iter.log; echo "c5 iter rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
for c in c4 c2 c3 c5 c4w; do python - <<PY
import json
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', {k:d.get(k) for k in ['value','ms_per_step','permute_warm_ms','layout_build_ms','layout_build_warm_ms','setup_warm_ms']}, d.get('roofline',{}).get('frac'), d.get('e2e',{}).get('value'), d.get('permuted_vs_unpermuted',{}).get('ratio'), d.get('clocks'))
PY
done
# launch list of the default bench command (kernel shares; cold-cache, serialised: not bench values)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/launches_bench_c4.log 2>&1; echo "ncu list rc=$?"
