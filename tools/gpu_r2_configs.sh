# round 2: bench lines of every config (C2, C3 at ~256M nnz, C5 iterative with fold=False), full-scale parity on
mkdir -p gpurun_out
for c in c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.log; echo "$c rc=$?"
  tail -3 gpurun_out/bench_$c.log
done
timeout 900 python bench.py --config c5 --iterative > gpurun_out/bench_c5_iter.json 2> gpurun_out/bench_c5_iter.log; echo "c5 rc=$?"
tail -3 gpurun_out/bench_c5_iter.log
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo "c5 spmv rc=$?"
tail -3 gpurun_out/bench_c5.log
