timeout 600 python -m pytest tests/test_gpu_iterative.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config c5 --iterative --warmup 3 2> gpurun_out/bench_c5.log | tee gpurun_out/bench_c5.json
tail -3 gpurun_out/bench_c5.log
