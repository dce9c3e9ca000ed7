timeout 600 python -m pytest tests/test_gpu_iterative.py tests/test_gpu_seg.py -x -q 2>&1 | tail -5
timeout 900 python bench.py --config c5 --iterative --warmup 3 2> gpurun_out/bench_c5.log > gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.log
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['value'], d['ms_per_step'], d['config'], d['eigenvalue'], d['amortisation'], d['gpu_launches'])"
