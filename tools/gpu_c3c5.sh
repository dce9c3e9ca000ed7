bash tools/gpu_c5.sh
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; tail -2 gpurun_out/bench_c3.log
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('c3', d['config']['kernel'], d['value'], d['ms_per_step'], d['roofline'], d['permuted_vs_unpermuted'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_seg -s 3 -c 3 -o gpurun_out/c3_seg python bench.py --config c3 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
