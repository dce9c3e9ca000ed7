# round 2: new full-scale parity tests, the bench with parity, the sharded path (2 ranks on one GPU, gloo)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q > gpurun_out/t_fullscale.log 2>&1; echo "fullscale rc=$?"
tail -5 gpurun_out/t_fullscale.log
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "bench rc=$?"
tail -5 gpurun_out/bench_c4.log
export BENCH_SINGLE_DEVICE=1 BENCH_DIST_BACKEND=gloo
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2r.json 2> gpurun_out/bench_2r.log; echo "2rank rc=$?"
grep -E "parity|rank|Error|error" gpurun_out/bench_2r.log | tail -8
