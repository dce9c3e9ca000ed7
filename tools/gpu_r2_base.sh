# round-2 re-entry baseline: full GPU suite, smoke, default bench (C4), reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_c4.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref.json
