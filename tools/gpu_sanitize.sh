# compute-sanitizer over the GPU parity suite (small cases): memcheck (OOB / misaligned
# / leaks on device allocations), racecheck + synccheck (shared-memory hazards, barriers)
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?"
tail -4 gpurun_out/sanitize_memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_seg.py tests/test_gpu_iterative.py tests/test_gpu_parity.py tests/test_gpu_hist.py -x -q -m gpu -k "hist or seg or fused or entropy or host" -p no:cacheprovider > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"
tail -4 gpurun_out/sanitize_racecheck.txt
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_seg.py tests/test_gpu_iterative.py tests/test_gpu_parity.py tests/test_gpu_hist.py -x -q -m gpu -k "hist or seg or fused or merge or sort" -p no:cacheprovider > gpurun_out/sanitize_synccheck.txt 2>&1; echo "synccheck rc=$?"
tail -4 gpurun_out/sanitize_synccheck.txt
