# compute-sanitizer over the round-2 code paths (int64 row_ptr twins, direct-store layout fill,
# K4 with gathered source starts, preload) on small cases
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_wide.py tests/test_gpu_seg.py tests/test_gpu_parity.py tests/test_gpu_r2_api.py tests/test_gpu_cache.py \
  -k "not above_2_31" > gpurun_out/r2_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2_memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_seg.py tests/test_gpu_wide.py -k "ballot or k4 or spmv_bitwise" > gpurun_out/r2_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r2_racecheck.txt
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_seg.py tests/test_gpu_wide.py -k "ballot or k4 or spmv_bitwise" > gpurun_out/r2_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/r2_synccheck.txt
