# compute-sanitizer over the late round-2 seg SpMV changes (ballot row-end slots, rotated chunk carry,
# L1-allocating 256-bit f64 stream) and the occupancy-wave sort grids, on small cases
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_seg.py tests/test_gpu_iterative.py tests/test_gpu_parity.py -k "not above_2_31" > gpurun_out/r2c_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2c_memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_seg.py tests/test_gpu_iterative.py > gpurun_out/r2c_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r2c_racecheck.txt
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_seg.py tests/test_gpu_iterative.py > gpurun_out/r2c_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/r2c_synccheck.txt
