# memcheck / racecheck of the later round-2 kernels: the CTA hybrid row sort, the fill prefetch
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
mkdir -p gpurun_out
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_r2_api.py tests/test_gpu_seg.py -k "cta or ballot or warp_medium" > gpurun_out/r2b_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/r2b_memcheck.txt
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_r2_api.py tests/test_gpu_seg.py -k "cta or ballot" > gpurun_out/r2b_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r2b_racecheck.txt
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q -p no:cacheprovider \
  tests/test_gpu_r2_api.py -k "cta" > gpurun_out/r2b_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/r2b_synccheck.txt
