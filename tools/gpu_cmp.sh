# seg row-total writes: staged in row order (mode 0) vs per-(lane,k) (mode 6), C4 and C3, alternating
timeout 600 python -m pytest tests/test_gpu_seg.py tests/test_gpu_iterative.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for rep in 1 2; do for m in 0 6; do
  timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode $m --iters 20 --reps 2 2>&1 | tail -2 | sed "s/^/c4 mode $m: /"
done; done
for m in 0 6; do timeout 300 python tools/prof_spmv.py --config c3 --kernel seg --seg-mode $m --iters 20 --reps 2 2>&1 | tail -2 | sed "s/^/c3 mode $m: /"; done
for m in 0 6; do timeout 300 python tools/prof_spmv.py --config c5 --kernel seg --seg-mode $m --iters 50 --reps 2 2>&1 | tail -2 | sed "s/^/c5 mode $m: /"; done
