# seg accumulate passes: load+store (mode 0) vs RED.ADD (mode 4), C4 and C3; alternating for fairness
for rep in 1 2; do for m in 0 4; do
  timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode $m --iters 20 --reps 2 --check 2>&1 | tail -3 | sed "s/^/c4 mode $m: /"
done; done
for m in 0 4; do timeout 300 python tools/prof_spmv.py --config c3 --kernel seg --seg-mode $m --iters 20 --reps 2 --check 2>&1 | tail -3 | sed "s/^/c3 mode $m: /"; done
