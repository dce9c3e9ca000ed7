# seg bound probe (stream + gathers, no reduction) and the seg SpMV vs persistent warp count
for w in 3552 4736 7104 9472; do timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode 3 --seg-warps $w --iters 20 --reps 2 2>&1 | tail -1 | sed "s/^/probe warps=$w /"; done
for w in 3552 4736; do timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-warps $w --iters 20 --reps 2 2>&1 | tail -1 | sed "s/^/seg warps=$w /"; done
