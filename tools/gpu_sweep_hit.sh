for H in 1.0 0.7 0.4 0; do for P in 7 8; do
timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-panels $P --seg-hit $H --iters 40 --reps 2 --preload 3 2>&1 | grep -v "^first"
done; done | tee gpurun_out/seg_hit.txt
