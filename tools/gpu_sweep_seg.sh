# sustained-load sweep of the seg kernel on C4 (panels x mode), clocks sampled mid-loop
for P in ${SEGP:-6 7 8 10}; do for M in ${SEGMODES:-0}; do
  timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode $M --seg-panels $P --iters 40 --reps 2 --preload 3 2>&1 | grep -v "^first"
done; done | tee gpurun_out/seg_sweep.txt
timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode 3 --seg-panels 8 --iters 40 --reps 2 --preload 3 2>&1 | grep -v "^first" | tee -a gpurun_out/seg_sweep.txt
