# seg layout: parity tests + C4/C2 timings (outputs in gpurun_out/)
timeout 600 python -m pytest tests/test_gpu_seg.py -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_seg.txt
for M in ${SEGMODES:-0 3}; do for P in ${SEGP:-8}; do timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-mode $M --seg-panels $P --iters 10 --reps 3 ${CHECK:---check}; done; done 2>&1 | grep -v "^first" | tee gpurun_out/seg_c4.txt
for M in ${SEGMODES:-0 3}; do timeout 300 python tools/prof_spmv.py --config c2 --kernel seg --seg-mode $M --seg-panels 1 --iters 50 --reps 2 --check; done 2>&1 | grep -v "^first" | tee -a gpurun_out/seg_c4.txt
for P in ${SEGP_SUS:-7 8}; do timeout 300 python tools/prof_spmv.py --config c4 --kernel seg --seg-panels $P --iters 40 --reps 2 --preload 3 2>&1 | grep -v "^first"; done | tee -a gpurun_out/seg_c4.txt
