# ncu --set full of C4 seg passes (one panel-0 pass, one accumulating pass)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_seg -s 8 -c 2 -o gpurun_out/c4_seg python tools/prof_spmv.py --config c4 --kernel seg --seg-panels ${SEGP:-8} --iters 1 > gpurun_out/ncu_c4_seg.log 2>&1
tail -3 gpurun_out/ncu_c4_seg.log
