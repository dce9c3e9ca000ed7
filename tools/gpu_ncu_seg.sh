# ncu of the C4 seg SpMV: (1) DRAM bytes, time, requests of all 8 passes of one step,
# (2) --set full of passes 0 and 1, (3) the bound probe's step metrics
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread"
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_spmv_seg|k_seg_probe" -s 16 -c 8 --csv --log-file gpurun_out/c4_seg_step8.csv python tools/prof_spmv.py --config c4 --kernel seg --seg-panels ${SEGP:-8} --iters 3 > gpurun_out/ncu_c4_seg_step.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_spmv_seg|k_seg_probe" -s 16 -c 8 --csv --log-file gpurun_out/c4_probe_step8.csv python tools/prof_spmv.py --config c4 --kernel seg --seg-mode 3 --seg-panels ${SEGP:-8} --iters 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_seg -s 16 -c 2 -o gpurun_out/c4_seg_v2 python tools/prof_spmv.py --config c4 --kernel seg --seg-panels ${SEGP:-8} --iters 3 > gpurun_out/ncu_c4_seg.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 300 tools/bin/gather_bench 8 64 100 400 > gpurun_out/gather_bench.txt 2>&1
tail -2 gpurun_out/ncu_c4_seg.log
