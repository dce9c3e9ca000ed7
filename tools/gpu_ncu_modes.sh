# per-mode request / wavefront counts of one C4 seg pass pair
for M in 0 1 2 3; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,lts__t_requests_srcunit_tex.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_spmv_seg|k_seg_probe" -s 16 -c 2 --csv --log-file gpurun_out/c4_mode$M.csv python tools/prof_spmv.py --config c4 --kernel seg --seg-mode $M --seg-panels 8 --iters 3 > /dev/null 2>&1
done
ls gpurun_out/c4_mode*.csv
