# ncu of the C4 seg SpMV with RED.ADD accumulation: step metrics (8 passes), --set full of passes 0+1,
# launch list of the bench command; then the bench line itself (no profiler)
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread"
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_spmv_seg" -s 16 -c 8 --csv --log-file gpurun_out/c4_seg_na_step8.csv python tools/prof_spmv.py --config c4 --kernel seg --iters 3 > gpurun_out/ncu_c4_red_step.log 2>&1
python tools/ncu_step_summary.py gpurun_out/c4_seg_na_step8.csv > gpurun_out/c4_seg_na_step8_summary.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_seg -s 16 -c 2 -o gpurun_out/c4_seg_na python tools/prof_spmv.py --config c4 --kernel seg --iters 3 > gpurun_out/ncu_c4_red.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_na.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
tail -2 gpurun_out/bench_c4.log
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['value'], d['ms_per_step'], d['roofline'], d['clocks'], d['e2e']['value'])"
