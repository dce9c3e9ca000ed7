mkdir -p gpurun_out
timeout 600 python -m pytest -q -x tests/test_gpu_seg.py tests/test_gpu_wide.py 2>&1 | tail -2
timeout 600 python tools/fill_direct_ab.py c4 2>&1 | tee gpurun_out/fill_ab.txt
timeout 600 python tools/fill_direct_ab.py c3 2>&1 | tee -a gpurun_out/fill_ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:k_seg_scatter_groups --csv --log-file gpurun_out/fill_direct_c4.csv python tools/seg_fill_profile.py > /dev/null 2>&1; echo ncu rc=$?
