mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_seg.py 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_seg --csv --log-file gpurun_out/segfill_c4.csv python tools/setup_breakdown.py c4 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/segfill_c4.csv 200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_seg --csv --log-file gpurun_out/segfill_c3.csv python tools/setup_breakdown.py c3 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/segfill_c3.csv 200
