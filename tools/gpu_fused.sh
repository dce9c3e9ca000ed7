timeout 900 python -m pytest -q -x tests/test_gpu_fused_seg.py 2>&1 | tail -3
timeout 600 python tools/fused_seg_ab.py c4 2>&1 | tee gpurun_out/fused_ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_seg|k_sort|k_map|k_scan" --csv --log-file gpurun_out/fused_c4.csv python tools/seg_fill_profile.py > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/fused_c4.csv 60
