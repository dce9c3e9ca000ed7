# K4 pre-map A/B (C4, C3), parity tests of K4, ncu launch list of the C4 setup
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_property.py tests/test_gpu_fullscale.py tests/test_gpu_rmat.py 2>&1 | tail -3
timeout 600 python tools/k4_premap_ab.py c4 > gpurun_out/k4_ab_c4.txt 2>&1; echo "ab c4 rc=$?"; cat gpurun_out/k4_ab_c4.txt
timeout 600 python tools/k4_premap_ab.py c3 > gpurun_out/k4_ab_c3.txt 2>&1; echo "ab c3 rc=$?"; cat gpurun_out/k4_ab_c3.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup3_c4.csv python tools/setup_breakdown.py c4 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/setup3_c4.csv 200 | grep -v "k_fy\|k_gg\|scan_apply"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sort_rows_warp -c 1 -o gpurun_out/k4_sort_full -f python tools/k4_profile.py 0 > gpurun_out/k4_ncu.log 2>&1; echo rc=$?
