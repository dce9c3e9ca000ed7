# setup kernels after the warp-medium sort and the coalesced seg fill: tests + ncu launch list
timeout 900 python -m pytest -q -x tests/test_gpu_r2_api.py tests/test_gpu_seg.py tests/test_gpu_parity.py tests/test_gpu_property.py tests/test_gpu_fullscale.py tests/test_gpu_rmat.py 2>&1 | tail -4
timeout 1000 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup2_c4.csv python tools/setup_breakdown.py c4 > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup2_c3.csv python tools/setup_breakdown.py c3 > /dev/null 2>&1; echo rc=$?
