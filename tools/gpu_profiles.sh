# round-1 profiles: full test suite, launch list of the bench command, full ncu captures of the
# dominant kernels (all 8 panel passes of one C4 SpMV), gather roofline
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/prof/pytest_gpu.txt; cat gpurun_out/prof/pytest_gpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/prof/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmv_stream -s 9 -c 8 -o gpurun_out/prof/c4_panel_step python tools/prof_spmv.py --config c4 --kernel panel --panels 8 --persist --iters 2 > gpurun_out/prof/c4_panel_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hist2d_csr -s 1 -c 1 -o gpurun_out/prof/c4_hist python tools/prof_hist.py > gpurun_out/prof/c4_hist.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_stream -s 1 -c 1 -o gpurun_out/prof/c3_stream python tools/prof_spmv.py --config c3 --kernel stream --iters 2 > gpurun_out/prof/c3_stream.log 2>&1
timeout 300 python tools/gather_roofline.py > gpurun_out/prof/gather_roofline.jsonl
ls gpurun_out/prof
