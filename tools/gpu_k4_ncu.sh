mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sort_rows_warp -c 1 -o gpurun_out/k4_sort_full -f python tools/k4_profile.py 0 > gpurun_out/k4_ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/k4_ncu.log
