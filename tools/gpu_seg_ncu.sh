mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_seg_scatter_groups -c 1 -o gpurun_out/seg_fill_full -f python tools/seg_fill_profile.py > gpurun_out/seg_ncu.log 2>&1; echo rc=$?
