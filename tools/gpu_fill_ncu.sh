# one full ncu capture (source counters) of the C4 seg layout fill and of the K4 row sort
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_seg_scatter_groups -c 1 \
  -o gpurun_out/fill_c4 python tools/seg_fill_profile.py > gpurun_out/fill_ncu.log 2>&1; echo ncu rc=$?
