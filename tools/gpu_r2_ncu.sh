# round-2 ncu evidence for the default bench command: launch list (durations, DRAM bytes) of
# every libsme kernel, and one --set full capture of a C4 seg pass
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sme::|k_" -c 3000 --csv --log-file gpurun_out/launches_bench_c4.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/launches_bench_c4.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_seg -s 8 -c 1 \
  -o gpurun_out/c4_seg_r2 python tools/prof_spmv.py --config c4 --kernel seg --iters 2 > gpurun_out/c4_seg_r2.log 2>&1; echo full rc=$?
