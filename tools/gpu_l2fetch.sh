mkdir -p gpurun_out
./tools/bin/l2fetch_bench 50 100 200 400 > gpurun_out/l2fetch.txt 2>&1; cat gpurun_out/l2fetch.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv --log-file gpurun_out/l2fetch_ncu.csv ./tools/bin/l2fetch_bench 200 > /dev/null 2>&1; echo ncu rc=$?
