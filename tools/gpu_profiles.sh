# profiles for round 1: launch list of the bench command, full captures of the dominant kernels
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/prof/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/prof/bench_c4_under_ncu.json 2> gpurun_out/prof/bench_c4_under_ncu.log
tail -2 gpurun_out/prof/bench_c4_under_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_stream -s 7 -c 1 -o gpurun_out/prof/c4_panel_pass python tools/prof_spmv.py --config c4 --kernel panel --panels 7 --persist --iters 1 > gpurun_out/prof/c4_panel_pass.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_vector -s 1 -c 1 -o gpurun_out/prof/c2_vector python tools/prof_spmv.py --config c2 --kernel vector --lanes 2 --iters 1 > gpurun_out/prof/c2_vector.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_vector -s 1 -c 1 -o gpurun_out/prof/c2u_vector python tools/prof_spmv.py --config c2 --kernel vector --lanes 1 --unpermuted --iters 1 > gpurun_out/prof/c2u_vector.log 2>&1
timeout 300 python tools/gather_roofline.py > gpurun_out/prof/gather_roofline.jsonl
ls -la gpurun_out/prof
