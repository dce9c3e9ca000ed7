# ncu captures of the merge SpMV kernels (C2 both modes, C4 TMA)
set -x
for m in 0 1; do timeout 300 python tools/prof_spmv.py --config c2 --mode $m --iters 20 --time; done
for m in 0 1; do timeout 300 python tools/prof_spmv.py --config c4 --mode $m --iters 5 --time; done
timeout 300 python tools/prof_spmv.py --config c2 --kernel vector --iters 20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_merge -s 2 -c 1 -o gpurun_out/c2_mode0 python tools/prof_spmv.py --config c2 --mode 0 --iters 2 > gpurun_out/ncu_c2_m0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_merge -s 2 -c 1 -o gpurun_out/c2_mode1 python tools/prof_spmv.py --config c2 --mode 1 --iters 2 > gpurun_out/ncu_c2_m1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_merge -s 1 -c 1 -o gpurun_out/c4_mode1 python tools/prof_spmv.py --config c4 --mode 1 --iters 1 > gpurun_out/ncu_c4_m1.log 2>&1
tail -3 gpurun_out/ncu_*.log
ls -la gpurun_out
