# quick GPU loop: tests + kernel timings (no ncu)
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for k in ${KERNELS:-stream}; do
  timeout 300 python tools/prof_spmv.py --config c2 --kernel $k --iters 50
  timeout 300 python tools/prof_spmv.py --config c2 --kernel $k --iters 50 --unpermuted
done
for P in ${PANELS:-1 2 3 4 6 8}; do timeout 300 python tools/prof_spmv.py --config c4 --kernel panel --panels $P --iters 5; done
