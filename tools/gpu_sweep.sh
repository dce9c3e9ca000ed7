timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "panel or power_law or golden" 2>&1 | tail -2
for P in 6 7 8; do timeout 300 python tools/prof_spmv.py --config c4 --kernel panel --panels $P --persist --iters 5; done
timeout 300 python tools/prof_spmv.py --config c2 --kernel stream --iters 50
