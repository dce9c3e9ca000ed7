for rc in 0 1 2 4; do timeout 300 python tools/prof_spmv.py --config c4 --kernel panel --panels 8 --persist --iters 10 --reps 3 --row-cost $rc; done
for rc in 0 2 4; do timeout 300 python tools/prof_spmv.py --config c2 --kernel stream --iters 50 --reps 2 --row-cost $rc; done
