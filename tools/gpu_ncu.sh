# ncu --set full of one kernel:  KREGEX=... ARGS="--config c2 --kernel stream" OUT=name bash tools/gpu_ncu.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-2} -c 1 -o gpurun_out/${OUT} python tools/prof_spmv.py ${ARGS} --iters 2 > gpurun_out/${OUT}.log 2>&1
tail -n 3 gpurun_out/${OUT}.log
