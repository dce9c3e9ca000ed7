# functional check of the N>1 path on one GPU: 2 ranks on cuda:0 over gloo
# (CONFIG / KERNEL select the workload; seg shards take the pipelined per-slot exchange)
export BENCH_SINGLE_DEVICE=1 BENCH_DIST_BACKEND=gloo
C=${CONFIG:-c2}; K=${KERNEL:-auto}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $C --kernel $K --steps 5 --warmup 3 > gpurun_out/bench_multi_${C}_$K.json 2> gpurun_out/bench_multi_${C}_$K.log
echo rc=$?
grep -E "rel err|Error|error" gpurun_out/bench_multi_${C}_$K.log | tail -5; cat gpurun_out/bench_multi_${C}_$K.json
