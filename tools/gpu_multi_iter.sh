# functional check of the multi-GPU C5 path on one GPU: 2 ranks on cuda:0 over gloo,
# CUDA IPC peer stores into the other process's buffers
export BENCH_SINGLE_DEVICE=1 BENCH_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --config c5 --iterative --warmup 3 > gpurun_out/bench_multi_c5.json 2> gpurun_out/bench_multi_c5.log
echo rc=$?; tail -3 gpurun_out/bench_multi_c5.log; cat gpurun_out/bench_multi_c5.json
