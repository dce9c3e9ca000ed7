# functional check of the N>1 path on one GPU: 2 ranks on cuda:0 over gloo
export BENCH_SINGLE_DEVICE=1 BENCH_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config c2 --steps 5 --warmup 3 > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.log
echo rc=$?
tail -5 gpurun_out/bench_multi.log; cat gpurun_out/bench_multi.json
