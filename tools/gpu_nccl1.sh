# the NCCL code paths of the multi-GPU bench with ONE rank (this pool leases one GPU):
# pipelined per-slot broadcasts, the single all_gather, and the fused-exchange power iteration
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1"
BENCH_FORCE_SHARDED=1 SME_PIPELINED_EXCHANGE=force timeout 600 $R --master-port 29601 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/nccl1_pipe.json 2> gpurun_out/nccl1_pipe.log; echo "pipelined rc=$?"
BENCH_FORCE_SHARDED=1 timeout 600 $R --master-port 29602 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/nccl1_ag.json 2> gpurun_out/nccl1_ag.log; echo "allgather rc=$?"
BENCH_FORCE_SHARDED=1 timeout 600 $R --master-port 29603 bench.py --gpus 1 --config c5 --iterative --warmup 3 > gpurun_out/nccl1_iter.json 2> gpurun_out/nccl1_iter.log; echo "iterative rc=$?"
for f in pipe ag iter; do tail -c 600 gpurun_out/nccl1_$f.json; echo; grep -iE "error|Traceback" gpurun_out/nccl1_$f.log | head -3; done
