# the multi-rank paths after the round-2 changes: 2 ranks on one GPU (gloo) for C2 and C4-class
# seg shards, and the NCCL code with one rank (pipelined exchange, all_gather, fused iteration)
mkdir -p gpurun_out
CONFIG=c2 bash tools/gpu_multi.sh
CONFIG=c5 bash tools/gpu_multi.sh
bash tools/gpu_nccl1.sh
