# LDG + TMA gather4 mix (tools/gather_mix_bench.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather_mix_bench tools/gather_mix_bench.cu -lcuda
for mb in ${MBS:-48}; do timeout 300 tools/bin/gather_mix_bench $mb; done
