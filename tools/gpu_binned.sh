# two-phase binned SpMV timing prototype (tools/binned_bench.cu), several tilings
cd tools
mk() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/bb_$1 binned_bench.cu $2; }
mk a "-DRB=4096 -DCELL=28 -DKC=64"
mk b "-DRB=4096 -DCELL=28 -DKC=64 -DEXU=4"
mk c "-DRB=8192 -DCELL=54 -DKC=32"
mk d "-DRB=4096 -DCELL=28 -DKC=64 -DP2T=256"
mk e "-DRB=4096 -DCB=8192 -DCELL=14 -DKC=128 -DP1T=512"
mk f "-DRB=2048 -DCELL=14 -DKC=128 -DP2T=256"
for v in a b c d e f; do echo "== $v"; timeout 120 bin/bb_$v; done 2>&1 | tee ../gpurun_out/binned.txt
