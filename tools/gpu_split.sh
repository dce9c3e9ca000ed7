# side-by-side pull (L2 gathers) + binned (HBM) feasibility (tools/split_bench.cu)
cd tools
mk() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/sb_$1 split_bench.cu -DRB=4096 -DCELL=28 -DKC=64 $2; }
mk a "-DPULL_CTAS=4 -DP1T=1024"
mk b "-DPULL_CTAS=3 -DP1T=256"
mk c "-DPULL_CTAS=3 -DP1T=512"
mk d "-DPULL_CTAS=2 -DP1T=512"
mk e "-DPULL_CTAS=3 -DP1T=256 -DCB=8192 -DCELL=14 -DKC=128"
for v in a b c d e; do echo "== $v"; timeout 120 bin/sb_$v 0.4; done 2>&1 | tee ../gpurun_out/split.txt
for f in 0.25 0.55; do echo "== c f=$f"; timeout 120 bin/sb_c $f; done 2>&1 | tee -a ../gpurun_out/split.txt
