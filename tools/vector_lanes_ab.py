"""CSR-vector lanes per row on a permuted matrix, alternated in one process (CUDA events
around `steps` SpMVs per setting).  Usage: vector_lanes_ab.py [c2|c5] [lanes, e.g. 1,2,4,8] [--unpermuted]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.kernels import default_lanes, spmv_into
from paper_2308_00106_b200.permute import axis_seed

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if args else "c2"
lanes_list = [int(v) for v in args[1].split(",")] if len(args) > 1 else [1, 2, 4, 8]
A = synth.laplacian5(2000 if cfg == "c2" else 2828)
n = A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
B = A if "--unpermuted" in sys.argv else P.permute_csr(A, p_r, p_c)
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
print(f"{cfg}: default lanes {default_lanes(B)}", flush=True)
res = {L: [] for L in lanes_list}
for rep in range(5):
    for L in lanes_list:
        for _ in range(5):
            spmv_into(B, x, y, "vector", lanes=L)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(200):
            spmv_into(B, x, y, "vector", lanes=L)
        e1.record()
        torch.cuda.synchronize()
        res[L].append(e0.elapsed_time(e1) / 200)
for L in lanes_list:
    v = sorted(res[L])
    print(f"lanes {L}: median {v[len(v) // 2]:.4f} ms  ({2 * B.nnz / v[len(v) // 2] / 1e6:.1f} GFLOP/s)")
