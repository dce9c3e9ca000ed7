"""128 x 128 tile histogram of the permuted C4 (or C3) matrix: CUDA events around 20
calls, median of 5 (cross-build A/B helper).  Usage: hist_ab.py [c4|c3]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
A = synth.random_rows(50_000_000, 50_000_000, 20) if cfg == "c4" else synth.rmat(24, 22, cap=1024)
B = P.permute_csr(A, P.random_permutation(A.n_rows, 1), P.random_permutation(A.n_cols, 2))
del A
ref = P.histogram_2d(B, 128, 128).counts
ts = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        h = P.histogram_2d(B, 128, 128)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 20)
assert (h.counts == ref).all()
print(f"{cfg} histogram_2d 128x128: median {sorted(ts)[2]:.4f} ms  {sorted(ts)}")
