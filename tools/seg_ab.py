"""A/B of seg kernel modes on one permuted matrix: interleaved rounds of K SpMVs per
mode (medians of CUDA-event times, after a preload to reach the power-capped clock);
results must be bitwise equal to mode 0.

python tools/seg_ab.py --config c4 --modes 0,7 --rounds 6 --k 10
"""
import argparse
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--modes", default="0,7")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--preload", type=float, default=2.0)
a = ap.parse_args()
modes = [int(m) for m in a.modes.split(",")]
_lib.call("sme_spmv_seg_set_mode", max(modes))  # occupancy of every variant in the layout's grid
if a.config == "c4":
    A = synth.random_rows(50_000_000, 50_000_000, 20)
elif a.config == "c3":
    A = synth.rmat(24, 22, cap=1024)
elif a.config == "c5":
    A = synth.laplacian5(2828)
else:
    A = synth.laplacian5(2000)
n = A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (A.n_cols, axis_seed(7, 1))])
B = P.permute_csr(A, p_r, p_c)
del A
torch.cuda.empty_cache()
lay = seg_of(B)
x = torch.rand(B.n_cols, dtype=B.dtype, device="cuda")
ys = {m: torch.empty(n, dtype=B.dtype, device="cuda") for m in modes}
for m in modes:
    _lib.call("sme_spmv_seg_set_mode", m)
    lay.spmv_into(x, ys[m])
torch.cuda.synchronize()
for m in modes:
    print(f"mode {m}: bitwise equal to mode {modes[0]}: {torch.equal(ys[m], ys[modes[0]])}", flush=True)
t_end = time.perf_counter() + a.preload
while time.perf_counter() < t_end:
    lay.spmv_into(x, ys[modes[0]])
    torch.cuda.synchronize()
res = {m: [] for m in modes}
for _ in range(a.rounds):
    for m in modes:
        _lib.call("sme_spmv_seg_set_mode", m)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.k):
            lay.spmv_into(x, ys[m])
        e1.record()
        torch.cuda.synchronize()
        res[m].append(e0.elapsed_time(e1) / a.k)
for m in modes:
    print(f"{a.config} P={lay.n_panels} warps={lay.n_warps} mode {m}: median {statistics.median(res[m]):.4f} ms "
          f"(min {min(res[m]):.4f}, max {max(res[m]):.4f}) nnz {B.nnz:,} -> "
          f"{2 * B.nnz / statistics.median(res[m]) / 1e6:.1f} GFLOP/s", flush=True)
