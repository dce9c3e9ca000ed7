"""C4 permuted-CSR build (K4, permute_csr) for ncu / timing: python tools/prof_permute.py [--reps 3]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=50_000_000)
a = ap.parse_args()
A = synth.random_rows(a.n, a.n, 20)
p_r, p_c = P.random_permutation(a.n, 1), P.random_permutation(a.n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018  (inverses outside the timing)
for i in range(a.reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    B = P.permute_csr(A, p_r, p_c)
    torch.cuda.synchronize()
    print(f"permute_csr: {(time.perf_counter() - t) * 1e3:.2f} ms (nnz {B.nnz:,})", flush=True)
    del B
