"""Permuted 128x128 histogram of a config's matrix: timing of both kernels (CUDA events),
and two plain calls for ncu.  python tools/prof_hist.py [--config c4|c2|c3] [--reps 10]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
A = {"c4": lambda: synth.random_rows(50_000_000, 50_000_000, 20), "c2": lambda: synth.laplacian5(2000),
     "c3": lambda: synth.rmat(24, 16, cap=1024)}[a.config]()
n = A.n_rows
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
ref = None
for mode, var, name in ((1, 0, "shared-atomic window"), (0, 0, "lanes default (864x4, CL 2)"), (0, 7, "lanes 512x8"), (0, 1, "lanes 768x4"),
                        (0, 2, "lanes 512x4+pf"), (0, 3, "lanes 768x2+pf"), (0, 4, "lanes 640x4+pf"), (0, 5, "lanes 864x4 (CL 0, previous default)"), (0, 6, "lanes 864x2"),
                        (0, 8, "lanes 864x4 conflict-free words"), (0, 9, "lanes 864x4 conflict-free words, shared atomics"),
                        (0, 10, "lanes 864x2 CL 2"), (0, 11, "lanes 640x4+pf CL 2"), (0, 12, "lanes 512x8 CL 2")):
    _lib.call("sme_hist2d_set_mode", mode)
    _lib.call("sme_hist2d_set_variant", var)
    h = P.histogram_2d(B, 128, 128).counts  # warm
    if ref is None:
        ref = h
    assert (h == ref).all()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(a.reps):
        P.histogram_2d(B, 128, 128)
    e[1].record()
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1]) / a.reps
    print(f"{a.config} hist2d 128x128 {name}: {ms:.3f} ms  ({B.nnz * 4 / ms / 1e6:.0f} GB/s of col_idx, "
          f"{B.nnz / ms / 1e6:.1f} G nnz/s)", flush=True)
_lib.call("sme_hist2d_set_mode", 0)
_lib.call("sme_hist2d_set_variant", 0)
