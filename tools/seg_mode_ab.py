"""k_spmv_seg variants (sme_spmv_seg_set_mode) on one permuted matrix, alternated in one
process: CUDA events around `steps` SpMVs per variant, y compared bit for bit with mode 0.
Usage: seg_mode_ab.py [c4|c5|c3] [modes, e.g. 0,8,9,10,11]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.kernels import spmv_into
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
modes = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 8]
A = (synth.random_rows(50_000_000, 50_000_000, 20) if cfg == "c4" else synth.laplacian5(2828) if cfg == "c5"
     else synth.rmat(24, 22, cap=1024))
n = A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (A.n_cols, axis_seed(7, 1))])
B = P.permute_csr(A, p_r, p_c)
del A
torch.cuda.empty_cache()
lay = seg_of(B)
x = torch.rand(B.n_cols, dtype=B.dtype, device="cuda")
y = torch.empty(B.n_rows, dtype=B.dtype, device="cuda")
steps = 20 if cfg == "c4" else 200
ref = None
res = {m: [] for m in modes}
for rep in range(4):
    for m in modes:
        _lib.call("sme_spmv_seg_set_mode", m)
        for _ in range(3):
            spmv_into(B, x, y, "seg")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            spmv_into(B, x, y, "seg")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[m].append(ms)
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(ref, y))
        rel_vs0 = float((y - ref).abs().max() / ref.abs().max()) if not same else 0.0
        print(f"{cfg} panels={lay.n_panels} rep={rep} mode={m}: {ms:.4f} ms/SpMV  {2 * B.nnz / ms / 1e6:.1f} GFLOP/s"
              f"  bitwise={same} rel_vs0={rel_vs0:.2e}", flush=True)
_lib.call("sme_spmv_seg_set_mode", 0)
for m in modes:
    print(f"mode {m}: median {sorted(res[m])[len(res[m]) // 2]:.4f} ms")
