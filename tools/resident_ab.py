"""Resident-wave grids (sme_set_resident_grids) vs the fixed per-SM caps for the
grid-stride setup kernels: K4 (permute_csr) and the seg layout build, alternated in
one process, CUDA events around each, outputs compared bit for bit.
Usage: resident_ab.py [c4|c3|c4w] [modes, e.g. 1,0: 0 = fixed caps, k = k resident waves] [hook]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg in ("c4", "c4w"):
    n = 50_000_000 if cfg == "c4" else 108_000_000
    A = synth.random_rows(n, n, 20)
else:
    A = synth.rmat(24, 22, cap=1024)
    n = A.n_rows
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse
ref = None


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


modes = [int(m) for m in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 0]
hook = sys.argv[3] if len(sys.argv) > 3 else "sme_set_resident_grids"
for rep in range(3 if cfg != "c4w" else 2):
    for on in modes:
        _lib.call(hook, on)
        B, t_k4 = timed(lambda: P.permute_csr(A, p_r, p_c))
        Pn = auto_seg_panels(B)
        lay, t_lay = timed(lambda: SegLayout(B, Pn))
        sig = (B.d_col_idx, B.d_values, lay.pk, lay.val, lay.hdr)
        if ref is None:
            ref = tuple(t.clone() for t in sig)
            same = ""
        else:
            same = f" identical={all(torch.equal(a, b) for a, b in zip(ref, sig))}"
        print(f"{cfg} rep={rep} {hook}={on}: K4 {t_k4:.2f} ms, layout ({Pn} panels) {t_lay:.2f} ms{same}", flush=True)
        del B, lay, sig
        if cfg == "c4w":
            torch.cuda.empty_cache()
_lib.call("sme_set_resident_grids", -1)
