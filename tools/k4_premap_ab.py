"""K4 at C4 (or C3) with and without the column-sliced pre-map, for several slice sizes
and with/without a persisting-L2 window: CUDA-event time and bit-identity."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
import paper_2308_00106_b200.permute as PM
from paper_2308_00106_b200 import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
A = synth.random_rows(50_000_000, 50_000_000, 20) if cfg == "c4" else synth.rmat(24, 22, cap=1024)
n = A.n_rows
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018
ref = None
VARIANTS = sys.argv[2] if len(sys.argv) > 2 else "slices"
if VARIANTS == "persist":  # the persisting-L2 window over each slice, 3-5 slices
    variants = [(True, mb, pers, False) for mb in (40, 48, 64) for pers in (False, True)]
else:
    variants = [(False, 0, False, False)] + [(True, mb, pers, fuse) for mb in (40, 48, 64)
                                              for pers in (False,) for fuse in (False, True)]
for rep in range(2):
    for on, mb, pers, fuse in variants:
        PM.PREMAP, PM.PREMAP_PERSIST, PM.PREMAP_FUSE_LAST = on, pers, fuse
        if mb:
            PM.PREMAP_SLICE_BYTES = mb << 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        B = P.permute_csr(A, p_r, p_c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ref is None:
            ref, same = B, True
        else:
            same = bool(torch.equal(ref.d_col_idx, B.d_col_idx) and torch.equal(ref.d_values, B.d_values)
                        and torch.equal(ref.d_row_ptr, B.d_row_ptr))
        print(f"rep {rep} premap={'on' if on else 'off'} slice={mb} MB persist={pers} fuse_last={fuse} slices={PM._premap_slices(A)}: "
              f"{ms:.2f} ms, identical: {same}", flush=True)
        if B is not ref:
            del B
