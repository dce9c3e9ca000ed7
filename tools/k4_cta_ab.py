"""K4 at C3 (R-MAT rows up to 1024) with the CTA hybrid row sort (sme_sort_rows_set_cta)
vs the all-shared-memory bitonic: CUDA events around permute_csr, bit-identity."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth

A = synth.rmat(24, 22, cap=1024)
n = A.n_rows
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018
ref = None
for rep in range(3):
    for cta in (1, 0):
        _lib.call("sme_sort_rows_set_cta", cta)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        B = P.permute_csr(A, p_r, p_c)
        e1.record()
        torch.cuda.synchronize()
        if ref is None:
            ref, same = B, True
        else:
            same = bool(torch.equal(ref.d_col_idx, B.d_col_idx) and torch.equal(ref.d_values, B.d_values))
        print(f"c3 rep {rep} cta={cta}: permute_csr {e0.elapsed_time(e1):.2f} ms, identical: {same}", flush=True)
        if B is not ref:
            del B
_lib.call("sme_sort_rows_set_cta", 1)
