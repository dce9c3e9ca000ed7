"""K4 at C4 with and without the column-sliced pre-map: time and bit-identity."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
import paper_2308_00106_b200.permute as PM
from paper_2308_00106_b200 import synth

n = 50_000_000
A = synth.random_rows(n, n, 20)
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018
ref = None
for share in (0.5, 0, 0.5, 0):
    PM.PREMAP_L2_SHARE = share
    torch.cuda.synchronize()
    t = time.perf_counter()
    B = P.permute_csr(A, p_r, p_c)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3
    if ref is None:
        ref = B
        same = True
    else:
        same = bool(torch.equal(ref.d_col_idx, B.d_col_idx) and torch.equal(ref.d_values, B.d_values)
                    and torch.equal(ref.d_row_ptr, B.d_row_ptr))
    print(f"premap={'on' if share else 'off'}: {ms:.2f} ms, identical to the first: {same}", flush=True)
    if B is not ref:
        del B
