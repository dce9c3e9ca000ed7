"""K4 at C4 / C3 with the source starts gathered once (permute.K4_STARTS) vs the row sort's
own row_ptr gathers: CUDA events around permute_csr, bit-identity of the results."""
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
for rep in range(3):
    for on in (True, False):
        PM.K4_STARTS = on
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        B = P.permute_csr(A, p_r, p_c)
        e1.record()
        torch.cuda.synchronize()
        if ref is None:
            ref, same = B, True
        else:
            same = bool(torch.equal(ref.d_col_idx, B.d_col_idx) and torch.equal(ref.d_values, B.d_values)
                        and torch.equal(ref.d_row_ptr, B.d_row_ptr))
        print(f"{cfg} rep {rep} starts={on}: permute_csr {e0.elapsed_time(e1):.2f} ms, identical: {same}", flush=True)
        if B is not ref:
            del B
