"""Seg layout build at C5 (permuted 5-pt Laplacian 2828^2, 2 panels): wall time of the build
and of its host-side steps, for a launch list under ncu."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
A = synth.laplacian5(2828) if cfg == "c5" else synth.random_rows(50_000_000, 50_000_000, 20)
n = A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
B = P.permute_csr(A, p_r, p_c)
Pn = auto_seg_panels(B)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lay = SegLayout(B, Pn)
    torch.cuda.synchronize()
    print(f"{cfg} seg layout build ({Pn} panels): {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
    del lay
