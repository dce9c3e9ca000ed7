"""C4 setup with and without the K4-fused seg layout build (permute.FUSE_SEG_LAYOUT):
CUDA events around permute_csr and around the first seg_of (the layout the SpMV uses)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import permute as PM
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.seg import seg_of

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = 50_000_000 if cfg == "c4" else 108_000_000
A = synth.random_rows(n, n, 20)
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018


def ev():
    return torch.cuda.Event(enable_timing=True)


for rep in range(3):
    for fuse in (True, False):
        PM.FUSE_SEG_LAYOUT = fuse
        e0, e1, e2 = ev(), ev(), ev()
        torch.cuda.synchronize()
        e0.record()
        B = P.permute_csr(A, p_r, p_c)
        e1.record()
        lay = seg_of(B)
        e2.record()
        torch.cuda.synchronize()
        k4, lb = e0.elapsed_time(e1), e1.elapsed_time(e2)
        print(f"{cfg} rep {rep} fused={fuse}: permute_csr {k4:.2f} ms + layout {lb:.2f} ms = {k4 + lb:.2f} ms "
              f"({lay.n_panels} panels)", flush=True)
        del B, lay
