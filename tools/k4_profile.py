"""One C4 K4 (permute_csr) for an ncu capture of its kernels; argv[1] = fuse_last 0/1."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
import paper_2308_00106_b200.permute as PM
from paper_2308_00106_b200 import synth

PM.PREMAP_FUSE_LAST = bool(int(sys.argv[1])) if len(sys.argv) > 1 else True
n = 50_000_000
A = synth.random_rows(n, n, 20)
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
p_r.d_inverse, p_c.d_inverse  # noqa: B018
B = P.permute_csr(A, p_r, p_c)
torch.cuda.synchronize()
print("done")
