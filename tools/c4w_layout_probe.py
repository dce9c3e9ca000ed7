"""C4-wide (108M rows, 2.16e9 nnz) seg layout build for an ncu launch list."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

n = 108_000_000
A = synth.random_rows(n, n, 20)
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
del A
torch.cuda.empty_cache()
for _ in range(2):
    lay = SegLayout(B, auto_seg_panels(B))
    torch.cuda.synchronize()
    del lay
print("done")
