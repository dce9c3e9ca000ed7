"""C4 permuted CSR + one seg layout build, for an ncu capture of the layout fill."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

n = 50_000_000
A = synth.random_rows(n, n, 20)
p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
B = P.permute_csr(A, p_r, p_c)
del A
torch.cuda.empty_cache()
lay = SegLayout(B, auto_seg_panels(B))
torch.cuda.synchronize()
print("done")
