"""C4 permuted 128x128 histogram, twice (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth

A = synth.random_rows(50_000_000, 50_000_000, 20)
n = A.n_rows
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
for _ in range(2):
    P.histogram_2d(B, 128, 128)
torch.cuda.synchronize()
