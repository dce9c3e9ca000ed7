"""Seg layout build time at C4 (the 'analysis' step, cached per matrix)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.seg import SegLayout

A = synth.random_rows(50_000_000, 50_000_000, 20)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lay = SegLayout(A, 8)
    torch.cuda.synchronize()
    print(f"seg layout build (8 panels, 1e9 nnz): {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    del lay
