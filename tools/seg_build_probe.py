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

from paper_2308_00106_b200 import _lib

for on in (0, 1, 0, 1):
    _lib.call("sme_seg_set_scatter_groups", on)
    torch.cuda.synchronize()
    t = time.perf_counter()
    lay = SegLayout(A, 8)
    torch.cuda.synchronize()
    print(f"scatter_groups={on}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    if on == 0:
        ref = (lay.pk.clone(), lay.val.clone(), lay.hdr.clone())
    else:
        print("  identical layout:", bool(torch.equal(ref[0], lay.pk) and torch.equal(ref[1], lay.val)
                                         and torch.equal(ref[2], lay.hdr)), flush=True)
    del lay
