"""Seg layout fill variants behind a test hook (e.g. sme_seg_set_fill_lut), alternated in
one process, CUDA events around the SegLayout build, layouts compared bit for bit.
Usage: fill_hook_ab.py [c4|c4w|c3] [hook] [modes, e.g. 1,0]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg in ("c4", "c4w"):
    n = 50_000_000 if cfg == "c4" else 108_000_000
    A = synth.random_rows(n, n, 20)
else:
    A = synth.rmat(24, 22, cap=1024)
    n = A.n_rows
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
del A
torch.cuda.empty_cache()
Pn = auto_seg_panels(B)
ref = None
hook = sys.argv[2] if len(sys.argv) > 2 else "sme_seg_set_fill_lut"
modes = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 0]
for rep in range(4 if cfg != "c4w" else 2):
    for mode in modes:
        _lib.call(hook, mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        lay = SegLayout(B, Pn)
        e1.record()
        torch.cuda.synchronize()
        same = ""
        if ref is None:
            ref = (lay.pk.clone(), lay.val.clone(), lay.hdr.clone())
        else:
            same = f" identical={bool(torch.equal(ref[0], lay.pk) and torch.equal(ref[1], lay.val) and torch.equal(ref[2], lay.hdr))}"
        print(f"{cfg} panels={Pn} rep={rep} {hook}={mode}: layout build {e0.elapsed_time(e1):.2f} ms{same}", flush=True)
        del lay
_lib.call(hook, 1)
