"""Breakdown of the first (cold) seg layout build of a process at C5: every libsme
call timed with a synchronising wall clock; the rest is host work and allocation."""
import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _cuda, _lib, synth
from paper_2308_00106_b200.seg import seg_of

_cuda.require_cuda()
A = synth.laplacian5(2828)
n = A.n_rows
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
torch.cuda.synchronize()

acc = defaultdict(float)
orig = _lib.call


def timed_call(name, *args):
    torch.cuda.synchronize()
    t = time.perf_counter()
    orig(name, *args)
    torch.cuda.synchronize()
    acc[name] += (time.perf_counter() - t) * 1e3


for rep in range(1):
    acc.clear()
    _lib.call = timed_call
    torch.cuda.synchronize()
    t = time.perf_counter()
    B._cache.pop(("seg", 2, True), None)
    lay = seg_of(B, full_last=True)
    torch.cuda.synchronize()
    total = (time.perf_counter() - t) * 1e3
    _lib.call = orig
    print(f"rep {rep}: seg layout {total:.1f} ms; libsme calls {sum(acc.values()):.1f} ms:",
          ", ".join(f"{k} {v:.1f}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])), flush=True)
    del lay

# which torch ops does the first build run (each first use of a torch kernel loads its module)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

C = synth.laplacian5(2000)
Bc = P.permute_csr(C, P.random_permutation(C.n_rows, 3), P.random_permutation(C.n_rows, 4))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU]) as prof:
    lay = seg_of(Bc, 3, full_last=False)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15))
