"""The first seg layout build of a bench process (bench.py's order: matrix, permutations,
K4 twice, histogram, entropy), phase by phase with synchronising wall clocks, then under
the torch profiler for a second process-first build of another shape.
Usage: bench_cold_layout_probe.py [c5|c4]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
A = synth.laplacian5(2828) if cfg == "c5" else synth.random_rows(50_000_000, 50_000_000, 20)
n = A.n_rows
torch.cuda.Stream()
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
B = P.permute_csr(A, p_r, p_c)
hB = P.histogram_2d(B, 128, 128)
B2 = P.permute_csr(A, p_r, p_c)
del B2
P.shannon_entropy(P.histogram_2d(A, 128, 128)), P.shannon_entropy(hB)
torch.cuda.synchronize()

orig = {k: getattr(SegLayout, k) for k in ("_geometry", "_allocate", "_finish")}
times = {}


def wrap(name):
    f = orig[name]

    def g(self, *a, **kw):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(self, *a, **kw)
        torch.cuda.synchronize()
        times[name] = (time.perf_counter() - t) * 1e3
        return r
    return g


for k in orig:
    setattr(SegLayout, k, wrap(k))
_call = _lib.call_rp


def call_rp(name, *a):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = _call(name, *a)
    torch.cuda.synchronize()
    times[name] = (time.perf_counter() - t) * 1e3
    return r


_lib.call_rp = call_rp
for rep in range(3):
    times.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    lay = SegLayout(B, auto_seg_panels(B))
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t) * 1e3
    print(f"{cfg} rep {rep}: layout {tot:.1f} ms  " + "  ".join(f"{k} {v:.1f}" for k, v in times.items()), flush=True)
    del lay
