"""Where does the C4 e2e step go?  spmv_csr_pipelined (H2D x_k+1 || SpMV x_k || D2H y_k-1)
timed (a) as is, (b) with the panel passes replaced by nothing (copies only), (c) with
only the SpMV (device-resident vectors), (d) H2D alone and D2H alone of the same buffers."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.seg import SegLayout, seg_of

n = 50_000_000
A = synth.random_rows(n, n, 20)
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
del A
lay = seg_of(B)
xs = [torch.rand(n, dtype=torch.float64).pin_memory() for _ in range(2)]
steps = 20
yr = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
ys = [yr[k & 1] for k in range(steps)]


def run(label):
    P.spmv_csr_pipelined(B, xs, ys[:2])
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.spmv_csr_pipelined(B, [xs[k & 1] for k in range(steps)], ys)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / steps * 1e3
    print(f"{label}: {ms:.3f} ms/step", flush=True)


import paper_2308_00106_b200.kernels as K

orig_pass = SegLayout._pass

for nb in (2, 3):
    K.PIPELINE_BUFFERS = nb
    run(f"pipelined e2e, {nb} buffers")
K.PIPELINE_BUFFERS = 2
for g in (1, 2, 4, 8):
    K.PIPELINE_H2D_COPIES = g
    run(f"pipelined e2e, 2 buffers, {g} H2D copies per x")
    SegLayout._pass = lambda self, p, xd, y: None
    run(f"copies only, {g} H2D copies per x")
    SegLayout._pass = orig_pass
K.PIPELINE_H2D_COPIES = 0
orig = SegLayout._pass
SegLayout._pass = lambda self, p, xd, y: None
for nb in (2, 3):
    K.PIPELINE_BUFFERS = nb
    run(f"copies only (no SpMV), {nb} buffers")
K.PIPELINE_BUFFERS = 2
SegLayout._pass = orig
xd, yd = xs[0].cuda(), torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    lay.spmv_into(xd, yd)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(steps):
    lay.spmv_into(xd, yd)
torch.cuda.synchronize()
print(f"SpMV only: {(time.perf_counter() - t) / steps * 1e3:.3f} ms/step", flush=True)
for name, fn in (("H2D 400 MB", lambda: xd.copy_(xs[0], non_blocking=True)),
                 ("D2H 400 MB", lambda: ys[0].copy_(yd, non_blocking=True))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 5 * 1e3:.3f} ms", flush=True)
