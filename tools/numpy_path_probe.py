"""The reference-shaped call with numpy vectors (what a KernelSpec plugin inside the
reference's run_experiment does): y = spmv_csr(m, x_numpy) -> numpy, at C4, broken down."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
A = synth.random_rows(n, n, 20)
B = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
del A
x = np.random.default_rng(0).random(n)
xd = torch.from_numpy(x).cuda()
yd = P.spmv_csr(B, xd)
torch.cuda.synchronize()


def t(label, fn, reps=5):
    r = None
    for _ in range(3):  # warm, keeping each result alive across the next call as a harness
        r = fn()        # does: the result pool then holds two page-locked mappings
    del r
    torch.cuda.synchronize()
    w = time.perf_counter()
    each = []
    for _ in range(reps):
        w1 = time.perf_counter()
        r = fn()
        each.append((time.perf_counter() - w1) * 1e3)
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - w) / reps * 1e3:.2f} ms  (calls: {' '.join(f'{e:.1f}' for e in each)})",
          flush=True)
    return r


y = t("spmv_csr(numpy x) -> numpy y", lambda: P.spmv_csr(B, x))
assert np.array_equal(y, yd.cpu().numpy())
y2 = P.spmv_csr(B, x * 2)
assert np.array_equal(y2, 2 * y) and y2 is not y  # fresh result, the first one intact
xt = torch.from_numpy(x)
t("spmv_csr(pageable CPU tensor x) -> CPU tensor y", lambda: P.spmv_csr(B, xt))
t("  numpy x -> device (torch.from_numpy(x).cuda())", lambda: torch.from_numpy(x).cuda())
t("  device y -> fresh numpy (y.cpu().numpy())", lambda: yd.cpu().numpy())
t("  SpMV only (device vectors)", lambda: P.spmv_csr(B, xd))
xp = torch.from_numpy(x).pin_memory()
t("spmv_csr(pinned x) -> pinned y", lambda: P.spmv_csr(B, xp))
t("  np.copyto into a pinned buffer (400 MB)", lambda: np.copyto(xp.numpy(), x))
t("  fresh np.empty + copy of 400 MB", lambda: np.array(x, copy=True))
t("  torch copy_ into pinned", lambda: xp.copy_(torch.from_numpy(x)))
print("torch threads", torch.get_num_threads())

# breakdown of the numpy-x call: staging + passes, then the result copy
from paper_2308_00106_b200 import hostio
from paper_2308_00106_b200.seg import seg_of

lay = seg_of(B)
xd2 = torch.empty(n, dtype=torch.float64, device="cuda")
yd2 = torch.empty(n, dtype=torch.float64, device="cuda")
src = torch.from_numpy(x)
for rep in range(3):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for p, ev in hostio.stage_in(src, xd2, lay.bounds_host):
        torch.cuda.current_stream().wait_event(ev)
        lay._window(p, xd2)
        lay._pass(p, xd2, yd2)
    w1 = time.perf_counter()
    lay._window(None, None)
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    out = hostio.to_host(yd2, np.float64, True)
    w3 = time.perf_counter()
    del out
    print(f"stage_in+enqueue {1e3 * (w1 - w0):.2f} ms, until passes done {1e3 * (w2 - w0):.2f} ms, "
          f"to_host {1e3 * (w3 - w2):.2f} ms", flush=True)
stage = hostio.pinned((n,), torch.float64, "in")
for rep in range(3):
    w0 = time.perf_counter()
    stage.copy_(src)
    print(f"copy_ numpy -> pinned stage, whole: {1e3 * (time.perf_counter() - w0):.2f} ms", flush=True)
for rep in range(3):
    w0 = time.perf_counter()
    for q in range(8):
        lo, hi = n * q // 8, n * (q + 1) // 8
        stage[lo:hi].copy_(src[lo:hi])
    print(f"copy_ numpy -> pinned stage, 8 slices: {1e3 * (time.perf_counter() - w0):.2f} ms", flush=True)

import cProfile
import pstats

print("per call:", flush=True)
for rep in range(4):
    w0 = time.perf_counter()
    r = P.spmv_csr(B, x)
    print(f"  {1e3 * (time.perf_counter() - w0):.2f} ms, pool {[(k, len(v)) for k, v in hostio._POOL.items()]}", flush=True)
pr = cProfile.Profile()
pr.enable()
for rep in range(3):
    r = P.spmv_csr(B, x)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
