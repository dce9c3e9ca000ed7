"""random_permutations at C4 (2 x 50M, the bench's device_perms) broken down: concurrent
host partners, pageable vs pinned H2D, GPU apply."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _cuda, _lib
from paper_2308_00106_b200._cuda import ptr, stream
from paper_2308_00106_b200.permute import axis_seed, pcg64_swap_partners

torch.zeros(1, device="cuda")
n = 50_000_000
specs = [(n, axis_seed(7, 0)), (n, axis_seed(7, 1))]
# first call, piece by piece (what bench.py's perm_gen_s sees once)
from paper_2308_00106_b200.permute import pcg64_swap_partners_device

torch.cuda.synchronize()
t0 = time.perf_counter()
bufs = [(torch.empty(n, dtype=torch.int32, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda"),
         _cuda.workspace(_lib.query_size("sme_fy_apply_workspace_size", n))) for _ in specs]
torch.cuda.synchronize()
t1 = time.perf_counter()
ss = [torch.cuda.Stream() for _ in specs]
t2 = time.perf_counter()
tt = {}


def one(k):
    a = time.perf_counter()
    with torch.cuda.stream(ss[k]):
        pcg64_swap_partners_device(np.random.PCG64(specs[k][1]), n, threads=4, out=bufs[k][0])
        b = time.perf_counter()
        _lib.call("sme_fy_apply", n, ptr(bufs[k][0]), ptr(bufs[k][1]), ptr(bufs[k][2]), bufs[k][2].numel(), stream())
    ss[k].synchronize()
    tt[k] = (b - a, time.perf_counter() - b)


with ThreadPoolExecutor(max_workers=2) as ex:
    list(ex.map(one, range(2)))
t3 = time.perf_counter()
print(f"first call: buffers {t1 - t0:.3f} s (ws {bufs[0][2].numel() / 1e6:.0f} MB each), streams {t2 - t1:.3f}, "
      f"partners+apply {t3 - t2:.3f} (per axis partners/apply: {tt})", flush=True)
del bufs
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = P.random_permutations(specs)
    torch.cuda.synchronize()
    print(f"random_permutations total: {time.perf_counter() - t0:.3f} s", flush=True)
    del p
for rep in range(2):
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=2) as ex:
        hs = list(ex.map(lambda a: pcg64_swap_partners(np.random.PCG64(a[1]), a[0], threads=4), specs))
    t1 = time.perf_counter()
    ds = [torch.from_numpy(h.view(np.int32)).to("cuda") for h in hs]
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    ws = _cuda.workspace(_lib.query_size("sme_fy_apply_workspace_size", n))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    for d in ds:
        _lib.call("sme_fy_apply", n, ptr(d), ptr(out), ptr(ws), ws.numel(), stream())
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"partners (2 concurrent) {t1 - t0:.3f} s, pageable H2D x2 {t2 - t1:.3f}, ws alloc {t3 - t2:.3f}, "
          f"apply x2 {t4 - t3:.3f}", flush=True)
    # the same partners into pre-faulted buffers
    bufs = [np.empty(n, dtype=np.uint32) for _ in range(2)]
    for b in bufs:
        b.fill(0)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=2) as ex:
        list(ex.map(lambda ab: pcg64_swap_partners(np.random.PCG64(ab[0][1]), ab[0][0], ab[1], threads=4),
                    zip(specs, bufs)))
    print(f"partners into pre-faulted buffers: {time.perf_counter() - t0:.3f} s", flush=True)
    pin = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
    for pb, h in zip(pin, hs):
        pb.numpy()[:] = h.view(np.int32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds = [pb.to("cuda", non_blocking=True) for pb in pin]
    torch.cuda.synchronize()
    print(f"pinned H2D x2 {time.perf_counter() - t0:.3f}", flush=True)

for rep in range(2):
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=2) as ex:
        djs = list(ex.map(lambda a: P.permute.pcg64_swap_partners_device(np.random.PCG64(a[1]), a[0], threads=4),
                          specs))
    torch.cuda.synchronize()
    print(f"partners streamed to the device (2 concurrent): {time.perf_counter() - t0:.3f} s", flush=True)
