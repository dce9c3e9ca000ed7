"""Where does device permutation generation spend its time? (pinned alloc, host partners,
H2D, GPU apply) vs the host full shuffle."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2308_00106_b200 import _cuda, _lib
from paper_2308_00106_b200._cuda import ptr, stream
from paper_2308_00106_b200.permute import pcg64_permutation, pcg64_swap_partners

torch.zeros(1, device="cuda")
for n in (8_000_000, 50_000_000):
    for threads in (1, 4, 8):
        t0 = time.perf_counter()
        h = torch.empty(n, dtype=torch.int32).pin_memory()
        t1 = time.perf_counter()
        pcg64_swap_partners(np.random.PCG64(1), n, h.numpy().view(np.uint32), threads)
        t2 = time.perf_counter()
        d = h.to("cuda", non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        ws = _cuda.workspace(_lib.query_size("sme_fy_apply_workspace_size", n))
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        _lib.call("sme_fy_apply", n, ptr(d), ptr(out), ptr(ws), ws.numel(), stream())
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        print(f"n={n} threads={threads}: pin {t1-t0:.3f} partners {t2-t1:.3f} h2d {t3-t2:.3f} alloc {t4-t3:.3f} "
              f"apply {t5-t4:.3f} s", flush=True)
    t = time.perf_counter()
    pcg64_permutation(np.random.PCG64(1), n)
    print(f"n={n}: host full shuffle {time.perf_counter() - t:.3f} s", flush=True)
