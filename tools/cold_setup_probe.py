"""Where a cold (first in the process) permuted-matrix setup spends its time: C5
(8M-row Laplacian) permutation + K4 + seg layout, timed three times in one process —
1st (cold: lazy kernel loading, allocator growth), 2nd (same sizes), 3rd — with
synchronising wall clocks around each step.  Run it with CUDA_MODULE_LOADING=EAGER
to separate the kernel-loading share."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
t0 = time.perf_counter()
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
print(f"context + torch init {time.perf_counter() - t0:.3f}s  (CUDA_MODULE_LOADING={os.environ.get('CUDA_MODULE_LOADING', 'default')})")
t0 = time.perf_counter()
from paper_2308_00106_b200 import _cuda  # noqa: E402

_cuda.require_cuda()  # sme_preload: libsme's kernel modules
print(f"require_cuda (sme_preload) {time.perf_counter() - t0:.3f}s")


def step(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3


for rep in range(3):
    A = (synth.laplacian5(2828) if cfg == "c5" else synth.rmat(24, 22, cap=1024) if cfg == "c3"
         else synth.random_rows(50_000_000, 50_000_000, 20))
    n = A.n_rows
    (p_r, p_c), t_gen = step("gen", lambda: P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))]))
    _, t_inv = step("inv", lambda: (p_r.d_inverse, p_c.d_inverse))
    B, t_k4 = step("k4", lambda: P.permute_csr(A, p_r, p_c))
    lay, t_seg = step("seg", lambda: seg_of(B, full_last=(cfg == "c5")))
    print(f"rep {rep}: generation {t_gen:.1f} ms, inverse {t_inv:.1f} ms, K4 {t_k4:.1f} ms, seg layout {t_seg:.1f} ms", flush=True)
    del A, B, lay, p_r, p_c
