timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or hist or c2_scale or reference_kats" 2>&1 | tail -2
timeout 600 python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
for name, A in (("c2", synth.laplacian5(2000)), ("c4", synth.random_rows(50_000_000, 50_000_000, 20))):
    for perm in (False, True):
        M = A
        if perm:
            n = A.n_rows
            M = P.permute_csr(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
        P.histogram_2d(M, 128, 128); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): h = P.histogram_2d(M, 128, 128)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(name, "perm" if perm else "unperm", f"{ms:.3f} ms", f"{M.nnz*4/ms/1e6:.0f} GB/s", h.total == M.nnz, flush=True)
PY
