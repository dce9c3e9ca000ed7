"""On-disk permuted-CSR cache (cache.py) measured at C2, C3 and C4: the miss (permute_csr +
seg layout + save), the hit (load incl. layout), the file size and rates, against rebuilding
(permutations + K4 + layout).  Files under $SME_CACHE_DIR (default /tmp/sme_cache)."""
import os
import shutil
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import cache, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

root = Path(os.environ.get("SME_CACHE_DIR", "/tmp/sme_cache"))
shutil.rmtree(root, ignore_errors=True)


def clock(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


for cfg in sys.argv[1:] or ["c2", "c3", "c4"]:
    A = (synth.laplacian5(2000) if cfg == "c2" else synth.rmat(24, 22, cap=1024) if cfg == "c3"
         else synth.random_rows(50_000_000, 50_000_000, 20))
    n = A.n_rows
    perms = lambda: P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])  # noqa: E731
    (p_r, p_c), _ = clock(perms)

    def rebuild():
        pr, pc = perms()
        B = P.permute_csr(A, pr, pc)
        seg_of(B)
        return B

    for _ in range(2):
        Bw, t_rebuild = clock(rebuild)  # warm: the steady-state cost of recomputing
    del Bw
    d = root / cfg
    _, t_miss = clock(lambda: cache.permute_csr_cached(A, p_r, p_c, d))
    f = next(d.glob("*.smecache"))
    size = f.stat().st_size
    hits = []
    for _ in range(3):
        B, t_hit = clock(lambda: cache.permute_csr_cached(A, p_r, p_c, d))
        hits.append(t_hit)
        del B
    print(f"{cfg}: file {size / 1e9:.2f} GB on {root}; miss (permute + layout + save) {t_miss:.3f} s; "
          f"hit (load + layout) {min(hits):.3f}-{max(hits):.3f} s = {size / min(hits) / 1e9:.1f} GB/s; "
          f"rebuild (permutations + K4 + layout, warm) {t_rebuild * 1e3:.1f} ms", flush=True)
    shutil.rmtree(d, ignore_errors=True)
    del A
    torch.cuda.empty_cache()
