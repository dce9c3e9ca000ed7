"""K4 (permute_csr) time per warp-sort level on C3 (ragged R-MAT rows), and the seg
layout build time on C4 and C3 (CUDA events, warm)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import _lib, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
        del r
    return statistics.median(out)


for cfg in sys.argv[1:] or ["c3", "c4"]:
    A = synth.rmat(24, 22, cap=1024) if cfg == "c3" else synth.random_rows(50_000_000, 50_000_000, 20)
    n = A.n_rows
    p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
    ref = P.permute_csr(A, p_r, p_c)
    levels = (0, 1, 2, 3, 4) if cfg == "c3" else (4,)
    for lv in levels:
        _lib.call("sme_sort_rows_set_wmed", lv)
        B = P.permute_csr(A, p_r, p_c)
        same = torch.equal(B.d_col_idx, ref.d_col_idx) and torch.equal(B.d_values, ref.d_values)
        del B
        print(f"{cfg} K4 wmed level {lv}: {timed(lambda: P.permute_csr(A, p_r, p_c)):.2f} ms  identical {same}",
              flush=True)
    _lib.call("sme_sort_rows_set_wmed", 4)
    del A
    torch.cuda.empty_cache()
    Pn = auto_seg_panels(ref)
    print(f"{cfg} seg layout build ({Pn} panels): {timed(lambda: SegLayout(ref, Pn)):.2f} ms", flush=True)
    del ref
    torch.cuda.empty_cache()
