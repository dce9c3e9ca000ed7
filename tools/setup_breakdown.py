"""C4 setup kernels for an ncu launch list: K4 (permute_csr) and the seg layout build,
each run twice (the second warm)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
A = synth.random_rows(50_000_000, 50_000_000, 20) if cfg == "c4" else synth.rmat(24, 22, cap=1024)
n = A.n_rows
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("k4")
for _ in range(2):
    B = P.permute_csr(A, p_r, p_c)
    torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
del A
torch.cuda.empty_cache()
torch.cuda.nvtx.range_push("seg")
for _ in range(2):
    lay = SegLayout(B, auto_seg_panels(B))
    torch.cuda.synchronize()
    del lay
torch.cuda.nvtx.range_pop()
print("done")
