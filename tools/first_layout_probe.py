"""The first seg layout of a process (C5 iterative operator), under the torch profiler
(CPU ops and CUDA runtime calls): what the first-use overhead is made of."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.iterative import PermutedOperator
from paper_2308_00106_b200.permute import axis_seed

A = synth.laplacian5(2828)
n = A.n_rows
torch.cuda.Stream()
p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU]) as prof:
    op = PermutedOperator(A, p_r, p_c)
    torch.cuda.synchronize()
print("== PermutedOperator (first K4)")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
with profile(activities=[ProfilerActivity.CPU]) as prof:
    op.fused_layout()
    torch.cuda.synchronize()
print("== fused_layout (first seg layout)")
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=18))
