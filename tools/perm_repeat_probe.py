"""Repeated ROW_COLUMN permutation pairs (seed 7 axes) at a size: wall time per call with
device syncs, to see the run-to-run spread of the generation (host partners + GPU)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200.permute import axis_seed

n = int(sys.argv[1]) if len(sys.argv) > 1 else 7_997_584
torch.cuda.Stream()
times = []
for rep in range(12):
    torch.cuda.synchronize()
    t = time.perf_counter()
    p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t) * 1e3)
    del p_r, p_c
print(f"n={n}: " + " ".join(f"{t:.1f}" for t in times) + " ms", flush=True)
