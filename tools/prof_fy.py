"""One 50M permutation through the GPU shuffle (sme_fy_apply) for an ncu launch list."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2308_00106_b200.permute import pcg64_permutation_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
for _ in range(2):
    p = pcg64_permutation_device(np.random.PCG64(7), n)
torch.cuda.synchronize()
print("ok", int(p[0]))
