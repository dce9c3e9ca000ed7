"""C3 fidelity: nnz of R-MAT scale 24 after dedupe + degree cap 1024 for several edge
factors (BASELINE configs[2] asks for ~256M nnz)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2308_00106_b200 import synth
for ef in (16, 20, 21, 22, 23, 24):
    A = synth.rmat(24, ef, cap=1024, dtype=np.float32)
    mx = int((A.d_row_ptr[1:] - A.d_row_ptr[:-1]).max())
    print(f"ef={ef} nnz={A.nnz:,} max_row={mx}", flush=True)
    del A
    torch.cuda.empty_cache()
