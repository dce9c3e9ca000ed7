import sys, torch
sys.path.insert(0, '.')
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth, _lib
from paper_2308_00106_b200.kernels import spmv_into, default_lanes
from paper_2308_00106_b200.iterative import VectorEpi
from paper_2308_00106_b200._cuda import ptr, stream
A = synth.laplacian5(2828); n = A.n_rows
x = torch.rand(n, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
L = default_lanes(A); ve = VectorEpi(A, L)
part = torch.zeros(ve.n_warps, dtype=torch.float64, device='cuda'); tk = torch.zeros(1, dtype=torch.int32, device='cuda'); res = torch.tensor([1.0, 0.0], dtype=torch.float64, device='cuda')
def t(f, k=200):
    for _ in range(5): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(k): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / k
print("lanes", L, "blocks", ve.n_warps)
print("vector     ", t(lambda: spmv_into(A, x, y, "vector")))
print("vector_epi ", t(lambda: ve.epi_pass(x, None, y, None, res, part, tk, res)))
print("vector_epi scale=None", t(lambda: _lib.call("sme_spmv_vector_epi", L, n, ptr(A.d_row_ptr), ptr(A.d_col_idx), ptr(A.d_values), ptr(x), ptr(y), None, None, ptr(part), ptr(tk), ptr(res), 0, stream())))
