"""C3 R-MAT construction (edges -> dedupe -> degree cap -> values) vs the numpy oracle,
and the SpMV kernels on its power-law rows."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,cap", [(10, 1024), (12, 48)])
def test_rmat_matches_oracle(scale, cap):
    m = synth.rmat(scale, 16, seed=123, cap=cap)
    ptr, col, val = O.rmat_csr(scale, 16, *synth.RMAT_ABC, 123, cap)
    assert np.array_equal(m.row_ptr, ptr)
    assert np.array_equal(m.col_idx, col)
    assert m.dtype == torch.float32
    assert np.array_equal(m.d_values.cpu().numpy(), val.astype(np.float32))
    # power law: the heaviest rows hit the cap, many rows are empty
    lens = np.diff(ptr)
    assert lens.max() == min(cap, lens.max()) and (lens == 0).sum() > 0


def test_rmat_spmv_kernels_f32():
    m = synth.rmat(14, 16, seed=7, cap=1024)
    x = torch.from_numpy(O.input_vector(0, m.n_cols).astype(np.float32)).cuda()
    ptr, col, val = m.row_ptr, m.col_idx, m.values
    want = O.spmv_csr(ptr, col, val, x.double().cpu().numpy())
    for kernel in ("merge", "stream", "vector"):
        y = P.spmv_csr(m, x, kernel)
        assert O.relative_error(y.double().cpu().numpy(), want) <= 1e-5, kernel
    # permuted (row+col) round trip at the f32 bar
    n = m.n_rows
    p_r, p_c = P.random_permutation(n, 1), P.random_permutation(n, 2)
    B = P.permute_csr(m, p_r, p_c)
    yb = P.spmv_csr(B, P.permute_vector(x, p_c), "merge")
    assert O.relative_error(yb.double().cpu().numpy(),
                            P.permute_vector(torch.from_numpy(want).cuda(), p_r).cpu().numpy()) <= 1e-5
