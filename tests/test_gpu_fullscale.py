"""Full-scale parity: whole bench-sized matrices against the oracle,
and the sharded multi-GPU setup (each rank builds only its rows) against the 1-GPU build.

Bars: permuted CSR bit-exact (row_ptr, col_idx, value bits) against the oracle's
coo_to_csr(permute_matrix(A, p_r, p_c)) (matio.py:281-294, permute.py:98-102);
SpMV normwise relative error <= 1e-12 (kernels.py:131-142, bench.py:34).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import rowshard, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _perms(n):
    return P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])


def test_c2_full_scale_bitexact_and_spmv():
    """C2 (4M rows, 19,992,000 nnz) in full: GPU perms == numpy, the whole permuted CSR
    == the oracle's, and y (auto kernel and seg with 8 panels) within 1e-12 of the
    oracle's reduceat SpMV on every row."""
    g = 2000
    n = g * g
    A = synth.laplacian5(g)
    p_r, p_c = _perms(n)
    fr, fc = O.random_permutation(n, axis_seed(7, 0)), O.random_permutation(n, axis_seed(7, 1))
    assert np.array_equal(p_r.forward, fr) and np.array_equal(p_c.forward, fc)
    B = P.permute_csr(A, p_r, p_c)
    ptr0, col0, val0 = O.laplacian5(g)
    pr, pc = O.permute_coo(O.csr_to_coo_rows(ptr0), col0, fr, fc)
    ptr_o, col_o, val_o = O.coo_to_csr(n, pr, pc, val0)
    assert np.array_equal(B.row_ptr, ptr_o)
    assert np.array_equal(B.col_idx, col_o)
    assert np.array_equal(B.values.view(np.uint64), val_o.view(np.uint64))
    x = O.permute_vector(O.input_vector(0, n), fc)
    y_o = O.spmv_csr(ptr_o, col_o, val_o, x)
    xd = torch.from_numpy(x).cuda()
    assert O.relative_error(P.spmv_csr(B, xd).cpu().numpy(), y_o) <= TOL
    y8 = torch.empty(n, dtype=torch.float64, device="cuda")
    seg_of(B, 8).spmv_into(xd, y8)
    assert O.relative_error(y8.cpu().numpy(), y_o) <= TOL


def test_random_10m_rows_seg8_sampled_bitexact_full_y():
    """A 10M-row C4-shaped matrix (8 random columns per row, 80M nnz) through seg with
    8 panels: 20,000 sampled permuted rows bit-exact against the oracle's restatement
    (bench.oracle_sample), and y on every row within 1e-12 of the oracle SpMV."""
    n, k = 10_000_000, 8
    cfg = dict(kind="random_rows", n=n, k=k, dtype="f64")
    A = synth.random_rows(n, n, k)
    p_r, p_c = _perms(n)
    fr, fc = p_r.forward, p_c.forward  # pinned == numpy by test_c2_* / test_gpu_shuffle
    B = P.permute_csr(A, p_r, p_c)
    R, rows = bench.sample_rows(n, n * k, seed=5, target_nnz=80_000, n_random=10_000)
    got = bench.device_rows(B, rows)
    want = bench.oracle_sample(cfg, fr, fc, rows)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    assert np.array_equal(got[2].view(np.uint64), want[2].view(np.uint64))
    x = O.permute_vector(O.input_vector(0, n), fc)
    xd = torch.from_numpy(x).cuda()
    lay = seg_of(B, 8)
    assert lay.n_panels == 8
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    lay.spmv_into(xd, y)
    y_o = O.spmv_csr(B.row_ptr, B.col_idx, B.values, x)  # the oracle SpMV over the (sample-verified) CSR
    assert O.relative_error(y.cpu().numpy(), y_o) <= TOL
    # and on the sampled rows against the fully oracle-built rows
    y_s = O.spmv_csr(want[0], want[1], want[2], x)
    assert O.relative_error(y.cpu().numpy()[rows], y_s) <= TOL


def test_random_rows_select_equals_rows_of_full_generator():
    n, k = 200_000, 20
    A = synth.random_rows(n, n, k)
    rows = torch.from_numpy(np.random.default_rng(1).permutation(n)[:5000].astype(np.int32)).cuda()
    S = synth.random_rows_select(rows, n, k)
    got = bench.device_rows(S, np.arange(5000))
    want = bench.device_rows(A, rows.cpu().numpy().astype(np.int64))
    for a, b in zip(got, want):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("kind,world", [("random_rows", 4), ("laplacian", 3)])
def test_sharded_setup_equals_rows_of_full_build(kind, world):
    """bench.build_shard (rank k builds only rows inverse(p_r)[lo:hi] and runs K4 on
    them) == rows [lo, hi) of the 1-GPU permute_csr(A, p_r, p_c), bit for bit, and the
    shard's seg SpMV equals those rows of the full SpMV bitwise."""
    cfg = (dict(kind="random_rows", n=1_000_000, k=20, dtype="f64") if kind == "random_rows"
           else dict(kind="laplacian", g=700, dtype="f64"))
    A = bench.build_matrix(cfg)
    n = A.n_rows
    p_r, p_c = _perms(n)
    B = P.permute_csr(A, p_r, p_c)
    plan = rowshard.ShardPlan(n, n, world)
    x = P.permute_vector(torch.from_numpy(P.input_vector(0, n)).cuda(), p_c)
    for rank in range(world):
        lo, hi = plan.row_range(rank)
        B_loc, _, _ = bench.build_shard(cfg, plan, rank, p_r, p_c)
        got = bench.device_rows(B_loc, np.arange(hi - lo))
        want = bench.device_rows(B, np.arange(lo, hi))
        for a, b in zip(got, want):
            assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
        sh = rowshard.RowShardedSpMV(B_loc, plan, rank, "vector", lanes=P.kernels.default_lanes(B), local=True)
        xf = torch.zeros(plan.world * plan.pad, dtype=torch.float64, device="cuda")
        for k in range(world):
            c0, c1 = plan.col_range(k)
            xf[k * plan.pad: k * plan.pad + c1 - c0] = x[c0:c1]
        y_loc = sh.spmv(xf)
        y_full = P.spmv_csr(B, x, "vector")
        assert torch.equal(y_loc, y_full[lo:hi])
