"""C5 iterative drivers on the permuted matrix vs the numpy oracle loops."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.iterative import ConjugateGradient, PermutedOperator, PowerIteration

pytestmark = pytest.mark.gpu


def bits(t):
    return t.detach().cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("fold", [True, False])
@pytest.mark.parametrize("kernel", ["auto", "stream", "merge"])
def test_power_iteration_rc_permuted_matches_oracle(kernel, fold):
    g = 20
    A = synth.laplacian5(g)
    n = A.n_rows
    p_r, p_c = P.random_permutation(n, 3), P.random_permutation(n, 4)  # independent (ROW_COLUMN_PERMUTE)
    op = PermutedOperator(A, p_r, p_c, kernel=kernel, fold=fold)
    assert op.folded == fold and (op.q is None) == fold
    x0 = O.input_vector(0, n)
    pi = PowerIteration(op, x0)
    pi.run(60)
    ptr, col, val = O.laplacian5(g)
    x_ref, lam_ref = O.power_iteration(ptr, col, val, x0, 60)
    assert abs(pi.eigenvalue - lam_ref) <= 1e-10 * lam_ref
    assert O.relative_error(pi.x().cpu().numpy(), x_ref) <= 1e-9


def test_power_iteration_graph_replay_is_bitwise_eager():
    A = synth.laplacian5(64)
    n = A.n_rows
    op = PermutedOperator(A, P.random_permutation(n, 1), P.random_permutation(n, 2))
    x0 = O.input_vector(5, n)
    eager = PowerIteration(op, x0)
    eager.run(41)
    graphed = PowerIteration(op, x0)
    graphed.capture(10)  # one eager warm-up step + a 10-step graph
    graphed.run(40)
    torch.cuda.synchronize()
    assert np.array_equal(bits(eager.z), bits(graphed.z))


def test_cg_symmetric_permutation_matches_oracle():
    g = 30
    A = synth.laplacian5(g)
    n = A.n_rows
    p = P.random_permutation(n, 9)
    op = PermutedOperator(A, p, p)  # B = P A P^T stays SPD
    b = O.input_vector(1, n)
    cg = ConjugateGradient(op, b)
    cg.capture(5)
    cg.run(200)
    ptr, col, val = O.laplacian5(g)
    x_ref, rr_ref = O.conjugate_gradient(ptr, col, val, b, 201)
    x = cg.solution().cpu().numpy()
    assert O.relative_error(x, x_ref) <= 1e-8
    # the solution solves A x = b
    assert O.relative_error(O.spmv_csr(ptr, col, val, x), b) <= 1e-6
    with pytest.raises(ValueError, match="symmetric"):
        ConjugateGradient(PermutedOperator(A, p, P.random_permutation(n, 10), fold=False), b)
    # a ROW_COLUMN pair folds into the symmetric permutation by p_r: CG applies
    cg2 = ConjugateGradient(PermutedOperator(A, p, P.random_permutation(n, 10)), b)
    cg2.run(201)
    assert O.relative_error(cg2.solution().cpu().numpy(), x_ref) <= 1e-8


def _seg_op(A, p_r, p_c, panels, fold=True):
    op = PermutedOperator(A, p_r, p_c, kernel="seg", fold=fold)
    op.B._cache["seg_panels"] = panels
    return op


@pytest.mark.parametrize("panels", [1, 3])
@pytest.mark.parametrize("perm", ["rc", "rc_unfolded", "symmetric", "none"])
def test_fused_power_iteration_matches_oracle(panels, perm):
    """sme_spmv_seg_epi: SpMV + scatter into permuted coordinates + deterministic
    norm in one launch; same eigenpair as the numpy loop over spmv_csr."""
    g = 24
    A = synth.laplacian5(g)
    n = A.n_rows
    if perm.startswith("rc"):
        p_r, p_c = P.random_permutation(n, 3), P.random_permutation(n, 4)
    elif perm == "symmetric":
        p_r = p_c = P.random_permutation(n, 5)
    else:
        p_r = p_c = None
    op = _seg_op(A, p_r, p_c, panels, fold=perm != "rc_unfolded")
    assert (op.q is not None) == (perm == "rc_unfolded")
    x0 = O.input_vector(0, n)
    pi = PowerIteration(op, x0, fused=True)
    assert pi.fused and pi.lay.n_panels == panels
    pi.run(60)
    ptr, col, val = O.laplacian5(g)
    x_ref, lam_ref = O.power_iteration(ptr, col, val, x0, 60)
    assert abs(pi.eigenvalue - lam_ref) <= 1e-10 * lam_ref
    assert O.relative_error(pi.x().cpu().numpy(), x_ref) <= 1e-9
    unfused = PowerIteration(op, x0, fused=False)
    unfused.run(60)
    assert abs(pi.eigenvalue - unfused.eigenvalue) <= 1e-12 * lam_ref


def test_fused_power_iteration_graph_is_bitwise_eager_and_deterministic():
    A = synth.random_rows(20_000, 20_000, 7, seed=3) if hasattr(synth, "random_rows") else synth.laplacian5(140)
    n = A.n_rows
    op = _seg_op(A, P.random_permutation(n, 1), P.random_permutation(n, 2), 2)
    x0 = O.input_vector(5, n)
    eager = PowerIteration(op, x0, fused=True)
    eager.run(41)
    graphed = PowerIteration(op, x0, fused=True)
    graphed.capture(10)  # one eager warm-up step + a 10-step graph
    graphed.run(40)
    again = PowerIteration(op, x0, fused=True)
    again.run(41)
    torch.cuda.synchronize()
    assert np.array_equal(bits(eager.x()), bits(graphed.x()))
    assert np.array_equal(bits(eager.x()), bits(again.x()))
    assert eager.eigenvalue == graphed.eigenvalue == again.eigenvalue
    with pytest.raises(ValueError, match="even"):
        PowerIteration(op, x0, fused=True).capture(3)


@pytest.mark.parametrize("panels", [1, 3])
def test_fused_cg_matches_oracle_and_unfused(panels):
    """sme_spmv_seg_epi_cg: p.Ap and alpha from the SpMV's last pass."""
    g = 30
    A = synth.laplacian5(g)
    n = A.n_rows
    p = P.random_permutation(n, 9)
    op = _seg_op(A, p, P.random_permutation(n, 11), panels)  # folded: symmetric by p
    b = O.input_vector(1, n)
    fused = ConjugateGradient(op, b, fused=True)
    assert fused.fused and fused.lay.n_panels == panels
    fused.capture(6)
    fused.run(198)
    unfused = ConjugateGradient(op, b, fused=False)
    unfused.run(199)
    ptr, col, val = O.laplacian5(g)
    x_ref, rr_ref = O.conjugate_gradient(ptr, col, val, b, 201)
    x = fused.solution().cpu().numpy()
    assert O.relative_error(x, x_ref) <= 1e-8
    assert O.relative_error(x, unfused.solution().cpu().numpy()) <= 1e-10
    assert O.relative_error(O.spmv_csr(ptr, col, val, x), b) <= 1e-6


@pytest.mark.parametrize("perm", ["none", "symmetric"])
def test_fused_vector_epilogue_power_and_cg(perm):
    """sme_spmv_vector_epi: the CSR-vector operator (banded / unpermuted) fused like seg."""
    g = 26
    A = synth.laplacian5(g)
    n = A.n_rows
    p = P.random_permutation(n, 4) if perm == "symmetric" else None
    op = PermutedOperator(A, p, p, kernel="vector")
    x0 = O.input_vector(0, n)
    pi = PowerIteration(op, x0, fused=True)
    assert pi.fused and pi.lay.n_panels == 1
    pi.capture(10)  # one eager step + a 10-step graph
    pi.run(50)
    ptr, col, val = O.laplacian5(g)
    x_ref, lam_ref = O.power_iteration(ptr, col, val, x0, 51)
    assert abs(pi.eigenvalue - lam_ref) <= 1e-10 * lam_ref
    assert O.relative_error(pi.x().cpu().numpy(), x_ref) <= 1e-9
    b = O.input_vector(1, n)
    cg = ConjugateGradient(op, b, fused=True)
    assert cg.fused
    cg.run(150)
    x_cg, _ = O.conjugate_gradient(ptr, col, val, b, 151)
    assert O.relative_error(cg.solution().cpu().numpy(), x_cg) <= 1e-8


def _hub_spd(n=3000):
    """SPD: 1-D Laplacian plus a hub (row/column 0 coupled to every node), diagonally dominant."""
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in (i - 1, i + 1):
            if 0 <= j < n:
                rows.append(i); cols.append(j); vals.append(-1.0)
    for j in range(2, n):  # hub couplings (0, j) and (j, 0), skipping the existing (0, 1)
        rows += [0, j]; cols += [j, 0]; vals += [-0.01, -0.01]
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals)
    diag = np.zeros(n)
    np.add.at(diag, rows, np.abs(vals))
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.arange(n)])
    vals = np.concatenate([vals, diag + 1.0])
    return O.coo_to_csr(n, rows, cols, vals)


def test_fused_iterations_on_split_row_layouts():
    """A dominant (hub) row makes the seg layout split rows; the fused power iteration and CG
    then run their epilogue as a row pass (sme_rows_epi) and still match the oracle."""
    ptr, col, val = _hub_spd()
    n = ptr.size - 1
    A = P.CsrMatrix(n, n, ptr, col, val)
    p = P.random_permutation(n, 21)
    op = PermutedOperator(A, p, p, kernel="seg")
    x0 = O.input_vector(0, n)
    pi = PowerIteration(op, x0, fused=True)
    assert pi.fused and pi.lay.split_rows
    pi.run(40)
    x_ref, lam_ref = O.power_iteration(ptr, col, val, x0, 40)
    assert abs(pi.eigenvalue - lam_ref) <= 1e-10 * lam_ref
    assert O.relative_error(pi.x().cpu().numpy(), x_ref) <= 1e-9
    b = O.input_vector(1, n)
    cg = ConjugateGradient(op, b, fused=True)
    cg.run(60)
    x_cg, _ = O.conjugate_gradient(ptr, col, val, b, 61)
    assert O.relative_error(cg.solution().cpu().numpy(), x_cg) <= 1e-8
