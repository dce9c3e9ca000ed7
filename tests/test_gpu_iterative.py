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


@pytest.mark.parametrize("kernel", ["auto", "stream", "merge"])
def test_power_iteration_rc_permuted_matches_oracle(kernel):
    g = 20
    A = synth.laplacian5(g)
    n = A.n_rows
    p_r, p_c = P.random_permutation(n, 3), P.random_permutation(n, 4)  # independent (ROW_COLUMN_PERMUTE)
    op = PermutedOperator(A, p_r, p_c, kernel=kernel)
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
        ConjugateGradient(PermutedOperator(A, p, P.random_permutation(n, 10)), b)
