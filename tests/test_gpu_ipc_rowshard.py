"""Multi-process power iteration with the iterate exchange fused into the SpMV
epilogue (sme_spmv_seg_epi_peers + CUDA IPC), run as 2 ranks on ONE GPU over gloo
(the stores that would cross NVLink land in the peer process's buffer on the same
device): same eigenpair as the one-GPU fused PowerIteration and the numpy oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

pytestmark = pytest.mark.gpu

G, STEPS = 40, 50


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, panels):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_00106_b200 as P
        from paper_2308_00106_b200 import synth
        from paper_2308_00106_b200.rowshard import DistributedPowerIteration

        A = synth.laplacian5(G)
        n = A.n_rows
        p = P.random_permutation(n, 3)
        x0 = O.input_vector(0, n)
        from paper_2308_00106_b200 import seg as S

        orig = S.auto_seg_panels
        S.auto_seg_panels = lambda m, *a, **k: panels  # several panels per shard
        try:
            dpi = DistributedPowerIteration(A, p, x0)
        finally:
            S.auto_seg_panels = orig
        assert dpi.lay.n_panels == panels
        dpi.run(STEPS)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), dpi.x().cpu().numpy())
        np.save(os.path.join(out_dir, f"lam{rank}.npy"), np.array([dpi.eigenvalue]))
        dpi.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("panels", [1, 2])
def test_fused_exchange_power_iteration_two_ranks(tmp_path, panels):
    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200 import synth
    from paper_2308_00106_b200.iterative import PermutedOperator, PowerIteration

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), panels), nprocs=world, join=True)
    xs = [np.load(tmp_path / f"x{r}.npy") for r in range(world)]
    lams = [float(np.load(tmp_path / f"lam{r}.npy")[0]) for r in range(world)]
    # every rank holds the same full iterate, bit for bit
    assert np.array_equal(xs[0].view(np.uint64), xs[1].view(np.uint64)) and lams[0] == lams[1]
    A = synth.laplacian5(G)
    n = A.n_rows
    op = PermutedOperator(A, P.random_permutation(n, 3), P.random_permutation(n, 3), kernel="seg")
    one = PowerIteration(op, O.input_vector(0, n), fused=True)
    one.run(STEPS)
    assert abs(lams[0] - one.eigenvalue) <= 1e-12 * one.eigenvalue
    assert O.relative_error(xs[0], one.x().cpu().numpy()) <= 1e-10
    ptr, col, val = O.laplacian5(G)
    x_ref, lam_ref = O.power_iteration(ptr, col, val, O.input_vector(0, n), STEPS)
    assert abs(lams[0] - lam_ref) <= 1e-10 * lam_ref
    assert O.relative_error(xs[0], x_ref) <= 1e-9
