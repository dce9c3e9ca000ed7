"""World-size-2 gloo run of the row-sharded SpMV's host logic on CPU: the shard
plan, the padded x all-gather and the column remap reproduce the unsharded
SpMV bitwise (the local SpMV here is the oracle; on GPUs it is libsme)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2308_00106_b200.rowshard import ShardPlan, allgather_padded, pipelined_exchange


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, ptr, col, val, x, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = ptr.size - 1
        plan = ShardPlan(n, n, world)
        lo, hi = plan.row_range(rank)
        c0, c1 = plan.col_range(rank)
        # this rank's x slice, padded, all-gathered over gloo
        chunk = plan.pad_slice(torch.from_numpy(x[c0:c1].copy()))
        x_full = torch.zeros(world * plan.pad, dtype=torch.float64)
        allgather_padded(x_full, chunk)
        assert torch.equal(plan.unpad(x_full), torch.from_numpy(x))
        # the pipelined exchange of the seg shards: in-order per-slot broadcasts;
        # when slot k is reported in place it already holds rank k's chunk
        x_pipe = torch.full((world * plan.pad,), float("nan"), dtype=torch.float64)
        seen = []

        def on_slot(k):
            assert torch.equal(x_pipe[k * plan.pad : (k + 1) * plan.pad], x_full[k * plan.pad : (k + 1) * plan.pad])
            seen.append(k)

        pipelined_exchange(x_pipe, chunk, rank, world, on_slot)
        assert seen == list(range(world)) and torch.equal(x_pipe, x_full)
        # local shard with columns remapped into the padded vector
        p0, p1 = ptr[lo], ptr[hi]
        lptr = ptr[lo : hi + 1] - p0
        lcol = plan.slot_of(col[p0:p1])
        y_local = O.spmv_csr(lptr, lcol, val[p0:p1], x_full.numpy())
        np.save(os.path.join(out_dir, f"y{rank}.npy"), y_local)
    finally:
        dist.destroy_process_group()


def test_rowshard_world2_gloo(tmp_path):
    rng = np.random.default_rng(3)
    n = 301
    dens = rng.random((n, n)) < 0.03
    rows, cols = np.nonzero(dens)
    vals = rng.random(rows.size) * 2 - 1
    ptr, col, val = O.coo_to_csr(n, rows, cols, vals)
    x = rng.random(n)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), ptr, col, val, x, str(tmp_path)), nprocs=world, join=True)
    y = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    assert np.array_equal(y.view(np.uint64), O.spmv_csr(ptr, col, val, x).view(np.uint64))


def test_rowshard_world3_gloo_pipelined(tmp_path):
    rng = np.random.default_rng(4)
    n = 250
    dens = rng.random((n, n)) < 0.04
    rows, cols = np.nonzero(dens)
    vals = rng.random(rows.size) * 2 - 1
    ptr, col, val = O.coo_to_csr(n, rows, cols, vals)
    x = rng.random(n)
    world = 3
    mp.spawn(_worker, args=(world, _free_port(), ptr, col, val, x, str(tmp_path)), nprocs=world, join=True)
    y = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    assert np.array_equal(y.view(np.uint64), O.spmv_csr(ptr, col, val, x).view(np.uint64))
