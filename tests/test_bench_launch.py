"""CPU tests of bench.py's harness logic: the N-rank self-launch
and the host side of the full-scale parity check."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


@pytest.mark.parametrize("n", [2, 3])
def test_self_launch_spawns_n_ranks(n):
    """`bench.py --gpus N` without WORLD_SIZE re-executes itself under
    torch.distributed.run with N ranks (rendezvous on 127.0.0.1, gloo all_reduce)."""
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--dry-run"], capture_output=True,
                       text=True, timeout=240, env=env, cwd="/tmp")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == n and out["all_reduce_ok"] is True


def test_world_mismatch_is_an_error(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--dry-run"])
    with pytest.raises(SystemExit, match="WORLD_SIZE=2"):
        bench.main()


def test_sample_rows_shape():
    R, rows = bench.sample_rows(100_000, 2_000_000, target_nnz=200_000, n_random=500)
    assert R == 10_000 and np.array_equal(rows[:R], np.arange(R))
    assert np.all(np.diff(rows) > 0) and rows[-1] < 100_000 and rows.size > R + 400


@pytest.mark.parametrize("kind", ["random_rows", "laplacian"])
def test_oracle_sample_equals_full_oracle_permutation(kind):
    """The vectorised sample builder equals rows of the oracle's full
    coo_to_csr(permute_matrix(A, p_r, p_c)) (matio.py:281-294, permute.py:98-102)."""
    if kind == "random_rows":
        cfg = dict(kind="random_rows", n=3000, k=7, dtype="f64")
        n = cfg["n"]
        cols, vals = O.random_rows(np.arange(n), n, cfg["k"], 0x5EED_C4)
        ptr = np.arange(n + 1, dtype=np.int64) * cfg["k"]
        col, val = cols.ravel(), vals.ravel()
    else:
        cfg = dict(kind="laplacian", g=40, dtype="f64")
        n = 1600
        ptr, col, val = O.laplacian5(cfg["g"])
    fr, fc = O.random_permutation(n, 11), O.random_permutation(n, 12)
    rows_full = O.csr_to_coo_rows(ptr)
    pr, pc = O.permute_coo(rows_full, col, fr, fc)
    ptr_b, col_b, val_b = O.coo_to_csr(n, pr, pc, val)
    R, rows = bench.sample_rows(n, int(ptr[-1]), target_nnz=int(ptr[-1]) // 10, n_random=50)
    got = bench.oracle_sample(cfg, fr, fc, rows)
    want = bench.gather_rows_host(ptr_b, col_b, val_b, rows)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g), np.asarray(w))


def test_cpu_baseline_run_matches_oracle_bitwise():
    ptr, col, val = O.laplacian5(30)
    x = O.input_vector(0, 900)
    res = bench.cpu_baseline_run(ptr, col, val, x, 900, steps=1, warmup=0)
    assert np.array_equal(res["y"], O.spmv_csr(ptr, col, val, x))
    assert res["kind"] in ("reference", "port")


def test_cpu_permute_hist_baseline_runs():
    ptr, col, val = O.laplacian5(30)
    out = bench.cpu_permute_hist_baseline(dict(kind="laplacian", g=30), (ptr, col, val), 900,
                                          O.random_permutation(900, 3))
    assert out["permute_nnz_per_s"] > 0 and out["hist_nnz_per_s"] > 0 and 0 < out["entropy_bits"] <= 14
