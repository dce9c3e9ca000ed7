"""Generate tests/golden/ref_vectors.npz by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference/pkg/src, which does
not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every array stored here is an output of the reference package `spmv_entropy`
(numpy 2.3.5) on seeded inputs; tests/test_oracle.py pins the CPU oracle to
these vectors and tests/test_gpu_parity.py pins the CUDA path to them.
Cases:
  c1   BASELINE config 1: make_random_coo(default_rng(0), 10000, 10000, 0.001),
       strategy ROW_COLUMN_PERMUTE seed 7, x = input_vector(0, n).
  sN   small matrices x all five strategies (ragged, empty rows, rectangular).
  long rows of length 1, 32, 33, 4096, 4097, 9000 (every sort path).
  ent  entropy known answers incl. natural base.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import spmv_entropy as se  # noqa: E402
from conftest import make_random_coo  # noqa: E402  (reference test generator)

OUT = Path(__file__).resolve().parent / "ref_vectors.npz"


def case(store: dict, name: str, m, strategy, seed: int, bins2d=None, x=None) -> None:
    p_r, p_c = se.build_strategy(m, strategy, seed, min(512, max(m.n_rows, m.n_cols)))
    perm = se.permute_matrix(m, p_r, p_c)
    csr0 = se.coo_to_csr(m)
    csr = se.coo_to_csr(perm)
    if x is None:
        x = se.bench.input_vector(0, m.n_cols)
    x_perm = se.permute_vector(x, p_c)
    y0 = se.spmv_csr(csr0, x)
    y = se.spmv_csr(csr, x_perm)
    br, bc = bins2d or (min(128, m.n_rows), min(128, m.n_cols))
    store[f"{name}/shape"] = np.array([m.n_rows, m.n_cols], dtype=np.int64)
    store[f"{name}/row"] = m.row_idx.astype(np.int32)
    store[f"{name}/col"] = m.col_idx.astype(np.int32)
    store[f"{name}/val"] = m.values
    store[f"{name}/p_r"] = p_r.forward.astype(np.int32)
    store[f"{name}/p_c"] = p_c.forward.astype(np.int32)
    store[f"{name}/perm_row"] = perm.row_idx.astype(np.int32)
    store[f"{name}/perm_col"] = perm.col_idx.astype(np.int32)
    store[f"{name}/csr0_ptr"] = csr0.row_ptr.astype(np.int32)
    store[f"{name}/csr0_col"] = csr0.col_idx.astype(np.int32)
    store[f"{name}/csr0_val"] = csr0.values
    store[f"{name}/csr_ptr"] = csr.row_ptr.astype(np.int32)
    store[f"{name}/csr_col"] = csr.col_idx.astype(np.int32)
    store[f"{name}/csr_val"] = csr.values
    store[f"{name}/x"] = x
    store[f"{name}/x_perm"] = x_perm
    store[f"{name}/y0"] = y0
    store[f"{name}/y"] = y
    store[f"{name}/y_expected"] = se.permute_vector(y0, p_r)
    store[f"{name}/bins2d"] = np.array([br, bc], dtype=np.int64)
    if perm.nnz:
        h0 = se.histogram_2d(m, br, bc)
        h = se.histogram_2d(perm, br, bc)
        store[f"{name}/hist0"] = h0.counts
        store[f"{name}/hist"] = h.counts
        store[f"{name}/H0"] = np.array(se.shannon_entropy(h0))
        store[f"{name}/H"] = np.array(se.shannon_entropy(h))
        b1r, b1c = min(512, m.n_rows), min(512, m.n_cols)
        store[f"{name}/rowhist"] = se.row_histogram(perm, b1r).counts
        store[f"{name}/colhist"] = se.col_histogram(perm, b1c).counts
    store[f"{name}/par4"] = se.spmv_csr_parallel(csr, x_perm, min(4, m.n_rows))


def main() -> None:
    store: dict[str, np.ndarray] = {}
    names = []
    S = se.StrategyKind

    # C1 (BASELINE.json configs[0])
    m = make_random_coo(np.random.default_rng(0), 10000, 10000, 0.001)
    case(store, "c1", m, S.ROW_COLUMN_PERMUTE, 7)
    names.append("c1")

    # small matrices x every strategy
    rng = np.random.default_rng(20240811)
    shapes = [(1, 1, 1.0), (3, 2, 0.5), (13, 17, 0.3), (40, 25, 0.2), (64, 64, 0.05), (200, 150, 0.02), (10, 1, 0.5)]
    k = 0
    for (nr, nc, dens) in shapes:
        for strat in se.TABLE_ORDER:
            mm = make_random_coo(rng, nr, nc, dens)
            name = f"s{k}"
            try:
                case(store, name, mm, strat, int(rng.integers(0, 2**31)))
            except ValueError:  # gradient strategies need >= 2 bins per axis
                continue
            names.append(name)
            k += 1
    # empty rows (matio KAT shape), column-major input, and an empty matrix
    for name, mm in [
        ("empty_rows", se.CooMatrix(3, 3, [0, 2], [1, 2], [5.0, 6.0])),
        ("colmajor", se.CooMatrix(2, 2, [0, 1, 0, 1], [0, 0, 1, 1], [1.0, 3.0, 2.0, 4.0])),
        ("nnz0", se.CooMatrix(3, 2, [], [], [])),
    ]:
        case(store, name, mm, S.ROW_COLUMN_PERMUTE, 11)
        names.append(name)

    # long / medium rows: every path of the segmented sort
    lengths = [1, 32, 33, 100, 4096, 4097, 9000, 0, 5]
    n_cols = 20000
    rows, cols = [], []
    r2 = np.random.default_rng(5)
    for r, L in enumerate(lengths):
        c = r2.choice(n_cols, size=L, replace=False)
        rows.append(np.full(L, r))
        cols.append(c)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    order = r2.permutation(rows.size)
    mm = se.CooMatrix(len(lengths), n_cols, rows[order], cols[order], r2.random(rows.size) * 2 - 1)
    case(store, "long", mm, S.ROW_COLUMN_PERMUTE, 3, bins2d=(3, 100))
    names.append("long")

    # entropy known answers (entropy.py:104-119 incl. base e)
    cnt = r2.integers(0, 50, size=300)
    store["ent/counts"] = cnt
    store["ent/H2"] = np.array(se.shannon_entropy(se.BinnedHistogram(cnt, (np.arange(301),))))
    store["ent/He"] = np.array(se.shannon_entropy(se.BinnedHistogram(cnt, (np.arange(301),)), base=np.e))
    store["ent/H10"] = np.array(se.shannon_entropy(se.BinnedHistogram(cnt, (np.arange(301),)), base=10.0))

    # permutation KATs (permute.py:71-81, bench.py:161-171)
    store["perm/rp_31_5"] = se.random_permutation(31, 5).forward
    store["perm/rp_1000_123"] = se.random_permutation(1000, 123).forward
    store["perm/axis_seed_7"] = np.array([se.permute._axis_seed(7, 0), se.permute._axis_seed(7, 1)], dtype=np.uint64)
    store["perm/derived_0_3"] = np.array([se.bench.derived_seed(0, 3)], dtype=np.uint64)
    store["perm/input_vector_0_17"] = se.bench.input_vector(0, 17)

    store["cases"] = np.array(names)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(names)} matrix cases)")


if __name__ == "__main__":
    main()
