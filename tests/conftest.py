"""Shared fixtures.  `gpu` tests need a B200 (run by the driver with -m gpu); the rest
run on CPU.  Golden vectors come from the reference itself (tests/golden/make_golden.py)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "ref_vectors.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def golden_cases(g):
    return [str(c) for c in g["cases"]]


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


def make_random_coo_arrays(rng, n_rows, n_cols, density):
    """The reference test generator (pkg/tests/conftest.py:10-16) as raw arrays."""
    total = n_rows * n_cols
    nnz = int(round(density * total))
    cells = rng.choice(total, size=nnz, replace=False)
    values = rng.random(nnz) * 2.0 - 1.0
    return cells // n_cols, cells % n_cols, values
