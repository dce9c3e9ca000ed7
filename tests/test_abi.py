"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/*.h declares; the product path fails loudly without CUDA."""

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2308_00106_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADERS = sorted((ROOT / "include").glob("*.h"))


def declared_symbols() -> set[str]:
    names = set()
    for h in HEADERS:
        for m in re.finditer(r"^\s*(?:const\s+char\s*\*|int)\s+(sme_\w+)\s*\(", h.read_text(), re.M):
            names.add(m.group(1))
    return names


def test_library_is_built_for_sm100a():
    lib = _lib.LIB_PATH
    assert lib.exists(), "run __graft_entry__.build() first"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_every_declared_symbol_is_exported_and_bound():
    decl = declared_symbols()
    assert len(decl) >= 30
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(sme_\w+)\b", nm))
    assert decl <= exported, f"declared but not exported: {sorted(decl - exported)}"
    assert decl <= set(_lib.SIGNATURES), f"declared but not bound: {sorted(decl - set(_lib.SIGNATURES))}"
    lib = _lib.load()
    for name in decl:
        assert hasattr(lib, name)


def test_library_reports_version_and_errors_without_gpu():
    lib = _lib.load()
    assert lib.sme_version() == 1
    # argument validation happens before any CUDA call
    with pytest.raises(ValueError, match="bin count"):
        _lib.call("sme_hist2d_csr", 10, 10, 5, None, None, 0, 4, None, None)
    with pytest.raises(ValueError, match="lanes"):
        _lib.call("sme_spmv_vector", 0, 3, 10, 10, None, None, None, None, None, 0, None)
    assert "lanes" in _lib.last_error()


def test_workspace_queries():
    assert _lib.query_size("sme_permute_csr_workspace_size", 1000, 5000, 0) > 1000 * 4
    assert _lib.query_size("sme_coo_to_csr_workspace_size", 1000, 5000, 10000) > 5000 * 12 + 10000 * 16
    assert _lib.query_i64("sme_spmv_merge_tiles", 10000, 100000) == -(-110000 // 2048)


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2308_00106_b200 as pkg

    with pytest.raises(RuntimeError, match="CUDA"):
        pkg.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 2.0])
    with pytest.raises(RuntimeError, match="CUDA"):
        pkg.Permutation([1, 0])


def _fastdiv(d: int):
    l = 0
    while (1 << l) < d:
        l += 1
    s = 32 + l
    m = -(-(1 << s) // d)
    return m, s


def test_fastdiv_magic_is_exact():
    """common.cuh make_fastdiv: q = (n * m) >> s == n // d for 0 <= n < 2^31, and n*m < 2^64."""
    rng = np.random.default_rng(1)
    divisors = [1, 2, 3, 7, 78, 128, 1000, 2**20 + 1, 2**30, 2**31 - 1] + rng.integers(1, 2**31 - 1, 50).tolist()
    for d in divisors:
        m, s = _fastdiv(int(d))
        ns = [0, 1, d - 1, d, d + 1, 2**31 - 1, 2**31 - 2] + rng.integers(0, 2**31 - 1, 200).tolist()
        for n in ns:
            if n < 0:
                continue
            assert n * m < 2**64
            assert (n * m) >> s == n // d, (n, d)
