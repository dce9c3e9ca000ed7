"""On-disk cache of permuted CSR + seg layout (the reference
persists permuted matrices through cmd_permute -> write_matrix_market, cli.py:173-230):
the round trip is bit-exact, the layout reloads without a rebuild and computes the
same y, and the cache key separates matrices and permutations."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import cache, synth
from paper_2308_00106_b200.permute import axis_seed
from paper_2308_00106_b200.seg import seg_of

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    return torch.equal(a.d_row_ptr, b.d_row_ptr) and torch.equal(a.d_col_idx, b.d_col_idx) and torch.equal(
        a.d_values.view(torch.uint8), b.d_values.view(torch.uint8))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_round_trip_bitexact_with_layout(tmp_path, monkeypatch, dtype):
    monkeypatch.setattr(cache, "CHUNK_BYTES", 1 << 20)  # many chunks through the double buffer
    n = 300_000
    A = synth.random_rows(n, n, 12, dtype=dtype)
    p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
    B = P.permute_csr(A, p_r, p_c)
    lay = seg_of(B, 4)
    x = torch.rand(n, dtype=B.dtype, device="cuda")
    y0 = torch.empty(n, dtype=B.dtype, device="cuda")
    lay.spmv_into(x, y0)
    f = cache.save(tmp_path / "b.smecache", B, layout=lay, key="k")
    C = cache.load(f, verify=True)
    assert _bits_equal(B, C)
    lay2 = C._cache[("seg", 4, False)]
    assert torch.equal(lay2.pk, lay.pk) and torch.equal(lay2.plans, lay.plans)
    y1 = torch.empty_like(y0)
    seg_of(C, 4).spmv_into(x, y1)  # the installed layout, no rebuild
    assert seg_of(C, 4) is lay2 and torch.equal(y0, y1)
    D = cache.load(f, with_layout=False)
    assert _bits_equal(B, D) and not any(isinstance(k, tuple) for k in D._cache)


def test_permute_csr_cached_hits_and_keys(tmp_path):
    g = 600
    A = synth.laplacian5(g)
    n = g * g
    p_r, p_c = P.random_permutations([(n, axis_seed(7, 0)), (n, axis_seed(7, 1))])
    B = P.permute_csr(A, p_r, p_c)
    C1 = cache.permute_csr_cached(A, p_r, p_c, tmp_path)  # miss: computed and stored
    files = list(tmp_path.glob("permuted-*.smecache"))
    assert len(files) == 1 and _bits_equal(B, C1)
    C2 = cache.permute_csr_cached(A, p_r, p_c, tmp_path, verify=True)  # hit
    assert _bits_equal(B, C2) and len(list(tmp_path.glob("*.smecache"))) == 1
    # another permutation or another matrix -> another key
    q = P.random_permutation(n, 99)
    C3 = cache.permute_csr_cached(A, q, p_c, tmp_path)
    assert _bits_equal(C3, P.permute_csr(A, q, p_c)) and len(list(tmp_path.glob("*.smecache"))) == 2
    assert cache.matrix_key(A, p_r, p_c) != cache.matrix_key(A, q, p_c) != cache.matrix_key(A, p_c, p_r)
    x = torch.from_numpy(P.input_vector(0, n)).cuda()
    assert torch.equal(P.spmv_csr(C2, x), P.spmv_csr(B, x))


def test_hash64_is_content_and_position_sensitive():
    t = torch.arange(1000, dtype=torch.int32, device="cuda")
    h = cache.hash64(t)
    assert h == cache.hash64(t.clone())
    u = t.clone()
    u[[3, 4]] = u[[4, 3]]  # same multiset, other order
    assert cache.hash64(u) != h
    u = t.clone()
    u[999] += 1
    assert cache.hash64(u) != h and cache.hash64(t, 1) != h


def test_corrupt_file_detected(tmp_path):
    A = synth.laplacian5(100)
    f = cache.save(tmp_path / "a.smecache", A)
    head, base = cache.read_header(f)
    raw = bytearray(f.read_bytes())
    raw[base + head["arrays"]["values"]["offset"] + 5] ^= 0x40
    f.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="values does not match"):
        cache.load(f, verify=True)
