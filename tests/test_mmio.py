"""Matrix Market I/O: the native parser / writer (mmio_host.cpp) against golden
cases produced by the REAL reference parser (tests/golden/make_mm_golden.py), a
large multithreaded parse, and the device CooMatrix path (gpu)."""

import io
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2308_00106_b200.mmio import MatrixMarketError, format_entries, parse_host_arrays

CASES = json.loads((Path(__file__).parent / "golden" / "mm_cases.json").read_text())
HOST_CASES = sorted(k for k, v in CASES.items() if not v.get("needs_gpu"))


def _src(case):
    data = case["input"].encode()
    return data, case["kind"] == "bytes"


@pytest.mark.parametrize("name", HOST_CASES)
@pytest.mark.parametrize("threads", [1, 4])
def test_parse_matches_reference_golden(name, threads):
    case = CASES[name]
    data, universal = _src(case)
    if "error" in case:
        with pytest.raises(MatrixMarketError) as ei:
            parse_host_arrays(data, universal, threads)
        assert str(ei.value) == case["error"] and ei.value.line_no == case["line_no"]
        return
    n_rows, n_cols, rows, cols, vals = parse_host_arrays(data, universal, threads)
    assert (n_rows, n_cols) == (case["n_rows"], case["n_cols"])
    assert rows.tolist() == case["rows"] and cols.tolist() == case["cols"]
    assert [float(v).hex() for v in vals] == case["vals"]


def _random_body(rng, n, n_rows, n_cols, crlf=False):
    r = rng.integers(1, n_rows + 1, n)
    c = rng.integers(1, n_cols + 1, n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n)
    nl = "\r\n" if crlf else "\n"
    lines = [f"{a} {b} {x!r}" for a, b, x in zip(r.tolist(), c.tolist(), v.tolist())]
    # sprinkle comments and blank lines
    for k in range(0, n, 997):
        lines.insert(k, "% comment" if k % 2 else "   ")
    text = f"%%MatrixMarket matrix coordinate real general{nl}{n_rows} {n_cols} {n}{nl}" + nl.join(lines) + nl
    return text.encode(), r - 1, c - 1, v


@pytest.mark.parametrize("crlf", [False, True])
def test_large_parse_is_exact_and_thread_invariant(crlf):
    rng = np.random.default_rng(11)
    data, r, c, v = _random_body(rng, 300_000, 70_000, 90_000, crlf)
    for threads in (1, 3, 8):
        n_rows, n_cols, rows, cols, vals = parse_host_arrays(data, True, threads)
        assert (n_rows, n_cols) == (70_000, 90_000)
        assert np.array_equal(rows, r) and np.array_equal(cols, c)
        assert np.array_equal(vals.view(np.uint64), v.view(np.uint64))


def test_large_parse_first_error_wins_across_threads():
    rng = np.random.default_rng(12)
    data, *_ = _random_body(rng, 200_000, 1000, 1000)
    lines = data.split(b"\n")
    lines[150_000] = b"5 5000 1.0"  # column out of range, late
    lines[90_000] = b"1 1 nope"  # malformed value, earlier: this one must be reported
    bad = b"\n".join(lines)
    for threads in (1, 8):
        with pytest.raises(MatrixMarketError) as ei:
            parse_host_arrays(bad, True, threads)
        assert ei.value.line_no == 90_001 and "malformed value: 'nope'" in str(ei.value)


def test_format_entries_matches_python_formatting():
    rng = np.random.default_rng(5)
    n = 20_000
    r = rng.integers(0, 10**9, n)
    c = rng.integers(0, 10**9, n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    v[:8] = [0.1, -0.0, 0.0, np.inf, -np.inf, np.nan, 5e-324, 1.7976931348623157e308]
    want = "".join(f"{i + 1} {j + 1} {x:.17g}\n" for i, j, x in zip(r.tolist(), c.tolist(), v.tolist())).encode()
    for threads in (1, 6):
        assert format_entries(r, c, v, threads) == want


def test_format_then_parse_roundtrip_bits():
    rng = np.random.default_rng(6)
    n = 50_000
    r, c = rng.integers(0, 5000, n), rng.integers(0, 7000, n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-200, 200, n)
    text = f"%%MatrixMarket matrix coordinate real general\n5000 7000 {n}\n".encode() + format_entries(r, c, v)
    _, _, rows, cols, vals = parse_host_arrays(text, True, 4)
    assert np.array_equal(rows, r) and np.array_equal(cols, c)
    assert np.array_equal(vals.view(np.uint64), v.view(np.uint64))


# ---------------------------------------------------------------------------- device
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dup", "dup_symmetric"])
def test_duplicate_entries_raise_reference_error(name):
    from paper_2308_00106_b200 import parse_matrix_market

    with pytest.raises(MatrixMarketError, match="duplicate") as ei:
        parse_matrix_market(CASES[name]["input"])
    assert str(ei.value) == CASES[name]["error"]


@pytest.mark.gpu
def test_parse_write_parse_on_device(tmp_path):
    from paper_2308_00106_b200 import load_matrix_market, parse_matrix_market, write_matrix_market

    m = parse_matrix_market(CASES["symmetric"]["input"])
    assert m.row_idx.tolist() == CASES["symmetric"]["rows"]
    buf = io.StringIO()
    write_matrix_market(m, buf)
    again = parse_matrix_market(buf.getvalue())
    assert again == m
    p = tmp_path / "m.mtx"
    write_matrix_market(m, p)
    assert load_matrix_market(p) == m
    m0 = parse_matrix_market(CASES["empty_body"]["input"])
    out = io.StringIO()
    write_matrix_market(m0, out)
    assert out.getvalue() == "%%MatrixMarket matrix coordinate real general\n3 4 0\n"
