"""Golden Matrix Market cases from the REAL reference parser (run in the build
container, where /root/reference exists): writes tests/golden/mm_cases.json with,
per case, the input (str or bytes), and either the parsed triplets (values as
float.hex for bit-exactness) or the MatrixMarketError message.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mm_golden.py
"""

import io
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402
from spmv_entropy.matio import MatrixMarketError, parse_matrix_market  # noqa: E402

H = "%%MatrixMarket matrix coordinate "
CASES = {
    # reference test_matio.py inputs
    "identity": H + "real general\n2 2 2\n1 1 1.0\n2 2 1.0\n",
    "comments_blank": H + "real general\n% a comment\n\n2 2 2\n% inside\n1 1 1.0\n\n   \n2 2 1.0\n",
    "symmetric": H + "real symmetric\n3 3 4\n1 1 1.0\n2 1 2.0\n3 3 3.0\n3 2 4.5\n",
    "pattern": H + "pattern general\n3 2 3\n1 1\n2 2\n3 1\n",
    "integer": H + "integer general\n2 2 3\n1 1 3\n2 1 -7\n2 2 +12\n",
    "integer_big": H + "integer general\n1 3 3\n1 1 123456789012345678901234567890\n1 2 -0\n1 3 9007199254740993\n",
    "real_forms": H + "real general\n1 9 9\n1 1 .5\n1 2 5.\n1 3 -1e-3\n1 4 +2.5E+10\n1 5 0.1\n"
                      "1 6 1e-310\n1 7 1.7976931348623157e308\n1 8 -0.0\n1 9 3.141592653589793238462643\n",
    "real_inf": H + "real general\n1 3 3\n1 1 inf\n1 2 -Infinity\n1 3 1e400\n",
    "whitespace": H + "real general\n2 2 2\n\t1\t1   1.5  \n  2 2\t\t-2.25\n",
    "case_banner": "%%matrixmarket MATRIX Coordinate REAL General\n1 1 1\n1 1 7\n",
    "empty_body": H + "real general\n3 4 0\n",
    "size_last_no_newline": H + "real general\n3 4 0",
    "no_final_newline": H + "real general\n2 2 2\n1 1 1.0\n2 2 1.0",
    "column_major": H + "real general\n3 3 4\n1 1 1\n2 1 2\n3 2 3\n1 3 4\n",
    # errors (test_matio.py:64-100 and more)
    "err_complex": H + "complex general\n1 1 1\n1 1 1 0\n",
    "err_array": "%%MatrixMarket matrix array real general\n2 2\n1.0\n",
    "err_hermitian": H + "real hermitian\n1 1 1\n1 1 1\n",
    "err_skew": H + "real skew-symmetric\n1 1 1\n1 1 1\n",
    "err_banner": "%%NotMatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "err_banner_vector": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "err_unknown_field": H + "quaternion general\n1 1 1\n1 1 1\n",
    "err_unknown_format": "%%MatrixMarket matrix sparse real general\n1 1 1\n1 1 1\n",
    "err_unknown_symmetry": H + "real diagonal\n1 1 1\n1 1 1\n",
    "err_row": H + "real general\n2 2 1\n3 1 1.0\n",
    "err_col": H + "real general\n2 2 1\n1 0 1.0\n",
    "err_declared": H + "real general\n2 2 3\n1 1 1.0\n2 2 1.0\n",
    "err_more_than": H + "real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
    "err_more_than_before_bad": H + "real general\n2 2 1\n1 1 1.0\nthis line is garbage\n",
    "err_bad_before_more": H + "real general\n2 2 2\n1 1 1.0\n1 x 1.0\n2 2 1.0\n",
    "err_value": H + "real general\n2 2 1\n1 1 abc\n",
    "err_value_hex": H + "real general\n2 2 1\n1 1 0x10\n",
    "err_value_nanparen": H + "real general\n2 2 1\n1 1 nan(1)\n",
    "err_int_value": H + "integer general\n2 2 1\n1 1 1.5\n",
    "err_size": H + "real general\nnot a size line\n",
    "err_size_range": H + "real general\n0 2 1\n",
    "err_missing_size": H + "real general\n% only comments\n\n",
    "err_empty": "",
    "err_fields": H + "real general\n2 2 1\n1 1\n",
    "err_fields_pattern": H + "pattern general\n2 2 1\n1 1 1.0\n",
    "err_index": H + "real general\n2 2 1\n1.0 1 1.0\n",
    "err_line_no": H + "real general\n% c\n2 2 2\n\n1 1 1.0\n% c\n2 3 1.0\n",
}
BYTES_CASES = {
    "crlf_bytes": (H + "real general\r\n% c\r\n2 2 2\r\n1 1 1.0\r\n2 2 2.0\r\n").encode(),
    "cr_only_bytes": (H + "real general\r2 2 2\r1 1 1.0\r2 2 2.0\r").encode(),
    "crlf_error_bytes": (H + "real general\r\n2 2 2\r\n1 1 1.0\r\n\r\n2 5 2.0\r\n").encode(),
    "identity_bytes": (H + "real general\n2 2 2\n1 1 1.0\n2 2 1.0\n").encode(),
}


def run(src):
    try:
        m = parse_matrix_market(src)
    except MatrixMarketError as e:
        return {"error": str(e), "line_no": e.line_no}
    return {"n_rows": m.n_rows, "n_cols": m.n_cols, "rows": m.row_idx.tolist(), "cols": m.col_idx.tolist(),
            "vals": [float(v).hex() for v in m.values]}


def main():
    out = {}
    for name, text in CASES.items():
        out[name] = {"input": text, "kind": "str", **run(text)}
    for name, data in BYTES_CASES.items():
        out[name] = {"input": data.decode(), "kind": "bytes", **run(io.BytesIO(data))}
    # duplicate cases need the GPU CooMatrix on our side; recorded for the gpu tests
    for name, text in {"dup": H + "real general\n2 2 2\n1 1 1.0\n1 1 2.0\n",
                       "dup_symmetric": H + "real symmetric\n2 2 2\n2 1 5\n1 2 5\n"}.items():
        out[name] = {"input": text, "kind": "str", "needs_gpu": True, **run(text)}
    path = Path(__file__).with_name("mm_cases.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print(f"wrote {len(out)} cases to {path} (numpy {np.__version__})")


if __name__ == "__main__":
    main()
