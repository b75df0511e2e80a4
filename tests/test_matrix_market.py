"""Matrix Market ingest of the C++ cgv:: shim (cgvariants/matrix_market.hpp,
host code, no GPU) against the reference parser (src/matrix_market.cpp):
the bundled fixtures parse to exactly the CSR arrays the reference parser
produced (tests/golden/mtx, made by scripts/make_golden.py through
oracle/_ref), write → parse round trips bit for bit, and small handwritten
inputs exercise every accepted form and every ParseError code — checked
against the reference parser itself when /root/reference is present."""
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_1905_01549_b200", "cpp", "mtx_tool")
REF_MTX = "/root/reference/proj/data/matrices"

# ParseError::Code (include/cgvariants/matrix_market.hpp)
MALFORMED_HEADER, NOT_SQUARE, NON_REAL, PATTERN, UNSUPPORTED_SYMMETRY, OUT_OF_BOUNDS, NOT_SYMMETRIC, \
    MALFORMED = range(8)


def fnv(arrays) -> int:
    h = 1469598103934665603
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h = ((h ^ byte) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def run_tool(path, *extra):
    if not os.path.exists(TOOL):
        pytest.skip("mtx_tool not built (python __graft_entry__.py)")
    out = subprocess.run([TOOL, path, *extra], capture_output=True, text=True, timeout=60)
    return out.returncode, out.stdout.split()


def ref_available():
    try:
        from oracle import oracle as O
        return O.reference_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.mark.parametrize("name", ["1138_bus", "494_bus", "bcsstk03", "bcsstm21", "bcsstm22", "model_48_8_3",
                                  "nos2", "nos4", "nos7"])
def test_fixture_matches_reference_parser(name):
    path = os.path.join(REF_MTX, name + ".mtx")
    if not os.path.exists(path):
        pytest.skip("reference fixtures not present")
    g = np.load(os.path.join(GOLDEN, "mtx", name + ".npz"))
    rc, out = run_tool(path, "--roundtrip")
    assert rc == 0, out
    n, nnz, h = int(out[0]), int(out[1]), int(out[2])
    assert (n, nnz) == (int(g["n"]), len(g["values"]))
    assert h == fnv([g["row_ptr"].astype(np.int64), g["col_idx"].astype(np.int64),
                     g["values"].astype(np.float64)])


# (text, expected): ("ok", n, row_ptr, col_idx, values) or ("error", code)
CASES = {
    "sym_coord_dups_zero_comments": (
        "%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n3 3 5\n"
        "1 1 4.0\n2 1 -1.0\n2 1 -0.5\n3 3 2.5D+00\n3 2 0.0\n",
        ("ok", 3, [0, 2, 3, 4], [0, 1, 0, 2], [4.0, -1.5, -1.5, 2.5])),  # (3,2) = 0 dropped
    "crlf_uppercase_banner": (
        "%%MATRIXMARKET MATRIX COORDINATE REAL GENERAL\r\n2 2 2\r\n  1 1 1.5\r\n2 2 2e0 \r\n",
        ("ok", 2, [0, 1, 2], [0, 1], [1.5, 2.0])),
    "general_array": (
        "%%MatrixMarket matrix array real general\n2 2\n3.0\n1.0\n1.0\n5.0\n",
        ("ok", 2, [0, 2, 4], [0, 1, 0, 1], [3.0, 1.0, 1.0, 5.0])),
    "symmetric_array": (
        "%%MatrixMarket matrix array real symmetric\n2 2\n3.0 1.0\n5.0\n",
        ("ok", 2, [0, 2, 4], [0, 1, 0, 1], [3.0, 1.0, 1.0, 5.0])),
    "empty": ("", ("error", MALFORMED_HEADER)),
    "bad_banner": ("%%MatrixMarkt matrix coordinate real general\n1 1 1\n1 1 1\n", ("error", MALFORMED_HEADER)),
    "short_banner": ("%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n", ("error", MALFORMED_HEADER)),
    "vector_object": ("%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n", ("error", MALFORMED_HEADER)),
    "unknown_format": ("%%MatrixMarket matrix sparse real general\n1 1 1\n1 1 1\n", ("error", MALFORMED_HEADER)),
    "pattern": ("%%MatrixMarket matrix coordinate pattern symmetric\n1 1 1\n1 1\n", ("error", PATTERN)),
    "integer": ("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 1\n", ("error", NON_REAL)),
    "complex": ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", ("error", NON_REAL)),
    "skew": ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
             ("error", UNSUPPORTED_SYMMETRY)),
    "missing_size": ("%%MatrixMarket matrix coordinate real general\n% only a comment\n", ("error", MALFORMED)),
    "not_square": ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", ("error", NOT_SQUARE)),
    "few_entries": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n", ("error", MALFORMED)),
    "bad_entry": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", ("error", MALFORMED)),
    "plus_sign": ("%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 +1.0\n", ("error", MALFORMED)),
    "index_zero": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n", ("error", OUT_OF_BOUNDS)),
    "index_high": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 1\n", ("error", OUT_OF_BOUNDS)),
    "not_symmetric": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n2 1 2\n",
                      ("error", NOT_SYMMETRIC)),
    "array_count": ("%%MatrixMarket matrix array real general\n2 2\n1 2 3\n", ("error", MALFORMED)),
    "array_value": ("%%MatrixMarket matrix array real general\n1 1\nx\n", ("error", MALFORMED)),
}


@pytest.mark.parametrize("case", list(CASES))
def test_handwritten_inputs(case, tmp_path):
    text, want = CASES[case]
    path = str(tmp_path / f"{case}.mtx")
    with open(path, "w", newline="") as f:
        f.write(text)
    rc, out = run_tool(path, "--roundtrip")
    assert rc == 0, out
    if want[0] == "error":
        assert out == ["error", str(want[1])], out
    else:
        _, n, rp, ci, va = want
        assert int(out[0]) == n and int(out[1]) == len(va)
        assert int(out[2]) == fnv([np.array(rp, np.int64), np.array(ci, np.int64), np.array(va, np.float64)])
    if ref_available():  # the reference parser agrees: same arrays, or an error too
        from oracle import oracle as O
        if want[0] == "error":
            with pytest.raises(ValueError):
                O.ref_read_mtx(path)
        else:
            n, rp, ci, va = O.ref_read_mtx(path).arrays()
            assert n == int(out[0]) and fnv([rp, ci, va]) == int(out[2])
