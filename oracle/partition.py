"""TEST INFRASTRUCTURE ONLY — CPU restatement of the row partition and halo
maps of a row-partitioned solve (the reference has no
distributed code, so these maps are pinned by this independent restatement),
plus a host-only distributed SpMV that follows the device data path (local
numbering, halo fill, rows summed in CSR order) for the multi-process tests.
"""
from __future__ import annotations

import numpy as np


def partition_rows(n: int, nparts: int, align: int = 1) -> np.ndarray:
    """Contiguous blocks of whole `align`-row planes, as even as possible."""
    units = n // align
    assert units * align == n
    return np.array([(r * units // nparts) * align for r in range(nparts + 1)], dtype=np.int64)


def halo_maps(A, lo, rank: int) -> dict:
    """From the GLOBAL CSR: the columns rank `rank` reads from its neighbours
    (sorted) and the local rows each neighbour reads from it (sorted)."""
    a, b = int(lo[rank]), int(lo[rank + 1])
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    mine = (rows >= a) & (rows < b)
    cols = A.col_idx[mine]
    lower = np.unique(cols[cols < a])
    upper = np.unique(cols[cols >= b])
    # rows of mine that a neighbour's rows reference (computed from THEIR rows)
    out = {"lower": lower, "upper": upper}
    for key, r in (("send_lo", rank - 1), ("send_hi", rank + 1)):
        if 0 <= r < len(lo) - 1:
            theirs = (rows >= lo[r]) & (rows < lo[r + 1])
            c = A.col_idx[theirs]
            out[key] = np.unique(c[(c >= a) & (c < b)]) - a
        else:
            out[key] = np.zeros(0, np.int64)
    return out


def local_matrix(A, lo, rank: int):
    """Local CSR in [own | lower halo | upper halo] numbering, entries in the
    global CSR order."""
    a, b = int(lo[rank]), int(lo[rank + 1])
    h = halo_maps(A, lo, rank)
    k0, k1 = int(A.row_ptr[a]), int(A.row_ptr[b])
    ci = A.col_idx[k0:k1]
    m, L = b - a, len(h["lower"])
    loc = np.where(ci < a, m + np.searchsorted(h["lower"], ci),
                   np.where(ci >= b, m + L + np.searchsorted(h["upper"], ci), ci - a))
    return A.row_ptr[a:b + 1] - k0, loc.astype(np.int64), A.values[k0:k1], h


def local_spmv(rp, ci, va, xloc) -> np.ndarray:
    """Row sums left to right in stored order (src/sparse_matrix.cpp:112-117)."""
    y = np.empty(len(rp) - 1)
    for i in range(len(rp) - 1):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s = s + va[k] * xloc[ci[k]]
        y[i] = s
    return y
