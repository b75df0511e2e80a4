"""The BASELINE.json problem configurations as seeded synthetic inputs
(SURVEY.md §8(d) and Appendix B), built by the host generator library
``libcgvkgen.so`` so the GPU path, the oracle and the CPU reference all see
the same CSR arrays, x* and b = A x* (reference spmv order), x0 = 0.

The reference's own measurements use Matrix Market matrices;
these configs are synthetic stand-ins of the shapes BASELINE.json names.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
GEN_PATH = os.path.join(_HERE, "libcgvkgen.so")
_gen_path = os.environ.get("CGVK_GEN_LIB") or GEN_PATH


class _CSR(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("values", C.c_void_p)]


def use_generator(path: str) -> None:
    """Load the generators from another build of csrc/cgvk_gen.c (bench.py's
    reference arm uses oracle/_build/libinputgen.so, so that process maps no
    library of this package). Only before the first generator call."""
    global _gen_path
    if _gen is not None and path != _gen_path:
        raise RuntimeError("generator library already loaded from " + _gen_path)
    _gen_path = path


def _load() -> C.CDLL:
    if not os.path.exists(_gen_path):
        raise ImportError(f"generator library not built: {_gen_path}")
    g = C.CDLL(_gen_path)
    g.cgvk_gen_poisson.restype = C.POINTER(_CSR)
    g.cgvk_gen_poisson.argtypes = [C.c_int, C.c_int64]
    g.cgvk_gen_varcoef.restype = C.POINTER(_CSR)
    g.cgvk_gen_varcoef.argtypes = [C.c_int64, C.c_uint64, C.c_double]
    g.cgvk_gen_random_spd.restype = C.POINTER(_CSR)
    g.cgvk_gen_random_spd.argtypes = [C.c_int64, C.c_int, C.c_int64, C.c_uint64]
    g.cgvk_csr_free.argtypes = [C.POINTER(_CSR)]
    g.cgvk_gen_xstar.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
    g.cgvk_gen_mt19937_64.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
    g.cgvk_gen_spmv.argtypes = [C.POINTER(_CSR), C.c_void_p, C.c_void_p]
    return g


_gen = None  # loaded on first use (see use_generator)


def _lib() -> C.CDLL:
    global _gen
    if _gen is None:
        _gen = _load()
    return _gen


@dataclass
class CSR:
    """Host CSR in the reference layout (inc/sparse_matrix.hpp:16-23)."""

    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col_idx: np.ndarray  # int64[nnz]
    values: np.ndarray  # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def spmv(self, x: np.ndarray) -> np.ndarray:
        """Host y = A x in the reference order (input synthesis only)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        c = _CSR(self.n, self.nnz, self.row_ptr.ctypes.data, self.col_idx.ctypes.data,
                 self.values.ctypes.data)
        _lib().cgvk_gen_spmv(C.byref(c), x.ctypes.data, y.ctypes.data)
        return y


def _take(p) -> CSR:
    if not p:
        raise ValueError("generator rejected its parameters")
    c = p.contents
    n, nnz = c.n, c.nnz
    rp = np.ctypeslib.as_array(C.cast(c.row_ptr, C.POINTER(C.c_int64)), (n + 1,)).copy()
    ci = np.ctypeslib.as_array(C.cast(c.col_idx, C.POINTER(C.c_int64)), (max(nnz, 1),))[:nnz].copy()
    va = np.ctypeslib.as_array(C.cast(c.values, C.POINTER(C.c_double)), (max(nnz, 1),))[:nnz].copy()
    _lib().cgvk_csr_free(p)
    return CSR(int(n), rp, ci, va)


def poisson2d(N: int) -> CSR:
    return _take(_lib().cgvk_gen_poisson(2, N))


def poisson3d(N: int) -> CSR:
    return _take(_lib().cgvk_gen_poisson(3, N))


def varcoef3d(N: int, seed: int = 11, sigma: float = 2.0) -> CSR:
    return _take(_lib().cgvk_gen_varcoef(N, seed, sigma))


def random_spd(n: int, per_row: int = 13, band: int = 4096, seed: int = 7) -> CSR:
    return _take(_lib().cgvk_gen_random_spd(n, per_row, band, seed))


def xstar(n: int, seed: int = 1) -> np.ndarray:
    out = np.empty(n)
    _lib().cgvk_gen_xstar(n, seed, out.ctypes.data)
    return out


def mt19937_64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _lib().cgvk_gen_mt19937_64(seed, count, out.ctypes.data)
    return out


@dataclass
class Problem:
    name: str
    A: CSR
    x_star: np.ndarray
    b: np.ndarray
    x0: np.ndarray


def make_problem(name: str, A: CSR, seed: int = 1) -> Problem:
    xs = xstar(A.n, seed)
    return Problem(name, A, xs, A.spmv(xs), np.zeros(A.n))


# BASELINE.json configs[0..4]
CONFIGS = {
    "p2d": lambda: poisson2d(256),        # n=65,536, nnz=326,656
    "p64": lambda: poisson3d(64),         # n=262,144, nnz=1,810,432
    "p128": lambda: poisson3d(128),       # n=2,097,152, nnz=14,581,760
    "v256": lambda: varcoef3d(256),       # n=16,777,216, nnz=117,047,296
    "r4m": lambda: random_spd(1 << 22),   # n=4,194,304, nnz=113,033,524
}


def config_problem(name: str) -> Problem:
    return make_problem(name, CONFIGS[name]())
