"""Shared cases of the extended-precision KATs (the reference's MPFR-based
tests restated: proj/tests/test_vector_ops.cpp exact-dot bound,
test_variants.cpp HS-vs-HighPrecCg on a 4x4 system and the exactly rounded
alpha_0)."""
import numpy as np

from paper_1905_01549_b200 import problems as pb

EPS = 2.0 ** -53


def hilbert_shift_4():
    """The 4x4 SPD system of the reference's HS-vs-HighPrecCg test:
    a_ij = 1/(i+j+1) + 0.1 [i == j], b = (1, -0.5, 0.25, 2), x0 = 0."""
    n = 4
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int64), n)
    va = np.array([1.0 / (i + j + 1) + (0.1 if i == j else 0.0) for i in range(n) for j in range(n)])
    return pb.CSR(n, rp, ci, va), np.array([1.0, -0.5, 0.25, 2.0]), np.zeros(n)
