"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

* ``Restatement`` wraps oracle/_build/liboracle.so (cgv_oracle.c, our C
  restatement of the reference algorithm; sequential or GPU-order dots).
* ``Reference`` wraps oracle/_ref/libcgvref.so (the reference's own sources,
  built unchanged by oracle/Makefile; present wherever it was built — it is
  git-ignored but travels to the GPU box with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product library never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_PATH = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_PATH = os.path.join(HERE, "_ref", "libcgvref.so")

DOT_SEQ, DOT_TREE, DOT_PART = 0, 1, 2
VEC_NAMES = ("x", "r", "p", "s", "w", "u", "t", "r_tilde", "s_tilde", "w_tilde", "u_tilde")
SCALAR_NAMES = ("alpha", "beta", "nu", "nu_prime", "mu", "delta", "delta_hat", "gamma", "eta")


class _DotCfg(C.Structure):
    _fields_ = [("mode", C.c_int), ("block", C.c_int), ("gmax", C.c_int), ("nparts", C.c_int),
                ("part_lo", C.c_void_p), ("order", C.c_int)]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def reference_available() -> bool:
    return os.path.exists(REFERENCE_PATH)


def _load_restatement():
    if not os.path.exists(RESTATEMENT_PATH):
        raise ImportError(f"oracle restatement not built: {RESTATEMENT_PATH}")
    L = C.CDLL(RESTATEMENT_PATH)
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    L.orc_dot.restype = D
    L.orc_dot.argtypes = [I64, P, P, C.POINTER(_DotCfg)]
    L.orc_spmv.argtypes = [I64, P, P, P, P, P]
    L.orc_block_spmv.argtypes = [I64, P, P, P, P, P, P, P]
    L.orc_jacobi.argtypes = [I64, P, P, P, P]
    L.orc_jacobi.restype = I
    L.orc_validate_csr.argtypes = [I64, P, P, I64]
    L.orc_validate_csr.restype = I
    L.orc_solver_create.restype = P
    L.orc_solver_create.argtypes = [I64, P, P, P, I, I, I, I, I, I, I, P, P,
                                    C.POINTER(_DotCfg), C.POINTER(I)]
    L.orc_solver_destroy.argtypes = [P]
    L.orc_solver_step.argtypes = [P]
    L.orc_solver_step.restype = I
    L.orc_solver_state.argtypes = [P, C.POINTER(I), P, P, P]
    L.orc_solver_vector.argtypes = [P, I, P]
    L.orc_solver_vector.restype = I
    L.orc_solve.argtypes = [P, P, I, D, P, P, I]
    L.orc_solve.restype = I
    L.orc_time_steps.argtypes = [P, I, C.POINTER(I)]
    L.orc_time_steps.restype = D
    L.orc_anorm_run.argtypes = [P, P, I, D, C.POINTER(I), C.POINTER(D), C.POINTER(I)]
    L.orc_anorm_run.restype = I
    L.orc_config_validate.argtypes = [I] * 6
    L.orc_config_validate.restype = I
    return L


def _load_reference():
    if not reference_available():
        return None
    L = C.CDLL(REFERENCE_PATH)
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    L.cgvref_last_error.restype = C.c_char_p
    L.cgvref_matrix_create.restype = P
    L.cgvref_matrix_create.argtypes = [I64, P, P, P]
    L.cgvref_matrix_destroy.argtypes = [P]
    L.cgvref_matrix_nnz.restype = I64
    L.cgvref_matrix_nnz.argtypes = [P]
    L.cgvref_matrix_n.restype = I64
    L.cgvref_matrix_n.argtypes = [P]
    L.cgvref_matrix_arrays.argtypes = [P, P, P, P]
    L.cgvref_read_mtx.restype = P
    L.cgvref_read_mtx.argtypes = [C.c_char_p]
    L.cgvref_validate_csr.argtypes = [P]
    L.cgvref_is_symmetric.argtypes = [P]
    L.cgvref_spmv.argtypes = [P, P, P]
    L.cgvref_block_spmv.argtypes = [P, P, P, P, P]
    L.cgvref_jacobi.argtypes = [P, P]
    L.cgvref_dot.restype = D
    L.cgvref_dot.argtypes = [I64, P, P]
    L.cgvref_config_validate.argtypes = [I] * 6
    L.cgvref_solver_create.restype = P
    L.cgvref_solver_create.argtypes = [P, I, I, I, I, I, I, I, P, P, C.POINTER(I)]
    L.cgvref_solver_destroy.argtypes = [P]
    L.cgvref_solver_step.argtypes = [P]
    L.cgvref_solver_state.argtypes = [P, C.POINTER(I), P, P, P]
    L.cgvref_solver_vector.argtypes = [P, I, P]
    L.cgvref_solve.restype = I
    L.cgvref_solve.argtypes = [P, P, I, D, P, P, I]
    L.cgvref_true_residual.restype = D
    L.cgvref_true_residual.argtypes = [P, P]
    L.cgvref_time_steps.restype = D
    L.cgvref_time_steps.argtypes = [P, I, C.POINTER(I)]
    L.cgvref_run.argtypes = [P, I, I, P, P, P, I, I, D, I, C.POINTER(I), C.POINTER(D),
                             C.POINTER(I), C.POINTER(I), I, P, P, P, P]
    L.cgvref_mt19937_64.argtypes = [C.c_uint64, I64, P]
    L.cgvref_run_records.restype = I
    L.cgvref_run_records.argtypes = [P, I, I, I, I, I, I, I, P, P, P, I, I, I, D, I, D, I, I, P,
                                     C.POINTER(I), C.POINTER(I), C.POINTER(D), C.POINTER(I), I, P,
                                     P, P]
    return L


_orc = _load_restatement()
_ref = _load_reference()


class _SolverBase:
    """Common accessors; subclasses provide _state / _vector / _step."""

    n: int

    def state(self) -> dict:
        k = C.c_int()
        st = np.zeros(4, np.int32)
        sc = np.zeros(9)
        stats = np.zeros(4, np.uint64)
        self._state(C.byref(k), st.ctypes.data, sc.ctypes.data, stats.ctypes.data)
        return {"k": k.value, "state": int(st[0]), "breakdown": int(st[1]),
                "criterion": int(st[2]), "allocated_vectors": int(st[3]),
                "scalars": dict(zip(SCALAR_NAMES, sc.tolist())),
                "stats": dict(zip(("spmv_calls", "block_spmv_calls", "precond_applies",
                                   "reductions"), stats.tolist()))}

    def vector(self, which: int):
        out = np.empty(max(self.n, 1))
        rc = self._vector(which, out.ctypes.data)
        return None if rc != 0 else out[: self.n]

    def solve(self, b, max_iter: int, tol: float = 0.0, true_cap: int = 0):
        b = _f64(b)
        upd = np.zeros(max_iter + 1)
        tru = np.zeros(max(true_cap, 1))
        taken = self._solve(b.ctypes.data, max_iter, tol, upd.ctypes.data, tru.ctypes.data,
                            true_cap)
        return taken, upd[: taken + 1], tru[: min(true_cap, taken + 1)]

    def time_steps(self, iters: int):
        taken = C.c_int()
        secs = self._time(iters, C.byref(taken))
        return secs, taken.value


class Restatement(_SolverBase):
    """orc_solver: the C restatement. dot = 'seq' | ('tree', block, gmax) |
    ('part', block, gmax, part_lo)."""

    def __init__(self, A, variant: int, precond: int, b, x0, dot="seq", nu_expr: int = -1,
                 recompute_nu=True, recompute_w=True, unsimplified_mu=False, track_delta=False):
        self._keep = (_i64(A.row_ptr), _i64(A.col_idx), _f64(A.values), _f64(b), _f64(x0))
        rp, ci, va, bb, xx = self._keep
        self._cfg, self._parts = make_dotcfg(dot)
        err = C.c_int()
        self._h = _orc.orc_solver_create(A.n, _p(rp), _p(ci), _p(va), variant, nu_expr,
                                         int(recompute_nu), int(recompute_w), int(unsimplified_mu),
                                         int(track_delta), precond, _p(bb), _p(xx),
                                         C.byref(self._cfg), C.byref(err))
        if not self._h:
            raise ValueError(f"oracle initialize rejected the inputs ({err.value})")
        self.n = A.n

    def __del__(self):
        if getattr(self, "_h", None):
            _orc.orc_solver_destroy(self._h)
            self._h = None

    def step(self) -> int:
        return _orc.orc_solver_step(self._h)

    def _state(self, *a):
        _orc.orc_solver_state(self._h, *a)

    def _vector(self, which, ptr):
        return _orc.orc_solver_vector(self._h, which, ptr)

    def _solve(self, *a):
        return _orc.orc_solve(self._h, *a)

    def _time(self, *a):
        return _orc.orc_time_steps(self._h, *a)

    def anorm_run(self, x_star, max_iter: int, threshold: float = 1e-5):
        """Table-3 protocol (run() + error-reduction stop, probes every step)."""
        xs = _f64(x_star)
        it, mle, fs = C.c_int(), C.c_double(), C.c_int()
        taken = _orc.orc_anorm_run(self._h, xs.ctypes.data, max_iter, threshold, C.byref(it),
                                   C.byref(mle), C.byref(fs))
        return {"taken": taken, "iters_to_1e5": it.value, "min_log10_err": mle.value,
                "final_state": fs.value}


class Reference(_SolverBase):
    """cgv_ref::SolverState driven through the reference's own initialize/step."""

    def __init__(self, A, variant: int, precond: int, b, x0, nu_expr: int = -1,
                 recompute_nu=True, recompute_w=True, unsimplified_mu=False, track_delta=False,
                 mat: "RefMatrix | None" = None):
        if _ref is None:
            raise ImportError("oracle/_ref/libcgvref.so not built")
        self._mat = mat if mat is not None else RefMatrix(A)  # A borrowed, as the reference does
        b, x0 = _f64(b), _f64(x0)
        self._keep = (b, x0)
        err = C.c_int()
        self._h = _ref.cgvref_solver_create(self._mat.h, variant, nu_expr, int(recompute_nu),
                                            int(recompute_w), int(unsimplified_mu),
                                            int(track_delta), precond, _p(b), _p(x0),
                                            C.byref(err))
        if not self._h:
            raise ValueError(_ref.cgvref_last_error().decode())
        self.n = A.n

    def __del__(self):
        if getattr(self, "_h", None):
            _ref.cgvref_solver_destroy(self._h)
            self._h = None

    def step(self) -> int:
        return _ref.cgvref_solver_step(self._h)

    def _state(self, *a):
        _ref.cgvref_solver_state(self._h, *a)

    def _vector(self, which, ptr):
        return _ref.cgvref_solver_vector(self._h, which, ptr)

    def _solve(self, *a):
        return _ref.cgvref_solve(self._h, *a)

    def _time(self, *a):
        return _ref.cgvref_time_steps(self._h, *a)

    def true_residual(self, b) -> float:
        b = _f64(b)
        return _ref.cgvref_true_residual(self._h, b.ctypes.data)


class RefMatrix:
    def __init__(self, A=None, handle=None):
        if handle is not None:
            self.h = handle
        else:
            rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
            self.h = _ref.cgvref_matrix_create(A.n, _p(rp), _p(ci), _p(va))

    def __del__(self):
        if getattr(self, "h", None):
            _ref.cgvref_matrix_destroy(self.h)
            self.h = None

    def arrays(self):
        n = _ref.cgvref_matrix_n(self.h)
        nnz = _ref.cgvref_matrix_nnz(self.h)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int64)
        va = np.empty(max(nnz, 1))
        _ref.cgvref_matrix_arrays(self.h, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
        return int(n), rp, ci[:nnz], va[:nnz]


def make_dotcfg(dot):
    cfg = _DotCfg()
    parts = None
    if dot == "seq":
        cfg.mode = DOT_SEQ
    elif dot[0] == "tree":  # ("tree", block, gmax[, order])
        cfg.mode, cfg.block, cfg.gmax = DOT_TREE, dot[1], dot[2]
        cfg.order = dot[3] if len(dot) > 3 else 0
    else:  # ("part", block, gmax, part_lo[, order])
        parts = _i64(dot[3])
        cfg.mode, cfg.block, cfg.gmax = DOT_PART, dot[1], dot[2]
        cfg.nparts = parts.shape[0] - 1
        cfg.part_lo = parts.ctypes.data
        cfg.order = dot[4] if len(dot) > 4 else 0
    return cfg, parts


# ------------------------------------------------------------ primitives

def dot(x, y, mode="seq") -> float:
    x, y = _f64(x), _f64(y)
    cfg, parts = make_dotcfg(mode)
    return _orc.orc_dot(x.shape[0], _p(x), _p(y), C.byref(cfg))


def spmv(A, x) -> np.ndarray:
    rp, ci, va, x = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values), _f64(x)
    y = np.empty(A.n)
    _orc.orc_spmv(A.n, _p(rp), _p(ci), _p(va), _p(x), _p(y))
    return y


def block_spmv(A, x1, x2):
    rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
    x1, x2 = _f64(x1), _f64(x2)
    y1, y2 = np.empty(A.n), np.empty(A.n)
    _orc.orc_block_spmv(A.n, _p(rp), _p(ci), _p(va), _p(x1), _p(x2), _p(y1), _p(y2))
    return y1, y2


def jacobi(A):
    rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
    d = np.empty(max(A.n, 1))
    rc = _orc.orc_jacobi(A.n, _p(rp), _p(ci), _p(va), d.ctypes.data)
    return None if rc else d[: A.n]


def config_valid(variant, nu_expr, recompute_nu=True, recompute_w=True, unsimplified_mu=False,
                 track_delta=False) -> bool:
    return _orc.orc_config_validate(variant, nu_expr, int(recompute_nu), int(recompute_w),
                                    int(unsimplified_mu), int(track_delta)) == 0


# ---------------------------------------------------- reference-only helpers

def ref_lib():
    return _ref


def ref_read_mtx(path: str):
    h = _ref.cgvref_read_mtx(path.encode())
    if not h:
        raise ValueError(_ref.cgvref_last_error().decode())
    return RefMatrix(handle=h)


RECORD_FIELDS = ("rel_err_a_norm", "true_res_norm", "upd_res_norm", "residual_gap_norm", "nu_gap",
                 "w_gap_norm", "s_gap_norm", "lanczos_res_norm", "succ_orth", "alpha", "beta", "nu",
                 "nu_prime")


def ref_run_records(A, variant: int, precond: int, b, x0, x_star=None, max_iter: int = 100,
                    stop=("fixed", 100), probes: bool = True, cadence: int = 1, nu_expr: int = -1,
                    recompute_nu=True, recompute_w=True, unsimplified_mu=False, track_delta=False,
                    rec_cap: int = 4096) -> dict:
    """The reference's run() (proj/src/runner.cpp:32-147) with every probe field.
    stop: ("fixed", count) | ("error", threshold) | ("stagnation", window, improvement)."""
    m = RefMatrix(A)
    b, x0 = _f64(b), _f64(x0)
    xs = _f64(x_star) if x_star is not None else None
    kind = {"fixed": 0, "error": 1, "stagnation": 2}[stop[0]]
    fixed = stop[1] if kind == 0 else 0
    thr = stop[1] if kind == 1 else 1e-5
    win = stop[1] if kind == 2 else 50
    imp = stop[2] if kind == 2 else 0.01
    fs = (C.c_int * 3)()
    hs, it, nrec = C.c_int(), C.c_int(), C.c_int()
    mle = C.c_double()
    rk = np.zeros(rec_cap, np.int32)
    rm = np.zeros(rec_cap, np.uint32)
    rv = np.zeros((rec_cap, 13))
    rc = _ref.cgvref_run_records(m.h, variant, nu_expr, int(recompute_nu), int(recompute_w),
                                 int(unsimplified_mu), int(track_delta), precond, _p(b), _p(x0),
                                 _p(xs) if xs is not None else None, max_iter, kind, fixed, thr, win,
                                 imp, int(probes), cadence, fs, C.byref(hs), C.byref(it),
                                 C.byref(mle), C.byref(nrec), rec_cap, rk.ctypes.data,
                                 rm.ctypes.data, rv.ctypes.data)
    if rc:
        raise ValueError(_ref.cgvref_last_error().decode())
    cnt = min(nrec.value, rec_cap)
    recs = []
    for q in range(cnt):
        r = {"k": int(rk[q])}
        for f, name in enumerate(RECORD_FIELDS):
            r[name] = float(rv[q, f]) if rm[q] >> f & 1 else None
        recs.append(r)
    return {"state": fs[0], "breakdown": fs[1], "criterion": fs[2], "records": recs,
            "summary": ({"iters_to_1e5": it.value if it.value >= 0 else None,
                         "min_log10_err": mle.value} if hs.value else None)}


def ref_mt19937_64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    _ref.cgvref_mt19937_64(seed, count, out.ctypes.data)
    return out


def ref_run(A, variant: int, precond: int, b, x0, x_star, max_iter: int, stop_kind: int,
            threshold: float = 1e-5, cadence: int = 1, rec_cap: int = 0):
    """The reference's run() (Table-3 protocol, tests/test_matrices.cpp:39-46)."""
    m = RefMatrix(A)
    b, x0, xs = _f64(b), _f64(x0), _f64(x_star)
    it, mle, fs, nrec = C.c_int(), C.c_double(), C.c_int(), C.c_int()
    cap = max(rec_cap, 1)
    rk = np.zeros(cap, np.int32)
    re, rt, ru = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    rc = _ref.cgvref_run(m.h, variant, precond, _p(b), _p(x0), _p(xs), max_iter, stop_kind,
                         threshold, cadence, C.byref(it), C.byref(mle), C.byref(fs),
                         C.byref(nrec), rec_cap, rk.ctypes.data, re.ctypes.data, rt.ctypes.data,
                         ru.ctypes.data)
    if rc:
        raise ValueError(_ref.cgvref_last_error().decode())
    k = min(nrec.value, rec_cap)
    return {"iters_to_1e5": it.value, "min_log10_err": mle.value, "final_state": fs.value,
            "n_records": nrec.value, "k": rk[:k], "err": re[:k], "true": rt[:k], "upd": ru[:k]}


# ------------------------------------------------ extended precision (extprec.c)
# The reference tests' MPFR oracles (proj/tests/oracles.hpp: exact_dot,
# exact_dot_ratio, HighPrecCg) restated in binary128; TEST INFRASTRUCTURE.
EXTPREC_PATH = os.path.join(HERE, "_build", "libextprec.so")
_xp = None


def _extprec():
    global _xp
    if _xp is None:
        L = C.CDLL(EXTPREC_PATH)
        P, I64, D = C.c_void_p, C.c_int64, C.c_double
        L.xp_dot.restype = D
        L.xp_dot.argtypes = [I64, P, P]
        L.xp_abs_dot.restype = D
        L.xp_abs_dot.argtypes = [I64, P, P]
        L.xp_ratio.restype = D
        L.xp_ratio.argtypes = [I64, P, P, P, P]
        L.xp_cg.restype = C.c_int
        L.xp_cg.argtypes = [I64, P, P, P, P, P, P, C.c_int, P]
        _xp = L
    return _xp


def exact_dot(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return _extprec().xp_dot(x.shape[0], _p(x), _p(y))


def abs_dot(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return _extprec().xp_abs_dot(x.shape[0], _p(x), _p(y))


def exact_ratio(a, b, c, d) -> float:
    a, b, c, d = _f64(a), _f64(b), _f64(c), _f64(d)
    return _extprec().xp_ratio(a.shape[0], _p(a), _p(b), _p(c), _p(d))


def high_prec_cg(A, b, x0, steps: int, inv_diag=None):
    """x_1 .. x_steps of PCG carried in binary128 (rows of the result)."""
    rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
    b, x0 = _f64(b), _f64(x0)
    d = None if inv_diag is None else _f64(inv_diag)
    xs = np.zeros((steps, A.n))
    k = _extprec().xp_cg(A.n, _p(rp), _p(ci), _p(va), _p(d) if d is not None else None, _p(b), _p(x0),
                         steps, _p(xs))
    return xs[:k]
