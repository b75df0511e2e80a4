"""ctypes binding of the cgvk C ABI (include/cgvk.h).

Python-side mirror of the reference's solver interface
(/root/reference/proj/include/cgvariants/{variants,runner,sparse_matrix,
preconditioner}.hpp): the same names, argument meaning and error behaviour, so
the parity tests read like the reference's own tests. There is no CPU fallback:
importing this module without the built CUDA library raises.

Error mapping (include/cgvk.h): CGVK_EINVAL -> InvalidArgument (a ValueError,
like std::invalid_argument), CGVK_ESTATE -> LogicError (std::logic_error),
CUDA/NCCL/OOM -> CgvkError (std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CGVK_LIB") or os.path.join(_HERE, "libcgvk.so")  # CGVK_LIB: A/B builds


HISTORY_CAP = 1 << 17  # CGVK_HISTORY_CAP (include/cgvk.h)


class CgvkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"cgvk error {code}: {msg}")
        self.code = code


class InvalidArgument(CgvkError, ValueError):
    pass


class LogicError(CgvkError):
    pass


class Variant(enum.IntEnum):  # inc/variants.hpp:17-25
    HS = 0
    CG_CG = 1
    M = 2
    PR = 3
    GV = 4
    PIPE_PR_M = 5
    PIPE_PR = 6


VARIANT_NAMES = {  # src/variants.cpp:49-60
    Variant.HS: "hs", Variant.CG_CG: "cg", Variant.M: "m", Variant.PR: "pr",
    Variant.GV: "gv", Variant.PIPE_PR_M: "pipe-pr-m", Variant.PIPE_PR: "pipe-pr",
}


def variant_from_name(name: str) -> Variant | None:  # src/variants.cpp:62-71
    alias = {"hs": Variant.HS, "cg": Variant.CG_CG, "cg-cg": Variant.CG_CG, "m": Variant.M,
             "pr": Variant.PR, "gv": Variant.GV, "pipe-pr-m": Variant.PIPE_PR_M,
             "pprm": Variant.PIPE_PR_M, "pipe-pr": Variant.PIPE_PR, "ppr": Variant.PIPE_PR}
    return alias.get(name)


class NuExpression(enum.IntEnum):  # inc/variants.hpp:28-32
    EXPANDED = 0
    SIMPLIFIED = 1
    MEURANT = 2


class Precond(enum.IntEnum):  # inc/preconditioner.hpp:13-14
    IDENTITY = 0
    JACOBI = 1


class State(enum.IntEnum):  # SolveStatus::State
    RUNNING = 0
    BREAKDOWN = 1
    MAX_ITERATIONS = 2
    CONVERGED = 3


class Breakdown(enum.IntEnum):
    NONE = 0
    NU_PRIME_NONPOSITIVE = 1
    NU_NONPOSITIVE = 2
    MU_NONPOSITIVE = 3
    NON_FINITE = 4


class ConvergedBy(enum.IntEnum):
    ZERO_RESIDUAL = 0
    ERROR_THRESHOLD = 1
    STAGNATION = 2
    TOLERANCE = 3


class Vec(enum.IntEnum):  # SolverState fields
    X = 0
    R = 1
    P = 2
    S = 3
    W = 4
    U = 5
    T = 6
    R_TILDE = 7
    S_TILDE = 8
    W_TILDE = 9
    U_TILDE = 10


class _Config(C.Structure):
    _fields_ = [(f, C.c_int) for f in ("variant", "nu_expression", "recompute_nu", "recompute_w",
                                       "unsimplified_mu", "track_delta")]


class _Status(C.Structure):
    _fields_ = [(f, C.c_int) for f in ("state", "breakdown", "criterion", "k",
                                       "allocated_vectors")]


class _Scalars(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("alpha", "beta", "nu", "nu_prime", "mu", "delta",
                                          "delta_hat", "gamma", "eta", "rr")]


class _Stats(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in ("spmv_calls", "block_spmv_calls", "precond_applies",
                                          "reductions")]


RECORD_FIELDS = ("rel_err_a_norm", "true_res_norm", "upd_res_norm", "residual_gap_norm", "nu_gap",
                 "w_gap_norm", "s_gap_norm", "lanczos_res_norm", "succ_orth", "alpha", "beta", "nu",
                 "nu_prime")


class _StopRule(C.Structure):
    _fields_ = [("kind", C.c_int), ("fixed_count", C.c_int), ("error_threshold", C.c_double),
                ("stagnation_window", C.c_int), ("stagnation_improvement", C.c_double)]


class _ProbeOptions(C.Structure):
    _fields_ = [("enabled", C.c_int), ("cadence", C.c_int), ("x_star", C.c_void_p)]


class _Record(C.Structure):
    _fields_ = [("k", C.c_int), ("mask", C.c_uint), ("v", C.c_double * len(RECORD_FIELDS))]


class _Summary(C.Structure):
    _fields_ = [("has", C.c_int), ("iters_to_1e5", C.c_int), ("min_log10_err", C.c_double)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"cgvk CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    pp = C.POINTER(C.c_void_p)
    sig = {
        "cgvk_last_error": (C.c_char_p, []),
        "cgvk_device_count": (I, [C.POINTER(I)]),
        "cgvk_variant_config_make": (_Config, [I]),
        "cgvk_variant_config_validate": (I, [C.POINTER(_Config)]),
        "cgvk_matrix_create_csr": (I, [I64, P, P, P, I, I, pp]),
        "cgvk_matrix_destroy": (I, [P]),
        "cgvk_matrix_info": (I, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I)]),
        "cgvk_matrix_engine": (I, [P, C.POINTER(I), C.POINTER(I)]),
        "cgvk_time_ops": (I, [P, I, P]),
        "cgvk_spmv": (I, [P, P, P]),
        "cgvk_block_spmv": (I, [P, P, P, P, P]),
        "cgvk_jacobi": (I, [P, P]),
        "cgvk_precond_apply": (I, [P, I, P, P]),
        "cgvk_dot": (I, [P, P, P, C.POINTER(D)]),
        "cgvk_reduction_config": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
        "cgvk_solver_create": (I, [P, C.POINTER(_Config), I, P, P, pp]),
        "cgvk_solver_destroy": (I, [P]),
        "cgvk_solver_set_tolerance": (I, [P, D]),
        "cgvk_solver_step": (I, [P, I]),
        "cgvk_solver_sync": (I, [P]),
        "cgvk_solver_status": (I, [P, C.POINTER(_Status), C.POINTER(_Scalars),
                                   C.POINTER(_Stats)]),
        "cgvk_solver_get_vector": (I, [P, I, P]),
        "cgvk_solver_get_vector_async": (I, [P, I, P]),
        "cgvk_solver_after": (I, [P, P]),
        "cgvk_solver_true_residual": (I, [P, C.POINTER(D)]),
        "cgvk_solver_history": (I, [P, P, I, C.POINTER(I)]),
        "cgvk_solver_stream": (P, [P]),
        "cgvk_solver_launches_per_iter": (I, [P]),
        "cgvk_solver_launches": (C.c_longlong, [P, I]),
        "cgvk_solver_time_steps": (I, [P, I, C.POINTER(D), C.POINTER(I)]),
        "cgvk_solver_profile": (I, [P, I, C.POINTER(D), C.POINTER(D), C.POINTER(I)]),
        "cgvk_run": (I, [P, C.POINTER(_Config), I, P, P, I, C.POINTER(_StopRule),
                         C.POINTER(_ProbeOptions), P, I, C.POINTER(I), C.POINTER(_Status),
                         C.POINTER(_Summary), P]),
        "cgvk_solve": (I, [P, C.POINTER(_Config), I, P, P, I, D, P, C.POINTER(_Status),
                           C.POINTER(_Scalars)]),
        "cgvk_host_register": (I, [P, C.c_uint64]),
        "cgvk_partition_rows": (I, [I64, I, I64, P]),
        "cgvk_halo_plan": (I, [I64, I, P, I, P, P, P, P, P, P, P]),
        "cgvk_matrix_create_rank": (I, [I64, I, I, P, P, P, P, I, pp]),
        "cgvk_comm_nccl_unique_id": (I, [P]),
        "cgvk_comm_create_nccl": (I, [P, I, I, I, pp]),
        "cgvk_comm_create_local": (I, [I, I, pp]),
        "cgvk_comm_destroy": (I, [P]),
        "cgvk_group_create": (I, [P, I, P, C.POINTER(_Config), I, P, P, P]),
        "cgvk_group_create_ex": (I, [P, I, P, C.POINTER(_Config), I, P, P, I, P]),
        "cgvk_group_transport": (I, [P]),
        "cgvk_rank_local_columns": (I, [I64, I, P, I, P, P, P, C.POINTER(I64)]),
        "cgvk_group_step": (I, [P, I, I]),
        "cgvk_group_true_residual": (I, [P, I, C.POINTER(D)]),
        "cgvk_host_unregister": (I, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()

# every symbol include/cgvk.h declares (checked by tests/test_abi.py)
EXPORTED = sorted(n for n in dir(_lib) if n.startswith("cgvk_"))


def lib() -> C.CDLL:
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.cgvk_last_error() or b"").decode()
    if rc == -1:
        raise InvalidArgument(rc, msg)
    if rc == -2:
        raise LogicError(rc, msg)
    raise CgvkError(rc, msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def device_count() -> int:
    n = C.c_int(0)
    _check(_lib.cgvk_device_count(C.byref(n)))
    return n.value


def device_count_safe() -> int:
    """0 when no CUDA driver/device is present (used to skip, never to fall back)."""
    try:
        return device_count()
    except CgvkError:
        return 0


@dataclass
class VariantConfig:
    """POD mirror of VariantConfig (inc/variants.hpp:34-57)."""

    variant: Variant = Variant.HS
    recompute_nu: bool = True
    recompute_w: bool = True
    nu_expression: NuExpression = NuExpression.SIMPLIFIED
    unsimplified_mu: bool = False
    track_delta: bool = False

    @staticmethod
    def make(v: Variant) -> "VariantConfig":  # src/variants.cpp:10-23
        c = _lib.cgvk_variant_config_make(int(v))
        return VariantConfig._from_c(c)

    @staticmethod
    def _from_c(c: _Config) -> "VariantConfig":
        return VariantConfig(Variant(c.variant), bool(c.recompute_nu), bool(c.recompute_w),
                             NuExpression(c.nu_expression), bool(c.unsimplified_mu),
                             bool(c.track_delta))

    def _to_c(self) -> _Config:
        return _Config(int(self.variant), int(self.nu_expression), int(self.recompute_nu),
                       int(self.recompute_w), int(self.unsimplified_mu), int(self.track_delta))

    def validate(self) -> None:  # src/variants.cpp:35-47
        c = self._to_c()
        _check(_lib.cgvk_variant_config_validate(C.byref(c)))

    def is_predictor(self) -> bool:
        return self.variant in (Variant.M, Variant.PR, Variant.PIPE_PR_M, Variant.PIPE_PR)

    def is_pipelined(self) -> bool:
        return self.variant in (Variant.GV, Variant.PIPE_PR_M, Variant.PIPE_PR)


class DeviceMatrix:
    """SparseMatrix resident on one GPU (int32 CSR + fp64 values)."""

    ENGINES = {None: 0, "csr": 2, "band": 4}

    def __init__(self, n: int, row_ptr, col_idx, values, device: int = 0,
                 check_symmetric: bool = False, engine: str | None = None):
        """engine: None = automatic (band for narrow-band long-row matrices,
        seg for stencil-like ones), or "csr" / "band" / "seg" (that engine
        whenever it applies)."""
        rp, ci, va = _i64(row_ptr), _i64(col_idx), _f64(values)
        if rp.shape[0] != n + 1:
            raise InvalidArgument(-1, "row_ptr length must be n+1")
        if ci.shape[0] != va.shape[0] or int(rp[-1]) != ci.shape[0]:
            raise InvalidArgument(-1, "row_ptr[n] must equal number of stored entries")
        h = C.c_void_p()
        _check(_lib.cgvk_matrix_create_csr(n, _ptr(rp), _ptr(ci) if ci.size else None,
                                           _ptr(va) if va.size else None, device,
                                           (1 if check_symmetric else 0) | self.ENGINES[engine],
                                           C.byref(h)))
        self._h = h
        self.n = int(n)
        self.nnz = int(ci.shape[0])
        self.device = device

    @classmethod
    def from_csr(cls, csr, device: int = 0, check_symmetric: bool = False,
                 engine: str | None = None) -> "DeviceMatrix":
        return cls(csr.n, csr.row_ptr, csr.col_idx, csr.values, device, check_symmetric, engine)

    def engine(self) -> tuple[str, int]:
        """("csr" | "band" | "seg", band: x-window half-width in 256-row
        tiles; seg: number of staged x-tile offsets; csr: 0)."""
        e, h = C.c_int(), C.c_int()
        _check(_lib.cgvk_matrix_engine(self._h, C.byref(e), C.byref(h)))
        return ("csr", "band")[e.value], h.value

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.cgvk_matrix_destroy(self._h)
            self._h = None

    __del__ = close

    def _vec(self, v) -> np.ndarray:
        a = _f64(v)
        if a.shape != (self.n,):
            raise InvalidArgument(-1, "vector dimension mismatch")
        return a

    def spmv(self, x) -> np.ndarray:
        x = self._vec(x)
        y = np.empty(self.n)
        _check(_lib.cgvk_spmv(self._h, _ptr(x), _ptr(y)))
        return y

    def block_spmv(self, x1, x2) -> tuple[np.ndarray, np.ndarray]:
        x1, x2 = self._vec(x1), self._vec(x2)
        y1, y2 = np.empty(self.n), np.empty(self.n)
        _check(_lib.cgvk_block_spmv(self._h, _ptr(x1), _ptr(x2), _ptr(y1), _ptr(y2)))
        return y1, y2

    def jacobi(self) -> np.ndarray:
        d = np.empty(self.n)
        _check(_lib.cgvk_jacobi(self._h, _ptr(d)))
        return d

    def precond_apply(self, kind: Precond, v) -> np.ndarray:
        v = self._vec(v)
        out = np.empty(self.n)
        _check(_lib.cgvk_precond_apply(self._h, int(kind), _ptr(v), _ptr(out)))
        return out

    def dot(self, x, y) -> float:
        x, y = self._vec(x), self._vec(y)
        out = C.c_double()
        _check(_lib.cgvk_dot(self._h, _ptr(x), _ptr(y), C.byref(out)))
        return out.value

    def time_ops(self, reps: int = 50) -> dict:
        """Device ms per launch of spmv, block_spmv, one dot, one vector copy."""
        ms = np.zeros(4)
        _check(_lib.cgvk_time_ops(self._h, int(reps), _ptr(ms)))
        return dict(zip(("spmv", "block_spmv", "dot", "copy"), ms.tolist()))

    def reduction_config(self) -> tuple[int, int, int]:
        """(rows per tile, CTA cap G, tile order) of the canonical dot tree."""
        b, g, o = C.c_int(), C.c_int(), C.c_int()
        _check(_lib.cgvk_reduction_config(self._h, C.byref(b), C.byref(g), C.byref(o)))
        return b.value, g.value, o.value


@dataclass
class SolveStatus:
    state: State
    breakdown: Breakdown
    criterion: ConvergedBy

    def running(self) -> bool:
        return self.state == State.RUNNING


SCALAR_NAMES = ("alpha", "beta", "nu", "nu_prime", "mu", "delta", "delta_hat", "gamma", "eta")


class Solver:
    """A device SolverState (inc/variants.hpp:101-143) created by initialize()."""

    def __init__(self, config: VariantConfig, A: DeviceMatrix, precond: Precond, b, x0,
                 _handle=None):
        self.A = A  # borrowed, kept alive
        self.config = config
        self.precond = Precond(precond)
        if _handle is not None:  # a rank of a group (created by Group)
            self._h = _handle
            self.n = A.n
            return
        b, x0 = _f64(b), _f64(x0)
        if b.shape != (A.n,) or x0.shape != (A.n,):
            raise InvalidArgument(-1, "right-hand side or initial guess dimension mismatch")
        c = config._to_c()
        h = C.c_void_p()
        _check(_lib.cgvk_solver_create(A.handle, C.byref(c), int(precond), _ptr(b), _ptr(x0),
                                       C.byref(h)))
        self._h = h
        self.n = A.n

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.cgvk_solver_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def set_tolerance(self, rel_tol: float) -> None:
        _check(_lib.cgvk_solver_set_tolerance(self._h, float(rel_tol)))

    def step(self, n_iters: int = 1) -> None:
        """step() n times (src/variants.cpp:446-458), enqueued asynchronously."""
        _check(_lib.cgvk_solver_step(self._h, int(n_iters)))

    def sync(self) -> None:
        _check(_lib.cgvk_solver_sync(self._h))

    def _status(self):
        st, sc, stats = _Status(), _Scalars(), _Stats()
        _check(_lib.cgvk_solver_status(self._h, C.byref(st), C.byref(sc), C.byref(stats)))
        return st, sc, stats

    @property
    def status(self) -> SolveStatus:
        st, _, _ = self._status()
        return SolveStatus(State(st.state), Breakdown(st.breakdown), ConvergedBy(st.criterion))

    @property
    def k(self) -> int:
        return self._status()[0].k

    def allocated_vectors(self) -> int:
        return self._status()[0].allocated_vectors

    def scalars(self) -> dict:
        _, sc, _ = self._status()
        out = {f: getattr(sc, f) for f in SCALAR_NAMES}
        out["rr"] = sc.rr
        return out

    def stats(self) -> dict:
        _, _, s = self._status()
        return {f: getattr(s, f) for f in ("spmv_calls", "block_spmv_calls", "precond_applies",
                                           "reductions")}

    def vector(self, which: Vec, out: np.ndarray | None = None) -> np.ndarray:
        """Download a state vector (SolverState field) into `out` (a float64
        array of n, e.g. one registered with host_register for a direct DMA)
        or a new array."""
        if out is None:
            out = np.empty(self.n)
        elif out.dtype != np.float64 or out.shape != (self.n,) or not out.flags.c_contiguous:
            raise InvalidArgument(-1, "out must be a contiguous float64 array of n")
        _check(_lib.cgvk_solver_get_vector(self._h, int(which), _ptr(out) if self.n else None))
        return out

    def after(self, prev: "Solver") -> None:
        """Work enqueued on this solver from now on starts after everything
        already enqueued on `prev` (cgvk_solver_after)."""
        _check(_lib.cgvk_solver_after(self._h, prev._h))

    def x_async(self, out: np.ndarray) -> None:
        """Enqueue the download of x into `out` (contiguous float64 of n,
        registered with host_register); valid after sync()."""
        if out.dtype != np.float64 or out.shape != (self.n,) or not out.flags.c_contiguous:
            raise InvalidArgument(-1, "out must be a contiguous float64 array of n")
        _check(_lib.cgvk_solver_get_vector_async(self._h, int(Vec.X), _ptr(out) if self.n else None))

    def has_vector(self, which: Vec) -> bool:
        try:
            self.vector(which)
            return True
        except InvalidArgument:
            return False

    def true_residual(self) -> float:
        out = C.c_double()
        _check(_lib.cgvk_solver_true_residual(self._h, C.byref(out)))
        return out.value

    def history(self) -> np.ndarray:
        ln = C.c_int()
        _check(_lib.cgvk_solver_history(self._h, None, 0, C.byref(ln)))
        out = np.empty(max(ln.value, 1))
        _check(_lib.cgvk_solver_history(self._h, _ptr(out), ln.value, C.byref(ln)))
        if self._h and self.k + 1 > ln.value and ln.value == HISTORY_CAP:
            raise CgvkError(-1, f"residual history holds the first {HISTORY_CAP} iterations; k = {self.k}")
        return out[: ln.value]

    def stream(self) -> int:
        return _lib.cgvk_solver_stream(self._h) or 0

    def launches_per_iter(self) -> int:
        return _lib.cgvk_solver_launches_per_iter(self._h)

    def launches(self, n_iters: int) -> int:
        """Kernel launches one step(n_iters) call makes on this rank."""
        return int(_lib.cgvk_solver_launches(self._h, int(n_iters)))

    def time_steps(self, n_iters: int) -> tuple[float, int]:
        """Device time (ms) of n_iters graph-replayed iterations, and how many ran."""
        ms, it = C.c_double(), C.c_int()
        _check(_lib.cgvk_solver_time_steps(self._h, int(n_iters), C.byref(ms), C.byref(it)))
        return ms.value, it.value

    def profile(self, n_iters: int) -> tuple[float, float, int]:
        """Summed device ms of the update kernel and the SpMV kernel over n_iters."""
        a, b, it = C.c_double(), C.c_double(), C.c_int()
        _check(_lib.cgvk_solver_profile(self._h, int(n_iters), C.byref(a), C.byref(b),
                                        C.byref(it)))
        return a.value, b.value, it.value

    # reference-named accessors
    @property
    def x(self):
        return self.vector(Vec.X)

    @property
    def r(self):
        return self.vector(Vec.R)


def initialize(config: VariantConfig, A: DeviceMatrix, precond: Precond, b, x0) -> Solver:
    """initialize() (inc/variants.hpp:149-150)."""
    return Solver(config, A, precond, b, x0)


def step(state: Solver) -> None:
    """step() (inc/variants.hpp:153): exactly one iteration, synchronised;
    LogicError on a terminated state (src/variants.cpp:447), also one that
    initialize() settled (creation is stream-ordered, so the status is read
    here)."""
    if not state.status.running():
        raise LogicError(-2, "step() on a terminated solver")
    state.step(1)
    state.sync()


def solve(A: DeviceMatrix, config: VariantConfig, precond: Precond, b, x0, max_iter: int,
          rel_tol: float = 0.0):
    """run() with StopRule::fixed and probes off (+ optional ||r||/||b|| stop)."""
    b, x0 = _f64(b), _f64(x0)
    x = np.empty(A.n)
    st, sc = _Status(), _Scalars()
    c = config._to_c()
    _check(_lib.cgvk_solve(A.handle, C.byref(c), int(precond), _ptr(b), _ptr(x0), int(max_iter),
                           float(rel_tol), _ptr(x), C.byref(st), C.byref(sc)))
    return x, SolveStatus(State(st.state), Breakdown(st.breakdown), ConvergedBy(st.criterion)), st.k


# ------------------------------------------------------ run() with probes

@dataclass
class StopRule:
    """StopRule (inc/runner.hpp:9-36); the default kind is ResidualStagnation."""
    kind: str = "stagnation"  # "fixed" | "error_reduction" | "stagnation"
    fixed_count: int = 0
    error_threshold: float = 1e-5
    stagnation_window: int = 50
    stagnation_improvement: float = 0.01

    @classmethod
    def fixed(cls, count: int) -> "StopRule":
        return cls("fixed", fixed_count=count)

    @classmethod
    def error_reduction(cls, threshold: float) -> "StopRule":
        return cls("error_reduction", error_threshold=threshold)

    @classmethod
    def stagnation(cls, window: int = 50, improvement: float = 0.01) -> "StopRule":
        return cls("stagnation", stagnation_window=window, stagnation_improvement=improvement)

    def _to_c(self) -> _StopRule:
        kind = {"fixed": 0, "error_reduction": 1, "stagnation": 2}[self.kind]
        return _StopRule(kind, self.fixed_count, self.error_threshold, self.stagnation_window,
                         self.stagnation_improvement)


@dataclass
class ProbeOptions:
    """ProbeOptions (inc/runner.hpp:38-42): record every `cadence`-th iteration
    (plus k = 0 and the last); x_star enables the A-norm error ratios."""
    cadence: int = 1
    x_star: np.ndarray | None = None
    enabled: bool = True


@dataclass
class IterationRecord:
    """IterationRecord (inc/diagnostics.hpp:16-29); absent fields are None."""
    k: int = 0
    rel_err_a_norm: float | None = None
    true_res_norm: float | None = None
    upd_res_norm: float | None = None
    residual_gap_norm: float | None = None
    nu_gap: float | None = None
    w_gap_norm: float | None = None
    s_gap_norm: float | None = None
    lanczos_res_norm: float | None = None
    succ_orth: float | None = None
    alpha: float | None = None
    beta: float | None = None
    nu: float | None = None
    nu_prime: float | None = None


@dataclass
class Summary:
    iters_to_1e5: int | None
    min_log10_err: float


@dataclass
class ConvergenceHistory:
    """ConvergenceHistory (inc/diagnostics.hpp:62-69) plus the final x."""
    config: VariantConfig
    precond: Precond
    records: list
    final_status: SolveStatus
    summary: Summary | None
    x: np.ndarray


def run(config: VariantConfig, A: DeviceMatrix, precond: Precond, b, x0, max_iter: int,
        stop: StopRule | None = None, probe: ProbeOptions | None = None,
        rec_cap: int | None = None) -> ConvergenceHistory:
    """run() (inc/runner.hpp:47-49, src/runner.cpp:32-147) on the device:
    every probe quantity from fresh device products and reductions."""
    stop = stop if stop is not None else StopRule()
    probe = probe if probe is not None else ProbeOptions()
    b, x0 = _f64(b), _f64(x0)
    xs = _f64(probe.x_star) if probe.x_star is not None else None
    cap = rec_cap if rec_cap is not None else max_iter + 2
    recs = (_Record * max(cap, 1))()
    nrec = C.c_int()
    st, summ = _Status(), _Summary()
    x = np.empty(A.n)
    c = config._to_c()
    sr = stop._to_c()
    po = _ProbeOptions(int(probe.enabled), int(probe.cadence), _ptr(xs) if xs is not None else None)
    _check(_lib.cgvk_run(A.handle, C.byref(c), int(precond), _ptr(b), _ptr(x0), int(max_iter),
                         C.byref(sr), C.byref(po), C.cast(recs, C.c_void_p), cap, C.byref(nrec),
                         C.byref(st), C.byref(summ), _ptr(x)))
    out = []
    for q in range(min(nrec.value, cap)):
        r = recs[q]
        vals = {f: (float(r.v[i]) if r.mask >> i & 1 else None) for i, f in enumerate(RECORD_FIELDS)}
        out.append(IterationRecord(k=r.k, **vals))
    summary = (Summary(summ.iters_to_1e5 if summ.iters_to_1e5 >= 0 else None, summ.min_log10_err)
               if summ.has else None)
    return ConvergenceHistory(config, Precond(precond), out,
                              SolveStatus(State(st.state), Breakdown(st.breakdown),
                                          ConvergedBy(st.criterion)), summary, x)


def host_register(arr: np.ndarray) -> None:
    _check(_lib.cgvk_host_register(_ptr(arr), arr.nbytes))


def host_unregister(arr: np.ndarray) -> None:
    _check(_lib.cgvk_host_unregister(_ptr(arr)))


# ------------------------------------------------- row-partitioned solves

def partition_rows(n: int, nparts: int, align: int = 1) -> np.ndarray:
    """Row blocks [lo[r], lo[r+1]) cut at multiples of `align` (z-slabs)."""
    lo = np.empty(nparts + 1, np.int64)
    _check(_lib.cgvk_partition_rows(int(n), int(nparts), int(align), _ptr(lo)))
    return lo


def local_rows(csr, lo, rank: int):
    """Rank `rank`'s rows of a global CSR: local row_ptr, global columns, values."""
    a, b = int(lo[rank]), int(lo[rank + 1])
    k0, k1 = int(csr.row_ptr[a]), int(csr.row_ptr[b])
    return (np.ascontiguousarray(csr.row_ptr[a:b + 1] - k0), np.ascontiguousarray(csr.col_idx[k0:k1]),
            np.ascontiguousarray(csr.values[k0:k1]))


def halo_plan(n: int, lo, rank: int, row_ptr, col_idx) -> dict:
    lo, rp, ci = _i64(lo), _i64(row_ptr), _i64(col_idx)
    sizes = np.zeros(4, np.int64)
    _check(_lib.cgvk_halo_plan(int(n), lo.shape[0] - 1, _ptr(lo), int(rank), _ptr(rp),
                               _ptr(ci) if ci.size else None, _ptr(sizes), None, None, None, None))
    arrs = [np.empty(max(int(s), 1), np.int64) for s in sizes]
    _check(_lib.cgvk_halo_plan(int(n), lo.shape[0] - 1, _ptr(lo), int(rank), _ptr(rp),
                               _ptr(ci) if ci.size else None, _ptr(sizes), *[_ptr(x) for x in arrs]))
    names = ("lower", "upper", "send_lo", "send_hi")
    return {k: a[: int(s)] for k, a, s in zip(names, arrs, sizes)}


def rank_local_columns(n: int, lo, rank: int, row_ptr, col_idx):
    """The device's rank-local numbering of `rank`'s rows (host only):
    (local column indices, hbase) — own columns first, the lower then upper
    halo from hbase (own rows rounded up to 32 when there is a halo)."""
    lo, rp, ci = _i64(lo), _i64(row_ptr), _i64(col_idx)
    out = np.empty(max(ci.shape[0], 1), np.int64)
    hb = C.c_int64()
    _check(_lib.cgvk_rank_local_columns(int(n), lo.shape[0] - 1, _ptr(lo), int(rank), _ptr(rp),
                                        _ptr(ci) if ci.size else None, _ptr(out), C.byref(hb)))
    return out[: ci.shape[0]], int(hb.value)


class RankMatrix(DeviceMatrix):
    """Rows [lo[rank], lo[rank+1]) of a global n x n matrix, local numbering
    [own | pad | lower halo | upper halo] (cgvk_matrix_create_rank)."""

    def __init__(self, n: int, lo, rank: int, row_ptr, col_idx, values, device: int = 0):
        lo, rp, ci, va = _i64(lo), _i64(row_ptr), _i64(col_idx), _f64(values)
        h = C.c_void_p()
        _check(_lib.cgvk_matrix_create_rank(int(n), lo.shape[0] - 1, int(rank), _ptr(lo), _ptr(rp),
                                            _ptr(ci) if ci.size else None,
                                            _ptr(va) if va.size else None, device, C.byref(h)))
        self._h = h
        self.n = int(lo[rank + 1] - lo[rank])
        self.nnz = int(ci.shape[0])
        self.device = device
        self.rank = rank
        self.lo = lo


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(_lib.cgvk_comm_nccl_unique_id(buf))
    return bytes(buf)


class Comm:
    """Transport of a row-partitioned solve: NCCL (one process per GPU) or
    'local' (all ranks in this process on one device)."""

    def __init__(self, nranks: int, rank: int = 0, device: int = 0, nccl_id: bytes | None = None):
        h = C.c_void_p()
        if nccl_id is None:
            _check(_lib.cgvk_comm_create_local(int(nranks), device, C.byref(h)))
            self.kind = "local"
        else:
            buf = (C.c_char * 128).from_buffer_copy(nccl_id)
            _check(_lib.cgvk_comm_create_nccl(buf, int(nranks), int(rank), device, C.byref(h)))
            self.kind = "nccl"
        self._h = h
        self.nranks, self.rank = nranks, rank

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.cgvk_comm_destroy(self._h)
            self._h = None

    __del__ = close


class Group:
    """initialize() of one solve over the ranks this process drives."""

    P2P = 1  # CGVK_GROUP_P2P: halos and rank totals through peer memory inside the kernels

    def __init__(self, comm: Comm, mats: list, config: VariantConfig, precond: Precond, bs: list,
                 x0s: list, p2p: bool = False):
        self.comm, self.mats = comm, mats
        bs = [_f64(b) for b in bs]
        x0s = [_f64(x) for x in x0s]
        nl = len(mats)
        hs = (C.c_void_p * nl)(*[m.handle for m in mats])
        bp = (C.c_void_p * nl)(*[_ptr(b) if b.size else None for b in bs])
        xp = (C.c_void_p * nl)(*[_ptr(x) if x.size else None for x in x0s])
        out = (C.c_void_p * nl)()
        c = config._to_c()
        _check(_lib.cgvk_group_create_ex(comm._h, nl, hs, C.byref(c), int(precond), bp, xp,
                                         self.P2P if p2p else 0, out))
        self._handles = out
        self.transport = "p2p" if _lib.cgvk_group_transport(out[0]) == self.P2P else comm.kind
        self.solvers = [Solver(config, m, precond, None, None, _handle=C.c_void_p(out[i]))
                        for i, m in enumerate(mats)]

    def step(self, n_iters: int = 1) -> None:
        _check(_lib.cgvk_group_step(self._handles, len(self.mats), int(n_iters)))

    def sync(self) -> None:
        for s in self.solvers:
            s.sync()

    def true_residual(self) -> float:
        out = C.c_double()
        _check(_lib.cgvk_group_true_residual(self._handles, len(self.mats), C.byref(out)))
        return out.value

    def vector(self, which: Vec) -> np.ndarray:
        """The global vector (concatenation of the ranks' own rows; local comm)."""
        return np.concatenate([s.vector(which) for s in self.solvers])

    def close(self) -> None:
        for s in self.solvers:
            s.close()
        self.solvers = []
