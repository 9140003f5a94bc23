"""Python mirror of the reference's ``ridgepath::`` solver API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/ridgepath/{sketch,spectrum,preconditioner,
path_solver,matrix}.hpp; every call runs on the GPU through
``libridgepath_b200.so`` (include/ridgepath_b200.h).  There is no CPU
fallback: without the library or a CUDA device the calls raise.

Exceptions: std::invalid_argument -> ValueError, BasisDivergedError,
SolverError (path_solver.hpp:18-27), thin_svd failure -> FactorizationError.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libridgepath_b200.so")

RP_HOST, RP_DEVICE, RP_HOST_STREAM = 0, 1, 2
SKETCH_KINDS = ("gaussian", "countsketch", "sjlt", "srht", "identity")
RHO_PROVENANCE = ("gaussian", "sjlt", "srht", "identity", "manual")


class BasisDivergedError(RuntimeError):
    """path_solver.hpp:18-21."""


class SolverError(RuntimeError):
    """path_solver.hpp:23-27."""


class FactorizationError(RuntimeError):
    """Shifted sketched Gram not positive definite (the reference's thin_svd
    runtime_error slot, matrix.cpp:227-228)."""


class DeviceError(RuntimeError):
    pass


class ParseError(RuntimeError):
    """data_io.hpp ParseError: "line L, column C: ..." with 1-based .line / .column."""

    def __init__(self, message: str, line: int = 0, column: int = 0):
        super().__init__(message)
        self.line = line
        self.column = column


# ---------------------------------------------------------------------------
# ctypes binding
# ---------------------------------------------------------------------------


class _SketchSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("s", ctypes.c_int32), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("seed", ctypes.c_uint64)]


class _PathConfig(ctypes.Structure):
    _fields_ = [("lambda_min", ctypes.c_double), ("lambda_max", ctypes.c_double),
                ("lambdas", ctypes.POINTER(ctypes.c_double)), ("num_lambdas", ctypes.c_int64),
                ("epsilon", ctypes.c_double), ("num_intervals", ctypes.c_int32)]


class _Rho(ctypes.Structure):
    _fields_ = [("rho1", ctypes.c_double), ("rho2", ctypes.c_double), ("provenance", ctypes.c_int32)]


class _SpectrumInfo(ctypes.Structure):
    _fields_ = [("effective_dimension", ctypes.c_double), ("sigma_max_sq", ctypes.c_double),
                ("dnorm_sq", ctypes.c_double), ("lambda0", ctypes.c_double), ("lanczos_steps", ctypes.c_int32)]


class _AdaptiveConfig(ctypes.Structure):
    _fields_ = [("gamma1", ctypes.c_double), ("gamma2", ctypes.c_double), ("gamma3", ctypes.c_double),
                ("epsilon", ctypes.c_double), ("m_initial", ctypes.c_int64), ("m_cap", ctypes.c_int64),
                ("iteration_cap", ctypes.c_int32)]


class _AdaptiveStep(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("f_before", ctypes.c_double), ("f_after", ctypes.c_double),
                ("step", ctypes.c_double), ("progress", ctypes.c_double), ("doubled", ctypes.c_int32)]


class _AdaptiveResult(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("iterations", ctypes.c_int32), ("doublings", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("stalled_at_cap", ctypes.c_int32), ("trace_len", ctypes.c_int64)]


class _Rate(ctypes.Structure):
    _fields_ = [("lambda0", ctypes.c_double), ("alpha", ctypes.c_double), ("kappa", ctypes.c_double),
                ("contraction", ctypes.c_double), ("k", ctypes.c_int32)]


class Timings(ctypes.Structure):
    _fields_ = [("setup_seconds", ctypes.c_double), ("eval_seconds", ctypes.c_double),
                ("total_seconds", ctypes.c_double), ("sketch_seconds", ctypes.c_double),
                ("factor_seconds", ctypes.c_double), ("basis_seconds", ctypes.c_double),
                ("copy_seconds", ctypes.c_double), ("retries", ctypes.c_int32), ("gram_mode", ctypes.c_int32),
                ("launches", ctypes.c_int64), ("gemm_seconds", ctypes.c_double), ("gemm_flops", ctypes.c_double),
                ("gemm_calls", ctypes.c_int64), ("linear_seconds", ctypes.c_double),
                ("gram_seconds", ctypes.c_double), ("precond_seconds", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None

_P = ctypes.c_void_p
_D = ctypes.c_double
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int32
_INT = ctypes.c_int

# Every symbol declared in include/ridgepath_b200.h with its signature.
SIGNATURES = {
    "rp_version": ([], ctypes.c_char_p),
    "rp_create": ([ctypes.POINTER(_P), _INT], _INT),
    "rp_destroy": ([_P], None),
    "rp_last_error": ([_P], ctypes.c_char_p),
    "rp_set_stream": ([_P, _P], _INT),
    "rp_synchronize": ([_P], _INT),
    "rp_set_option": ([_P, ctypes.c_char_p, _I64], _INT),
    "rp_launch_count": ([], _I64),
    "rp_comm_unique_id": ([_P], _INT),
    "rp_comm_init": ([_P, _INT, _INT, _P], _INT),
    "rp_comm_init_host": ([_P, _INT, _INT, _P, _P, _P], _INT),
    "rp_set_dense": ([_P, _I64, _I64, _P, _I64, _INT], _INT),
    "rp_set_dense_rows": ([_P, _I64, _I64, _I64, _I64, _P, _I64, _INT], _INT),
    "rp_set_dense_cols": ([_P, _I64, _I64, _I64, _I64, _P, _I64, _INT], _INT),
    "rp_set_csr": ([_P, _I64, _I64, _P, _P, _P, _INT], _INT),
    "rp_set_csr_rows": ([_P, _I64, _I64, _I64, _I64, _P, _P, _P, _INT], _INT),
    "rp_apply": ([_P, _P, _I64, _P, _INT], _INT),
    "rp_apply_transpose": ([_P, _P, _I64, _P, _INT], _INT),
    "rp_gram_apply": ([_P, _P, _I64, _P, _INT], _INT),
    "rp_losses": ([_P, _P, _I64, _I64, _P, _P, _P, _INT], _INT),
    "rp_last_device_seconds": ([_P, ctypes.POINTER(_D)], _INT),
    "rp_sketch_apply": ([_P, ctypes.POINTER(_SketchSpec), _INT, _P, _INT], _INT),
    "rp_precond_build": ([_P, _P, _I64, _I64, _D, _INT, ctypes.POINTER(_P)], _INT),
    "rp_precond_reshift": ([_P, _P, _D, ctypes.POINTER(_P)], _INT),
    "rp_precond_apply": ([_P, _P, _P, _I64, _P, _INT], _INT),
    "rp_precond_destroy": ([_P], None),
    "rp_ihs_basis": ([_P, _P, _P, _I64, _D, _I32, _P, _INT], _INT),
    "rp_ihs_basis_core": ([_P, _P, _P, _I64, _D, _I32, _INT, _P, _INT], _INT),
    "rp_ihs_compose": ([_P, _P, _I64, _I64, _I32, _D, _D, _P, _INT], _INT),
    "rp_ihs_bin_path": ([_P, _P, _I64, ctypes.POINTER(_PathConfig), ctypes.POINTER(_SketchSpec),
                         ctypes.POINTER(_Rho), _P, _P, _INT, ctypes.POINTER(Timings)], _INT),
    "rp_dual_path": ([_P, _P, _I64, ctypes.POINTER(_PathConfig), ctypes.POINTER(_SketchSpec),
                      ctypes.POINTER(_Rho), _P, _P, _INT, ctypes.POINTER(Timings)], _INT),
    "rp_log_grid": ([_D, _D, _I32, _P], _INT),
    "rp_tune_interval": ([_D, _D, ctypes.POINTER(_Rho), _P, _D, ctypes.POINTER(_Rate)], _INT),
    "rp_auto_interval_count": ([_D, _D], _I32),
    "rp_interval_split": ([_D, _D, _I32, _P, ctypes.POINTER(_I32)], _INT),
    "rp_draw_u64": ([_P, _U64, _U64, _I64, _P, _INT], _INT),
    "rp_draw_uniform01": ([_P, _U64, _I64, _P, _INT], _INT),
    "rp_draw_sign": ([_P, _U64, _I64, _P, _INT], _INT),
    "rp_draw_uniform_index": ([_P, _U64, _U64, _I64, _P, _INT], _INT),
    "rp_draw_normals": ([_P, _U64, _I64, _I64, _D, _P, _INT], _INT),
    "rp_gaussian_window": ([_P, _U64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _INT], _INT),
    "rp_count_draws": ([_P, ctypes.POINTER(_SketchSpec), _P, _P, _INT], _INT),
    "rp_srht_draws": ([_P, ctypes.POINTER(_SketchSpec), _P, _P, _INT], _INT),
    "rp_mt_selfcheck": ([_U64, _U64], _INT),
    "rp_warm_cg_path": ([_P, _P, ctypes.POINTER(_PathConfig), _P, _INT, _P, _P, _P], _INT),
    "rp_warm_ihs_path": ([_P, _P, ctypes.POINTER(_PathConfig), ctypes.POINTER(_SketchSpec), ctypes.POINTER(_Rho), _P,
                          _INT, _P, _P, _P], _INT),
    "rp_direct_path": ([_P, _P, ctypes.POINTER(_PathConfig), _P, _INT, _P, _P], _INT),
    "rp_svd_path": ([_P, _P, ctypes.POINTER(_PathConfig), _P, _INT, _P, _P], _INT),
    "rp_libsvm_parse": ([ctypes.c_char_p, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P], _INT),
    "rp_write_csv": ([_I64, _P, _P, _P, _P, _P, _P, _P, ctypes.c_char_p, _I64, _P], _INT),
    "rp_adaptive_sketch_dim": ([_P, _P, _D, ctypes.POINTER(_AdaptiveConfig), ctypes.POINTER(_SketchSpec), _P, _P, _INT,
                                ctypes.POINTER(_AdaptiveResult), _P, _I64], _INT),
    "rp_last_gemm_profile": ([_P, _P, _P, _P, _I64, _P], _INT),
    "rp_derive_rho": ([_P, ctypes.POINTER(_SketchSpec), _INT, _D, _D, ctypes.POINTER(_Rho),
                       ctypes.POINTER(_SpectrumInfo)], _INT),
    "rp_effective_dimension": ([_P, _I64, _D, _P], _INT),
    "rp_rho_gaussian": ([_D, _D, _D, _I64, ctypes.POINTER(_Rho), _P], _INT),
    "rp_rho_srht": ([_D, _D, _I64, _D, ctypes.POINTER(_Rho), _P], _INT),
    "rp_rho_sjlt": ([_D, _D, _D, _D, ctypes.POINTER(_Rho), _P, _P], _INT),
}


def lib():
    """Loads libridgepath_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() (make -C paper_2210_12212_b200)")
    L = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


_ERRORS = {1: ValueError, 2: BasisDivergedError, 3: SolverError, 4: FactorizationError, 5: DeviceError,
           6: DeviceError, 7: MemoryError}


def _check(st: int, ctx=None):
    if st != 0:
        msg = lib().rp_last_error(ctx).decode() if ctx is not None else lib().rp_last_error(None).decode()
        raise _ERRORS.get(st, DeviceError)(msg or f"rp status {st}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------------
# Value types (sketch.hpp, spectrum.hpp, path_solver.hpp)
# ---------------------------------------------------------------------------


@dataclass
class SketchSpec:
    """sketch.hpp:17-29."""
    kind: str = "identity"
    m: int = 0
    n: int = 0
    s: int = 1
    seed: int = 0

    def c(self) -> _SketchSpec:
        if self.kind not in SKETCH_KINDS:
            raise ValueError("unknown sketch kind: " + str(self.kind))
        return _SketchSpec(SKETCH_KINDS.index(self.kind), int(self.s), int(self.m), int(self.n), int(self.seed))

    def with_m(self, m):
        return SketchSpec(self.kind, m, self.n, self.s, self.seed)

    def with_seed(self, seed):
        return SketchSpec(self.kind, self.m, self.n, self.s, seed)


@dataclass
class RhoBounds:
    """spectrum.hpp:32-40."""
    rho1: float = 1.0
    rho2: float = 1.0
    provenance: str = "identity"

    def c(self) -> _Rho:
        return _Rho(float(self.rho1), float(self.rho2), RHO_PROVENANCE.index(self.provenance))

    @staticmethod
    def identity():
        return RhoBounds(1.0, 1.0, "identity")

    @staticmethod
    def manual(rho1, rho2):
        if not rho2 > 0.0:
            raise ValueError("rho bounds: rho2 must be positive")
        if not rho1 >= rho2:
            raise ValueError("rho bounds: rho1 must be >= rho2")
        return RhoBounds(float(rho1), float(rho2), "manual")


@dataclass
class PathConfig:
    """spectrum.hpp:14-22 (num_intervals None = auto)."""
    lambda_min: float = 0.0
    lambda_max: float = 0.0
    lambdas: Sequence[float] = field(default_factory=list)
    epsilon: float = 1e-6
    num_intervals: Optional[int] = None

    def c(self):
        arr = np.ascontiguousarray(np.asarray(self.lambdas, dtype=np.float64))
        cfg = _PathConfig(float(self.lambda_min), float(self.lambda_max),
                          arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(arr.shape[0]),
                          float(self.epsilon), int(self.num_intervals) if self.num_intervals is not None else 0)
        if self.num_intervals is not None and self.num_intervals < 1:
            raise ValueError("path config: L must be >= 1")
        return cfg, arr


@dataclass
class RateParams:
    lambda0: float
    alpha: float
    kappa: float
    contraction: float
    k: int


@dataclass
class Csr:
    """CsrMatrix (matrix.hpp:16-50): int64 offsets/columns, float64 values."""
    rows: int
    cols: int
    offsets: np.ndarray
    indices: np.ndarray
    values: np.ndarray

    @property
    def shape(self):
        return (self.rows, self.cols)


@dataclass
class SketchedMatrix:
    product: np.ndarray
    spec: SketchSpec


@dataclass
class BinomialBasis:
    """path_solver.hpp:34-44: k blocks of dim x K."""
    terms: List[np.ndarray]
    tau: float = 0.0
    lambda_lo: float = 0.0
    lambda_hi: float = 0.0
    flavor: str = "ihs"

    @property
    def k(self):
        return len(self.terms)


@dataclass
class PathPoint:
    lam: float
    solution: np.ndarray
    seconds: float = 0.0
    train_loss: float = 0.0  # 0.5 ||A x - b||^2 + 0.5 lam ||x||^2  (path_solver.cpp:425-439)
    test_loss: Optional[float] = None  # 0.5 ||A_test x - b_test||^2 when a test set is given
    iterations: int = 0  # inner iterations (the iterative baselines, baselines.cpp:25-38)


@dataclass
class RegPathResult:
    solver: str
    points: List[PathPoint]
    setup_seconds: float = 0.0
    total_seconds: float = 0.0
    timings: Optional[dict] = None


# ---------------------------------------------------------------------------
# Scalar tuning (host code of the library; bit-identical to spectrum.cpp)
# ---------------------------------------------------------------------------


def log_grid(lambda_min: float, lambda_max: float, count: int) -> List[float]:
    out = np.empty(max(int(count), 1), dtype=np.float64)
    _check(lib().rp_log_grid(lambda_min, lambda_max, int(count), _ptr(out)))
    return out[:count].tolist()


def tune_interval(lambda_lo, lambda_hi, rho: RhoBounds, sigma_d=None, eps=1e-6) -> RateParams:
    r = _Rate()
    sd = ctypes.c_double(sigma_d) if sigma_d is not None else None
    _check(lib().rp_tune_interval(lambda_lo, lambda_hi, ctypes.byref(rho.c()),
                                  ctypes.cast(ctypes.byref(sd), _P) if sd is not None else None, eps, ctypes.byref(r)))
    return RateParams(r.lambda0, r.alpha, r.kappa, r.contraction, r.k)


def _rho_py(r: "_Rho") -> RhoBounds:
    return RhoBounds(r.rho1, r.rho2, RHO_PROVENANCE[r.provenance])


def effective_dimension(sigma, lambda0: float) -> float:
    """spectrum.cpp:87-103 (host)."""
    sig = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64).reshape(-1))
    out = ctypes.c_double(0.0)
    _check(lib().rp_effective_dimension(_ptr(sig) if sig.size else None, sig.size, float(lambda0),
                                        ctypes.cast(ctypes.byref(out), _P)))
    return out.value


def rho_gaussian(rho, eta, dnorm_sq, m=None):
    """spectrum.cpp:105-128 -> (RhoBounds, success_probability or None)."""
    r, p = _Rho(), ctypes.c_double(0.0)
    _check(lib().rp_rho_gaussian(rho, eta, dnorm_sq, int(m) if m is not None else 0, ctypes.byref(r),
                                 ctypes.cast(ctypes.byref(p), _P)))
    return _rho_py(r), (p.value if m is not None else None)


def rho_srht(rho, dnorm_sq, n_and_de=None):
    """spectrum.cpp:130-148 -> (RhoBounds, recommended_m or None)."""
    r, rec = _Rho(), _I64(0)
    n, de = n_and_de if n_and_de is not None else (0, 0.0)
    _check(lib().rp_rho_srht(rho, dnorm_sq, int(n), float(de), ctypes.byref(r), ctypes.cast(ctypes.byref(rec), _P)))
    return _rho_py(r), (rec.value if n_and_de is not None else None)


def rho_sjlt(eps, alpha_delta_de=None):
    """spectrum.cpp:150-169 -> (RhoBounds, recommended_m or None, recommended_s or None)."""
    r, rm, rs = _Rho(), _I64(0), _I32(0)
    alpha, delta, de = alpha_delta_de if alpha_delta_de is not None else (0.0, 0.0, 0.0)
    _check(lib().rp_rho_sjlt(eps, float(alpha), float(delta), float(de), ctypes.byref(r), ctypes.cast(ctypes.byref(rm), _P),
                             ctypes.cast(ctypes.byref(rs), _P)))
    if alpha_delta_de is None:
        return _rho_py(r), None, None
    return _rho_py(r), rm.value, rs.value


def derive_rho(spec: "SketchSpec", a, lambda_min: float, lambda_max: float, ctx: Optional["Context"] = None,
               transpose_op: bool = False):
    """The CLI's plug-in envelope (tools/ridgepath_main.cpp:218-279) on the
    device: returns (RhoBounds, info dict).  Identity sketches return identity
    bounds without sketching."""
    ctx = ctx or default_context()
    if spec.kind != "identity":
        ctx.set_operator(a)
    r, info = _Rho(), _SpectrumInfo()
    ctx.check(lib().rp_derive_rho(ctx.handle, ctypes.byref(spec.c()), int(bool(transpose_op)), float(lambda_min),
                                  float(lambda_max), ctypes.byref(r), ctypes.byref(info)))
    if spec.kind == "identity":
        return _rho_py(r), {}
    return _rho_py(r), dict(effective_dimension=info.effective_dimension, sigma_max_sq=info.sigma_max_sq,
                            dnorm_sq=info.dnorm_sq, lambda0=info.lambda0, lanczos_steps=info.lanczos_steps)


def auto_interval_count(lambda_min, lambda_max) -> int:
    v = lib().rp_auto_interval_count(lambda_min, lambda_max)
    if v < 0:
        raise ValueError(lib().rp_last_error(None).decode())
    return v


def interval_split(lambda_min, lambda_max, num_intervals=None):
    cnt = _I32(0)
    _check(lib().rp_interval_split(lambda_min, lambda_max, int(num_intervals or 0), None, ctypes.byref(cnt)))
    edges = np.empty(2 * cnt.value, dtype=np.float64)
    _check(lib().rp_interval_split(lambda_min, lambda_max, int(num_intervals or 0), _ptr(edges), ctypes.byref(cnt)))
    return [(edges[2 * i], edges[2 * i + 1]) for i in range(cnt.value)]


def hadamard_pad(n: int) -> int:
    """sketch.cpp:190-193."""
    p = 1
    while p < max(n, 1):
        p <<= 1
    return p


# ---------------------------------------------------------------------------
# Context
# ---------------------------------------------------------------------------


class Context:
    """One GPU (rp_ctx).  Holds the data operator resident in HBM."""

    def __init__(self, device: int = 0):
        self._h = _P()
        _check(lib().rp_create(ctypes.byref(self._h), int(device)))
        self.device = device
        self._op_key = None
        self._keep = None

    def __del__(self):
        try:
            if self._h:
                lib().rp_destroy(self._h)
                self._h = _P()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def check(self, st):
        _check(st, self._h)

    def set_option(self, key: str, value: int):
        self.check(lib().rp_set_option(self._h, key.encode(), int(value)))

    def set_stream(self, stream_ptr: Optional[int]):
        self.check(lib().rp_set_stream(self._h, _P(stream_ptr) if stream_ptr else None))

    def synchronize(self):
        self.check(lib().rp_synchronize(self._h))

    # -- operator ------------------------------------------------------------
    def set_operator(self, a, force: bool = False):
        """Dense (numpy, n x d) or Csr; a torch CUDA tensor is used in place
        (column-major: pass A.T-contiguous storage, i.e. a tensor whose
        transpose is contiguous).

        Host operators (numpy, Csr) are uploaded on every call, like the
        reference reads A on every call: a caller may change them in place
        between calls.  A device tensor is used in place (its current contents
        are what the kernels read), so re-registering the same storage is
        skipped."""
        key = None
        if _is_torch_cuda(a):
            key = (a.data_ptr(), tuple(a.shape), tuple(a.stride()))
            if not force and key == self._op_key:
                return
        if isinstance(a, Csr):
            off = np.ascontiguousarray(a.offsets, dtype=np.int64)
            idx = np.ascontiguousarray(a.indices, dtype=np.int64)
            val = np.ascontiguousarray(a.values, dtype=np.float64)
            self.check(lib().rp_set_csr(self._h, a.rows, a.cols, _ptr(off), _ptr(idx), _ptr(val), RP_HOST))
            self._keep = None
        elif _is_torch_cuda(a):
            n, d = a.shape
            ld = _torch_colmajor_ld(a)
            self.check(lib().rp_set_dense(self._h, n, d, _P(a.data_ptr()), ld, RP_DEVICE))
            self._keep = a
        else:
            af = _f64(a)
            n, d = af.shape
            self.check(lib().rp_set_dense(self._h, n, d, _ptr(af), max(n, 1), RP_HOST))
            self._keep = None
        self._op_key = key
        self._op = a

    def draws_u64(self, seed, count, skip=0):
        out = np.empty(max(count, 1), dtype=np.uint64)
        self.check(lib().rp_draw_u64(self._h, seed, skip, count, _ptr(out), RP_HOST))
        return out[:count]


def _is_torch_cuda(a) -> bool:
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _torch_colmajor_ld(a) -> int:
    n, d = a.shape
    st = a.stride()
    if st[0] == 1 and (d <= 1 or st[1] >= max(n, 1)):
        return int(st[1]) if d > 1 else max(n, 1)
    raise ValueError("device operator must be column-major (A.t() contiguous)")


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(int(os.environ.get("RP_DEVICE", "0")))
    return _default


def _rows(a):
    return a.rows if isinstance(a, Csr) else a.shape[0]


def _cols(a):
    return a.cols if isinstance(a, Csr) else a.shape[1]


# ---------------------------------------------------------------------------
# matrix.hpp
# ---------------------------------------------------------------------------


def apply(a, x, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    x2 = _f64(np.asarray(x).reshape(np.asarray(x).shape[0], -1))
    if x2.shape[0] != _cols(a):
        raise ValueError("apply: dimension mismatch")
    out = np.empty((_rows(a), x2.shape[1]), order="F")
    ctx.check(lib().rp_apply(ctx.handle, _ptr(x2), x2.shape[1], _ptr(out), RP_HOST))
    return out.reshape((_rows(a),) + np.asarray(x).shape[1:])


def apply_transpose(a, y, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    y2 = _f64(np.asarray(y).reshape(np.asarray(y).shape[0], -1))
    if y2.shape[0] != _rows(a):
        raise ValueError("apply_transpose: dimension mismatch")
    out = np.empty((_cols(a), y2.shape[1]), order="F")
    ctx.check(lib().rp_apply_transpose(ctx.handle, _ptr(y2), y2.shape[1], _ptr(out), RP_HOST))
    return out.reshape((_cols(a),) + np.asarray(y).shape[1:])


def gram_apply(a, x, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    x2 = _f64(np.asarray(x).reshape(np.asarray(x).shape[0], -1))
    if x2.shape[0] != _cols(a):
        raise ValueError("gram_apply: dimension mismatch")
    out = np.empty((_cols(a), x2.shape[1]), order="F")
    ctx.check(lib().rp_gram_apply(ctx.handle, _ptr(x2), x2.shape[1], _ptr(out), RP_HOST))
    return out.reshape((_cols(a),) + np.asarray(x).shape[1:])


# ---------------------------------------------------------------------------
# sketch.hpp
# ---------------------------------------------------------------------------


def sketch_apply(spec: SketchSpec, a, ctx: Optional[Context] = None, transpose_op: bool = False) -> SketchedMatrix:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    d = _rows(a) if transpose_op else _cols(a)
    if spec.m < 1:
        raise ValueError("sketch: m must be positive")
    out = np.empty((spec.m, d), order="F")
    cs = spec.c()
    ctx.check(lib().rp_sketch_apply(ctx.handle, ctypes.byref(cs), int(transpose_op), _ptr(out), RP_HOST))
    return SketchedMatrix(out, spec)


# ---------------------------------------------------------------------------
# preconditioner.hpp
# ---------------------------------------------------------------------------


class Preconditioner:
    """(SA^T SA + lambda0 I)^{-1}, preconditioner.hpp:24-34."""

    def __init__(self, handle, ctx: Context, m: int, d: int, lambda0: float):
        self._h = handle
        self._ctx = ctx
        self.m, self.d, self._lambda0 = m, d, lambda0

    def __del__(self):
        try:
            if self._h:
                lib().rp_precond_destroy(self._h)
                self._h = _P()
        except Exception:
            pass

    @staticmethod
    def build(sa, lambda0: float, ctx: Optional[Context] = None) -> "Preconditioner":
        ctx = ctx or default_context()
        prod = sa.product if isinstance(sa, SketchedMatrix) else sa
        p = _f64(prod)
        h = _P()
        ctx.check(lib().rp_precond_build(ctx.handle, _ptr(p), p.shape[0], p.shape[1], float(lambda0), RP_HOST,
                                         ctypes.byref(h)))
        return Preconditioner(h, ctx, p.shape[0], p.shape[1], float(lambda0))

    def reshift(self, new_lambda0: float) -> "Preconditioner":
        h = _P()
        self._ctx.check(lib().rp_precond_reshift(self._ctx.handle, self._h, float(new_lambda0), ctypes.byref(h)))
        return Preconditioner(h, self._ctx, self.m, self.d, float(new_lambda0))

    def apply(self, v) -> np.ndarray:
        v = np.asarray(v)
        v2 = _f64(v.reshape(v.shape[0], -1))
        if v2.shape[0] != self.d:
            raise ValueError("preconditioner apply: dimension mismatch")
        out = np.empty_like(v2, order="F")
        self._ctx.check(lib().rp_precond_apply(self._ctx.handle, self._h, _ptr(v2), v2.shape[1], _ptr(out), RP_HOST))
        return out.reshape(v.shape)

    def lambda0(self):
        return self._lambda0

    def dim(self):
        return self.d

    def sketch_rows(self):
        return self.m


# ---------------------------------------------------------------------------
# path_solver.hpp
# ---------------------------------------------------------------------------


def _terms_from(buf: np.ndarray, dim: int, K: int, k: int) -> List[np.ndarray]:
    flat = buf.reshape(-1, order="F")
    return [flat[j * dim * K:(j + 1) * dim * K].reshape((dim, K), order="F").copy() for j in range(k)]


def ihs_basis(a, b, p: Preconditioner, tau: float, k: int, ctx: Optional[Context] = None) -> BinomialBasis:
    """path_solver.hpp:89-96 (vector b); ihs_basis_matrix for a matrix b."""
    ctx = ctx or p._ctx
    ctx.set_operator(a)
    b = np.asarray(b)
    if b.shape[0] != _rows(a):
        raise ValueError("ihs_basis: dimension mismatch")
    b2 = _f64(b.reshape(b.shape[0], -1))
    K = b2.shape[1]
    dim = _cols(a)
    out = np.empty(dim * K * max(k, 1))
    ctx.check(lib().rp_ihs_basis(ctx.handle, p._h, _ptr(b2), K, float(tau), int(k), _ptr(out), RP_HOST))
    return BinomialBasis(_terms_from(out, dim, K, k), float(tau))


ihs_basis_matrix = ihs_basis


def ihs_compose(basis: BinomialBasis, lam: float, ctx: Optional[Context] = None) -> np.ndarray:
    """path_solver.hpp:98-101: tau * sum_j (tau lambda)^j u_j (Horner)."""
    if basis.flavor != "ihs":
        raise ValueError("ihs_compose: wrong basis flavor")
    ctx = ctx or default_context()
    dim, K = basis.terms[0].shape
    terms = np.concatenate([np.asfortranarray(t).reshape(-1, order="F") for t in basis.terms])
    out = np.empty((dim, K), order="F")
    ctx.check(lib().rp_ihs_compose(ctx.handle, _ptr(terms), dim, K, basis.k, float(basis.tau), float(lam), _ptr(out),
                                   RP_HOST))
    return out[:, 0] if K == 1 else out


def ihs_compose_matrix(basis: BinomialBasis, lam: float, ctx: Optional[Context] = None) -> np.ndarray:
    out = ihs_compose(basis, lam, ctx)
    return out.reshape(basis.terms[0].shape)


def losses(a, b, x, lambdas=None, ctx: Optional[Context] = None) -> np.ndarray:
    """losses / losses_matrix (path_solver.cpp:425-454) for T solutions at once:
    x is d x K x T (or d x T for K = 1), b is n x K; returns
    0.5 ||A X_t - B||_F^2 (+ 0.5 lambda_t ||X_t||_F^2 when lambdas is given)."""
    ctx = ctx or default_context()
    ctx.set_operator(a)
    b2 = _f64(np.asarray(b).reshape(np.asarray(b).shape[0], -1))
    K = b2.shape[1]
    x = np.asarray(x, dtype=np.float64)
    d = _cols(a)
    T = x.size // (d * K) if x.size else 0
    if b2.shape[0] != _rows(a) or x.size != d * K * T:
        raise ValueError("losses: dimension mismatch")
    xs = np.ascontiguousarray(x.reshape(d, K, T).transpose(2, 1, 0)).reshape(-1)  # t-major, column-major d x K
    lam = _f64(np.asarray(lambdas, dtype=np.float64)) if lambdas is not None else None
    out = np.empty(max(T, 1))
    ctx.check(lib().rp_losses(ctx.handle, _ptr(b2.reshape(-1, order="F").copy()), K, T, _ptr(xs),
                              _ptr(lam) if lam is not None else None, _ptr(out), RP_HOST))
    return out[:T]


def _run_path(dual: bool, a, b, config: PathConfig, spec: SketchSpec, rho: RhoBounds, sigma_d=None,
              ctx: Optional[Context] = None, return_timings=False, a_test=None, b_test=None) -> RegPathResult:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    b = np.asarray(b)
    if b.shape[0] != _rows(a):
        raise ValueError(("dual_path" if dual else "ihs_bin_path") + ": dimension mismatch")
    b2 = _f64(b.reshape(b.shape[0], -1))
    K = b2.shape[1]
    T = len(config.lambdas)
    dim = _cols(a)
    out = np.empty(dim * K * max(T, 1))
    cfg, keep = config.c()
    cs, cr = spec.c(), rho.c()
    sd = ctypes.c_double(sigma_d) if sigma_d is not None else None
    tm = Timings()
    fn = lib().rp_dual_path if dual else lib().rp_ihs_bin_path
    ctx.check(fn(ctx.handle, _ptr(b2), K, ctypes.byref(cfg), ctypes.byref(cs), ctypes.byref(cr),
                 ctypes.cast(ctypes.byref(sd), _P) if sd is not None else None, _ptr(out), RP_HOST,
                 ctypes.byref(tm)))
    del keep
    # per-point losses as the reference's loss callbacks (path_solver.cpp:298-303,
    # 318-323, 342-347): train always, test when a test set is given
    lam = np.asarray(config.lambdas, dtype=np.float64)
    primal_dim = _cols(a)
    train = _losses_flat(ctx, b2, K, T, out, lam) if T else np.empty(0)
    test = None
    if a_test is not None and b_test is not None and T:
        bt = _f64(np.asarray(b_test).reshape(np.asarray(b_test).shape[0], -1))
        if _cols(a_test) != primal_dim or bt.shape[1] != K or bt.shape[0] != _rows(a_test):
            raise ValueError("losses: test dimension mismatch")
        ctx.set_operator(a_test)
        test = _losses_flat(ctx, bt, K, T, out, None)
        ctx.set_operator(a)
    pts = []
    for t in range(T):
        x = out[t * dim * K:(t + 1) * dim * K].reshape((dim, K), order="F").copy()
        pts.append(PathPoint(float(config.lambdas[t]), x, train_loss=float(train[t]),
                             test_loss=float(test[t]) if test is not None else None))
    return RegPathResult("dual" if dual else "ihs-bin", pts, tm.setup_seconds, tm.total_seconds, tm.as_dict())


def _losses_flat(ctx, b2, K, T, x_flat, lam):
    out = np.empty(max(T, 1))
    ctx.check(lib().rp_losses(ctx.handle, _ptr(np.asfortranarray(b2).reshape(-1, order="F").copy()), K, T,
                              _ptr(x_flat), _ptr(lam) if lam is not None else None, _ptr(out), RP_HOST))
    return out[:T]


def ihs_bin_path(a, b, config: PathConfig, spec: SketchSpec, rho: RhoBounds, sigma_d=None,
                 ctx: Optional[Context] = None, a_test=None, b_test=None) -> RegPathResult:
    """path_solver.hpp:109-114 (vector b) / 116-121 (matrix b)."""
    if spec.n != _rows(a):
        raise ValueError("ihs_bin_path: spec.n must equal A.rows")
    return _run_path(False, a, b, config, spec, rho, sigma_d, ctx, a_test=a_test, b_test=b_test)


ihs_bin_path_matrix = ihs_bin_path


def dual_path(a, b, config: PathConfig, spec: SketchSpec, rho: RhoBounds, sigma_d=None,
              ctx: Optional[Context] = None, a_test=None, b_test=None) -> RegPathResult:
    """path_solver.hpp:134-139; a matrix b runs K independent dual paths."""
    if spec.n != _cols(a):
        raise ValueError("dual_path: spec.n must equal A.cols (the dual operator is A^T)")
    return _run_path(True, a, b, config, spec, rho, sigma_d, ctx, a_test=a_test, b_test=b_test)


# ---------------------------------------------------------------------------
# Comparison baselines (baselines.hpp; baselines.cpp:80-226)
# ---------------------------------------------------------------------------


def _baseline(name, fn, a, b, config: PathConfig, ctx, a_test, b_test, *extra, iterative=True) -> RegPathResult:
    ctx = ctx or default_context()
    ctx.set_operator(a)
    b = np.asarray(b)
    if b.ndim != 1 and not (b.ndim == 2 and b.shape[1] == 1):
        raise ValueError(f"{name}_path: b must be a vector")
    b1 = _f64(b.reshape(-1))
    if b1.shape[0] != _rows(a):
        raise ValueError(f"{name}_path: dimension mismatch")
    T = len(config.lambdas)
    d = _cols(a)
    out = np.empty(d * max(T, 1))
    cfg, keep = config.c()
    iters = np.zeros(max(T, 1), dtype=np.int32)
    secs = np.zeros(max(T, 1))
    st = np.zeros(2)
    args = [ctx.handle, _ptr(b1), ctypes.byref(cfg), *extra, _ptr(out), RP_HOST]
    args += [_ptr(iters), _ptr(secs), _ptr(st)] if iterative else [_ptr(secs), _ptr(st)]
    ctx.check(fn(*args))
    del keep
    lam = np.asarray(config.lambdas, dtype=np.float64)
    b2 = b1.reshape(-1, 1)
    train = _losses_flat(ctx, b2, 1, T, out, lam) if T else np.empty(0)
    test = None
    if a_test is not None and b_test is not None and T:
        bt = _f64(np.asarray(b_test).reshape(-1, 1))
        if _cols(a_test) != d or bt.shape[0] != _rows(a_test):
            raise ValueError("losses: test dimension mismatch")
        ctx.set_operator(a_test)
        test = _losses_flat(ctx, bt, 1, T, out, None)
        ctx.set_operator(a)
    pts = [PathPoint(float(config.lambdas[t]), out[t * d:(t + 1) * d].reshape(d, 1).copy(), seconds=float(secs[t]),
                     train_loss=float(train[t]), test_loss=float(test[t]) if test is not None else None,
                     iterations=int(iters[t])) for t in range(T)]
    return RegPathResult(name, pts, float(st[0]), float(st[1]))


def warm_cg_path(a, b, config: PathConfig, ctx: Optional[Context] = None, a_test=None, b_test=None) -> RegPathResult:
    """baselines.hpp: CG on the normal equations, descending warm-started sweep."""
    return _baseline("cg", lib().rp_warm_cg_path, a, b, config, ctx, a_test, b_test)


def warm_ihs_path(a, b, config: PathConfig, spec: SketchSpec, rho: RhoBounds, ctx: Optional[Context] = None,
                  a_test=None, b_test=None) -> RegPathResult:
    """baselines.hpp: warm-started sketched Newton iterations per lambda."""
    if spec.n != _rows(a):
        raise ValueError("warm_ihs_path: spec.n must equal A.rows")
    return _baseline("ihs", lib().rp_warm_ihs_path, a, b, config, ctx, a_test, b_test, ctypes.byref(spec.c()),
                     ctypes.byref(rho.c()))


def direct_path(a, b, config: PathConfig, ctx: Optional[Context] = None, a_test=None, b_test=None) -> RegPathResult:
    """baselines.hpp: A^T A once, (A^T A + lambda I)^{-1} A^T b per lambda."""
    return _baseline("direct", lib().rp_direct_path, a, b, config, ctx, a_test, b_test, iterative=False)


def svd_path(a, b, config: PathConfig, ctx: Optional[Context] = None, a_test=None, b_test=None) -> RegPathResult:
    """baselines.hpp: one thin SVD of A, x = V diag(s / (s^2 + lambda)) U^T b per lambda."""
    return _baseline("svd", lib().rp_svd_path, a, b, config, ctx, a_test, b_test, iterative=False)


# ---------------------------------------------------------------------------
# Adaptive sketch dimension (adaptive.hpp; adaptive.cpp:19-137)
# ---------------------------------------------------------------------------


@dataclass
class AdaptiveConfig:
    """adaptive.hpp AdaptiveConfig (m_initial / m_cap 0 = the reference defaults)."""
    gamma1: float = 0.5
    gamma2: float = 1e-4
    gamma3: float = 0.9
    epsilon: float = 1e-8
    m_initial: int = 0
    m_cap: int = 0
    iteration_cap: int = 200

    def c(self):
        return _AdaptiveConfig(self.gamma1, self.gamma2, self.gamma3, self.epsilon, int(self.m_initial),
                               int(self.m_cap), int(self.iteration_cap))


@dataclass
class AdaptiveStep:
    m: int
    f_before: float
    f_after: float
    step: float
    progress: float
    doubled: bool


@dataclass
class AdaptiveResult:
    m: int
    x: np.ndarray
    iterations: int = 0
    doublings: int = 0
    converged: bool = False
    stalled_at_cap: bool = False
    trace: List[AdaptiveStep] = field(default_factory=list)


def adaptive_sketch_dim(a, b, lambda_min: float, config: AdaptiveConfig, spec_template: "SketchSpec", x0=None,
                        ctx: Optional[Context] = None) -> AdaptiveResult:
    """adaptive_sketch_dim (adaptive.hpp) on the device."""
    ctx = ctx or default_context()
    ctx.set_operator(a)
    b1 = _f64(np.asarray(b).reshape(-1))
    if b1.shape[0] != _rows(a):
        raise ValueError("adaptive: dimension mismatch")
    d = _cols(a)
    x = np.empty(d)
    xv = _f64(np.asarray(x0).reshape(-1)) if x0 is not None else None
    if xv is not None and xv.shape[0] != d:
        raise ValueError("adaptive: x0 dimension mismatch")
    res = _AdaptiveResult()
    cap = 4 * int(config.iteration_cap) + 8
    tr = (_AdaptiveStep * cap)()
    ctx.check(lib().rp_adaptive_sketch_dim(ctx.handle, _ptr(b1), float(lambda_min), ctypes.byref(config.c()),
                                           ctypes.byref(spec_template.c()), _ptr(xv) if xv is not None else None,
                                           _ptr(x), RP_HOST, ctypes.byref(res), ctypes.cast(tr, _P), cap))
    steps = [AdaptiveStep(t.m, t.f_before, t.f_after, t.step, t.progress, bool(t.doubled))
             for t in tr[:min(cap, res.trace_len)]]
    return AdaptiveResult(res.m, x, res.iterations, res.doublings, bool(res.converged), bool(res.stalled_at_cap), steps)


# ---------------------------------------------------------------------------
# Draw contract (device RNG)
# ---------------------------------------------------------------------------


def draw_u64(seed, count, skip=0, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(count, 1), dtype=np.uint64)
    ctx.check(lib().rp_draw_u64(ctx.handle, seed, skip, count, _ptr(out), RP_HOST))
    return out[:count]


def draw_uniform01(seed, count, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(count, 1))
    ctx.check(lib().rp_draw_uniform01(ctx.handle, seed, count, _ptr(out), RP_HOST))
    return out[:count]


def draw_sign(seed, count, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(count, 1))
    ctx.check(lib().rp_draw_sign(ctx.handle, seed, count, _ptr(out), RP_HOST))
    return out[:count]


def draw_uniform_index(seed, bound, count, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(count, 1), dtype=np.uint64)
    ctx.check(lib().rp_draw_uniform_index(ctx.handle, seed, bound, count, _ptr(out), RP_HOST))
    return out[:count]


def draw_normals(seed, count, first=0, scale=1.0, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(count, 1))
    ctx.check(lib().rp_draw_normals(ctx.handle, seed, first, count, scale, _ptr(out), RP_HOST))
    return out[:count]


def gaussian_window(seed, m, n, r0, rc, j0, jc, ctx=None):
    ctx = ctx or default_context()
    out = np.empty(max(rc * jc, 1))
    ctx.check(lib().rp_gaussian_window(ctx.handle, seed, m, n, r0, rc, j0, jc, _ptr(out), RP_HOST))
    return out[:rc * jc].reshape(rc, jc)


def count_draws(spec: SketchSpec, ctx=None):
    ctx = ctx or default_context()
    blocks = spec.s if spec.kind == "sjlt" else 1
    h = np.empty(blocks * spec.n, dtype=np.int64)
    sg = np.empty(blocks * spec.n)
    cs = spec.c()
    ctx.check(lib().rp_count_draws(ctx.handle, ctypes.byref(cs), _ptr(h), _ptr(sg), RP_HOST))
    return h.reshape(blocks, spec.n), sg.reshape(blocks, spec.n)


def srht_draws(spec: SketchSpec, ctx=None):
    ctx = ctx or default_context()
    signs = np.empty(spec.n)
    rows = np.empty(spec.m, dtype=np.int64)
    cs = spec.c()
    ctx.check(lib().rp_srht_draws(ctx.handle, ctypes.byref(cs), _ptr(signs), _ptr(rows), RP_HOST))
    return signs, rows


def launch_count() -> int:
    return int(lib().rp_launch_count())


# ---------------------------------------------------------------------------
# Device-resident entry points (operator / b / x already in HBM)
# ---------------------------------------------------------------------------


def set_dense_rows_device(ctx: Context, n_global: int, row0: int, n_local: int, d: int, ptr: int, lda: int):
    """rp_set_dense_rows with a device pointer (the shard's first row)."""
    ctx.check(lib().rp_set_dense_rows(ctx.handle, n_global, row0, n_local, d, _P(ptr), lda, RP_DEVICE))
    ctx._op_key = ("device", ptr, n_global, row0, n_local, d)


def set_dense_rows_host(ctx: Context, n_global: int, row0: int, n_local: int, d: int, ptr: int, lda: int,
                        stream: bool = False):
    """rp_set_dense_rows from host memory (pinned for full-speed DMA).  With
    stream=True (RP_HOST_STREAM) the upload runs asynchronously in column
    chunks and the next path call consumes them as they land; the host buffer
    must stay valid until that call returns."""
    ctx.check(lib().rp_set_dense_rows(ctx.handle, n_global, row0, n_local, d, _P(ptr), lda,
                                      RP_HOST_STREAM if stream else RP_HOST))
    ctx._op_key = ("host", ptr, n_global, row0, n_local, d)


def set_dense_cols_device(ctx: Context, n: int, d_global: int, col0: int, d_local: int, ptr: int, lda: int):
    ctx.check(lib().rp_set_dense_cols(ctx.handle, n, d_global, col0, d_local, _P(ptr), lda, RP_DEVICE))
    ctx._op_key = ("device-cols", ptr, n, d_global, col0, d_local)


def set_dense_cols_host(ctx: Context, n: int, d_global: int, col0: int, d_local: int, ptr: int, lda: int):
    """rp_set_dense_cols from host memory: columns [col0, col0 + d_local) of
    the n x d_global operator (dual route, column-sharded)."""
    ctx.check(lib().rp_set_dense_cols(ctx.handle, n, d_global, col0, d_local, _P(ptr), lda, RP_HOST))
    ctx._op_key = ("host-cols", ptr, n, d_global, col0, d_local)


def set_csr_rows(ctx: Context, n_global: int, row0: int, shard: "Csr"):
    """rp_set_csr_rows: `shard` holds rows [row0, row0 + shard.rows) of the
    n_global x shard.cols CSR operator (offsets local, starting at 0)."""
    off = np.ascontiguousarray(shard.offsets, dtype=np.int64)
    idx = np.ascontiguousarray(shard.indices, dtype=np.int64)
    val = np.ascontiguousarray(shard.values, dtype=np.float64)
    ctx.check(lib().rp_set_csr_rows(ctx.handle, n_global, row0, shard.rows, shard.cols, _ptr(off), _ptr(idx),
                                    _ptr(val), RP_HOST))
    ctx._op_key = None


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().rp_comm_unique_id(buf))
    return buf.raw


def comm_init(ctx: Context, rank: int, world: int, uid: bytes):
    buf = ctypes.create_string_buffer(uid, 128)
    ctx.check(lib().rp_comm_init(ctx.handle, rank, world, buf))


_HOST_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, _P, ctypes.POINTER(ctypes.c_double), _I64)
_HOST_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, _P, ctypes.POINTER(ctypes.c_double), _I64,
                                   ctypes.POINTER(ctypes.c_double))


def comm_init_host(ctx: Context, rank: int, world: int, allreduce, allgather):
    """rp_comm_init_host: the context's collectives run through Python
    callables on host numpy arrays -- `allreduce(buf)` sums `buf` over ranks in
    place, `allgather(send, recv)` fills recv (world x len(send)) with every
    rank's send.  A raised exception fails the library call (RP_ENCCL)."""

    def ar(_user, ptr, count):
        try:
            allreduce(np.ctypeslib.as_array(ptr, shape=(int(count),)))
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def ag(_user, send, count, recv):
        try:
            allgather(np.ctypeslib.as_array(send, shape=(int(count),)),
                      np.ctypeslib.as_array(recv, shape=(int(world), int(count))))
            return 0
        except Exception:  # noqa: BLE001
            return 1

    cb = (_HOST_ALLREDUCE(ar), _HOST_ALLGATHER(ag))
    ctx._host_comm = cb  # keep the thunks alive with the context
    ctx.check(lib().rp_comm_init_host(ctx.handle, rank, world, ctypes.cast(cb[0], _P), ctypes.cast(cb[1], _P), None))


def comm_init_torch_host(ctx: Context, group=None):
    """Host communicator over an initialised torch.distributed process group
    (e.g. gloo): several ranks may then share one GPU, or run without NCCL."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def allreduce(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t, group=group)

    def allgather(send, recv):
        outs = [torch.from_numpy(recv[r]) for r in range(world)]
        dist.all_gather(outs, torch.from_numpy(send.copy()), group=group)

    comm_init_host(ctx, dist.get_rank(group), world, allreduce, allgather)


def path_raw(ctx: Context, b_ptr: int, K: int, config: PathConfig, spec: SketchSpec, rho: RhoBounds, x_ptr: int,
             where: int = RP_DEVICE, dual: bool = False, sigma_d=None) -> Timings:
    """rp_ihs_bin_path / rp_dual_path on raw pointers (device or host)."""
    cfg, keep = config.c()
    cs, cr = spec.c(), rho.c()
    sd = ctypes.c_double(sigma_d) if sigma_d is not None else None
    tm = Timings()
    fn = lib().rp_dual_path if dual else lib().rp_ihs_bin_path
    ctx.check(fn(ctx.handle, _P(b_ptr), K, ctypes.byref(cfg), ctypes.byref(cs), ctypes.byref(cr),
                 ctypes.cast(ctypes.byref(sd), _P) if sd is not None else None, _P(x_ptr), where, ctypes.byref(tm)))
    del keep
    return tm


def gram_apply_raw(ctx: Context, x_ptr: int, ncols: int, out_ptr: int, where: int = RP_DEVICE):
    """rp_gram_apply on raw pointers: out = A^T (A x) for the context's operator."""
    ctx.check(lib().rp_gram_apply(ctx.handle, _P(x_ptr), ncols, _P(out_ptr), where))


def last_gemm_profile(ctx: Context):
    """Per-GEMM (seconds, flops, bytes) arrays of the last profiled path call."""
    cnt = _I64(0)
    ctx.check(lib().rp_last_gemm_profile(ctx.handle, None, None, None, 0, ctypes.cast(ctypes.byref(cnt), _P)))
    n = cnt.value
    sec, fl, by = np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1))
    ctx.check(lib().rp_last_gemm_profile(ctx.handle, _ptr(sec), _ptr(fl), _ptr(by), n,
                                         ctypes.cast(ctypes.byref(cnt), _P)))
    return sec[:n], fl[:n], by[:n]


def last_device_seconds(ctx: Context) -> float:
    """Device seconds of the last apply_transpose / gram_apply (profile option on)."""
    v = ctypes.c_double(0.0)
    ctx.check(lib().rp_last_device_seconds(ctx.handle, ctypes.byref(v)))
    return v.value


def apply_transpose_raw(ctx: Context, y_ptr: int, ncols: int, out_ptr: int, where: int = RP_DEVICE):
    """rp_apply_transpose on raw pointers: out = A^T y."""
    ctx.check(lib().rp_apply_transpose(ctx.handle, _P(y_ptr), ncols, _P(out_ptr), where))


# ---------------------------------------------------------------------------
# data_io.hpp: the formats either side of the path
# ---------------------------------------------------------------------------


def parse_libsvm(text, feature_override: Optional[int] = None):
    """parse_libsvm (data_io.cpp:50-127) -> (Csr, labels).  `text` is str or bytes."""
    raw = text.encode() if isinstance(text, str) else bytes(text)
    fo = -1 if feature_override is None else int(feature_override)
    if feature_override is not None and fo < 0:
        raise ValueError("parse_libsvm: negative feature dimension")
    rows, cols, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    el, ec = ctypes.c_int64(), ctypes.c_int64()
    L = lib()

    def call(*arrays):
        st = L.rp_libsvm_parse(raw, len(raw), fo, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(nnz),
                               *arrays, ctypes.byref(el), ctypes.byref(ec))
        if st == 8:
            raise ParseError(L.rp_last_error(None).decode(), el.value, ec.value)
        _check(st)

    call(None, None, None, None)
    off = np.empty(rows.value + 1, dtype=np.int64)
    idx = np.empty(nnz.value, dtype=np.int64)
    val = np.empty(nnz.value)
    lab = np.empty(rows.value)
    call(_ptr(off), _ptr(idx), _ptr(val), _ptr(lab))
    return Csr(rows.value, cols.value, off, idx, val), lab


def _g17(v: float) -> str:
    return "%.17g" % float(v)  # format_double (data_io.cpp:338-342)


def write_libsvm(a, labels) -> str:
    """write_libsvm (data_io.cpp:129-149): dense operators go through CSR
    (explicit zeros dropped); indices 1-based, 17 significant digits."""
    labels = np.asarray(labels, dtype=np.float64).reshape(-1)
    if not isinstance(a, Csr):
        d = np.asarray(a, dtype=np.float64)
        off, idx, val = [0], [], []
        for r in range(d.shape[0]):
            nz = np.nonzero(d[r])[0]
            idx.extend(nz.tolist())
            val.extend(d[r, nz].tolist())
            off.append(len(val))
        a = Csr(d.shape[0], d.shape[1], np.asarray(off), np.asarray(idx, dtype=np.int64), np.asarray(val))
    if labels.shape[0] != a.rows:
        raise ValueError("write_libsvm: label count mismatch")
    lines = []
    for r in range(a.rows):
        parts = [_g17(labels[r])]
        for p in range(int(a.offsets[r]), int(a.offsets[r + 1])):
            parts.append(f"{int(a.indices[p]) + 1}:{_g17(a.values[p])}")
        lines.append(" ".join(parts) + "\n")
    return "".join(lines)


def write_csv(results: List[RegPathResult]) -> str:
    """write_csv (data_io.cpp:344-364): every point of every result, sorted
    stably by lambda then solver name, header lambda,train_loss,test_loss,time_s,solver."""
    names = [r.solver.encode() for r in results]
    c_names = (ctypes.c_char_p * max(len(names), 1))(*names)
    npts = np.asarray([len(r.points) for r in results] or [0], dtype=np.int64)
    pts = [p for r in results for p in r.points]
    lam = np.asarray([p.lam for p in pts] or [0.0], dtype=np.float64)
    tr = np.asarray([p.train_loss for p in pts] or [0.0], dtype=np.float64)
    te = np.asarray([p.test_loss if p.test_loss is not None else 0.0 for p in pts] or [0.0], dtype=np.float64)
    has = np.asarray([p.test_loss is not None for p in pts] or [0], dtype=np.uint8)
    sec = np.asarray([p.seconds for p in pts] or [0.0], dtype=np.float64)
    need = ctypes.c_int64()
    args = [len(results), ctypes.cast(c_names, _P), _ptr(npts), _ptr(lam), _ptr(tr), _ptr(te), _ptr(has), _ptr(sec)]
    _check(lib().rp_write_csv(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().rp_write_csv(*args, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()
