"""CPU oracle: numpy restatement of the reference IHS-BIN path.

TEST INFRASTRUCTURE ONLY.  The product (paper_2210_12212_b200/) never imports
this module; tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs use it as the checker.

Parity status: the integer draw contract is pinned against the reference's own
``rng.hpp`` compiled in place (oracle/_ref, tests/test_oracle_pins.py) and the
KATs of SURVEY.md section 8(c).  The floating-point algorithm is pinned against
the reference's own doctest KATs (scalar basis 0.75/-0.25, tune_interval
lambda0=10/kappa=100/alpha=20/101, L=9 for beta=100, dual hand example, ...)
re-stated in tests/test_oracle_pins.py.  The reference's Eigen-dependent code
cannot be compiled here (no Eigen), so the GEMM/SVD rounding of this oracle is
numpy/LAPACK's, not Eigen's.

Reference citations: ref = /root/reference/proj/core.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# --------------------------------------------------------------------------
# C part (draw contract), built by oracle/Makefile
# --------------------------------------------------------------------------

_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = os.path.join(_HERE, "liboracle.so")
    if not os.path.exists(path):
        subprocess.check_call(["make", "-s", "-C", _HERE, os.path.join(_HERE, "liboracle.so")])
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    u64, i64, dbl, cint = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    sig = {
        "or_fill_u64": [u64, u64, i64, P],
        "or_fill_uniform01": [u64, i64, P],
        "or_fill_uniform_index": [u64, u64, i64, P],
        "or_fill_normals": [u64, i64, dbl, P],
        "or_gaussian_window": [u64, i64, i64, i64, i64, i64, i64, P],
        "or_count_draws": [u64, i64, i64, cint, dbl, P, P],
        "or_count_apply_dense": [u64, i64, i64, i64, cint, dbl, P, i64, P],
        "or_count_apply_csr": [u64, i64, i64, i64, cint, dbl, P, P, P, P],
        "or_srht_draws": [u64, i64, i64, P, P],
        "or_srht_apply": [u64, i64, i64, i64, P, i64, P, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = None
    lib.or_hadamard_pad.argtypes = [i64]
    lib.or_hadamard_pad.restype = i64
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def fill_u64(seed: int, count: int, skip: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _load().or_fill_u64(seed, skip, count, _ptr(out))
    return out


def fill_uniform01(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _load().or_fill_uniform01(seed, count, _ptr(out))
    return out


def fill_uniform_index(seed: int, bound: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _load().or_fill_uniform_index(seed, bound, count, _ptr(out))
    return out


def fill_normals(seed: int, count: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _load().or_fill_normals(seed, count, scale, _ptr(out))
    return out


def hadamard_pad(n: int) -> int:
    """sketch.cpp:190-193 (smallest power of two >= max(n, 1))."""
    return int(_load().or_hadamard_pad(n))


# --------------------------------------------------------------------------
# Errors (path_solver.hpp:18-27); std::invalid_argument -> ValueError
# --------------------------------------------------------------------------


class BasisDivergedError(RuntimeError):
    pass


class SolverError(RuntimeError):
    pass


def _require(cond: bool, msg: str):
    if not cond:
        raise ValueError(msg)


# --------------------------------------------------------------------------
# Matrix types (matrix.hpp:16-73)
# --------------------------------------------------------------------------


@dataclass
class Csr:
    rows: int
    cols: int
    offsets: np.ndarray  # int64, rows+1
    indices: np.ndarray  # int64, nnz (strictly increasing per row)
    values: np.ndarray  # float64, nnz
    _sp: object = None

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.indices = np.ascontiguousarray(self.indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        # matrix.cpp:22-50 structural checks
        _require(self.offsets.shape[0] == self.rows + 1, "csr: row_offsets length must be rows+1")
        _require(self.offsets[0] == 0, "csr: row_offsets must start at 0")
        _require(self.offsets[-1] == self.values.shape[0], "csr: row_offsets must end at nnz")
        _require(self.indices.shape[0] == self.values.shape[0], "csr: col_indices and values length mismatch")

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def nnz(self):
        return int(self.values.shape[0])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols))
        row_of = np.repeat(np.arange(self.rows), np.diff(self.offsets))
        out[row_of, self.indices] = self.values
        return out

    def transposed(self) -> "Csr":
        row_of = np.repeat(np.arange(self.rows), np.diff(self.offsets))
        order = np.lexsort((row_of, self.indices))
        cols_t = row_of[order]
        vals_t = self.values[order]
        offs = np.zeros(self.cols + 1, dtype=np.int64)
        np.add.at(offs, self.indices + 1, 1)
        return Csr(self.cols, self.rows, np.cumsum(offs), cols_t, vals_t)

    @staticmethod
    def from_dense(a: np.ndarray, drop_tol: float = 0.0) -> "Csr":
        mask = np.abs(a) > drop_tol
        offs = np.concatenate([[0], np.cumsum(mask.sum(axis=1))])
        r, c = np.nonzero(mask)
        return Csr(a.shape[0], a.shape[1], offs, c, a[r, c])


def is_csr(a) -> bool:
    return isinstance(a, Csr)


def _rows(a):
    return a.rows if is_csr(a) else a.shape[0]


def _cols(a):
    return a.cols if is_csr(a) else a.shape[1]


def _scipy(a):
    import scipy.sparse as sp

    if getattr(a, "_sp", None) is None:
        a._sp = sp.csr_matrix((a.values, a.indices, a.offsets), shape=(a.rows, a.cols))
    return a._sp


def apply(a, x: np.ndarray) -> np.ndarray:
    """matrix.cpp:140-152 / 174-188 (CSR: row-wise sums, scipy's CSR kernel)."""
    _require(x.shape[0] == _cols(a), "apply: dimension mismatch")
    if not is_csr(a):
        return a @ x
    return np.asarray(_scipy(a) @ x)


def apply_transpose(a, y: np.ndarray) -> np.ndarray:
    """matrix.cpp:154-166 / 190-201."""
    _require(y.shape[0] == _rows(a), "apply_transpose: dimension mismatch")
    if not is_csr(a):
        return a.T @ y
    return np.asarray(_scipy(a).T @ y)


_gram_count = 0


def gram_apply(a, x: np.ndarray) -> np.ndarray:
    """matrix.cpp:168-172: A^T (A x), evaluation order apply_transpose(apply)."""
    global _gram_count
    _gram_count += 1 if x.ndim == 1 else x.shape[1]
    return apply_transpose(a, apply(a, x))


def transpose(a):
    return a.transposed() if is_csr(a) else np.ascontiguousarray(a.T)


def thin_svd(m: np.ndarray):
    """matrix.cpp:213-234 (LAPACK gesdd here instead of Eigen Jacobi/BDC)."""
    _require(m.shape[0] >= 1 and m.shape[1] >= 1, "thin_svd: empty matrix")
    _require(bool(np.all(np.isfinite(m))), "thin_svd: non-finite entries")
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    return u, s, vt


# --------------------------------------------------------------------------
# Sketches (sketch.hpp / sketch.cpp)
# --------------------------------------------------------------------------

SKETCH_KINDS = ("gaussian", "countsketch", "sjlt", "srht", "identity")


@dataclass
class SketchSpec:
    kind: str = "identity"
    m: int = 0
    n: int = 0
    s: int = 1
    seed: int = 0

    def validate(self):
        """sketch.cpp:202-212."""
        _require(self.kind in SKETCH_KINDS, "unknown sketch kind: " + str(self.kind))
        _require(self.n >= 1, "sketch: n must be positive")
        _require(self.m >= 1, "sketch: m must be positive")
        if self.kind == "sjlt":
            _require(self.s >= 1, "sjlt: sparsity must be >= 1")
            _require(self.m % self.s == 0, "sjlt: sparsity must divide m")
        if self.kind == "identity":
            _require(self.m == self.n, "identity sketch: m must equal n")


def gaussian_scale(m: int) -> float:
    return 1.0 / math.sqrt(float(m))


def gaussian_sketch_matrix(spec: SketchSpec) -> np.ndarray:
    """Row-major realization of S (sketch.cpp:94-95, 255-261)."""
    s = fill_normals(spec.seed, spec.m * spec.n, gaussian_scale(spec.m))
    return s.reshape(spec.m, spec.n)


def count_draws(spec: SketchSpec):
    blocks = spec.s if spec.kind == "sjlt" else 1
    entry = 1.0 / math.sqrt(float(spec.s)) if spec.kind == "sjlt" else 1.0
    h = np.empty(blocks * spec.n, dtype=np.int64)
    sg = np.empty(blocks * spec.n, dtype=np.float64)
    _load().or_count_draws(spec.seed, spec.n, spec.m // blocks, blocks, entry, _ptr(h), _ptr(sg))
    return h.reshape(blocks, spec.n), sg.reshape(blocks, spec.n)


def srht_draws(spec: SketchSpec):
    signs = np.empty(spec.n, dtype=np.float64)
    rows = np.empty(spec.m, dtype=np.int64)
    _load().or_srht_draws(spec.seed, spec.n, spec.m, _ptr(signs), _ptr(rows))
    return signs, rows


def sketch_apply(spec: SketchSpec, a) -> np.ndarray:
    """sketch.cpp:225-248.  Returns S*A as an m x d array."""
    spec.validate()
    _require(_rows(a) == spec.n, "sketch_apply: spec.n must match A.rows")
    d = _cols(a)
    lib = _load()
    if spec.kind == "identity":
        return a.to_dense() if is_csr(a) else np.array(a, dtype=np.float64)
    if spec.kind == "gaussian":
        s = gaussian_sketch_matrix(spec)
        return s @ (a.to_dense() if is_csr(a) else a)
    if spec.kind in ("countsketch", "sjlt"):
        blocks = spec.s if spec.kind == "sjlt" else 1
        entry = 1.0 / math.sqrt(float(spec.s)) if spec.kind == "sjlt" else 1.0
        out = np.empty((d, spec.m), dtype=np.float64)  # column-major m x d
        if is_csr(a):
            lib.or_count_apply_csr(spec.seed, spec.m, spec.n, d, blocks, entry, _ptr(a.offsets),
                                   _ptr(a.indices), _ptr(a.values), _ptr(out))
        else:
            af = np.asfortranarray(a, dtype=np.float64)
            lib.or_count_apply_dense(spec.seed, spec.m, spec.n, d, blocks, entry, _ptr(af), spec.n, _ptr(out))
        return out.T.copy()
    # srht
    out = np.empty((d, spec.m), dtype=np.float64)
    if is_csr(a):
        lib.or_srht_apply(spec.seed, spec.m, spec.n, d, None, 0, _ptr(a.offsets), _ptr(a.indices),
                          _ptr(a.values), _ptr(out))
    else:
        af = np.asfortranarray(a, dtype=np.float64)
        lib.or_srht_apply(spec.seed, spec.m, spec.n, d, _ptr(af), spec.n, None, None, None, _ptr(out))
    return out.T.copy()


def realize_dense(spec: SketchSpec) -> np.ndarray:
    """sketch.cpp:250-300 (guarded to m*n <= 1e6)."""
    spec.validate()
    _require(spec.m * spec.n <= 1_000_000, "realize_dense: m*n exceeds the materialization guard")
    s = np.zeros((spec.m, spec.n))
    if spec.kind == "identity":
        return np.eye(spec.m, spec.n)
    if spec.kind == "gaussian":
        return gaussian_sketch_matrix(spec)
    if spec.kind in ("countsketch", "sjlt"):
        h, sg = count_draws(spec)
        blocks = h.shape[0]
        rpb = spec.m // blocks
        for b in range(blocks):
            s[b * rpb + h[b], np.arange(spec.n)] = sg[b]
        return s
    signs, rows = srht_draws(spec)
    npad = hadamard_pad(spec.n)
    scale = math.sqrt(npad / spec.m) / math.sqrt(npad)
    j = np.arange(spec.n, dtype=np.uint64)
    for r in range(spec.m):
        par = np.array([bin(int(v)).count("1") & 1 for v in (np.uint64(rows[r]) & j)])
        s[r] = scale * np.where(par == 1, -1.0, 1.0) * signs
    return s


# --------------------------------------------------------------------------
# Spectrum (spectrum.cpp)
# --------------------------------------------------------------------------

K_MAX_BUDGET = 64
K_MIN_BUDGET = 2


@dataclass
class PathConfig:
    lambda_min: float = 0.0
    lambda_max: float = 0.0
    lambdas: List[float] = field(default_factory=list)
    epsilon: float = 1e-6
    num_intervals: Optional[int] = None

    def validate(self):
        """spectrum.cpp:20-36."""
        _require(self.lambda_min > 0.0 and self.lambda_max > 0.0, "path config: lambda bounds must be positive")
        _require(self.lambda_min < self.lambda_max, "path config: lambda_min must be below lambda_max")
        _require(len(self.lambdas) > 0, "path config: empty evaluation grid")
        _require(0.0 < self.epsilon < 1.0, "path config: epsilon not in (0,1)")
        prev = self.lambda_min
        for l in self.lambdas:
            _require(l >= prev, "path config: grid must be sorted ascending")
            prev = l
        _require(self.lambdas[0] >= self.lambda_min and self.lambdas[-1] <= self.lambda_max,
                 "path config: grid must lie within [lambda_min, lambda_max]")
        if self.num_intervals is not None:
            _require(self.num_intervals >= 1, "path config: L must be >= 1")


@dataclass
class RhoBounds:
    rho1: float = 1.0
    rho2: float = 1.0
    provenance: str = "identity"

    def validate(self):
        """spectrum.cpp:71-76."""
        _require(self.rho2 > 0.0, "rho bounds: rho2 must be positive")
        _require(self.rho1 >= self.rho2, "rho bounds: rho1 must be >= rho2")
        if self.provenance == "identity":
            _require(self.rho1 == 1.0 and self.rho2 == 1.0, "identity rho bounds must be (1,1)")

    @staticmethod
    def identity():
        return RhoBounds(1.0, 1.0, "identity")

    @staticmethod
    def manual(rho1, rho2):
        b = RhoBounds(rho1, rho2, "manual")
        b.validate()
        return b


@dataclass
class RateParams:
    lambda0: float = 0.0
    alpha: float = 0.0
    kappa: float = 1.0
    contraction: float = 0.0
    k: int = 1


def effective_dimension(sigma, lambda0: float) -> float:
    """spectrum.cpp:87-103: ||D||_F^2 / ||D||_2^2 with D_ii^2 = s^2 / (s^2 + lambda0)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    _require(sigma.shape[0] > 0, "effective_dimension: empty spectrum")
    _require(lambda0 >= 0.0, "effective_dimension: negative shift")
    fro = 0.0
    top = 0.0
    for s in sigma.tolist():
        _require(s >= 0.0, "effective_dimension: negative singular value")
        if s == 0.0:
            continue
        dii_sq = s * s / (s * s + lambda0)
        fro += dii_sq
        top = max(top, dii_sq)
    _require(top > 0.0, "effective_dimension: all-zero spectrum")
    return fro / top


def rho_gaussian(rho: float, eta: float, dnorm_sq: float, m=None):
    """spectrum.cpp:105-128 -> (RhoBounds, success_probability or None)."""
    _require(0.0 < rho < 1.0, "rho_gaussian: rho not in (0,1)")
    eta_cap = (1.0 - math.sqrt(rho)) * (1.0 - math.sqrt(rho)) / 4.0
    _require(0.0 < eta < eta_cap, "rho_gaussian: eta outside (0, (1-sqrt(rho))^2/4)")
    _require(0.0 < dnorm_sq <= 1.0, "rho_gaussian: ||D||^2 must lie in (0,1]")
    sq_eta = math.sqrt(eta)
    c_eta = math.pow((1.0 + sq_eta) / (1.0 - sq_eta), 2.0)
    up = (1.0 + math.sqrt(rho)) * (1.0 + sq_eta)
    down = 1.0 - math.sqrt(c_eta * rho)
    b = RhoBounds(1.0 - dnorm_sq + dnorm_sq * up * up, 1.0 - dnorm_sq + dnorm_sq * down * down, "gaussian")
    b.validate()
    prob = None
    if m is not None:
        prob = 1.0 - 16.0 * math.exp(-eta * eta * rho * float(m) / 2.0)
    return b, prob


def rho_srht(rho: float, dnorm_sq: float, n_and_de=None):
    """spectrum.cpp:130-148 -> (RhoBounds, recommended_m or None)."""
    _require(0.0 < rho < 1.0, "rho_srht: rho not in (0,1)")
    _require(dnorm_sq > 0.0, "rho_srht: ||D||^2 must be positive")
    _require(dnorm_sq * rho < 1.0, "rho_srht: ||D||^2 * rho must be below 1")
    b = RhoBounds(1.0 + dnorm_sq * rho, 1.0 - dnorm_sq * rho, "srht")
    rec = None
    if n_and_de is not None:
        n, de = n_and_de
        _require(n >= 1 and de >= 1.0, "rho_srht: bad (n, d_e)")
        c = 16.0 / 3.0 * math.pow(1.0 + math.sqrt(8.0 * math.log(de * float(n)) / de), 2.0)
        rec = int(math.ceil(c * de * math.log(de) / rho))
    return b, rec


def rho_sjlt(eps: float, alpha_delta_de=None):
    """spectrum.cpp:150-169 -> (RhoBounds, recommended_m or None, recommended_s or None)."""
    _require(0.0 < eps < 0.5, "rho_sjlt: eps not in (0, 1/2)")
    b = RhoBounds(1.0 + eps, 1.0 - eps, "sjlt")
    rec_m = rec_s = None
    if alpha_delta_de is not None:
        alpha, delta, de = alpha_delta_de
        _require(alpha > 2.0, "rho_sjlt: alpha must exceed 2")
        _require(0.0 < delta < 0.5, "rho_sjlt: delta not in (0, 1/2)")
        _require(de >= 1.0, "rho_sjlt: d_e must be >= 1")
        log_alpha = math.log(de / delta) / math.log(alpha)
        rec_s = int(math.ceil(log_alpha / eps))
        rec_m = int(math.ceil(alpha * de * log_alpha / (eps * eps)))
    return b, rec_m, rec_s


def derive_rho(spec: "SketchSpec", a, lambda_min: float, lambda_max: float):
    """tools/ridgepath_main.cpp:218-279 (the CLI's plug-in envelope): sketch A,
    thin SVD of SA, effective dimension at lambda0 = sqrt(lo*hi), then the
    family's bound.  Returns (RhoBounds, info dict)."""
    if spec.kind == "identity":
        return RhoBounds.identity(), {}
    sa = sketch_apply(spec, a)
    _, sigma, _ = thin_svd(sa)
    lambda0 = math.sqrt(lambda_min * lambda_max)
    de = effective_dimension(sigma, lambda0)
    top = float(sigma[0]) * float(sigma[0])
    dnorm_sq = top / (top + lambda0)
    m = float(spec.m)
    bounds = RhoBounds.identity()
    if spec.kind == "gaussian":
        rho = min(0.95, de / m)
        eta = 0.5 * (1.0 - math.sqrt(rho)) * (1.0 - math.sqrt(rho)) / 4.0
        bounds, _ = rho_gaussian(rho, eta, dnorm_sq, spec.m)
    elif spec.kind == "srht":
        c = 16.0 / 3.0 * math.pow(1.0 + math.sqrt(8.0 * math.log(de * float(spec.n)) / de), 2.0)
        rho = c * de * max(1.0, math.log(de)) / m
        rho = min(rho, 0.95 / max(dnorm_sq, 1e-12))
        rho = min(max(rho, 1e-6), 0.95)
        bounds, _ = rho_srht(rho, dnorm_sq)
    elif spec.kind in ("countsketch", "sjlt"):
        alpha, delta = 4.0, 0.1
        log_term = math.log(max(de / delta, 1.5)) / math.log(alpha)
        eps = math.sqrt(alpha * de * log_term / m)
        eps = min(max(eps, 1e-6), 0.49)
        bounds, _, _ = rho_sjlt(eps, (alpha, delta, de))
    return bounds, dict(effective_dimension=de, sigma_max_sq=top, dnorm_sq=dnorm_sq, lambda0=lambda0)


def log_grid(lambda_min: float, lambda_max: float, count: int) -> List[float]:
    """spectrum.cpp:38-53."""
    _require(count >= 1, "log_grid: count must be >= 1")
    _require(lambda_min > 0.0 and lambda_max >= lambda_min, "log_grid: bad range")
    if count == 1:
        return [lambda_min]
    lr = math.log(lambda_max / lambda_min)
    grid = [lambda_min * math.exp(lr * float(i) / (count - 1)) for i in range(count)]
    grid[0] = lambda_min
    grid[-1] = lambda_max
    return grid


def tune_interval(lambda_lo, lambda_hi, rho: RhoBounds, sigma_d, eps) -> RateParams:
    """spectrum.cpp:171-203."""
    _require(lambda_lo > 0.0, "tune_interval: lambda_lo must be positive")
    _require(lambda_lo <= lambda_hi, "tune_interval: interval ordering violated")
    _require(0.0 < eps < 1.0, "tune_interval: eps not in (0,1)")
    rho.validate()
    shift = sigma_d * sigma_d if sigma_d is not None else 0.0
    _require(shift >= 0.0, "tune_interval: sigma_d must be nonnegative")
    lo = lambda_lo + shift
    hi = lambda_hi + shift
    out = RateParams()
    out.lambda0 = math.sqrt(lo * hi) - shift
    out.kappa = rho.rho1 * hi / (rho.rho2 * lo)
    out.alpha = 2.0 * math.sqrt(lo * hi) / (lo / rho.rho1 + hi / rho.rho2)
    rate = (out.kappa - 1.0) / (out.kappa + 1.0)
    out.contraction = rate * rate
    if out.contraction <= 0.0:
        out.k = K_MIN_BUDGET
    else:
        per_step = -math.log(rate)
        raw = math.ceil(math.log(1.0 / eps) / per_step)
        out.k = int(min(max(raw, float(K_MIN_BUDGET)), float(K_MAX_BUDGET)))
    return out


def auto_interval_count(lambda_min, lambda_max) -> int:
    """spectrum.cpp:205-211."""
    _require(lambda_min > 0.0 and lambda_min < lambda_max, "interval_split: need 0 < lambda_min < lambda_max")
    beta = lambda_max / lambda_min
    return max(1, int(math.floor(2.0 * math.log(beta))))


def interval_split(lambda_min, lambda_max, num_intervals=None):
    """spectrum.cpp:213-233."""
    _require(lambda_min > 0.0 and lambda_min < lambda_max, "interval_split: need 0 < lambda_min < lambda_max")
    count = num_intervals if num_intervals is not None else auto_interval_count(lambda_min, lambda_max)
    _require(count >= 1, "interval_split: L must be >= 1")
    log_beta = math.log(lambda_max / lambda_min)
    edges = [lambda_min * math.exp(log_beta * float(i) / count) for i in range(count + 1)]
    edges[0] = lambda_min
    edges[-1] = lambda_max
    return [(edges[i], edges[i + 1]) for i in range(count)]


# --------------------------------------------------------------------------
# Preconditioner (preconditioner.cpp)
# --------------------------------------------------------------------------


class Preconditioner:
    """P_S = (SA^T SA + lambda0 I)^{-1} from one SVD of SA (preconditioner.cpp:12-65)."""

    def __init__(self, vt, sigma, lambda0, m, d, projection_form):
        self.vt = vt
        self.sigma = sigma
        self.lambda0 = lambda0
        self.m = m
        self.d = d
        self.projection_form = projection_form
        self._refresh_weights()

    @staticmethod
    def build(sa: np.ndarray, lambda0: float) -> "Preconditioner":
        return Preconditioner.build_from_svd(thin_svd(sa), sa.shape[0], sa.shape[1], lambda0)

    @staticmethod
    def build_from_svd(svd, m, d, lambda0) -> "Preconditioner":
        if lambda0 <= 0.0:
            raise ValueError("preconditioner: shift must be positive")
        _, s, vt = svd
        full = s.shape[0]
        smax = s[0] if full > 0 else 0.0
        r = 0
        while r < full and s[r] > 1e-12 * smax:
            r += 1
        return Preconditioner(vt[:r].copy(), s[:r].copy(), lambda0, m, d, (m >= d) and (r == d))

    def reshift(self, new_lambda0: float) -> "Preconditioner":
        if new_lambda0 <= 0.0:
            raise ValueError("preconditioner: shift must be positive")
        return Preconditioner(self.vt, self.sigma, new_lambda0, self.m, self.d, self.projection_form)

    def _refresh_weights(self):
        inv = 1.0 / (self.sigma * self.sigma + self.lambda0)
        self.weights = inv if self.projection_form else inv - 1.0 / self.lambda0

    def apply(self, v: np.ndarray) -> np.ndarray:
        if v.shape[0] != self.d:
            raise ValueError("preconditioner apply: dimension mismatch")
        coeffs = self.vt @ v
        coeffs = coeffs * (self.weights if v.ndim == 1 else self.weights[:, None])
        if self.projection_form:
            return self.vt.T @ coeffs
        return v / self.lambda0 + self.vt.T @ coeffs

    def rank(self):
        return self.sigma.shape[0]

    def dense(self) -> np.ndarray:
        return self.apply(np.eye(self.d))


# --------------------------------------------------------------------------
# Path solver (path_solver.cpp)
# --------------------------------------------------------------------------


@dataclass
class BinomialBasis:
    terms: List[np.ndarray]  # k blocks, each dim x K
    tau: float = 0.0
    lambda_lo: float = 0.0
    lambda_hi: float = 0.0
    flavor: str = "ihs"

    @property
    def k(self):
        return len(self.terms)


def ihs_basis_core(op, c: np.ndarray, p: Preconditioner, tau: float, k: int,
                   gram: Optional[Callable] = None) -> np.ndarray:
    """path_solver.cpp:27-53.  Returns tilde (dim x k)."""
    dim = c.shape[0]
    _require(k >= 1, "ihs_basis: k must be >= 1")
    _require(tau > 0.0, "ihs_basis: tau must be positive")
    _require(_cols(op) == dim, "ihs_basis: operator/right-hand-side mismatch")
    _require(p.d == dim, "ihs_basis: preconditioner dimension mismatch")
    gram = gram or (lambda w: gram_apply(op, w))
    gen = np.zeros((dim, k))
    tilde = np.zeros((dim, k))
    gen[:, 0] = p.apply(c.copy())
    tilde[:, 0] = gen[:, 0]
    for g in range(1, k):
        w = gen[:, :g].copy()
        args = np.empty((dim, g + 1))
        args[:, :g] = tau * gram(w)
        for j in range(1, g):
            args[:, j] += w[:, j - 1]
        args[:, g] = w[:, g - 1]
        applied = p.apply(args)
        gen[:, :g] -= applied[:, :g]
        gen[:, g] = -applied[:, g]
        if not np.all(np.isfinite(gen[:, :g + 1])):
            raise BasisDivergedError("basis recursion diverged (step too large)")
        tilde[:, :g + 1] += gen[:, :g + 1]
    return tilde


_compose_count = 0


def compose_horner(basis: BinomialBasis, t: float) -> np.ndarray:
    """path_solver.cpp:64-74: x = u_{k-1}; x = u_j + t x; x *= tau."""
    global _compose_count
    k = basis.k
    x = basis.terms[k - 1].copy()
    for j in range(k - 2, -1, -1):
        x = basis.terms[j] + t * x
    x = x * basis.tau
    _compose_count += k * x.shape[1]
    return x


@dataclass
class IntervalPlan:
    lo: float
    hi: float
    params: RateParams
    grid: List[float]


def plan_intervals(config: PathConfig, rho: RhoBounds, sigma_d) -> List[IntervalPlan]:
    """path_solver.cpp:85-108."""
    splits = interval_split(config.lambda_min, config.lambda_max, config.num_intervals)
    plans = []
    cursor = 0
    for i, (lo, hi) in enumerate(splits):
        params = tune_interval(lo, hi, rho, sigma_d, config.epsilon)
        last = i + 1 == len(splits)
        grid = []
        while cursor < len(config.lambdas) and (last or config.lambdas[cursor] <= hi):
            grid.append(config.lambdas[cursor])
            cursor += 1
        plans.append(IntervalPlan(lo, hi, params, grid))
    return plans


def build_interval_basis_matrix(op, c: np.ndarray, p: Preconditioner, plan: IntervalPlan,
                                gram: Optional[Callable] = None) -> BinomialBasis:
    """path_solver.cpp:110-141 (per-RHS-column loop, tau/2 retry)."""

    def attempt(tau):
        k = plan.params.k
        per_col = [ihs_basis_core(op, c[:, col], p, tau, k, gram) for col in range(c.shape[1])]
        terms = [np.stack([pc[:, j] for pc in per_col], axis=1) for j in range(k)]
        return BinomialBasis(terms, tau, plan.lo, plan.hi, "ihs")

    try:
        return attempt(plan.params.alpha)
    except BasisDivergedError:
        try:
            return attempt(plan.params.alpha / 2.0)
        except BasisDivergedError:
            raise SolverError("interval basis diverged twice, even at tau/2")


@dataclass
class PathPoint:
    lam: float
    solution: np.ndarray
    seconds: float = 0.0
    iterations: int = 0


@dataclass
class RegPathResult:
    solver: str
    points: List[PathPoint]
    setup_seconds: float = 0.0
    total_seconds: float = 0.0
    bases: List[BinomialBasis] = field(default_factory=list)
    sa: Optional[np.ndarray] = None


def run_path(solver_name, op, c: np.ndarray, config: PathConfig, spec: SketchSpec, rho: RhoBounds,
             sigma_d=None, recover=None, interval_subset: Optional[Sequence[int]] = None,
             keep_bases: bool = False) -> RegPathResult:
    """path_solver.cpp:147-190.  `interval_subset` restricts the basis build and
    the composes to the listed intervals (each interval is independent in the
    reference, :168-186, so a subset is exact); used for bounded CPU samples."""
    import time
    t_total = time.perf_counter()
    config.validate()
    rho.validate()
    t_setup = time.perf_counter()
    sa = sketch_apply(spec, op)
    svd = thin_svd(sa)
    plans = plan_intervals(config, rho, sigma_d)
    pre = Preconditioner.build_from_svd(svd, sa.shape[0], sa.shape[1], plans[0].params.lambda0)
    setup = time.perf_counter() - t_setup
    points = []
    bases = []
    for idx, plan in enumerate(plans):
        if interval_subset is not None and idx not in interval_subset:
            continue
        t_setup = time.perf_counter()
        pre = pre.reshift(plan.params.lambda0)
        basis = build_interval_basis_matrix(op, c, pre, plan)
        setup += time.perf_counter() - t_setup
        if keep_bases:
            bases.append(basis)
        for lam in plan.grid:
            t_eval = time.perf_counter()
            x = compose_horner(basis, basis.tau * lam)
            secs = time.perf_counter() - t_eval
            points.append(PathPoint(lam, recover(x) if recover else x, secs))
    return RegPathResult(solver_name, points, setup, time.perf_counter() - t_total, bases, sa)


def ihs_bin_path(a, b: np.ndarray, config: PathConfig, spec: SketchSpec, rho: RhoBounds, sigma_d=None,
                 **kw) -> RegPathResult:
    """path_solver.cpp:289-305 (vector b) and 307-326 (matrix B)."""
    b2 = b.reshape(b.shape[0], -1)
    _require(b2.shape[0] == _rows(a), "ihs_bin_path: dimension mismatch")
    _require(spec.n == _rows(a), "ihs_bin_path: spec.n must equal A.rows")
    c = apply_transpose(a, b2)
    return run_path("ihs-bin", a, c, config, spec, rho, sigma_d, None, **kw)


ihs_bin_path_matrix = ihs_bin_path


def dual_path(a, b: np.ndarray, config: PathConfig, spec: SketchSpec, rho: RhoBounds, sigma_d=None,
              **kw) -> RegPathResult:
    """path_solver.cpp:328-351.  Matrix B is handled column by column, i.e. K
    dual_path calls."""
    b2 = b.reshape(b.shape[0], -1)
    _require(b2.shape[0] == _rows(a), "dual_path: dimension mismatch")
    _require(spec.n == _cols(a), "dual_path: spec.n must equal A.cols (the dual operator is A^T)")
    at = transpose(a)
    c = b2.copy()
    return run_path("dual", at, c, config, spec, rho, sigma_d, lambda z: apply(at, z), **kw)


def ihs_basis(a, b: np.ndarray, p: Preconditioner, tau: float, k: int) -> BinomialBasis:
    """path_solver.cpp:242-251."""
    _require(b.shape[0] == _rows(a), "ihs_basis: dimension mismatch")
    c = apply_transpose(a, b)
    tilde = ihs_basis_core(a, c, p, tau, k)
    return BinomialBasis([tilde[:, j:j + 1].copy() for j in range(k)], tau)


def ihs_compose(basis: BinomialBasis, lam: float) -> np.ndarray:
    """path_solver.cpp:253-256."""
    return compose_horner(basis, basis.tau * lam)[:, 0]


def ihs_basis_matrix(a, b: np.ndarray, p: Preconditioner, tau: float, k: int) -> BinomialBasis:
    """path_solver.cpp:258-281."""
    per_col = [ihs_basis_core(a, apply_transpose(a, b[:, col].copy()), p, tau, k) for col in range(b.shape[1])]
    return BinomialBasis([np.stack([pc[:, j] for pc in per_col], axis=1) for j in range(k)], tau)


def ihs_compose_matrix(basis: BinomialBasis, lam: float) -> np.ndarray:
    return compose_horner(basis, basis.tau * lam)


# --------------------------------------------------------------------------
# Comparison baselines (baselines.hpp; baselines.cpp:51-226)
# --------------------------------------------------------------------------

def _descending_order(grid):
    """baselines.cpp:40-47 (std::sort with '>' -- ties are never present in a
    validated grid except repeated lambdas, kept in index order here)."""
    return sorted(range(len(grid)), key=lambda i: -grid[i])


def svd_path(a, b: np.ndarray, config: PathConfig) -> RegPathResult:
    """baselines.cpp:51-78: one thin SVD of A, a diagonal solve per lambda."""
    config.validate()
    _require(b.shape[0] == _rows(a), "svd_path: dimension mismatch")
    dense = a.to_dense() if is_csr(a) else a
    u, s, vt = thin_svd(dense)
    utb = u.T @ b
    pts = [PathPoint(lam, vt.T @ (s * utb / (s * s + lam))) for lam in config.lambdas]
    return RegPathResult("svd", pts)


def direct_path(a, b: np.ndarray, config: PathConfig) -> RegPathResult:
    """baselines.cpp:80-118: A^T A once, Cholesky of A^T A + lambda I per lambda."""
    config.validate()
    _require(b.shape[0] == _rows(a), "direct_path: dimension mismatch")
    d = _cols(a)
    gram = apply_transpose(a, apply(a, np.eye(d))) if is_csr(a) else a.T @ a
    atb = apply_transpose(a, b)
    pts = []
    for lam in config.lambdas:
        sh = gram + lam * np.eye(d)
        try:
            lo = np.linalg.cholesky(sh)
        except np.linalg.LinAlgError:
            raise SolverError("direct_path: Cholesky factorization failed")
        y = np.linalg.solve(lo, atb)
        pts.append(PathPoint(lam, np.linalg.solve(lo.T, y)))
    return RegPathResult("direct", pts)


def warm_cg_path(a, b: np.ndarray, config: PathConfig) -> RegPathResult:
    """baselines.cpp:120-162: CG on (A^T A + lambda I) x = A^T b, swept from the
    largest lambda down with warm starts; stop at ||r|| <= eps ||A^T b||; cap 10 d."""
    config.validate()
    _require(b.shape[0] == _rows(a), "warm_cg_path: dimension mismatch")
    atb = apply_transpose(a, b)
    rhs_norm = float(np.linalg.norm(atb))
    d = _cols(a)
    cap = 10 * d
    tol = config.epsilon * (rhs_norm if rhs_norm > 0.0 else 1.0)
    pts = [None] * len(config.lambdas)
    x = np.zeros(d)
    for idx in _descending_order(config.lambdas):
        lam = config.lambdas[idx]
        r = atb - gram_apply(a, x) - lam * x
        p = r.copy()
        rr = float(r @ r)
        iters = 0
        while math.sqrt(rr) > tol:
            if iters >= cap:
                raise SolverError("warm_cg_path: iteration cap (10 d) reached")
            q = gram_apply(a, p) + lam * p
            alpha = rr / float(p @ q)
            x = x + alpha * p
            r = r - alpha * q
            rr_next = float(r @ r)
            p = r + (rr_next / rr) * p
            rr = rr_next
            iters += 1
        pts[idx] = PathPoint(lam, x.copy(), iterations=iters)
    return RegPathResult("cg", pts)


def warm_ihs_path(a, b: np.ndarray, config: PathConfig, spec: SketchSpec, rho: RhoBounds) -> RegPathResult:
    """baselines.cpp:164-224: warm-started preconditioned iterations per lambda
    with the shift pinned to the active lambda, step 2 / (1/rho1 + 1/rho2),
    stop at ||grad|| <= eps ||A^T b||, cap 1000, one tau/2 retry."""
    config.validate()
    rho.validate()
    _require(b.shape[0] == _rows(a), "warm_ihs_path: dimension mismatch")
    _require(spec.n == _rows(a), "warm_ihs_path: spec.n must equal A.rows")
    sa = sketch_apply(spec, a)
    pre = Preconditioner.build_from_svd(thin_svd(sa), sa.shape[0], sa.shape[1], config.lambdas[-1])
    atb = apply_transpose(a, b)
    rhs_norm = float(np.linalg.norm(atb))
    tau_nominal = 2.0 / (1.0 / rho.rho1 + 1.0 / rho.rho2)
    tol = config.epsilon * (rhs_norm if rhs_norm > 0.0 else 1.0)
    cap = 1000
    pts = [None] * len(config.lambdas)
    x = np.zeros(_cols(a))
    for idx in _descending_order(config.lambdas):
        lam = config.lambdas[idx]
        pre = pre.reshift(lam)
        tau = tau_nominal
        xs = x.copy()
        iters = 0
        retried = False
        while True:
            grad = gram_apply(a, xs) + lam * xs - atb
            if float(np.linalg.norm(grad)) <= tol:
                break
            if iters >= cap:
                raise SolverError("warm_ihs_path: iteration cap reached")
            xs = xs - tau * pre.apply(grad)
            iters += 1
            if not np.all(np.isfinite(xs)):
                if retried:
                    raise SolverError("warm_ihs_path: diverged twice, even at tau/2")
                retried = True
                tau /= 2.0
                xs = x.copy()
                iters = 0
        x = xs
        pts[idx] = PathPoint(lam, x.copy(), iterations=iters)
    return RegPathResult("ihs", pts)


# --------------------------------------------------------------------------
# Adaptive sketch dimension (adaptive.hpp; adaptive.cpp:19-137)
# --------------------------------------------------------------------------

@dataclass
class AdaptiveConfig:
    gamma1: float = 0.5
    gamma2: float = 1e-4
    gamma3: float = 0.9
    epsilon: float = 1e-8
    m_initial: int = 0
    m_cap: int = 0
    iteration_cap: int = 200

    def initial_m(self, d):
        return self.m_initial if self.m_initial > 0 else max(16, d // 64)

    def cap_m(self, d):
        return self.m_cap if self.m_cap > 0 else d

    def validate(self, d):
        """adaptive.cpp:19-28."""
        _require(0.0 < self.gamma1 < 1.0, "adaptive: gamma1 not in (0,1)")
        _require(0.0 < self.gamma2 < 1.0, "adaptive: gamma2 not in (0,1)")
        _require(0.0 < self.gamma3 < 1.0, "adaptive: gamma3 not in (0,1)")
        _require(self.epsilon > 0.0, "adaptive: epsilon must be positive")
        _require(self.initial_m(d) >= 1, "adaptive: m_initial must be >= 1")
        _require(self.cap_m(d) <= d, "adaptive: m_cap must not exceed d")
        _require(self.initial_m(d) <= self.cap_m(d), "adaptive: m_initial above m_cap")
        _require(self.iteration_cap >= 1, "adaptive: iteration cap must be >= 1")


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


def armijo_step(f, x, direction, dir_dot_grad, gamma1, gamma2) -> float:
    """adaptive.cpp:39-51."""
    _require(dir_dot_grad > 0.0, "armijo: direction is not a descent direction")
    fx = f(x)
    step = 1.0
    for _ in range(51):
        if f(x - step * direction) <= fx - gamma2 * step * dir_dot_grad:
            return step
        step *= gamma1
    raise SolverError("armijo: no acceptable step within 50 backtracks")


def adaptive_sketch_dim(a, b, lambda_min: float, config: AdaptiveConfig, spec_template: SketchSpec,
                        x0=None) -> AdaptiveResult:
    """adaptive.cpp:53-135: sketched Newton steps at lambda_min with Armijo
    steps, doubling m (fresh seed per doubling) when d.grad stalls."""
    _require(lambda_min > 0.0, "adaptive: lambda_min must be positive")
    _require(b.shape[0] == _rows(a), "adaptive: dimension mismatch")
    d = _cols(a)
    config.validate(d)
    atb = apply_transpose(a, b)

    def objective(x):
        r = apply(a, x) - b
        return 0.5 * float(r @ r) + 0.5 * lambda_min * float(x @ x)

    def gradient(x):
        return gram_apply(a, x) + lambda_min * x - atb

    res = AdaptiveResult(config.initial_m(d), np.array(x0, dtype=np.float64) if x0 is not None else np.zeros(d))
    m_cap = config.cap_m(d)

    def make_pre(m, resample):
        seed = (spec_template.seed + 0x9E3779B97F4A7C15 * resample) % (1 << 64)
        spec = SketchSpec(spec_template.kind, m, spec_template.n, spec_template.s, seed)
        if spec.kind == "identity":
            spec.m = spec.n
        if spec.kind == "sjlt" and spec.m % spec.s != 0:
            spec.m += spec.s - spec.m % spec.s
        return Preconditioner.build(sketch_apply(spec, a), lambda_min)

    pre = make_pre(res.m, 0)
    grad = gradient(res.x)
    direction = pre.apply(grad)
    progress = float(direction @ grad)
    loop_guard = 0
    while progress >= config.epsilon:
        loop_guard += 1
        if res.iterations >= config.iteration_cap or loop_guard > 4 * config.iteration_cap:
            break
        step = armijo_step(objective, res.x, direction, progress, config.gamma1, config.gamma2)
        x_next = res.x - step * direction
        grad_next = gradient(x_next)
        dir_next = pre.apply(grad_next)
        progress_next = float(dir_next @ grad_next)
        rec = AdaptiveStep(res.m, objective(res.x), objective(x_next), step, progress, False)
        if progress_next >= config.gamma3 * progress and res.m < m_cap:
            res.m = min(2 * res.m, m_cap)
            res.doublings += 1
            rec.doubled = True
            pre = make_pre(res.m, res.doublings)
            grad = gradient(res.x)
            direction = pre.apply(grad)
            progress = float(direction @ grad)
        else:
            res.x = x_next
            grad, direction, progress = grad_next, dir_next, progress_next
            res.iterations += 1
        res.trace.append(rec)
    res.converged = progress < config.epsilon
    res.stalled_at_cap = (not res.converged) and res.m >= m_cap
    return res


def losses(a, b, x, lam, a_test=None, b_test=None):
    """path_solver.cpp:425-438."""
    resid = apply(a, x) - b
    train = 0.5 * float(np.sum(resid * resid)) + 0.5 * lam * float(np.sum(x * x))
    test = None
    if a_test is not None and b_test is not None:
        tr = apply(a_test, x) - b_test
        test = 0.5 * float(np.sum(tr * tr))
    return train, test


# --------------------------------------------------------------------------
# Test-support oracles (tests/test_support.hpp:15-106)
# --------------------------------------------------------------------------


def random_dense(rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """test_support.hpp:15-21 (row-major draws) for a fresh SeededRng(seed)."""
    return fill_normals(seed, rows * cols, scale).reshape(rows, cols)


def ridge_solve_oracle(a: np.ndarray, b: np.ndarray, lam: float) -> np.ndarray:
    normal = a.T @ a + lam * np.eye(a.shape[1])
    return np.linalg.solve(normal, a.T @ b)


def dense_preconditioner_oracle(sa: np.ndarray, lambda0: float) -> np.ndarray:
    return np.linalg.inv(sa.T @ sa + lambda0 * np.eye(sa.shape[1]))


def ihs_iterate_oracle(a, b, p_dense, tau, lam, steps):
    x = np.zeros(a.shape[1])
    for _ in range(steps):
        grad = a.T @ (a @ x - b) + lam * x
        x = x - tau * (p_dense @ grad)
    return x


def rel_error(got, want) -> float:
    denom = float(np.linalg.norm(want))
    if denom == 0.0:
        return float(np.linalg.norm(got))
    return float(np.linalg.norm(np.asarray(got) - np.asarray(want)) / denom)


# ---- data_io.cpp: LIBSVM and CSV (host formats either side of the path) ----


class ParseError(RuntimeError):
    """data_io.hpp ParseError (data_io.cpp:41-48): 'line L, column C: ...'."""

    def __init__(self, msg, line, column):
        super().__init__(f"line {line}, column {column}: {msg}")
        self.line, self.column = line, column


_C_SPACE = " \t\n\v\f\r"


def _parse_real(tok, line, col):
    """parse_real (data_io.cpp:23-39): std::stod on the whole token, finite only.
    (Python's float() stands in for strtod on decimal input; hex floats and
    ERANGE underflow are the C side's.)"""
    import re

    m = re.match(r"[+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan)", tok, re.IGNORECASE)
    if not m:  # strtod converts nothing
        raise ParseError(f"malformed number '{tok}'", line, col)
    if m.end() != len(tok):  # strtod stops early: std::stod's `used` falls short
        raise ParseError(f"trailing characters in number '{tok}'", line, col)
    v = float(m.group(0))
    if not math.isfinite(v):
        raise ParseError(f"non-finite value '{tok}'", line, col)
    return v


def parse_libsvm(text, feature_override=None):
    """parse_libsvm (data_io.cpp:50-127) -> (Csr, labels)."""
    offsets, cols, vals, labels = [0], [], [], []
    max_index = 0
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for line_no, raw in enumerate(lines, start=1):
        line = raw.split("#", 1)[0]
        pos = 0

        def token():
            nonlocal pos
            while pos < len(line) and line[pos] in _C_SPACE:
                pos += 1
            start = pos
            while pos < len(line) and line[pos] not in _C_SPACE:
                pos += 1
            return line[start:pos], start + 1

        lab, lcol = token()
        if not lab:
            continue
        labels.append(_parse_real(lab, line_no, lcol))
        prev = 0
        while True:
            tok, col = token()
            if not tok:
                break
            colon = tok.find(":")
            if colon <= 0 or colon + 1 == len(tok):
                raise ParseError(f"expected index:value, got '{tok}'", line_no, col)
            part = tok[:colon]
            if not (part.isdigit() or (part[:1] == "-" and part[1:].isdigit())) or not part.isascii():
                raise ParseError(f"malformed feature index '{part}'", line_no, col)
            idx = int(part)
            if idx < 1:
                raise ParseError(f"feature index must be >= 1, got {idx}", line_no, col)
            if idx <= prev:
                raise ParseError(f"non-increasing feature index {idx}", line_no, col)
            vals.append(_parse_real(tok[colon + 1:], line_no, col + colon + 1))
            cols.append(idx - 1)
            prev = idx
            max_index = max(max_index, idx)
        offsets.append(len(vals))
    if feature_override is not None and feature_override < max_index:
        raise ValueError(f"parse_libsvm: declared dimension {feature_override} below max index {max_index}")
    ncols = max_index if feature_override is None else feature_override
    return (Csr(len(labels), ncols, np.asarray(offsets, dtype=np.int64), np.asarray(cols, dtype=np.int64),
                np.asarray(vals, dtype=np.float64)), np.asarray(labels, dtype=np.float64))


def write_csv(results):
    """write_csv (data_io.cpp:344-364) -> str."""
    rows = [(p.lam, r.solver, p) for r in results for p in r.points]
    rows.sort(key=lambda t: (t[0], t[1].encode()))  # (Python's sort is stable, like std::stable_sort)
    out = ["lambda,train_loss,test_loss,time_s,solver\n"]
    for lam, solver, p in rows:
        test = "%.17g" % p.test_loss if getattr(p, "test_loss", None) is not None else ""
        out.append(f"{'%.17g' % lam},{'%.17g' % p.train_loss},{test},{'%.17g' % p.seconds},{solver}\n")
    return "".join(out)
