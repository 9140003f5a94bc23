"""Seeded synthetic stand-ins for BASELINE.json's five configs (C1-C5).

No public dataset is involved: each generator reproduces the shapes, sizes and
value distributions the config states, with numpy's
PCG64 as the data RNG (data seed 0 unless given).  `scale` shrinks the row /
column counts for CPU-feasible parity runs while keeping the structure.

Every workload also pins the solver tuning the reference CLI would otherwise
derive (derive_rho makes these configs diverge):
epsilon = 1e-6, L = auto, rho = Marchenko-Pastur ((1 +- sqrt(d/m))^2) for
C1-C3, and a small-rho2 contractive envelope for the m < d_e configs C4/C5
(parity-only workloads).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Workload:
    name: str
    a: object                    # dense (n x d, Fortran order) or dict CSR
    b: np.ndarray                # n x K
    sketch: dict                 # kind, m, n, s, seed
    lambda_min: float
    lambda_max: float
    T: int
    rho: tuple
    dual: bool = False
    epsilon: float = 1e-6
    meta: dict = field(default_factory=dict)

    def lambdas(self, log_grid):
        """The evaluation grid, built with the caller's log_grid (the product's
        rp.log_grid or the oracle's; both restate spectrum.cpp:38-53)."""
        return log_grid(self.lambda_min, self.lambda_max, self.T)


def mp_envelope(d, m):
    r = math.sqrt(d / m)
    return (1.0 + r) ** 2, (1.0 - r) ** 2


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def c1(seed=0, scale=1.0):
    """4096 x 256, A_ij ~ N(0,1) j^-1/2 (j 1-indexed), Gaussian m=512, T=100 in [1e-3, 1e2]."""
    n, d, m = int(4096 * scale), max(8, int(256 * scale)), max(16, int(512 * scale))
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1)))
    x = g.standard_normal(d)
    b = a @ x + 0.1 * g.standard_normal(n)
    return Workload("C1", a, b.reshape(n, 1), dict(kind="gaussian", m=m, n=n, s=1, seed=0), 1e-3, 1e2, 100,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c2(seed=0, scale=1.0):
    """65536 x 1024, A = U diag(0.99^j) V^T (Haar U, V; j 0-based), SRHT m=2048, T=1000 in [1e-4, 1e3]."""
    n, d, m = int(65536 * scale), max(8, int(1024 * scale)), max(16, int(2048 * scale))
    g = _rng(seed)
    u, _ = np.linalg.qr(g.standard_normal((n, d)))
    v, _ = np.linalg.qr(g.standard_normal((d, d)))
    sig = 0.99 ** np.arange(d)
    a = np.asfortranarray((u * sig) @ v.T)
    x = g.standard_normal(d)
    b = a @ x + 0.01 * g.standard_normal(n)
    return Workload("C2", a, b.reshape(n, 1), dict(kind="srht", m=m, n=n, s=1, seed=0), 1e-4, 1e3, 1000,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c3(seed=0, scale=1.0):
    """1,048,576 x 2048, A_ij ~ N(0,1)/(1+j) (j 0-based), Gaussian m=4096, T=1000 in [1e-3, 1e2]."""
    n, d, m = int(1048576 * scale), max(8, int(2048 * scale)), max(16, int(4096 * scale))
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / (1.0 + np.arange(d)))
    x = g.standard_normal(d)
    b = a @ x + 0.1 * g.standard_normal(n)
    return Workload("C3", a, b.reshape(n, 1), dict(kind="gaussian", m=m, n=n, s=1, seed=0), 1e-3, 1e2, 1000,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c4(seed=0, scale=1.0, nnz_per_row=16):
    """4,194,304 x 65,536 CSR, 16 distinct sorted columns per row, N(0,1) values;
    CountSketch m=8192 (Woodbury m x m), T=500 in [1e-2, 1e2]."""
    n, d, m = int(4194304 * scale), max(64, int(65536 * scale)), max(16, int(8192 * scale))
    g = _rng(seed)
    k = min(nnz_per_row, d)
    # uniform k-subsets: draw k columns per row, redraw rows with a repeat
    cols = g.integers(0, d, size=(n, k))
    cols.sort(axis=1)
    bad = (np.diff(cols, axis=1) == 0).any(axis=1)
    while bad.any():
        idx = np.nonzero(bad)[0]
        redo = g.integers(0, d, size=(idx.shape[0], k))
        redo.sort(axis=1)
        cols[idx] = redo
        bad = np.zeros(n, dtype=bool)
        bad[idx] = (np.diff(redo, axis=1) == 0).any(axis=1)
    vals = g.standard_normal(n * k)
    offsets = np.arange(0, n * k + 1, k, dtype=np.int64)
    x = g.standard_normal(d)
    av = (vals.reshape(n, k) * x[cols]).sum(axis=1)
    b = av + 0.1 * g.standard_normal(n)
    csr = dict(rows=n, cols=d, offsets=offsets, indices=cols.reshape(-1), values=vals)
    return Workload("C4", csr, b.reshape(n, 1), dict(kind="countsketch", m=m, n=n, s=1, seed=0), 1e-2, 1e2, 500,
                    (1.0, 1e-5), meta=dict(n=n, d=d, nnz=n * k))


def c5(seed=0, scale=1.0, K=16):
    """16384 x 131072, A_ij ~ N(0,1)/sqrt(d), B = A X* + 0.1 E (K=16), dual route,
    Gaussian sketch of A^T with m=4096, T=200 in [1e-3, 1e1]."""
    n, d, m = int(16384 * scale), max(16, int(131072 * scale)), max(16, int(4096 * scale))
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / math.sqrt(d))
    x = g.standard_normal((d, K))
    b = a @ x + 0.1 * g.standard_normal((n, K))
    return Workload("C5", a, np.asfortranarray(b), dict(kind="gaussian", m=m, n=d, s=1, seed=0), 1e-3, 1e1, 200,
                    (1.0, 1e-5), dual=True, meta=dict(n=n, d=d, K=K))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def get(name: str, seed: int = 0, scale: float = 1.0) -> Workload:
    return CONFIGS[name.lower()](seed=seed, scale=scale)
