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


def c1(seed=0, scale=1.0, n_rows=None):
    """4096 x 256, A_ij ~ N(0,1) j^-1/2 (j 1-indexed), Gaussian m=512, T=100 in [1e-3, 1e2].
    `n_rows` (every generator): that many rows (of the sketched operator) with d and m unchanged --
    the CPU baseline's row subsample."""
    n, d, m = int(4096 * scale), max(8, int(256 * scale)), max(16, int(512 * scale))
    n = n_rows or n
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1)))
    x = g.standard_normal(d)
    b = a @ x + 0.1 * g.standard_normal(n)
    return Workload("C1", a, b.reshape(n, 1), dict(kind="gaussian", m=m, n=n, s=1, seed=0), 1e-3, 1e2, 100,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c2(seed=0, scale=1.0, n_rows=None):
    """65536 x 1024, A = U diag(0.99^j) V^T (Haar U, V; j 0-based), SRHT m=2048, T=1000 in [1e-4, 1e3]."""
    n, d, m = int(65536 * scale), max(8, int(1024 * scale)), max(16, int(2048 * scale))
    n = n_rows or n
    g = _rng(seed)
    u, _ = np.linalg.qr(g.standard_normal((n, d)))
    v, _ = np.linalg.qr(g.standard_normal((d, d)))
    sig = 0.99 ** np.arange(d)
    a = np.asfortranarray((u * sig) @ v.T)
    x = g.standard_normal(d)
    b = a @ x + 0.01 * g.standard_normal(n)
    return Workload("C2", a, b.reshape(n, 1), dict(kind="srht", m=m, n=n, s=1, seed=0), 1e-4, 1e3, 1000,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c3(seed=0, scale=1.0, n_rows=None):
    """1,048,576 x 2048, A_ij ~ N(0,1)/(1+j) (j 0-based), Gaussian m=4096, T=1000 in [1e-3, 1e2]."""
    n, d, m = int(1048576 * scale), max(8, int(2048 * scale)), max(16, int(4096 * scale))
    n = n_rows or n
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / (1.0 + np.arange(d)))
    x = g.standard_normal(d)
    b = a @ x + 0.1 * g.standard_normal(n)
    return Workload("C3", a, b.reshape(n, 1), dict(kind="gaussian", m=m, n=n, s=1, seed=0), 1e-3, 1e2, 1000,
                    mp_envelope(d, m), meta=dict(n=n, d=d))


def c4(seed=0, scale=1.0, nnz_per_row=16, n_rows=None):
    """4,194,304 x 65,536 CSR, 16 distinct sorted columns per row, N(0,1) values;
    CountSketch m=8192 (Woodbury m x m), T=500 in [1e-2, 1e2]."""
    n, d, m = int(4194304 * scale), max(64, int(65536 * scale)), max(16, int(8192 * scale))
    n = n_rows or n
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


def c5(seed=0, scale=1.0, K=16, n_rows=None):
    """16384 x 131072, A_ij ~ N(0,1)/sqrt(d), B = A X* + 0.1 E (K=16), dual route,
    Gaussian sketch of A^T with m=4096, T=200 in [1e-3, 1e1].  (`n_rows` sets the
    columns of A: the rows of the sketched dual operator A^T.)"""
    n, d, m = int(16384 * scale), max(16, int(131072 * scale)), max(16, int(4096 * scale))
    d = n_rows or d
    g = _rng(seed)
    a = np.asfortranarray(g.standard_normal((n, d)) / math.sqrt(d))
    x = g.standard_normal((d, K))
    b = a @ x + 0.1 * g.standard_normal((n, K))
    return Workload("C5", a, np.asfortranarray(b), dict(kind="gaussian", m=m, n=d, s=1, seed=0), 1e-3, 1e1, 200,
                    (1.0, 1e-5), dual=True, meta=dict(n=n, d=d, K=K))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def get(name: str, seed: int = 0, scale: float = 1.0, n_rows=None) -> Workload:
    return CONFIGS[name.lower()](seed=seed, scale=scale, n_rows=n_rows)


# ---------------------------------------------------------------------------
# Device-side generation (bench.py at full size, 1..8 ranks)
# ---------------------------------------------------------------------------
#
# The large configs are generated on the GPU with torch in fixed chunks of
# rows (columns of A for the dual C5), each chunk from its own generator
# seeded by (seed, chunk): a rank generates only the chunks of its shard and
# the global matrix is the same for every world size.  Shards are whole
# chunks, contiguous, as equal as the chunk count allows.  C1/C2 reuse the
# numpy generators above (the same data as the tests) and upload the shard.

CHUNK_ROWS = 65536       # C3 / C4 rows per chunk
CHUNK_COLS_C5 = 8192     # C5 columns (rows of the dual operator A^T) per chunk


@dataclass
class DeviceWorkload:
    name: str
    route: str                   # "rows" (primal, row shards) or "cols" (dual, column shards of A)
    sparse: bool
    n: int                       # rows of A
    d: int                       # columns of A
    K: int
    lo: int                      # shard [lo, hi): rows of A ("rows") or columns of A ("cols")
    hi: int
    a_t: object = None           # dense: torch (d, n_loc) == A_loc column-major, or (d_loc, n) for "cols"
    csr: tuple = None            # sparse: (offsets int64 [n_loc+1], cols int64, vals f64) on the device
    b: object = None             # torch (K, rows of b) == b column-major (local rows; all n for "cols")
    sketch: dict = None
    lambda_min: float = 0.0
    lambda_max: float = 0.0
    T: int = 0
    rho: tuple = ()
    epsilon: float = 1e-6
    desc: str = ""

    @property
    def local(self):
        return self.hi - self.lo


def chunk_shard(total, chunk, world, rank):
    """[lo, hi) of `rank`'s whole-chunk shard of `total` items."""
    nch = -(-total // chunk)
    c0, c1 = (rank * nch) // world, ((rank + 1) * nch) // world
    return min(total, c0 * chunk), min(total, c1 * chunk)


def _gen(torch, dev, seed, chunk):
    return torch.Generator(device=dev).manual_seed(seed * 1_000_003 + chunk + 1)


def device_workload(name, rank=0, world=1, dev=None, seed=0, allreduce=None):
    """The full-size workload `name` for `rank` of `world`, resident on `dev`.
    `allreduce(tensor)` sums a tensor over ranks (C5's B = sum_p A_p X*_p)."""
    import torch

    dev = dev or torch.device("cuda")
    f64 = dict(dtype=torch.float64, device=dev)
    name = name.lower()
    if name in ("c1", "c2"):
        w = get(name, seed=seed)
        n, d = w.a.shape
        lo, hi = (rank * n) // world, ((rank + 1) * n) // world
        a_t = torch.from_numpy(np.ascontiguousarray(w.a[lo:hi].T)).to(dev)
        b = torch.from_numpy(np.ascontiguousarray(w.b[lo:hi].T)).to(dev)
        return DeviceWorkload(w.name, "rows", False, n, d, 1, lo, hi, a_t=a_t, b=b, sketch=w.sketch,
                              lambda_min=w.lambda_min, lambda_max=w.lambda_max, T=w.T, rho=w.rho,
                              epsilon=w.epsilon, desc=_desc(w.name, n, d, w, "dense"))
    if name == "c3":
        n, d, m = 1048576, 2048, 4096
        lo, hi = chunk_shard(n, CHUNK_ROWS, world, rank)
        scale = 1.0 / (1.0 + torch.arange(d, **f64))
        xs = torch.randn(d, generator=_gen(torch, dev, seed, 1 << 20), **f64)
        a_t = torch.empty((d, hi - lo), **f64)
        b = torch.empty((1, hi - lo), **f64)
        for r0 in range(lo, hi, CHUNK_ROWS):
            c = r0 // CHUNK_ROWS
            rows = min(CHUNK_ROWS, hi - r0)
            g = _gen(torch, dev, seed, c)
            blk = torch.randn((d, rows), generator=g, **f64) * scale[:, None]
            a_t[:, r0 - lo:r0 - lo + rows] = blk
            b[0, r0 - lo:r0 - lo + rows] = blk.T @ xs + 0.1 * torch.randn(rows, generator=g, **f64)
        sk = dict(kind="gaussian", m=m, n=n, s=1, seed=0)
        w = Workload("C3", None, None, sk, 1e-3, 1e2, 1000, mp_envelope(d, m))
        return DeviceWorkload("C3", "rows", False, n, d, 1, lo, hi, a_t=a_t, b=b, sketch=sk, lambda_min=1e-3,
                              lambda_max=1e2, T=1000, rho=w.rho, desc=_desc("C3", n, d, w, "dense"))
    if name == "c4":
        n, d, m, k = 4194304, 65536, 8192, 16
        lo, hi = chunk_shard(n, CHUNK_ROWS, world, rank)
        xs = torch.randn(d, generator=_gen(torch, dev, seed, 1 << 20), **f64)
        cols_l, vals_l, b_l = [], [], []
        for r0 in range(lo, hi, CHUNK_ROWS):
            c = r0 // CHUNK_ROWS
            rows = min(CHUNK_ROWS, hi - r0)
            g = _gen(torch, dev, seed, c)
            cols = torch.randint(0, d, (rows, k), generator=g, device=dev, dtype=torch.int64)
            cols, _ = torch.sort(cols, dim=1)
            bad = (cols[:, 1:] == cols[:, :-1]).any(dim=1)
            while bool(bad.any()):  # uniform k-subsets: redraw rows with a repeated column
                idx = torch.nonzero(bad).flatten()
                redo, _ = torch.sort(torch.randint(0, d, (idx.numel(), k), generator=g, device=dev,
                                                   dtype=torch.int64), dim=1)
                cols[idx] = redo
                bad = torch.zeros_like(bad)
                bad[idx] = (redo[:, 1:] == redo[:, :-1]).any(dim=1)
            vals = torch.randn((rows, k), generator=g, **f64)
            b_l.append((vals * xs[cols]).sum(dim=1) + 0.1 * torch.randn(rows, generator=g, **f64))
            cols_l.append(cols.reshape(-1))
            vals_l.append(vals.reshape(-1))
        offsets = torch.arange(0, (hi - lo) * k + 1, k, device=dev, dtype=torch.int64)
        csr = (offsets, torch.cat(cols_l), torch.cat(vals_l))
        b = torch.cat(b_l).reshape(1, -1)
        sk = dict(kind="countsketch", m=m, n=n, s=1, seed=0)
        w = Workload("C4", None, None, sk, 1e-2, 1e2, 500, (1.0, 1e-5))
        return DeviceWorkload("C4", "rows", True, n, d, 1, lo, hi, csr=csr, b=b, sketch=sk, lambda_min=1e-2,
                              lambda_max=1e2, T=500, rho=(1.0, 1e-5), desc=_desc("C4", n, d, w, "CSR 16 nnz/row"))
    if name == "c5":
        n, d, m, K = 16384, 131072, 4096, 16
        lo, hi = chunk_shard(d, CHUNK_COLS_C5, world, rank)
        a_t = torch.empty((hi - lo, n), **f64)  # columns [lo, hi) of A, column-major (ld n)
        part = torch.zeros((K, n), **f64)       # B^T partial = (A_p X*_p)^T
        for c0 in range(lo, hi, CHUNK_COLS_C5):
            c = c0 // CHUNK_COLS_C5
            cols = min(CHUNK_COLS_C5, hi - c0)
            g = _gen(torch, dev, seed, c)
            blk = torch.randn((cols, n), generator=g, **f64) / math.sqrt(d)
            a_t[c0 - lo:c0 - lo + cols] = blk
            xs = torch.randn((K, cols), generator=g, **f64)
            part += xs @ blk
        if allreduce is not None and world > 1:
            allreduce(part)
        b = part + 0.1 * torch.randn((K, n), generator=_gen(torch, dev, seed, 1 << 20), **f64)
        sk = dict(kind="gaussian", m=m, n=d, s=1, seed=0)
        w = Workload("C5", None, None, sk, 1e-3, 1e1, 200, (1.0, 1e-5), dual=True)
        return DeviceWorkload("C5", "cols", False, n, d, K, lo, hi, a_t=a_t, b=b, sketch=sk, lambda_min=1e-3,
                              lambda_max=1e1, T=200, rho=(1.0, 1e-5),
                              desc=_desc("C5", n, d, w, "dense, dual (A^T sketched), K=16"))
    raise ValueError(f"unknown config {name}")


def _desc(name, n, d, w, layout):
    return (f"{name}: {n}x{d} {layout}, {w.sketch['kind']} m={w.sketch['m']}, T={w.T} log-spaced "
            f"[{w.lambda_min:g},{w.lambda_max:g}], eps={w.epsilon:g}, L=auto, rho=({w.rho[0]:.4g},{w.rho[1]:.4g})")
