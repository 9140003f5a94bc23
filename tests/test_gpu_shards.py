"""Shard arithmetic of the library on one GPU, no communicator.

A context holding rows [row0, row1) of A (rp_set_dense_rows / rp_set_csr_rows)
or columns [col0, col1) (rp_set_dense_cols, the dual route) computes its
rank's partial products -- without a communicator the all-reduce is a no-op --
so the partial sketch S[:, rows] A[rows, :] is observable directly:

* per shard, bit for bit: the partial sketch equals the oracle's sketch of A
  with every row outside the shard zeroed, for CountSketch, SJLT and SRHT
  (same draws, same accumulation / butterfly order; the zero rows add exact
  zeros), and within 1e-13 for the Gaussian sketch (GEMM summation order) --
  so the MT stream offsets r*n + row0, the global CountSketch draw stream and
  the local SRHT rows are exercised at row0 > 0;
* summed over the shards: the unsharded oracle sketch within 1e-13;
* the linear term A_p^T b_p and the Gram product A_p^T (A_p W) sum to the
  unsharded ones within 1e-13.

Reference: sketch.cpp:83-136, 138-173 (draw order), matrix.cpp:140-172.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _shards(n, parts):
    return [((p * n) // parts, ((p + 1) * n) // parts) for p in range(parts)]


def _zeroed(a, r0, r1):
    z = np.zeros_like(a)
    z[r0:r1] = a[r0:r1]
    return np.asfortranarray(z)


def _rel(x, ref):
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("kind,m,s", [("countsketch", 64, 1), ("sjlt", 64, 4), ("srht", 64, 1),
                                      ("gaussian", 48, 1)])
@pytest.mark.parametrize("parts", [2, 3, 4])
def test_dense_row_shards_sketch(rp, oracle, kind, m, s, parts):
    n, d = 700, 24  # n not a power of two: SRHT pads to 1024 across the shard boundaries
    a = oracle.random_dense(n, d, 11) / np.sqrt(np.arange(1, d + 1))
    spec_o = oracle.SketchSpec(kind, m, n, s, 7)
    full = oracle.sketch_apply(spec_o, a)
    total = np.zeros_like(full)
    for r0, r1 in _shards(n, parts):
        ctx = rp.Context(0)
        loc = np.asfortranarray(a[r0:r1])
        rp.set_dense_rows_host(ctx, n, r0, r1 - r0, d, loc.ctypes.data, r1 - r0)
        out = np.empty((m, d), order="F")
        cs = rp.SketchSpec(kind, m, n, s, 7).c()
        ctx.check(rp.lib().rp_sketch_apply(ctx.handle, rp.ctypes.byref(cs), 0, rp._ptr(out), rp.RP_HOST))
        want = oracle.sketch_apply(spec_o, _zeroed(a, r0, r1))
        if kind == "gaussian":
            assert _rel(out, want) <= 1e-13, (r0, r1)
        else:
            assert np.array_equal(out, want), (kind, r0, r1, int(np.count_nonzero(out != want)))
        total += out
    assert _rel(total, full) <= 1e-13


@pytest.mark.parametrize("kind,s", [("countsketch", 1), ("sjlt", 2), ("gaussian", 1)])
def test_csr_row_shards_sketch(rp, oracle, kind, s):
    n, d, m = 900, 40, 32
    rng = np.random.default_rng(5)
    dense = np.where(rng.random((n, d)) < 0.15, rng.standard_normal((n, d)), 0.0)
    spec_o = oracle.SketchSpec(kind, m, n, s, 4)
    full = oracle.sketch_apply(spec_o, np.asfortranarray(dense))
    total = np.zeros_like(full)
    for r0, r1 in _shards(n, 3):
        blk = dense[r0:r1]
        nz = blk != 0
        off = np.concatenate([[0], np.cumsum(nz.sum(axis=1))]).astype(np.int64)
        cols = np.nonzero(nz)[1].astype(np.int64)
        vals = blk[nz]
        ctx = rp.Context(0)
        rp.set_csr_rows(ctx, n, r0, rp.Csr(r1 - r0, d, off, cols, vals))
        out = np.empty((m, d), order="F")
        cs = rp.SketchSpec(kind, m, n, s, 4).c()
        ctx.check(rp.lib().rp_sketch_apply(ctx.handle, rp.ctypes.byref(cs), 0, rp._ptr(out), rp.RP_HOST))
        want = oracle.sketch_apply(spec_o, _zeroed(dense, r0, r1))
        if kind == "gaussian":
            assert _rel(out, want) <= 1e-13
        else:
            assert np.array_equal(out, want), (kind, r0, r1)
        total += out
    assert _rel(total, full) <= 1e-13


@pytest.mark.parametrize("kind", ["gaussian", "countsketch", "srht"])
def test_dual_column_shards_sketch(rp, oracle, kind):
    """Dual route: the operator is A^T, sharded by columns of A (rows of A^T)."""
    n, d, m = 40, 520, 32
    a = oracle.random_dense(n, d, 13)
    at = np.asfortranarray(a.T)
    spec_o = oracle.SketchSpec(kind, m, d, 1, 9)
    full = oracle.sketch_apply(spec_o, at)
    total = np.zeros_like(full)
    for c0, c1 in _shards(d, 3):
        ctx = rp.Context(0)
        loc = np.asfortranarray(a[:, c0:c1])
        rp.set_dense_cols_host(ctx, n, d, c0, c1 - c0, loc.ctypes.data, n)
        out = np.empty((m, n), order="F")
        cs = rp.SketchSpec(kind, m, d, 1, 9).c()
        ctx.check(rp.lib().rp_sketch_apply(ctx.handle, rp.ctypes.byref(cs), 1, rp._ptr(out), rp.RP_HOST))
        want = oracle.sketch_apply(spec_o, _zeroed(at, c0, c1))
        if kind == "gaussian":
            assert _rel(out, want) <= 1e-13
        else:
            assert np.array_equal(out, want), (kind, c0, c1)
        total += out
    assert _rel(total, full) <= 1e-13


def test_row_shards_linear_term_and_gram(rp, oracle):
    n, d, W = 1000, 36, 5
    a = oracle.random_dense(n, d, 17)
    b = oracle.fill_normals(18, n)
    w = np.asfortranarray(oracle.random_dense(d, W, 19))
    c_tot = np.zeros(d)
    g_tot = np.zeros((d, W), order="F")
    for r0, r1 in _shards(n, 3):
        ctx = rp.Context(0)
        loc = np.asfortranarray(a[r0:r1])
        rp.set_dense_rows_host(ctx, n, r0, r1 - r0, d, loc.ctypes.data, r1 - r0)
        c = np.empty(d)
        bl = np.ascontiguousarray(b[r0:r1])
        ctx.check(rp.lib().rp_apply_transpose(ctx.handle, rp._ptr(bl), 1, rp._ptr(c), rp.RP_HOST))
        g = np.empty((d, W), order="F")
        ctx.check(rp.lib().rp_gram_apply(ctx.handle, rp._ptr(w), W, rp._ptr(g), rp.RP_HOST))
        assert _rel(c, loc.T @ bl) <= 1e-13
        assert _rel(g, loc.T @ (loc @ w)) <= 1e-13
        c_tot += c
        g_tot += g
    assert _rel(c_tot, a.T @ b) <= 1e-13
    assert _rel(g_tot, a.T @ (a @ w)) <= 1e-13
