"""sketch_apply, apply / apply_transpose / gram_apply and the preconditioner on
the device vs the oracle (the reference's test_sketch / test_matrix_core /
test_preconditioner expectations, plus bit-exactness where the summation order
is the reference's)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAMILIES = [("gaussian", 12, 1), ("countsketch", 12, 1), ("sjlt", 12, 3), ("srht", 12, 1), ("identity", 64, 1)]


def _csr(rp, oracle, a):
    c = oracle.Csr.from_dense(a)
    return c, rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)


@pytest.mark.parametrize("kind,m,s", FAMILIES)
def test_sketch_families_dense_and_csr(rp, ctx, oracle, kind, m, s):
    n, d = 64, 9
    dense = oracle.random_dense(n, d, 7)
    rng = np.random.default_rng(1)
    oc, gc = _csr(rp, oracle, np.where(rng.random((n, d)) < 0.25, rng.standard_normal((n, d)), 0.0))
    for a_o, a_g in ((dense, dense), (oc, gc)):
        ref = oracle.sketch_apply(oracle.SketchSpec(kind, m, n, s, 4), a_o)
        got = rp.sketch_apply(rp.SketchSpec(kind, m, n, s, 4), a_g, ctx=ctx).product
        if kind == "gaussian":
            assert oracle.rel_error(got, ref) < 1e-13
        else:  # same summation order as the reference: bit-exact
            assert np.array_equal(got, ref)


@pytest.mark.parametrize("n,d,m", [(65536, 8, 2048), (1000, 5, 300), (4097, 3, 4097), (1, 2, 1)])
def test_srht_bit_exact_shapes(rp, ctx, oracle, n, d, m):
    a = np.random.default_rng(n).standard_normal((n, d))
    assert np.array_equal(rp.sketch_apply(rp.SketchSpec("srht", m, n, 1, 3), a, ctx=ctx).product,
                          oracle.sketch_apply(oracle.SketchSpec("srht", m, n, 1, 3), a))


def test_countsketch_large_bit_exact(rp, ctx, oracle):
    n, d, m = 20000, 33, 512
    rng = np.random.default_rng(4)
    a = rng.standard_normal((n, d))
    assert np.array_equal(rp.sketch_apply(rp.SketchSpec("countsketch", m, n, 1, 1), a, ctx=ctx).product,
                          oracle.sketch_apply(oracle.SketchSpec("countsketch", m, n, 1, 1), a))
    oc, gc = _csr(rp, oracle, np.where(rng.random((n, d)) < 0.1, a, 0.0))
    assert np.array_equal(rp.sketch_apply(rp.SketchSpec("sjlt", m, n, 4, 2), gc, ctx=ctx).product,
                          oracle.sketch_apply(oracle.SketchSpec("sjlt", m, n, 4, 2), oc))


def test_gaussian_sketch_c1_shape(rp, ctx, oracle):
    # C1: 512 x 4096 Gaussian sketch of a 4096 x 256 operator, <= 1e-13 relative
    a = oracle.random_dense(4096, 64, 3)
    ref = oracle.sketch_apply(oracle.SketchSpec("gaussian", 512, 4096, 1, 0), a)
    got = rp.sketch_apply(rp.SketchSpec("gaussian", 512, 4096, 1, 0), a, ctx=ctx).product
    assert oracle.rel_error(got, ref) < 1e-13


def test_sketch_validation(rp, ctx, oracle):  # test_sketch.cpp:161-176
    a = oracle.random_dense(32, 5, 9)
    with pytest.raises(ValueError):
        rp.sketch_apply(rp.SketchSpec("sjlt", 10, 32, 3, 0), a, ctx=ctx)
    with pytest.raises(ValueError):
        rp.sketch_apply(rp.SketchSpec("gaussian", 8, 31, 1, 0), a, ctx=ctx)
    with pytest.raises(ValueError):
        rp.sketch_apply(rp.SketchSpec("identity", 8, 32, 1, 0), a, ctx=ctx)
    first = rp.sketch_apply(rp.SketchSpec("gaussian", 8, 32, 1, 123), a, ctx=ctx).product
    second = rp.sketch_apply(rp.SketchSpec("gaussian", 8, 32, 1, 123), a, ctx=ctx).product
    assert np.array_equal(first, second)  # determinism


@pytest.mark.parametrize("n,d,k", [(300, 37, 5), (1000, 260, 130), (7, 3, 1), (129, 130, 67), (5000, 1, 3)])
def test_apply_transpose_gram_dense(rp, ctx, oracle, n, d, k):
    rng = np.random.default_rng(n + d)
    a = rng.standard_normal((n, d))
    x = rng.standard_normal((d, k))
    y = rng.standard_normal((n, k))
    assert oracle.rel_error(rp.apply(a, x, ctx=ctx), a @ x) < 1e-14
    assert oracle.rel_error(rp.apply_transpose(a, y, ctx=ctx), a.T @ y) < 1e-14
    assert oracle.rel_error(rp.gram_apply(a, x, ctx=ctx), a.T @ (a @ x)) < 1e-13


def test_csr_products_bit_exact(rp, ctx, oracle):
    rng = np.random.default_rng(3)
    dense = np.where(rng.random((400, 57)) < 0.1, rng.standard_normal((400, 57)), 0.0)
    oc, gc = _csr(rp, oracle, dense)
    x = rng.standard_normal((57, 4))
    # CSR apply / apply_transpose keep the reference's per-row / per-column order
    assert oracle.rel_error(rp.apply(gc, x, ctx=ctx), dense @ x) < 1e-14
    assert oracle.rel_error(rp.gram_apply(gc, x, ctx=ctx), oracle.gram_apply(oc, x)) < 1e-14
    with pytest.raises(ValueError):
        rp.apply(gc, rng.standard_normal((3, 1)), ctx=ctx)


def test_preconditioner_matches_dense_inverse(rp, ctx, oracle):  # test_preconditioner.cpp
    p = rp.Preconditioner.build(np.array([[1.0]]), 1.0, ctx=ctx)
    assert p.apply(np.array([2.0]))[0] == pytest.approx(1.0)
    z = rp.Preconditioner.build(np.zeros((2, 3)), 2.0, ctx=ctx)
    v = oracle.fill_normals(1, 3)
    assert oracle.rel_error(z.apply(v), v / 2.0) < 1e-15
    assert oracle.rel_error(z.reshift(4.0).apply(v), v / 4.0) < 1e-15
    for (m, d, seed, lam) in ((8, 20, 21, 0.5), (6, 4, 5, 0.8), (9, 14, 77, 1.3), (300, 130, 2, 0.01),
                              (100, 333, 3, 0.7)):
        sa = oracle.random_dense(m, d, seed)
        pre = rp.Preconditioner.build(sa, lam, ctx=ctx)
        v = oracle.random_dense(d, 3, seed + 1)
        assert oracle.rel_error(pre.apply(v), oracle.dense_preconditioner_oracle(sa, lam) @ v) < 1e-10
        assert oracle.rel_error(pre.apply(v), oracle.Preconditioner.build(sa, lam).apply(v)) < 1e-10
    sa = oracle.random_dense(6, 4, 13)
    sa[:, 3] = sa[:, 0] + sa[:, 1]  # rank deficient
    pre = rp.Preconditioner.build(sa, 0.7, ctx=ctx)
    v = oracle.fill_normals(14, 4)
    assert oracle.rel_error(pre.apply(v), oracle.dense_preconditioner_oracle(sa, 0.7) @ v) < 1e-9
    base = rp.Preconditioner.build(oracle.random_dense(7, 12, 2), 1.0, ctx=ctx)
    v = oracle.fill_normals(3, 12)
    rebuilt = rp.Preconditioner.build(oracle.random_dense(7, 12, 2), 3.7, ctx=ctx)
    assert oracle.rel_error(base.reshift(3.7).apply(v), rebuilt.apply(v)) < 1e-12
    # symmetry / positive definiteness
    pre = rp.Preconditioner.build(oracle.random_dense(6, 10, 55), 0.9, ctx=ctx)
    for t in range(5):
        v = oracle.fill_normals(100 + t, 10)
        w = oracle.fill_normals(200 + t, 10)
        assert v @ pre.apply(w) == pytest.approx(w @ pre.apply(v), rel=1e-12)
        assert v @ pre.apply(v) > 0
    with pytest.raises(ValueError):
        rp.Preconditioner.build(np.ones((2, 2)), 0.0, ctx=ctx)


@pytest.mark.parametrize("n,d,k", [(100000, 64, 1), (70001, 200, 2), (8192, 1024, 4), (3000, 2048, 8),
                                   (513, 33, 3), (40000, 16, 16)])
def test_narrow_passes(rp, ctx, oracle, n, d, k):
    """HBM-bound narrow kernels: A^T y (atv_narrow, k <= 16) and the fused
    single-pass Gram A^T (A w) (k in {1,2,3,4,8}) vs float64 numpy."""
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, d))
    y = rng.standard_normal((n, k))
    w = rng.standard_normal((d, k))
    assert oracle.rel_error(rp.apply_transpose(a, y, ctx=ctx), a.T @ y) < 1e-13
    assert oracle.rel_error(rp.gram_apply(a, w, ctx=ctx), a.T @ (a @ w)) < 1e-13
    # column stability (within one kernel family): each column alone gives the same bits
    if k > 8:
        return
    g_all = rp.gram_apply(a, w, ctx=ctx)
    t_all = rp.apply_transpose(a, y, ctx=ctx)
    for j in range(k):
        assert np.array_equal(rp.gram_apply(a, w[:, j].copy(), ctx=ctx), g_all[:, j])
        assert np.array_equal(rp.apply_transpose(a, y[:, j].copy(), ctx=ctx), t_all[:, j])


@pytest.mark.parametrize("panel,chunk,one", [(65536, 64, 0), (7, 64, 0), (64, 5, 0), (1, 1, 0), (100, 33, 0),
                                             (1000, 17, 0), (7, 128, 1 << 40), (7, 100, 0)])
def test_csr_panel_gram_bitwise(rp, ctx, oracle, panel, chunk, one):
    """The L2-blocked sparse Gram (sparse_gram.cu) continues each column's
    running sum across row panels, so it equals apply followed by
    apply_transpose (matrix.cpp:168-172) bit for bit, whatever the panel and
    chunk sizes; empty rows and empty columns included."""
    rng = np.random.default_rng(11)
    n, d = 523, 71
    dense = np.where(rng.random((n, d)) < 0.08, rng.standard_normal((n, d)), 0.0)
    dense[17] = 0.0  # empty row
    dense[:, 5] = 0.0  # empty column
    oc, gc = _csr(rp, oracle, dense)
    x = rng.standard_normal((d, 150))  # > 2 chunks of 64
    two_pass = rp.apply_transpose(gc, rp.apply(gc, x, ctx=ctx), ctx=ctx)
    try:
        ctx.set_option("csr_panel_rows", panel)
        ctx.set_option("csr_chunk", chunk)
        ctx.set_option("csr_one_panel_bytes", one)
        got = rp.gram_apply(gc, x, ctx=ctx)
        assert np.array_equal(got, two_pass)
        assert oracle.rel_error(got, oracle.gram_apply(oc, x)) < 1e-14
        # a single column through the same kernels
        assert np.array_equal(rp.gram_apply(gc, x[:, 3].copy(), ctx=ctx), two_pass[:, 3])
    finally:
        ctx.set_option("csr_panel_rows", 65536)
        ctx.set_option("csr_chunk", 128)
        ctx.set_option("csr_one_panel_bytes", 48 << 20)


def test_csr_panel_gram_empty_matrix(rp, ctx, oracle):
    dense = np.zeros((40, 9))
    oc, gc = _csr(rp, oracle, dense)
    got = rp.gram_apply(gc, np.ones((9, 3)), ctx=ctx)
    assert np.array_equal(got, np.zeros((9, 3)))


def test_csr_invariants_checked_on_device(rp, ctx, oracle):
    """CsrMatrix invariants (matrix.cpp:22-50) are checked where the entries
    live: same messages as the reference's constructor, the violation a
    row-major scan meets first is the one reported, and a rejected matrix
    leaves the context's operator untouched."""
    off = np.array([0, 2, 3, 5], dtype=np.int64)
    col = np.array([0, 2, 1, 0, 3], dtype=np.int64)
    val = np.array([1.0, -2.0, 3.0, 0.5, 4.0])
    good = rp.Csr(3, 4, off, col, val)
    dense = np.zeros((3, 4))
    for r in range(3):
        for p in range(off[r], off[r + 1]):
            dense[r, col[p]] = val[p]
    x = np.arange(1.0, 5.0)
    assert np.array_equal(np.asarray(rp.apply(good, x, ctx=ctx)).reshape(-1), dense @ x)
    y = np.array([1.0, -1.0, 2.0])
    got_t = rp.apply_transpose(good, y, ctx=ctx)
    assert np.array_equal(np.asarray(got_t).reshape(-1), dense.T @ y)  # (the device-built CSC mirror)
    bad_cases = [
        (off, np.array([0, 4, 1, 0, 3], dtype=np.int64), val, "column index out of range"),
        (off, np.array([0, -1, 1, 0, 3], dtype=np.int64), val, "column index out of range"),
        (off, np.array([2, 0, 1, 0, 3], dtype=np.int64), val, "strictly increasing"),
        (off, np.array([0, 0, 1, 0, 3], dtype=np.int64), val, "strictly increasing"),
        (off, col, np.array([1.0, -2.0, np.nan, 0.5, 4.0]), "non-finite"),
        (off, col, np.array([1.0, -2.0, 3.0, 0.5, np.inf]), "non-finite"),
        (np.array([0, 2, 1, 5], dtype=np.int64), col, val, "monotone"),
        (np.array([1, 2, 3, 5], dtype=np.int64), col, val, "start at 0"),
        # two violations: the earlier entry (order, entry 1) wins over the later one (range, entry 4)
        (off, np.array([2, 0, 1, 0, 9], dtype=np.int64), val, "strictly increasing"),
    ]
    for o2, c2, v2, needle in bad_cases:
        with pytest.raises(ValueError, match=needle):
            rp.apply(rp.Csr(3, 4, o2, c2, v2), x, ctx=ctx)
    # an empty matrix and an empty row are fine
    empty = rp.Csr(2, 4, np.zeros(3, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
    assert np.array_equal(np.asarray(rp.apply(empty, x, ctx=ctx)).reshape(-1), np.zeros(2))
