"""adaptive_sketch_dim (adaptive.cpp:53-135) on the device vs the oracle's
restatement and the expectations of test_adaptive.cpp.  The run is a chain of
discrete decisions (Armijo acceptances, doublings) on floating-point
comparisons; on these instances every decision matches the oracle, so the
(m, iterations, doublings) trace is equal and x agrees to rounding."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ab(oracle, seed, rows, cols):
    z = oracle.fill_normals(seed, rows * cols + rows)
    return z[: rows * cols].reshape(rows, cols), z[rows * cols:]


def _specs(rp, oracle, kind, n, seed, s=1):
    m = n if kind == "identity" else 1
    return rp.SketchSpec(kind, m, n, s, seed), oracle.SketchSpec(kind, m, n, s, seed)


def _same(got, ref, oracle, tol=1e-10):
    assert (got.m, got.iterations, got.doublings, got.converged, got.stalled_at_cap) == \
        (ref.m, ref.iterations, ref.doublings, ref.converged, ref.stalled_at_cap)
    assert oracle.rel_error(got.x, ref.x) < tol or np.linalg.norm(ref.x - got.x) < 1e-14
    assert len(got.trace) == len(ref.trace)
    for p, q in zip(got.trace, ref.trace):
        assert (p.m, p.doubled) == (q.m, q.doubled) and p.step == q.step
        assert p.f_after == pytest.approx(q.f_after, rel=1e-10, abs=1e-14)


def test_adaptive_immediate_stop(rp, ctx, oracle):  # test_adaptive.cpp:65-83
    a, b = _ab(oracle, 1, 20, 6)
    xs = oracle.ridge_solve_oracle(a, b, 0.7)
    gs, os_ = _specs(rp, oracle, "gaussian", 20, 3)
    got = rp.adaptive_sketch_dim(a, b, 0.7, rp.AdaptiveConfig(epsilon=1e-6, m_initial=4), gs, xs, ctx=ctx)
    assert (got.iterations, got.m, got.converged) == (0, 4, True)
    _same(got, oracle.adaptive_sketch_dim(a, b, 0.7, oracle.AdaptiveConfig(epsilon=1e-6, m_initial=4), os_, xs), oracle)


def test_adaptive_identity_never_doubles(rp, ctx, oracle):  # test_adaptive.cpp:85-114
    a, b = _ab(oracle, 2, 40, 10)
    gs, os_ = _specs(rp, oracle, "identity", 40, 5)
    got = rp.adaptive_sketch_dim(a, b, 1.0, rp.AdaptiveConfig(epsilon=1e-10, m_initial=8), gs, ctx=ctx)
    assert got.doublings == 0 and got.converged and got.m == 8 and got.iterations <= 200
    prev = np.inf
    for st in got.trace:
        if st.doubled:
            continue
        assert st.f_after <= st.f_before - 1e-4 * st.step * st.progress + 1e-15
        assert st.f_before <= prev + 1e-12
        prev = st.f_after
    _same(got, oracle.adaptive_sketch_dim(a, b, 1.0, oracle.AdaptiveConfig(epsilon=1e-10, m_initial=8), os_), oracle)


def test_adaptive_flat_spectrum_doubles(rp, ctx, oracle):  # test_adaptive.cpp:116-142
    raw, b = _ab(oracle, 7, 64, 20)
    q, _ = np.linalg.qr(raw)
    a = np.ascontiguousarray(5.0 * q)
    gs, os_ = _specs(rp, oracle, "gaussian", 64, 11)
    got = rp.adaptive_sketch_dim(a, b, 0.01, rp.AdaptiveConfig(epsilon=1e-8, m_initial=1), gs, ctx=ctx)
    assert got.doublings >= 1 and got.m <= 20
    assert all(s1.m <= s2.m for s1, s2 in zip(got.trace, got.trace[1:]))
    _same(got, oracle.adaptive_sketch_dim(a, b, 0.01, oracle.AdaptiveConfig(epsilon=1e-8, m_initial=1), os_), oracle,
          tol=1e-9)


@pytest.mark.parametrize("kind,s", [("countsketch", 1), ("sjlt", 3), ("srht", 1), ("gaussian", 1)])
def test_adaptive_reproducible_and_parity(rp, ctx, oracle, kind, s):  # test_adaptive.cpp:144-160
    a, b = _ab(oracle, 21, 300, 24)
    gs, os_ = _specs(rp, oracle, kind, 300, 77, s)
    cfg = rp.AdaptiveConfig(epsilon=1e-9, m_initial=2, iteration_cap=60)
    first = rp.adaptive_sketch_dim(a, b, 0.5, cfg, gs, ctx=ctx)
    second = rp.adaptive_sketch_dim(a, b, 0.5, cfg, gs, ctx=ctx)
    assert (first.m, first.iterations, first.doublings) == (second.m, second.iterations, second.doublings)
    assert np.array_equal(first.x, second.x)
    ref = oracle.adaptive_sketch_dim(a, b, 0.5, oracle.AdaptiveConfig(epsilon=1e-9, m_initial=2, iteration_cap=60), os_)
    _same(first, ref, oracle, tol=1e-9)


def test_adaptive_csr_and_validation(rp, ctx, oracle):
    rng = np.random.default_rng(6)
    dense = np.where(rng.random((500, 40)) < 0.25, rng.standard_normal((500, 40)), 0.0)
    c = oracle.Csr.from_dense(dense)
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    b = rng.standard_normal(500)
    gs, os_ = _specs(rp, oracle, "countsketch", 500, 9)
    got = rp.adaptive_sketch_dim(gc, b, 0.3, rp.AdaptiveConfig(epsilon=1e-9, m_initial=2, iteration_cap=60), gs, ctx=ctx)
    _same(got, oracle.adaptive_sketch_dim(c, b, 0.3, oracle.AdaptiveConfig(epsilon=1e-9, m_initial=2, iteration_cap=60),
                                          os_), oracle,
          tol=1e-9)
    a, b2 = _ab(oracle, 3, 30, 10)
    gs, _ = _specs(rp, oracle, "gaussian", 30, 1)
    for bad in (rp.AdaptiveConfig(gamma1=1.5), rp.AdaptiveConfig(m_cap=20), rp.AdaptiveConfig(m_initial=8, m_cap=4)):
        with pytest.raises(ValueError):
            rp.adaptive_sketch_dim(a, b2, 0.5, bad, gs, ctx=ctx)
    with pytest.raises(ValueError):
        rp.adaptive_sketch_dim(a, b2, 0.0, rp.AdaptiveConfig(), gs, ctx=ctx)
