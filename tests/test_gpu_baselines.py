"""The reference's comparison baselines (baselines.cpp:80-226) on the device vs
the oracle's restatement, plus the expectations of test_baselines.cpp.

warm_cg / warm_ihs run the same iteration as the reference, so the iteration
counts must agree exactly and the solutions to rounding; direct_path solves
with the explicit (G + lambda I)^{-1} instead of an LLT solve (same operator).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ab(oracle, seed, rows, cols):
    z = oracle.fill_normals(seed, rows * cols + rows)
    return z[: rows * cols].reshape(rows, cols), z[rows * cols:]


def _cfgs(rp, oracle, lo, hi, grid, eps):
    return rp.PathConfig(lo, hi, list(grid), eps), oracle.PathConfig(lo, hi, list(grid), eps, None)


def _same(got, ref, oracle, tol, iters=True):
    assert len(got.points) == len(ref.points)
    for p, q in zip(got.points, ref.points):
        assert p.lam == q.lam
        assert oracle.rel_error(p.solution[:, 0], q.solution) < tol
        if iters:
            assert p.iterations == q.iterations


def test_direct_matches_normal_equations(rp, ctx, oracle):  # test_baselines.cpp:52-66
    a, b = _ab(oracle, 3, 30, 8)
    gcfg, ocfg = _cfgs(rp, oracle, 0.5, 20.0, oracle.log_grid(0.5, 20.0, 6), 1e-8)
    got = rp.direct_path(a, b, gcfg, ctx=ctx)
    for p in got.points:
        assert oracle.rel_error(p.solution[:, 0], oracle.ridge_solve_oracle(a, b, p.lam)) < 1e-10
    _same(got, oracle.direct_path(a, b, ocfg), oracle, 1e-12, iters=False)
    for p in got.points:
        tr, _ = oracle.losses(a, b, p.solution[:, 0], p.lam)
        assert p.train_loss == pytest.approx(tr, rel=1e-12)


def test_warm_cg_kats_and_parity(rp, ctx, oracle):  # test_baselines.cpp:68-100
    a, b = _ab(oracle, 9, 25, 6)
    gcfg, _ = _cfgs(rp, oracle, 2.0, 3.0, [2.5, 2.5], 1e-10)
    assert rp.warm_cg_path(a, b, gcfg, ctx=ctx).points[1].iterations == 0
    be = oracle.fill_normals(9, 25 * 6 + 25 + 12)[25 * 6 + 25:]
    gcfg, _ = _cfgs(rp, oracle, 1.0, 2.0, [1.5], 1e-10)
    assert rp.warm_cg_path(np.eye(12), be, gcfg, ctx=ctx).points[0].iterations == 1
    a, b = _ab(oracle, 10, 100, 30)
    gcfg, ocfg = _cfgs(rp, oracle, 1.0, 100.0, oracle.log_grid(1.0, 100.0, 10), 1e-8)
    got = rp.warm_cg_path(a, b, gcfg, ctx=ctx)
    for p, q in zip(got.points, oracle.svd_path(a, b, ocfg).points):
        assert oracle.rel_error(p.solution[:, 0], q.solution) < 1e-6
    _same(got, oracle.warm_cg_path(a, b, ocfg), oracle, 1e-10)


def test_warm_ihs_kats_and_parity(rp, ctx, oracle):  # test_baselines.cpp:102-131
    a, b = _ab(oracle, 12, 30, 7)
    ident = rp.SketchSpec("identity", 30, 30, 1, 0)
    gcfg, _ = _cfgs(rp, oracle, 1.0, 2.0, [1.5], 1e-8)
    assert rp.warm_ihs_path(a, b, gcfg, ident, rp.RhoBounds.identity(), ctx=ctx).points[0].iterations == 1
    gcfg, _ = _cfgs(rp, oracle, 1.0, 2.0, [1.5, 1.5], 1e-8)
    assert rp.warm_ihs_path(a, b, gcfg, ident, rp.RhoBounds.identity(), ctx=ctx).points[1].iterations == 0
    a, b = _ab(oracle, 14, 80, 12)
    gcfg, ocfg = _cfgs(rp, oracle, 1.0, 50.0, oracle.log_grid(1.0, 50.0, 8), 1e-8)
    # m = 36 diverges under the reference's own draws (see test_oracle_pins.py): the cap fires
    with pytest.raises(rp.SolverError):
        rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("gaussian", 36, 80, 1, 5), rp.RhoBounds.manual(1.6, 0.55), ctx=ctx)
    got = rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("gaussian", 200, 80, 1, 5), rp.RhoBounds.manual(1.6, 0.55),
                           ctx=ctx)
    ref = oracle.warm_ihs_path(a, b, ocfg, oracle.SketchSpec("gaussian", 200, 80, 1, 5),
                               oracle.RhoBounds.manual(1.6, 0.55))
    _same(got, ref, oracle, 1e-9)
    for p, q in zip(got.points, oracle.svd_path(a, b, ocfg).points):
        assert oracle.rel_error(p.solution[:, 0], q.solution) < 1e-6


def test_warm_ihs_tau_half_retry(rp, ctx, oracle):
    """Identity sketch (P (A^T A + lambda I) = I) with rho = (3.5, 3.5): tau = 3.5
    multiplies the error by -2.5 per step and overflows after ~775 steps (below
    the 1000 cap), which triggers the single tau/2 retry (baselines.cpp:201-208);
    tau = 1.75 then contracts by 0.75 per step."""
    a, b = _ab(oracle, 12, 30, 7)
    gcfg, ocfg = _cfgs(rp, oracle, 1.0, 2.0, [1.5], 1e-8)
    got = rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("identity", 30, 30, 1, 0), rp.RhoBounds.manual(3.5, 3.5), ctx=ctx)
    ref = oracle.warm_ihs_path(a, b, ocfg, oracle.SketchSpec("identity", 30, 30, 1, 0), oracle.RhoBounds.manual(3.5, 3.5))
    assert 0 < ref.points[0].iterations < 200
    _same(got, ref, oracle, 1e-12)
    # rho = (9, 9): tau and tau/2 both diverge -> SolverError
    with pytest.raises(rp.SolverError):
        rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("identity", 30, 30, 1, 0), rp.RhoBounds.manual(9.0, 9.0), ctx=ctx)


def test_all_baselines_agree_pairwise(rp, ctx, oracle):  # test_baselines.cpp:133-151
    a, b = _ab(oracle, 20, 60, 15)
    eps = 1e-8
    gcfg, ocfg = _cfgs(rp, oracle, 1.0, 30.0, oracle.log_grid(1.0, 30.0, 7), eps)
    allp = [oracle.svd_path(a, b, ocfg).points,
            [p for p in rp.direct_path(a, b, gcfg, ctx=ctx).points],
            [p for p in rp.warm_cg_path(a, b, gcfg, ctx=ctx).points],
            [p for p in rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("gaussian", 240, 60, 1, 8),
                                         rp.RhoBounds.manual(1.6, 0.55), ctx=ctx).points]]
    tol = max(10 * eps, 1e-8)
    for i in range(4):
        for j in range(i + 1, 4):
            for p, q in zip(allp[i], allp[j]):
                assert oracle.rel_error(np.ravel(p.solution), np.ravel(q.solution)) < 10 * tol


def test_baselines_csr(rp, ctx, oracle):
    rng = np.random.default_rng(4)
    dense = np.where(rng.random((400, 30)) < 0.3, rng.standard_normal((400, 30)), 0.0)
    c = oracle.Csr.from_dense(dense)
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    b = rng.standard_normal(400)
    gcfg, ocfg = _cfgs(rp, oracle, 0.1, 10.0, oracle.log_grid(0.1, 10.0, 6), 1e-9)
    _same(rp.warm_cg_path(gc, b, gcfg, ctx=ctx), oracle.warm_cg_path(c, b, ocfg), oracle, 1e-10)
    _same(rp.direct_path(gc, b, gcfg, ctx=ctx), oracle.direct_path(c, b, ocfg), oracle, 1e-11, iters=False)
    spec_g, spec_o = rp.SketchSpec("countsketch", 200, 400, 1, 2), oracle.SketchSpec("countsketch", 200, 400, 1, 2)
    _same(rp.warm_ihs_path(gc, b, gcfg, spec_g, rp.RhoBounds.manual(1.8, 0.4), ctx=ctx),
          oracle.warm_ihs_path(c, b, ocfg, spec_o, oracle.RhoBounds.manual(1.8, 0.4)), oracle, 1e-9)


def test_baselines_errors(rp, ctx, oracle):
    a, b = _ab(oracle, 3, 30, 8)
    gcfg, _ = _cfgs(rp, oracle, 0.5, 20.0, [1.0], 1e-8)
    with pytest.raises(ValueError):
        rp.warm_cg_path(a, b[:-1], gcfg, ctx=ctx)
    with pytest.raises(ValueError):
        rp.warm_ihs_path(a, b, gcfg, rp.SketchSpec("gaussian", 20, 29, 1, 0), rp.RhoBounds.identity(), ctx=ctx)
    with pytest.raises(ValueError):  # unsorted grid (PathConfig::validate)
        rp.direct_path(a, b, rp.PathConfig(0.5, 20.0, [2.0, 1.0], 1e-8), ctx=ctx)


# ---- svd_path (baselines.cpp:51-78) -----------------------------------------


def test_svd_path_scalar_kat(rp, ctx, oracle):  # the 1 x 1 case of test_oracle_pins: x = 2*4 / (4 + lambda)
    got = rp.svd_path(np.array([[2.0]]), np.array([4.0]), rp.PathConfig(1.0, 1e7, [1.0, 1e7], 1e-8), ctx=ctx)
    assert got.solver == "svd"
    assert got.points[0].solution[0, 0] == pytest.approx(8.0 / 5.0, rel=1e-15)
    assert got.points[1].solution[0, 0] == pytest.approx(8.0 / (4.0 + 1e7), rel=1e-15)


@pytest.mark.parametrize("rows,cols", [(200, 24), (24, 200), (64, 64), (1, 5)])
def test_svd_path_tall_wide_square(rp, ctx, oracle, rows, cols):
    a, b = _ab(oracle, rows + cols, rows, cols)
    gcfg, ocfg = _cfgs(rp, oracle, 1e-3, 1e3, oracle.log_grid(1e-3, 1e3, 25), 1e-8)
    got = rp.svd_path(a, b, gcfg, ctx=ctx)
    _same(got, oracle.svd_path(a, b, ocfg), oracle, 1e-10, iters=False)
    for p in got.points:
        assert oracle.rel_error(p.solution[:, 0], oracle.ridge_solve_oracle(a, b, p.lam)) < 1e-9
        tr, _ = oracle.losses(a, b, p.solution[:, 0], p.lam)
        assert p.train_loss == pytest.approx(tr, rel=1e-10)


def test_svd_path_rank_deficient_and_csr(rp, ctx, oracle):
    a, b = _ab(oracle, 9, 120, 10)
    a = np.hstack([a, a[:, :4]])  # 14 columns, rank 10: zero singular values
    gcfg, ocfg = _cfgs(rp, oracle, 0.01, 100.0, oracle.log_grid(0.01, 100.0, 9), 1e-8)
    _same(rp.svd_path(a, b, gcfg, ctx=ctx), oracle.svd_path(a, b, ocfg), oracle, 1e-10, iters=False)
    rng = np.random.default_rng(12)
    dense = np.where(rng.random((300, 40)) < 0.2, rng.standard_normal((300, 40)), 0.0)
    c = oracle.Csr.from_dense(dense)
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    bb = rng.standard_normal(300)
    _same(rp.svd_path(gc, bb, gcfg, ctx=ctx), oracle.svd_path(c, bb, ocfg), oracle, 1e-10, iters=False)


def test_svd_path_c1_full_size(rp, ctx, oracle):
    """C1 (the reference's CPU-runnable config) at full size: the device thin SVD
    path against the oracle's LAPACK SVD."""
    import workloads

    w = workloads.get("c1")
    grid = list(w.lambdas(oracle.log_grid))
    gcfg, ocfg = _cfgs(rp, oracle, w.lambda_min, w.lambda_max, grid, w.epsilon)
    b = np.ravel(w.b)
    got = rp.svd_path(w.a, b, gcfg, ctx=ctx)
    _same(got, oracle.svd_path(w.a, b, ocfg), oracle, 1e-10, iters=False)


def test_svd_path_errors(rp, ctx, oracle):
    a, b = _ab(oracle, 3, 30, 8)
    with pytest.raises(ValueError):
        rp.svd_path(a, b[:-1], rp.PathConfig(0.5, 20.0, [1.0], 1e-8), ctx=ctx)
    with pytest.raises(ValueError):  # unsorted grid (PathConfig::validate)
        rp.svd_path(a, b, rp.PathConfig(0.5, 20.0, [2.0, 1.0], 1e-8), ctx=ctx)
