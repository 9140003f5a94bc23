"""IHS-BIN basis and path on the device vs the oracle.

Parity bar (north_star): x(lambda) within 1e-8 relative l2 of the reference
algorithm's CPU output for every lambda of the grid, FP64 throughout.  The
reference's own test_path_solver.cpp expectations are restated on the device.
"""
import math

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-8  # relative l2, every lambda (BASELINE.json north_star)


def _mirror(rp, oracle, w):
    """(oracle args, device args) for a workloads.Workload."""
    if isinstance(w.a, dict):
        oa = oracle.Csr(w.a["rows"], w.a["cols"], w.a["offsets"], w.a["indices"], w.a["values"])
        ga = rp.Csr(w.a["rows"], w.a["cols"], w.a["offsets"], w.a["indices"], w.a["values"])
    else:
        oa = ga = w.a
    sk = w.sketch
    grid = w.lambdas(oracle.log_grid)
    ocfg = oracle.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    gcfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    ospec = oracle.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
    gspec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
    return (oa, ocfg, ospec, oracle.RhoBounds.manual(*w.rho)), (ga, gcfg, gspec, rp.RhoBounds.manual(*w.rho))


def _worst(got_points, ref_points, oracle, lams=None):
    ref = {p.lam: p.solution for p in ref_points}
    worst = 0.0
    n = 0
    for p in got_points:
        if p.lam in ref and (lams is None or p.lam in lams):
            worst = max(worst, oracle.rel_error(p.solution, ref[p.lam]))
            n += 1
    return worst, n


# ---------------------------------------------------------------------------
# reference test_path_solver.cpp expectations
# ---------------------------------------------------------------------------


def test_scalar_basis_kat(rp, ctx):  # :80-100
    a = np.array([[1.0]])
    p = rp.Preconditioner.build(np.array([[1.0]]), 1.0, ctx=ctx)
    basis = rp.ihs_basis(a, np.ones(1), p, 1.0, 2, ctx=ctx)
    assert basis.terms[0][0, 0] == pytest.approx(0.75) and basis.terms[1][0, 0] == pytest.approx(-0.25)
    assert rp.ihs_compose(basis, 0.0, ctx=ctx)[0] == pytest.approx(0.75)
    assert rp.ihs_compose(basis, 1.0, ctx=ctx)[0] == pytest.approx(0.5)  # two explicit steps, dense inverse
    assert rp.ihs_basis(a, np.ones(1), p, 1.0, 1, ctx=ctx).terms[0][0, 0] == pytest.approx(0.5)
    zero = rp.ihs_basis(a, np.zeros(1), p, 1.0, 3, ctx=ctx)
    assert all(np.linalg.norm(t) == 0 for t in zero.terms)


def test_basis_iterate_identity(rp, ctx, oracle):  # :102-145
    rng = np.random.default_rng(2024)
    kinds = ["identity", "gaussian", "countsketch", "sjlt", "srht"]
    for trial in range(25):
        n = 20 + int(rng.integers(0, 81))
        d = 5 + int(rng.integers(0, 26))
        a = oracle.random_dense(n, d, 1000 + trial)
        b = oracle.fill_normals(2000 + trial, n)
        kind = kinds[trial % 5]
        m = n if kind == "identity" else max(4, (d * 3) // 2)
        sa = rp.sketch_apply(rp.SketchSpec(kind, m, n, 1, 100 + trial), a, ctx=ctx)
        lam0 = 0.2 + 4.0 * rng.random()
        p = rp.Preconditioner.build(sa, lam0, ctx=ctx)
        pd = oracle.dense_preconditioner_oracle(sa.product, lam0)
        lam = 0.1 + 9.0 * rng.random()
        w = np.linalg.eigvals(pd @ (a.T @ a + lam * np.eye(d))).real.max()
        tau = 2.0 / w * (0.15 + 0.75 * rng.random())
        k = 1 + int(rng.integers(0, 10))
        basis = rp.ihs_basis(a, b, p, tau, k, ctx=ctx)
        assert oracle.rel_error(rp.ihs_compose(basis, lam, ctx=ctx),
                                oracle.ihs_iterate_oracle(a, b, pd, tau, lam, k)) < 1e-10


def test_matrix_basis_equals_vector_runs_bitwise(rp, ctx, oracle):  # :212-237
    a = oracle.random_dense(25, 7, 11)
    rhs = oracle.random_dense(25, 3, 12)
    for mode in (0, 1):
        ctx.set_option("gram_mode", mode)
        p = rp.Preconditioner.build(a, 2.0, ctx=ctx)
        joint = rp.ihs_basis_matrix(a, rhs, p, 0.4, 5, ctx=ctx)
        for col in range(3):
            solo = rp.ihs_basis(a, rhs[:, col].copy(), p, 0.4, 5, ctx=ctx)
            for j in range(5):
                assert np.array_equal(joint.terms[j][:, col], solo.terms[j][:, 0])
            assert np.array_equal(rp.ihs_compose_matrix(joint, 3.0, ctx=ctx)[:, col],
                                  rp.ihs_compose(solo, 3.0, ctx=ctx))
        zero = rp.ihs_basis_matrix(a, np.zeros((25, 2)), p, 0.4, 4, ctx=ctx)
        assert np.linalg.norm(rp.ihs_compose_matrix(zero, 1.0, ctx=ctx)) == 0.0
    ctx.set_option("gram_mode", -1)


def test_matrix_path_columns_equal_vector_paths(rp, ctx, oracle):
    """With the "stable_columns" option (default on) the path's GEMMs split K
    by K alone, so a matrix path's columns equal the vector paths bit for bit
    (as the basis API, test_path_solver.cpp:212-237); with it off the split
    follows the problem width and columns agree to rounding."""
    w = workloads.c1(scale=0.25)
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    B = np.asfortranarray(np.column_stack([w.b[:, 0], 2 * w.b[:, 0] + 1, np.zeros(w.b.shape[0])]))
    for stable in (1, 0):
        ctx.set_option("stable_columns", stable)
        joint = rp.ihs_bin_path_matrix(ga, B, gcfg, gspec, grho, ctx=ctx)
        for col in range(3):
            solo = rp.ihs_bin_path(ga, B[:, col].copy(), gcfg, gspec, grho, ctx=ctx)
            for pj, ps in zip(joint.points, solo.points):
                if stable:
                    assert np.array_equal(pj.solution[:, col], ps.solution[:, 0])
                else:
                    assert oracle.rel_error(pj.solution[:, col], ps.solution[:, 0]) < 1e-12 or \
                        np.linalg.norm(ps.solution[:, 0]) == 0.0
    ctx.set_option("stable_columns", 1)


def test_single_point_path_equals_manual_pipeline(rp, ctx, oracle):  # :256-276
    a = oracle.random_dense(45, 9, 31)
    b = oracle.fill_normals(32, 45)
    cfg = rp.PathConfig(4.0, 6.0, [5.0], 1e-8, 1)
    spec = rp.SketchSpec("identity", 45, 45, 1, 0)
    path = rp.ihs_bin_path(a, b, cfg, spec, rp.RhoBounds.identity(), ctx=ctx)
    assert len(path.points) == 1
    prm = rp.tune_interval(4.0, 6.0, rp.RhoBounds.identity(), None, 1e-8)
    p = rp.Preconditioner.build(rp.sketch_apply(spec, a, ctx=ctx), prm.lambda0, ctx=ctx)
    basis = rp.ihs_basis(a, b, p, prm.alpha, prm.k, ctx=ctx)
    assert oracle.rel_error(path.points[0].solution[:, 0], rp.ihs_compose(basis, 5.0, ctx=ctx)) < 1e-14


def test_identity_path_matches_direct(rp, ctx, oracle):  # :278-299
    a = oracle.random_dense(200, 50, 7, 0.3)
    b = oracle.fill_normals(8, 200)
    grid = rp.log_grid(1.0, 100.0, 25)
    path = rp.ihs_bin_path(a, b, rp.PathConfig(1.0, 100.0, grid, 1e-6), rp.SketchSpec("identity", 200, 200, 1, 0),
                           rp.RhoBounds.identity(), ctx=ctx)
    assert len(path.points) == 25
    for pt in path.points:
        assert oracle.rel_error(pt.solution[:, 0], oracle.ridge_solve_oracle(a, b, pt.lam)) < 1e-5


def test_unstable_envelope_raises_solver_error(rp, ctx, oracle):  # :301-310
    a = oracle.random_dense(30, 6, 13)
    b = oracle.fill_normals(14, 30)
    cfg = rp.PathConfig(1.0, 100.0, [1.0, 10.0, 100.0], 1e-6, 2)
    with pytest.raises(rp.SolverError):
        rp.ihs_bin_path(a, b, cfg, rp.SketchSpec("identity", 30, 30, 1, 0), rp.RhoBounds.manual(1e9, 1e8), ctx=ctx)


def test_tau_half_retry_matches_oracle(rp, ctx, oracle):  # path_solver.cpp:132-140
    # an inflated envelope (rho = 6) makes the first attempt overflow while the
    # tau/2 retry stays finite (found with the oracle; same on both sides)
    a = np.array([[1.0]])
    b = np.array([1e285])
    grid = [1.0, 1.0001]
    rho = (6.0, 6.0)
    ref = oracle.ihs_bin_path(a, b, oracle.PathConfig(1.0, 1.0001, grid, 1e-300, 1),
                              oracle.SketchSpec("identity", 1, 1, 1, 0), oracle.RhoBounds.manual(*rho))
    got = rp.ihs_bin_path(a, b, rp.PathConfig(1.0, 1.0001, grid, 1e-300, 1), rp.SketchSpec("identity", 1, 1, 1, 0),
                          rp.RhoBounds.manual(*rho), ctx=ctx)
    assert got.timings["retries"] == 1
    assert all(np.isfinite(p.solution).all() for p in got.points)
    worst, n = _worst(got.points, ref.points, oracle)
    assert n == 2 and worst < 1e-12


def test_dual_hand_example_and_primal_agreement(rp, ctx, oracle):  # :312-375
    path = rp.dual_path(np.array([[1.0, 0.0]]), np.ones(1), rp.PathConfig(0.5, 2.0, [1.0], 1e-10, 1),
                        rp.SketchSpec("identity", 2, 2, 1, 0), rp.RhoBounds.identity(), ctx=ctx)
    assert path.points[0].solution[0, 0] == pytest.approx(0.5, rel=1e-9)
    assert abs(path.points[0].solution[1, 0]) < 1e-12
    for n, d, seed in ((12, 12, 17), (10, 40, 18)):
        a = oracle.random_dense(n, d, seed)
        b = oracle.fill_normals(seed + 100, n)
        cfg = rp.PathConfig(1.0, 50.0, rp.log_grid(1.0, 50.0, 6), 1e-10)
        path = rp.dual_path(a, b, cfg, rp.SketchSpec("identity", d, d, 1, 0), rp.RhoBounds.identity(), ctx=ctx)
        for pt in path.points:
            assert oracle.rel_error(pt.solution[:, 0], oracle.ridge_solve_oracle(a, b, pt.lam)) < 1e-8
    zero = rp.dual_path(oracle.random_dense(5, 9, 3), np.zeros(5), rp.PathConfig(1.0, 2.0, [1.0, 2.0], 1e-8),
                        rp.SketchSpec("identity", 9, 9, 1, 0), rp.RhoBounds.identity(), ctx=ctx)
    assert all(np.linalg.norm(p.solution) == 0 for p in zero.points)


def test_path_validation(rp, ctx, oracle):
    a = oracle.random_dense(30, 5, 1)
    b = oracle.fill_normals(2, 30)
    spec = rp.SketchSpec("identity", 30, 30, 1, 0)
    rho = rp.RhoBounds.identity()
    for cfg in (rp.PathConfig(1.0, 0.5, [1.0], 1e-6), rp.PathConfig(1.0, 2.0, [], 1e-6),
                rp.PathConfig(1.0, 2.0, [1.5, 1.2], 1e-6), rp.PathConfig(1.0, 2.0, [1.5], 1.5),
                rp.PathConfig(1.0, 2.0, [2.5], 1e-6)):
        with pytest.raises(ValueError):
            rp.ihs_bin_path(a, b, cfg, spec, rho, ctx=ctx)
    with pytest.raises(ValueError):
        rp.ihs_bin_path(a, b, rp.PathConfig(1.0, 2.0, [1.5], 1e-6), rp.SketchSpec("identity", 29, 29, 1, 0), rho,
                        ctx=ctx)
    with pytest.raises(ValueError):
        rp.dual_path(a, b, rp.PathConfig(1.0, 2.0, [1.5], 1e-6), spec, rho, ctx=ctx)


# ---------------------------------------------------------------------------
# Parity on the BASELINE configs (full size where the oracle finishes in
# seconds, structure-preserving scaled versions otherwise)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("mode", [0, 1])
def test_c1_full_parity(rp, ctx, oracle, mode):
    w = workloads.c1()
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    ref = oracle.ihs_bin_path(oa, w.b, ocfg, ospec, orho)
    ctx.set_option("gram_mode", mode)
    try:
        got = rp.ihs_bin_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    finally:
        ctx.set_option("gram_mode", -1)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"C1 full (gram_mode={mode}): {n} lambdas, max rel err {worst:.3e}")
    assert n == 100 and worst < TOL


@pytest.mark.parametrize("name,scale", [("c2", 1 / 8), ("c3", 1 / 64)])
def test_scaled_dense_parity(rp, ctx, oracle, name, scale):
    w = workloads.get(name, scale=scale)
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    ref = oracle.ihs_bin_path(oa, w.b, ocfg, ospec, orho)
    got = rp.ihs_bin_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"{name} scale {scale}: {n} lambdas, max rel err {worst:.3e}")
    assert n == w.T and worst < TOL


def test_c2_full_size_interval_subset_parity(rp, ctx, oracle):
    """Full C2 (65536 x 1024, SRHT m=2048): the device path against the oracle
    on the first and last interval (each interval is independent,
    path_solver.cpp:168-186, so a subset is exact)."""
    w = workloads.c2()
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    L = len(oracle.interval_split(w.lambda_min, w.lambda_max))
    ref = oracle.ihs_bin_path(oa, w.b, ocfg, ospec, orho, interval_subset=[0, L - 1])
    got = rp.ihs_bin_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    # the sketch itself is bit-exact (SRHT keeps the reference's butterfly order)
    assert np.array_equal(rp.sketch_apply(gspec, ga, ctx=ctx).product, ref.sa)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"C2 full, intervals 0 and {L-1}: {n} lambdas, max rel err {worst:.3e}")
    assert n >= 40 and worst < TOL


@pytest.mark.parametrize("mode", [-1, 0])
def test_c4_scaled_csr_countsketch_woodbury(rp, ctx, oracle, mode):
    w = workloads.c4(scale=1 / 1024)
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    assert w.sketch["m"] < w.meta["d"]  # m < d: Woodbury branch
    ref = oracle.ihs_bin_path(oa, w.b, ocfg, ospec, orho)
    ctx.set_option("gram_mode", mode)
    try:
        got = rp.ihs_bin_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    finally:
        ctx.set_option("gram_mode", -1)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"C4 scaled: {n} lambdas, max rel err {worst:.3e}")
    assert n == w.T and worst < TOL


def test_c5_scaled_dual_matrix_rhs(rp, ctx, oracle):
    w = workloads.c5(scale=1 / 64, K=4)
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    ocfg.lambdas = ocfg.lambdas[::4]
    gcfg.lambdas = list(ocfg.lambdas)
    ref = oracle.dual_path(oa, w.b, ocfg, ospec, orho)
    got = rp.dual_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"C5 scaled dual K=4: {n} lambdas, max rel err {worst:.3e}")
    assert n == len(ocfg.lambdas) and worst < TOL


@pytest.mark.parametrize("kind,s", [("sjlt", 4), ("countsketch", 1), ("identity", 1), ("gaussian", 1)])
def test_other_families_parity(rp, ctx, oracle, kind, s):
    n, d = 2000, 40
    a = oracle.random_dense(n, d, 5) / np.sqrt(np.arange(1, d + 1))
    b = oracle.fill_normals(6, n)
    m = n if kind == "identity" else 200
    rho = (1.0, 1.0) if kind == "identity" else workloads.mp_envelope(d, m)
    grid = oracle.log_grid(1e-2, 1e2, 40)
    ref = oracle.ihs_bin_path(a, b, oracle.PathConfig(1e-2, 1e2, grid, 1e-6, None), oracle.SketchSpec(kind, m, n, s, 3),
                              oracle.RhoBounds.manual(*rho) if kind != "identity" else oracle.RhoBounds.identity())
    got = rp.ihs_bin_path(a, b, rp.PathConfig(1e-2, 1e2, grid, 1e-6), rp.SketchSpec(kind, m, n, s, 3),
                          rp.RhoBounds.manual(*rho) if kind != "identity" else rp.RhoBounds.identity(), ctx=ctx)
    worst, n_ = _worst(got.points, ref.points, oracle)
    assert n_ == 40 and worst < TOL


def test_grid_edge_cases(rp, ctx, oracle):
    a = oracle.random_dense(300, 12, 9)
    b = oracle.fill_normals(10, 300)
    spec_o, spec_g = oracle.SketchSpec("gaussian", 60, 300, 1, 1), rp.SketchSpec("gaussian", 60, 300, 1, 1)
    rho = workloads.mp_envelope(12, 60)
    edges = [e for pair in oracle.interval_split(0.1, 10.0, 3) for e in pair]
    for grid, L in (([0.1], None), ([10.0], 1), (sorted(set(edges)), 3), ([0.1, 0.1, 5.0, 10.0], None)):
        ref = oracle.ihs_bin_path(a, b, oracle.PathConfig(0.1, 10.0, grid, 1e-6, L), spec_o, oracle.RhoBounds.manual(*rho))
        got = rp.ihs_bin_path(a, b, rp.PathConfig(0.1, 10.0, grid, 1e-6, L), spec_g, rp.RhoBounds.manual(*rho), ctx=ctx)
        assert len(got.points) == len(grid)
        for gp, rp_ in zip(got.points, ref.points):
            assert gp.lam == rp_.lam
            assert oracle.rel_error(gp.solution, rp_.solution) < TOL


def test_path_losses_match_oracle(rp, ctx, oracle):
    """Per-point train/test losses (path_solver.cpp:298-303, 318-323, 342-347,
    425-454): every PathPoint of the device path carries the reference's
    losses of its own solution."""
    rng = np.random.default_rng(17)
    n, d, nt = 300, 20, 90
    a = rng.standard_normal((n, d))
    b = a @ rng.standard_normal(d) + 0.1 * rng.standard_normal(n)
    at = rng.standard_normal((nt, d))
    bt = at @ rng.standard_normal(d)
    grid = rp.log_grid(1e-2, 1e1, 7)
    cfg = rp.PathConfig(1e-2, 1e1, grid, 1e-6)
    spec = rp.SketchSpec("gaussian", 60, n, 1, 3)
    rho = rp.RhoBounds.manual(*oracle.mp_rho(d, 60)) if hasattr(oracle, "mp_rho") else rp.RhoBounds.manual(
        (1 + (d / 60) ** 0.5) ** 2, (1 - (d / 60) ** 0.5) ** 2)
    path = rp.ihs_bin_path(a, b, cfg, spec, rho, ctx=ctx, a_test=at, b_test=bt)
    for p in path.points:
        tr, te = oracle.losses(a, b, p.solution[:, 0], p.lam, at, bt)
        assert p.train_loss == pytest.approx(tr, rel=1e-12)
        assert p.test_loss == pytest.approx(te, rel=1e-12)
    # matrix right-hand side (losses_matrix: Frobenius norms)
    B = np.stack([b, -2 * b + 0.3], axis=1)
    BT = np.stack([bt, bt], axis=1)
    pm = rp.ihs_bin_path(a, B, cfg, spec, rho, ctx=ctx, a_test=at, b_test=BT)
    for p in pm.points:
        tr, te = oracle.losses(a, B, p.solution, p.lam, at, BT)
        assert p.train_loss == pytest.approx(tr, rel=1e-12)
        assert p.test_loss == pytest.approx(te, rel=1e-12)
    # sparse operator, no test set
    c = oracle.Csr.from_dense(np.where(rng.random((n, d)) < 0.3, a, 0.0))
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    x = rng.standard_normal((d, 5))
    lams = np.linspace(0.1, 2.0, 5)
    got = rp.losses(gc, b, x, lams, ctx=ctx)
    for t in range(5):
        assert got[t] == pytest.approx(oracle.losses(c, b, x[:, t], lams[t])[0], rel=1e-12)
    assert np.allclose(rp.losses(gc, b, x, None, ctx=ctx),
                       [oracle.losses(c, b, x[:, t], 0.0)[0] for t in range(5)], rtol=1e-12)
    # dual path: losses of the recovered solution against the primal data
    aw = rng.standard_normal((40, 120))
    bw = rng.standard_normal(40)
    dpath = rp.dual_path(aw, bw, rp.PathConfig(1e-1, 1e1, rp.log_grid(1e-1, 1e1, 4), 1e-6),
                         rp.SketchSpec("gaussian", 80, 120, 1, 5), rp.RhoBounds.manual(1.0, 1e-5), ctx=ctx)
    for p in dpath.points:
        assert p.train_loss == pytest.approx(oracle.losses(aw, bw, p.solution[:, 0], p.lam)[0], rel=1e-12)


def test_dual_csr_path_matches_oracle(rp, ctx, oracle):
    """dual_path on a CSR operator (path_solver.cpp:329-351): the dual Gram
    A A^T runs through the panel sparse passes on the transposed structure."""
    rng = np.random.default_rng(21)
    n, d = 60, 300
    dense = np.where(rng.random((n, d)) < 0.1, rng.standard_normal((n, d)), 0.0)
    b = rng.standard_normal(n)
    c = oracle.Csr.from_dense(dense)
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    grid = oracle.log_grid(1e-1, 1e1, 12)
    ref = oracle.dual_path(c, b, oracle.PathConfig(1e-1, 1e1, grid, 1e-6, None),
                           oracle.SketchSpec("countsketch", 40, d, 1, 4), oracle.RhoBounds.manual(1.0, 1e-5))
    try:
        ctx.set_option("csr_panel_rows", 37)
        ctx.set_option("csr_one_panel_bytes", 0)
        got = rp.dual_path(gc, b, rp.PathConfig(1e-1, 1e1, list(grid), 1e-6), rp.SketchSpec("countsketch", 40, d, 1, 4),
                           rp.RhoBounds.manual(1.0, 1e-5), ctx=ctx)
    finally:
        ctx.set_option("csr_panel_rows", 65536)
        ctx.set_option("csr_one_panel_bytes", 48 << 20)
    worst, npts = _worst(got.points, ref.points, oracle)
    assert npts == len(grid) and worst < TOL


def test_c2_full_size_every_interval_parity(rp, ctx, oracle):
    """Full C2 on every interval: all 1000 grid points of the bench workload
    against the oracle (the CPU side is the bench's reference arm run to the
    end, ~1-2 minutes on the box's host cores)."""
    w = workloads.c2()
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    ref = oracle.ihs_bin_path(oa, w.b, ocfg, ospec, orho)
    got = rp.ihs_bin_path(ga, w.b, gcfg, gspec, grho, ctx=ctx)
    worst, n = _worst(got.points, ref.points, oracle)
    print(f"C2 full, every interval: {n} lambdas, max rel err {worst:.3e}")
    assert n == w.T and worst < TOL


_VSPLIT_CHILD = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import workloads
from paper_2210_12212_b200 import ridgepath as rp
w = workloads.get({name!r}, scale={scale!r})
grid = w.lambdas(rp.log_grid)
sk = w.sketch
got = rp.ihs_bin_path(w.a, w.b, rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon),
                      rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"]), rp.RhoBounds.manual(*w.rho))
np.save({out!r}, np.stack([p.solution for p in got.points]))
"""


@pytest.mark.parametrize("name,scale", [("c2", 1.0), ("c1", 4.0)])
def test_virtual_split_bitwise(name, scale, tmp_path):
    """The GEMM virtual split (a column-stable split product run as one CTA
    per tile with its K chunks accumulated separately and added in chunk
    order, fused epilogue) gives x(lambda) bit-identical to the real split
    (partials + consumer kernel): the two processes differ only in
    RP_GEMM_VSPLIT."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    xs = []
    for flag in ("1", "0"):  # (the virtual split is opt-in: RP_GEMM_VSPLIT=1)
        out = str(tmp_path / f"x{flag}.npy")
        code = _VSPLIT_CHILD.format(root=root, name=name, scale=scale, out=out)
        env = dict(os.environ, RP_GEMM_VSPLIT=flag)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        xs.append(np.load(out))
    assert np.array_equal(xs[0], xs[1])


def test_compose_gemm_matches_horner(rp, ctx, oracle):
    """x(lambda) composed as a batched DMMA GEMM (interval basis times the
    interval's coefficient block tau (tau lambda)^j, the default) against the
    reference's Horner order (option compose_gemm = 0; compose_horner,
    path_solver.cpp:64-74): same sums in another order -- 1e-12 -- for a
    matrix right-hand side, a grid that leaves intervals empty and a
    one-point grid."""
    w = workloads.c1(scale=0.25)
    (oa, ocfg, ospec, orho), (ga, gcfg, gspec, grho) = _mirror(rp, oracle, w)
    B = np.asfortranarray(np.column_stack([w.b[:, 0], 2 * w.b[:, 0] + 1, w.b[:, 0] ** 2]))
    full = list(gcfg.lambdas)
    for grid in (full, full[:3] + full[-2:], [full[len(full) // 2]]):
        cfg = rp.PathConfig(gcfg.lambda_min, gcfg.lambda_max, grid, gcfg.epsilon, gcfg.num_intervals)
        out = []
        for flag in (1, 0):
            ctx.set_option("compose_gemm", flag)
            out.append(rp.ihs_bin_path_matrix(ga, B, cfg, gspec, grho, ctx=ctx))
        ctx.set_option("compose_gemm", 1)
        assert len(out[0].points) == len(grid)
        for pg, ph in zip(out[0].points, out[1].points):
            assert pg.lam == ph.lam
            assert oracle.rel_error(pg.solution, ph.solution) < 1e-12
