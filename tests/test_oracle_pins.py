"""Pins the CPU oracle (oracle/) before anything is checked against it.

1. Draw contract: bit-exact against tests/golden/ref_draws.npz, generated from
   the reference's own rng.hpp (oracle/_ref, tests/golden/make_golden.py), the
   SURVEY.md section 8(c) KATs, and -- when oracle/_ref was built here -- the
   reference library itself on fresh seeds.
2. Floating-point algorithm: the reference's own doctest expectations
   (ref/proj/tests/test_{spectrum,preconditioner,path_solver,sketch,
   matrix_core}.cpp), restated against the oracle.
"""
import ctypes
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libref_rng.so")


# ---------------------------------------------------------------------------
# 1. Draw contract
# ---------------------------------------------------------------------------


def test_mt19937_64_standard_check(oracle, kats):
    # ISO C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(oracle.fill_u64(5489, 1, skip=9999)[0]) == int(kats["mt19937_64_default_10000th"]["value"])


def test_seed0_kats(oracle, kats):
    assert [int(v) for v in oracle.fill_u64(0, 3)] == [int(v) for v in kats["seed0_u64"]["value"]]
    assert oracle.fill_uniform01(0, 2).tolist() == kats["seed0_uniform01"]["value"]
    assert oracle.fill_normals(0, 2).tolist() == kats["seed0_normals"]["value"]


def test_c1_gaussian_kats(oracle, kats):
    s = oracle.gaussian_sketch_matrix(oracle.SketchSpec("gaussian", 512, 4096, 1, 0))
    assert s[0, :6].tolist() == kats["c1_gaussian_S_row0_0to5"]["value"]
    assert s[1, 0] == kats["c1_gaussian_S_1_0"]["value"]


def test_c4_countsketch_kats(oracle, kats):
    h, sg = oracle.count_draws(oracle.SketchSpec("countsketch", 8192, 5, 1, 0))
    assert [[int(a), int(b)] for a, b in zip(h[0], sg[0])] == kats["c4_countsketch_rows0to4"]["value"]


def test_c2_srht_kats(oracle, kats):
    signs, rows = oracle.srht_draws(oracle.SketchSpec("srht", 2048, 65536, 1, 0))
    assert signs[:8].tolist() == kats["c2_srht_signs_0to7"]["value"]
    assert rows[:6].tolist() == kats["c2_srht_rows_0to5"]["value"]
    assert int(rows[2047]) == kats["c2_srht_rows_2047"]["value"]


def test_golden_draw_vectors(oracle, golden):
    g = golden
    assert np.array_equal(oracle.fill_u64(0, 2048), g["u64_seed0"])
    assert np.array_equal(oracle.fill_u64(12345, 1024, skip=1_000_003), g["u64_seed12345_skip1000003"])
    assert np.array_equal(oracle.fill_uniform01(0, 1024), g["uniform01_seed0"])
    assert np.array_equal(oracle.fill_uniform_index(3, (1 << 63) + 1, 512), g["uindex_seed3_bound2p63p1"])
    assert np.array_equal(oracle.fill_uniform_index(4, 1000, 512), g["uindex_seed4_bound1000"])
    assert np.array_equal(oracle.fill_normals(0, 8192), g["normals_seed0"])
    s = oracle.gaussian_sketch_matrix(oracle.SketchSpec("gaussian", 512, 4096, 1, 0))
    assert np.array_equal(s[:2], g["c1_S_rows01"]) and np.array_equal(s[511], g["c1_S_row511"])
    assert np.array_equal(oracle.gaussian_sketch_matrix(oracle.SketchSpec("gaussian", 7, 33, 1, 9)),
                          g["gauss_m7_n33_seed9"])
    h, sg = oracle.count_draws(oracle.SketchSpec("countsketch", 8192, 4096, 1, 0))
    assert np.array_equal(h[0], g["count_m8192_seed0_h"]) and np.array_equal(sg[0], g["count_m8192_seed0_sign"])
    h, sg = oracle.count_draws(oracle.SketchSpec("sjlt", 12, 64, 3, 6))
    assert np.array_equal(h.reshape(-1), g["sjlt_m12_s3_n64_seed6_h"])
    assert np.array_equal(sg.reshape(-1), g["sjlt_m12_s3_n64_seed6_sign"])
    signs, rows = oracle.srht_draws(oracle.SketchSpec("srht", 2048, 65536, 1, 0))
    assert np.array_equal(np.packbits(signs > 0), g["srht_n65536_m2048_seed0_signbits"])
    assert np.array_equal(rows, g["srht_n65536_m2048_seed0_rows"])
    signs, rows = oracle.srht_draws(oracle.SketchSpec("srht", 4, 13, 1, 77))
    assert np.array_equal(signs, g["srht_n13_m4_seed77_signs"]) and np.array_equal(rows, g["srht_n13_m4_seed77_rows"])


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_reference_rng_fresh_seeds(oracle):
    L = ctypes.CDLL(REF_LIB)
    P, u64, i64, dbl = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
    L.ref_fill_u64.argtypes = [u64, u64, i64, P]
    L.ref_fill_normals.argtypes = [u64, i64, dbl, P]
    L.ref_count_draws.argtypes = [u64, i64, i64, ctypes.c_int, dbl, P, P]
    for seed in (1, 99, 2**40 + 3):
        ref = np.empty(5000, np.uint64)
        L.ref_fill_u64(seed, 17, 5000, ref.ctypes.data_as(P))
        assert np.array_equal(oracle.fill_u64(seed, 5000, skip=17), ref)
        refn = np.empty(3001, np.float64)
        L.ref_fill_normals(seed, 3001, 0.25, refn.ctypes.data_as(P))
        assert np.array_equal(oracle.fill_normals(seed, 3001, 0.25), refn)
        h = np.empty(2 * 300, np.int64)
        s = np.empty(2 * 300, np.float64)
        L.ref_count_draws(seed, 300, 5, 2, 1 / math.sqrt(2), h.ctypes.data_as(P), s.ctypes.data_as(P))
        oh, osg = oracle.count_draws(oracle.SketchSpec("sjlt", 10, 300, 2, seed))
        assert np.array_equal(oh.reshape(-1), h) and np.array_equal(osg.reshape(-1), s)


# ---------------------------------------------------------------------------
# 2. The reference's doctest expectations, restated against the oracle
# ---------------------------------------------------------------------------


def test_tune_interval_kats(oracle):  # test_spectrum.cpp:108-129
    p = oracle.tune_interval(1.0, 100.0, oracle.RhoBounds.identity(), None, 1e-6)
    assert p.lambda0 == pytest.approx(10.0, rel=1e-14)
    assert p.kappa == pytest.approx(100.0, rel=1e-14)
    assert p.alpha == pytest.approx(20.0 / 101.0, rel=1e-14)
    assert math.sqrt(p.contraction) == pytest.approx(99.0 / 101.0, rel=1e-14)
    dg = oracle.tune_interval(5.0, 5.0, oracle.RhoBounds.identity(), None, 1e-6)
    assert dg.kappa == pytest.approx(1.0) and dg.contraction == pytest.approx(0.0)
    # test_spectrum.cpp:119 expects alpha = 1/5 here, but spectrum.cpp:187 gives
    # 2 sqrt(lo hi) / (lo/rho1 + hi/rho2) = 1 for lo = hi = 5 with identity
    # bounds; the oracle follows the code, not that expectation.
    assert dg.alpha == pytest.approx(1.0, rel=1e-14) and dg.k == 2
    sh = oracle.tune_interval(1.0, 100.0, oracle.RhoBounds.identity(), math.sqrt(10.0), 1e-6)
    assert sh.lambda0 == pytest.approx(math.sqrt(1210.0) - 10.0, rel=1e-14)
    assert sh.kappa == pytest.approx(10.0, rel=1e-14)
    assert math.sqrt(sh.contraction) == pytest.approx(9.0 / 11.0, rel=1e-14)
    assert oracle.tune_interval(1.0, 1e9, oracle.RhoBounds.identity(), None, 1e-12).k == 64  # clamp


def test_tune_interval_balancing(oracle):  # test_spectrum.cpp:131-155
    state = 12345

    def nxt():
        nonlocal state
        state = (state * 6364136223846793005 + 1442695040888963407) % 2**64
        return (state >> 11) / 9007199254740992.0

    for trial in range(50):
        lo = 0.1 + 10.0 * nxt()
        hi = lo * (1.0 + 50.0 * nxt())
        rho2 = 0.2 + nxt()
        rho1 = rho2 + nxt()
        shift = 0.0 if trial % 2 == 0 else 3.0 * nxt()
        p = oracle.tune_interval(lo, hi, oracle.RhoBounds.manual(rho1, rho2),
                                 math.sqrt(shift) if shift > 0 else None, 1e-8)
        center = p.lambda0 + shift
        r_hi = abs(1.0 - p.alpha * (hi + shift) / center / rho2)
        r_lo = abs(1.0 - p.alpha * (lo + shift) / center / rho1)
        assert abs(r_hi - r_lo) < 1e-12
        assert r_hi == pytest.approx(math.sqrt(p.contraction), rel=1e-10)


def test_interval_split_ladder(oracle):  # test_spectrum.cpp:182-206
    autos = oracle.interval_split(1.0, 100.0)
    assert len(autos) == 9
    assert autos[0][1] == pytest.approx(100.0 ** (1 / 9), rel=1e-12)
    two = oracle.interval_split(1.0, 100.0, 2)
    assert two[0][1] == pytest.approx(10.0, rel=1e-14)
    assert len(oracle.interval_split(1.0, 1.0 + 1e-12)) == 1
    many = oracle.interval_split(0.5, 350.0, 11)
    ratio = many[0][1] / many[0][0]
    for lo, hi in many:
        assert hi / lo == pytest.approx(ratio, rel=1e-12)
    with pytest.raises(ValueError):
        oracle.interval_split(2.0, 1.0)
    with pytest.raises(ValueError):
        oracle.interval_split(0.0, 1.0)


def test_scalar_ihs_basis_kat(oracle):  # test_path_solver.cpp:80-100
    a = np.array([[1.0]])
    p = oracle.Preconditioner.build(np.array([[1.0]]), 1.0)
    basis = oracle.ihs_basis(a, np.ones(1), p, 1.0, 2)
    assert basis.terms[0][0, 0] == pytest.approx(0.75) and basis.terms[1][0, 0] == pytest.approx(-0.25)
    assert oracle.ihs_basis(a, np.ones(1), p, 1.0, 1).terms[0][0, 0] == pytest.approx(0.5)
    assert all(np.linalg.norm(t) == 0 for t in oracle.ihs_basis(a, np.zeros(1), p, 1.0, 3).terms)


def test_basis_iterate_identity(oracle):  # test_path_solver.cpp:102-145
    rng = np.random.default_rng(2024)
    kinds = ["identity", "gaussian", "countsketch", "sjlt", "srht"]
    for trial in range(25):
        n = 20 + int(rng.integers(0, 81))
        d = 5 + int(rng.integers(0, 26))
        a = oracle.random_dense(n, d, 1000 + trial)
        b = oracle.fill_normals(2000 + trial, n)
        kind = kinds[trial % 5]
        m = n if kind == "identity" else max(4, (d * 3) // 2)
        sa = oracle.sketch_apply(oracle.SketchSpec(kind, m, n, 1, 100 + trial), a)
        lam0 = 0.2 + 4.0 * rng.random()
        p = oracle.Preconditioner.build(sa, lam0)
        pd = oracle.dense_preconditioner_oracle(sa, lam0)
        lam = 0.1 + 9.0 * rng.random()
        w = np.linalg.eigvals(pd @ (a.T @ a + lam * np.eye(d))).real.max()
        tau = 2.0 / w * (0.15 + 0.75 * rng.random())
        k = 1 + int(rng.integers(0, 10))
        basis = oracle.ihs_basis(a, b, p, tau, k)
        assert oracle.rel_error(oracle.ihs_compose(basis, lam),
                                oracle.ihs_iterate_oracle(a, b, pd, tau, lam, k)) < 1e-10


def test_matrix_basis_equals_vector_runs(oracle):  # test_path_solver.cpp:212-237
    a = oracle.random_dense(25, 7, 11)
    rhs = oracle.random_dense(25, 3, 12)
    p = oracle.Preconditioner.build(a, 2.0)
    joint = oracle.ihs_basis_matrix(a, rhs, p, 0.4, 5)
    for col in range(3):
        solo = oracle.ihs_basis(a, rhs[:, col].copy(), p, 0.4, 5)
        for j in range(5):
            assert np.array_equal(joint.terms[j][:, col], solo.terms[j][:, 0])


def test_single_point_path_equals_manual_pipeline(oracle):  # test_path_solver.cpp:256-276
    a = oracle.random_dense(45, 9, 31)
    b = oracle.fill_normals(32, 45)
    cfg = oracle.PathConfig(4.0, 6.0, [5.0], 1e-8, 1)
    spec = oracle.SketchSpec("identity", 45, 45, 1, 0)
    path = oracle.ihs_bin_path(a, b, cfg, spec, oracle.RhoBounds.identity())
    prm = oracle.tune_interval(4.0, 6.0, oracle.RhoBounds.identity(), None, 1e-8)
    p = oracle.Preconditioner.build(oracle.sketch_apply(spec, a), prm.lambda0)
    basis = oracle.ihs_basis(a, b, p, prm.alpha, prm.k)
    assert oracle.rel_error(path.points[0].solution[:, 0], oracle.ihs_compose(basis, 5.0)) < 1e-14


def test_identity_path_matches_direct(oracle):  # test_path_solver.cpp:278-299
    a = oracle.random_dense(200, 50, 7, 0.3)
    b = oracle.fill_normals(8, 200)
    cfg = oracle.PathConfig(1.0, 100.0, oracle.log_grid(1.0, 100.0, 25), 1e-6, None)
    path = oracle.ihs_bin_path(a, b, cfg, oracle.SketchSpec("identity", 200, 200, 1, 0), oracle.RhoBounds.identity())
    for pt in path.points:
        assert oracle.rel_error(pt.solution[:, 0], oracle.ridge_solve_oracle(a, b, pt.lam)) < 1e-5


def test_absurd_envelope_raises_solver_error(oracle):  # test_path_solver.cpp:301-310
    a = oracle.random_dense(30, 6, 13)
    b = oracle.fill_normals(14, 30)
    cfg = oracle.PathConfig(1.0, 100.0, [1.0, 10.0, 100.0], 1e-6, 2)
    with pytest.raises(oracle.SolverError):
        oracle.ihs_bin_path(a, b, cfg, oracle.SketchSpec("identity", 30, 30, 1, 0), oracle.RhoBounds.manual(1e9, 1e8))


def test_dual_hand_example_and_primal_agreement(oracle):  # test_path_solver.cpp:312-375
    path = oracle.dual_path(np.array([[1.0, 0.0]]), np.ones(1), oracle.PathConfig(0.5, 2.0, [1.0], 1e-10, 1),
                            oracle.SketchSpec("identity", 2, 2, 1, 0), oracle.RhoBounds.identity())
    assert path.points[0].solution[0, 0] == pytest.approx(0.5, rel=1e-9)
    assert path.points[0].solution[1, 0] == pytest.approx(0.0, abs=1e-12)
    for n, d, seed in ((12, 12, 17), (10, 40, 18)):
        a = oracle.random_dense(n, d, seed)
        b = oracle.fill_normals(seed + 100, n)
        cfg = oracle.PathConfig(1.0, 50.0, oracle.log_grid(1.0, 50.0, 6), 1e-10, None)
        path = oracle.dual_path(a, b, cfg, oracle.SketchSpec("identity", d, d, 1, 0), oracle.RhoBounds.identity())
        for pt in path.points:
            assert oracle.rel_error(pt.solution[:, 0], oracle.ridge_solve_oracle(a, b, pt.lam)) < 1e-8


def test_preconditioner_oracles(oracle):  # test_preconditioner.cpp:38-141
    p = oracle.Preconditioner.build(np.array([[1.0]]), 1.0)
    assert p.apply(np.array([2.0]))[0] == pytest.approx(1.0)
    z = oracle.Preconditioner.build(np.zeros((2, 3)), 2.0)
    v = oracle.fill_normals(1, 3)
    assert oracle.rel_error(z.apply(v), v / 2.0) < 1e-15
    for (m, d, seed, lam) in ((8, 20, 21, 0.5), (6, 4, 5, 0.8), (9, 14, 77, 1.3)):
        sa = oracle.random_dense(m, d, seed)
        pre = oracle.Preconditioner.build(sa, lam)
        v = oracle.fill_normals(seed + 1, d)
        assert oracle.rel_error(pre.apply(v), oracle.dense_preconditioner_oracle(sa, lam) @ v) < 1e-10
    sa = oracle.random_dense(6, 4, 13)
    sa[:, 3] = sa[:, 0] + sa[:, 1]  # rank-deficient tall sketch
    pre = oracle.Preconditioner.build(sa, 0.7)
    v = oracle.fill_normals(14, 4)
    assert oracle.rel_error(pre.apply(v), oracle.dense_preconditioner_oracle(sa, 0.7) @ v) < 1e-9
    base = oracle.Preconditioner.build(oracle.random_dense(7, 12, 2), 1.0)
    v = oracle.fill_normals(3, 12)
    assert oracle.rel_error(base.reshift(3.7).apply(v),
                            oracle.Preconditioner.build(oracle.random_dense(7, 12, 2), 3.7).apply(v)) < 1e-12


def test_sketch_apply_equals_realized_operator(oracle):  # test_sketch.cpp:74-94
    n, d = 64, 9
    dense = oracle.random_dense(n, d, 7)
    rng = np.random.default_rng(0)
    sp = oracle.Csr.from_dense(np.where(rng.random((n, d)) < 0.25, rng.standard_normal((n, d)), 0.0))
    for kind, m, s, seed in (("gaussian", 12, 1, 4), ("countsketch", 12, 1, 5), ("sjlt", 12, 3, 6),
                             ("srht", 12, 1, 7), ("identity", n, 1, 8)):
        spec = oracle.SketchSpec(kind, m, n, s, seed)
        S = oracle.realize_dense(spec)
        for a in (dense, sp):
            ad = a.to_dense() if isinstance(a, oracle.Csr) else a
            assert oracle.rel_error(oracle.sketch_apply(spec, a), S @ ad) < 1e-12


def test_sketch_validation(oracle):  # test_sketch.cpp:161-176
    a = oracle.random_dense(32, 5, 9)
    with pytest.raises(ValueError):
        oracle.sketch_apply(oracle.SketchSpec("sjlt", 10, 32, 3, 0), a)
    with pytest.raises(ValueError):
        oracle.sketch_apply(oracle.SketchSpec("gaussian", 8, 31, 1, 0), a)
    with pytest.raises(ValueError):
        oracle.realize_dense(oracle.SketchSpec("gaussian", 2000, 2000, 1, 0))
    with pytest.raises(ValueError):
        oracle.sketch_apply(oracle.SketchSpec("identity", 8, 32, 1, 0), a)
    assert [oracle.hadamard_pad(v) for v in (1, 2, 3, 1000)] == [1, 2, 4, 1024]


def test_gram_is_composition(oracle):  # test_matrix_core.cpp:68-76
    rng = np.random.default_rng(3)
    m = oracle.Csr.from_dense(np.where(rng.random((15, 7)) < 0.4, rng.standard_normal((15, 7)), 0.0))
    x = rng.standard_normal(7)
    assert np.array_equal(oracle.gram_apply(m, x), oracle.apply_transpose(m, oracle.apply(m, x)))
    lower = np.array([[1.0, 0.0], [1.0, 1.0]])
    assert oracle.gram_apply(lower, np.ones(2)).tolist() == [3.0, 2.0]


# ---- derive_rho pieces: spectrum.cpp:87-169 against test_spectrum.cpp:9-106 ----

def test_effective_dimension_kats(oracle):  # test_spectrum.cpp:9-38
    assert oracle.effective_dimension([1.0, 1.0], 1.0) == pytest.approx(2.0)
    assert oracle.effective_dimension([2.0, 1.0], 3.0) == pytest.approx(23.0 / 16.0)
    assert oracle.effective_dimension([3.0, 0.0], 1.0) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        oracle.effective_dimension([0.0, 0.0, 0.0], 1.0)
    sigma = [5.0, 2.0, 1.0, 0.5]
    prev = oracle.effective_dimension(sigma, 0.0)
    assert prev == pytest.approx(4.0)
    for shift in (0.1, 1.0, 10.0, 100.0):
        cur = oracle.effective_dimension(sigma, shift)
        assert 1.0 <= cur <= prev + 1e-12
        prev = cur


def test_rho_envelope_kats(oracle):  # test_spectrum.cpp:40-106
    b, _ = oracle.rho_gaussian(0.25, 0.01, 1.0)
    assert b.rho1 == pytest.approx(2.7225, rel=1e-12)
    assert b.rho2 == pytest.approx(49.0 / 324.0, rel=1e-14)
    b, _ = oracle.rho_gaussian(0.25, 0.01, 1e-12)
    assert b.rho1 == pytest.approx(1.0, rel=1e-9) and b.rho2 == pytest.approx(1.0, rel=1e-9)
    b, _ = oracle.rho_gaussian(0.04, 0.04, 0.5)
    assert b.rho1 == pytest.approx(1.5368, rel=1e-12) and b.rho2 == pytest.approx(0.745, rel=1e-12)
    _, p = oracle.rho_gaussian(0.25, 0.01, 1.0, 8000)
    assert p == pytest.approx(1.0 - 16.0 * math.exp(-0.01 * 0.01 * 0.25 * 4000.0))
    for bad in ((0.25, 0.2, 1.0), (1.5, 0.01, 1.0)):
        with pytest.raises(ValueError):
            oracle.rho_gaussian(*bad)
    b, _ = oracle.rho_srht(0.5, 1.0)
    assert (b.rho1, b.rho2) == (1.5, 0.5)
    b, _ = oracle.rho_srht(0.2, 0.8)
    assert b.rho1 == pytest.approx(1.16, rel=1e-12) and b.rho2 == pytest.approx(0.84, rel=1e-12)
    _, rec = oracle.rho_srht(0.5, 1.0, (1024, 50.0))
    c = 16.0 / 3.0 * (1.0 + math.sqrt(8.0 * math.log(50.0 * 1024.0) / 50.0)) ** 2
    assert rec == math.ceil(c * 50.0 * math.log(50.0) / 0.5)
    with pytest.raises(ValueError):
        oracle.rho_srht(0.9, 1.2)
    b, _, _ = oracle.rho_sjlt(0.25)
    assert (b.rho1, b.rho2) == (1.25, 0.75)
    _, rm, rs = oracle.rho_sjlt(0.25, (4.0, 0.1, 100.0))
    assert rs == 20 and rm == 31891
    with pytest.raises(ValueError):
        oracle.rho_sjlt(0.6)


def test_derive_rho_oracle_families(oracle):
    """derive_rho (ridgepath_main.cpp:218-279) on a small problem: every family
    yields a valid envelope; identity short-circuits without sketching."""
    a = oracle.random_dense(600, 20, 3) / np.sqrt(np.arange(1, 21))
    for kind, m, s in (("gaussian", 120, 1), ("srht", 120, 1), ("countsketch", 120, 1), ("sjlt", 120, 3)):
        b, info = oracle.derive_rho(oracle.SketchSpec(kind, m, 600, s, 7), a, 1e-3, 1e2)
        b.validate()
        assert b.provenance == ("sjlt" if kind == "countsketch" else kind)
        assert 1.0 <= info["effective_dimension"] <= 20.0
    b, info = oracle.derive_rho(oracle.SketchSpec("identity", 600, 600, 1, 0), a, 1e-3, 1e2)
    assert (b.rho1, b.rho2, b.provenance, info) == (1.0, 1.0, "identity", {})


# ---- comparison baselines: baselines.cpp against test_baselines.cpp ----

def _ab(oracle, seed, rows, cols):
    """random_dense then random_vector from one SeededRng (test_support.hpp:15-27)."""
    z = oracle.fill_normals(seed, rows * cols + rows)
    return z[: rows * cols].reshape(rows, cols), z[rows * cols:]


def _cfg(oracle, lo, hi, grid, eps):
    return oracle.PathConfig(lo, hi, list(grid), eps, None)


def test_baselines_oracle_kats(oracle):  # test_baselines.cpp:42-131
    p = oracle.svd_path(np.array([[2.0]]), np.array([4.0]), _cfg(oracle, 1.0, 1e7, [1.0, 1e7], 1e-8))
    assert p.points[0].solution[0] == pytest.approx(1.6) and abs(p.points[1].solution[0]) < 1e-5
    a, b = _ab(oracle, 3, 30, 8)
    cfg = _cfg(oracle, 0.5, 20.0, oracle.log_grid(0.5, 20.0, 6), 1e-8)
    for path in (oracle.svd_path(a, b, cfg), oracle.direct_path(a, b, cfg)):
        for pt in path.points:
            assert oracle.rel_error(pt.solution, oracle.ridge_solve_oracle(a, b, pt.lam)) < 1e-10
    a, b = _ab(oracle, 9, 25, 6)
    assert oracle.warm_cg_path(a, b, _cfg(oracle, 2.0, 3.0, [2.5, 2.5], 1e-10)).points[1].iterations == 0
    be = oracle.fill_normals(9, 25 * 6 + 25 + 12)[25 * 6 + 25:]
    assert oracle.warm_cg_path(np.eye(12), be, _cfg(oracle, 1.0, 2.0, [1.5], 1e-10)).points[0].iterations == 1
    a, b = _ab(oracle, 10, 100, 30)
    cfg = _cfg(oracle, 1.0, 100.0, oracle.log_grid(1.0, 100.0, 10), 1e-8)
    for p, q in zip(oracle.warm_cg_path(a, b, cfg).points, oracle.svd_path(a, b, cfg).points):
        assert p.lam == q.lam and oracle.rel_error(p.solution, q.solution) < 1e-6
    a, b = _ab(oracle, 12, 30, 7)
    ident = oracle.SketchSpec("identity", 30, 30, 1, 0)
    assert oracle.warm_ihs_path(a, b, _cfg(oracle, 1.0, 2.0, [1.5], 1e-8), ident,
                                oracle.RhoBounds.identity()).points[0].iterations == 1
    assert oracle.warm_ihs_path(a, b, _cfg(oracle, 1.0, 2.0, [1.5, 1.5], 1e-8), ident,
                                oracle.RhoBounds.identity()).points[1].iterations == 0
    # test_baselines.cpp:119-131 expects convergence with a Gaussian m = 36
    # sketch of an 80 x 12 matrix under rho = (1.6, 0.55), but with the
    # reference's own draws lambda_max(P (A^T A + lambda I)) reaches 3.67, so
    # tau * lambda_max = 3.0 > 2: the iterate grows by ~2x per step and the
    # 1000-step cap (baselines.cpp:203-204) fires long before the non-finite
    # test that would trigger the tau/2 retry.  The oracle follows the code.
    a, b = _ab(oracle, 14, 80, 12)
    cfg = _cfg(oracle, 1.0, 50.0, oracle.log_grid(1.0, 50.0, 8), 1e-8)
    with pytest.raises(oracle.SolverError):
        oracle.warm_ihs_path(a, b, cfg, oracle.SketchSpec("gaussian", 36, 80, 1, 5), oracle.RhoBounds.manual(1.6, 0.55))
    # the same instance with an oversampled sketch (m = 200 > 16 d) converges
    ihs = oracle.warm_ihs_path(a, b, cfg, oracle.SketchSpec("gaussian", 200, 80, 1, 5), oracle.RhoBounds.manual(1.6, 0.55))
    for p, q in zip(ihs.points, oracle.svd_path(a, b, cfg).points):
        assert oracle.rel_error(p.solution, q.solution) < 1e-6


def test_baselines_oracle_agree_pairwise(oracle):  # test_baselines.cpp:133-151
    a, b = _ab(oracle, 20, 60, 15)
    eps = 1e-8
    cfg = _cfg(oracle, 1.0, 30.0, oracle.log_grid(1.0, 30.0, 7), eps)
    allp = [oracle.svd_path(a, b, cfg), oracle.direct_path(a, b, cfg), oracle.warm_cg_path(a, b, cfg),
            # (m = 30 as in test_baselines.cpp:143 diverges for the same reason
            # as above; an oversampled sketch stands in)
            oracle.warm_ihs_path(a, b, cfg, oracle.SketchSpec("gaussian", 240, 60, 1, 8), oracle.RhoBounds.manual(1.6, 0.55))]
    tol = max(10 * eps, 1e-8)
    for i in range(4):
        for j in range(i + 1, 4):
            for p, q in zip(allp[i].points, allp[j].points):
                assert oracle.rel_error(p.solution, q.solution) < 10 * tol


# ---- adaptive sketch dimension: adaptive.cpp against test_adaptive.cpp ----

def _tspec(oracle, kind, n, seed):
    return oracle.SketchSpec(kind, n if kind == "identity" else 1, n, 1, seed)


def test_armijo_oracle_kats(oracle):  # test_adaptive.cpp:25-63
    f = lambda x: 0.5 * float(x @ x)  # noqa: E731
    assert oracle.armijo_step(f, np.ones(1), np.ones(1), 1.0, 0.5, 1e-4) == pytest.approx(1.0)
    g = lambda x: 50.0 * float(x @ x)  # noqa: E731
    j = next(j for j in range(51) if g(np.full(1, 1.0 - 0.5 ** j)) <= g(np.ones(1)) - 1e-4 * 0.5 ** j * 100.0)
    assert oracle.armijo_step(g, np.ones(1), np.ones(1), 100.0, 0.5, 1e-4) == pytest.approx(0.5 ** j)
    with pytest.raises(ValueError):
        oracle.armijo_step(f, np.ones(1), np.ones(1), -1.0, 0.5, 1e-4)
    # test_adaptive.cpp:57-62 expects SolverError for a constant objective, but
    # in double arithmetic fx - gamma2 * step * 1 rounds to fx once
    # 1e-4 * 2^-j drops below half an ulp of 1 (j = 41), so the code at
    # adaptive.cpp:44-48 accepts that step; the oracle follows the code
    j = next(j for j in range(51) if 1.0 <= 1.0 - 1e-4 * 0.5 ** j * 1.0)
    assert j == 41
    assert oracle.armijo_step(lambda x: 1.0, np.ones(1), np.ones(1), 1.0, 0.5, 1e-4) == 0.5 ** j
    with pytest.raises(oracle.SolverError):  # a rising objective never qualifies
        oracle.armijo_step(lambda x: 1.0 + float(np.abs(x - 1).sum()), np.ones(1), np.ones(1), 1.0, 0.5, 1e-4)


def test_adaptive_oracle_kats(oracle):  # test_adaptive.cpp:65-171
    a, b = _ab(oracle, 1, 20, 6)
    xs = oracle.ridge_solve_oracle(a, b, 0.7)
    r = oracle.adaptive_sketch_dim(a, b, 0.7, oracle.AdaptiveConfig(epsilon=1e-6, m_initial=4),
                                   _tspec(oracle, "gaussian", 20, 3), xs)
    assert (r.iterations, r.m, r.converged) == (0, 4, True)
    a, b = _ab(oracle, 2, 40, 10)
    cfg = oracle.AdaptiveConfig(epsilon=1e-10, m_initial=8)
    r = oracle.adaptive_sketch_dim(a, b, 1.0, cfg, _tspec(oracle, "identity", 40, 5))
    assert r.doublings == 0 and r.converged and r.m == 8 and r.iterations <= cfg.iteration_cap
    prev = math.inf
    for st in r.trace:
        if st.doubled:
            continue
        assert st.f_after <= st.f_before - cfg.gamma2 * st.step * st.progress + 1e-15
        assert st.f_before <= prev + 1e-12
        prev = st.f_after
    raw, b = _ab(oracle, 7, 64, 20)
    q, _ = np.linalg.qr(raw)
    r = oracle.adaptive_sketch_dim(5.0 * q, b, 0.01, oracle.AdaptiveConfig(epsilon=1e-8, m_initial=1),
                                   _tspec(oracle, "gaussian", 64, 11))
    assert r.doublings >= 1 and r.m <= 20
    assert all(s1.m <= s2.m for s1, s2 in zip(r.trace, r.trace[1:]))
    a, b = _ab(oracle, 21, 30, 8)
    cfg = oracle.AdaptiveConfig(epsilon=1e-9, m_initial=2)
    r1 = oracle.adaptive_sketch_dim(a, b, 0.5, cfg, _tspec(oracle, "countsketch", 30, 77))
    r2 = oracle.adaptive_sketch_dim(a, b, 0.5, cfg, _tspec(oracle, "countsketch", 30, 77))
    assert (r1.m, r1.iterations, r1.doublings) == (r2.m, r2.iterations, r2.doublings)
    assert np.array_equal(r1.x, r2.x)
    with pytest.raises(ValueError):
        oracle.AdaptiveConfig(gamma1=1.5).validate(10)
    with pytest.raises(ValueError):
        oracle.AdaptiveConfig(m_cap=20).validate(10)
