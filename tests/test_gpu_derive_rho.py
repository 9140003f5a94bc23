"""derive_rho (the CLI's plug-in envelope, tools/ridgepath_main.cpp:218-279) on
the device vs the oracle's restatement (sketch + LAPACK thin SVD + the
spectrum.cpp:87-169 formulas).

The device reads the two spectral sums without an SVD (trace of H (H+l0 I)^-1
and Lanczos for s_max^2), so agreement is to rounding: the envelope within
1e-10 relative, and the interval budgets k it induces identical.
"""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def _check(rp, oracle, got, ref, lo, hi):
    (gb, gi), (ob, oi) = got, ref
    assert gb.provenance == ob.provenance
    assert abs(gb.rho1 - ob.rho1) <= RTOL * abs(ob.rho1)
    assert abs(gb.rho2 - ob.rho2) <= RTOL * abs(ob.rho2)
    assert abs(gi["effective_dimension"] - oi["effective_dimension"]) <= RTOL * oi["effective_dimension"]
    assert abs(gi["sigma_max_sq"] - oi["sigma_max_sq"]) <= 1e-12 * oi["sigma_max_sq"]
    # the plans the envelope drives are the same
    for a, b in oracle.interval_split(lo, hi):
        kg = oracle.tune_interval(a, b, oracle.RhoBounds(gb.rho1, gb.rho2, "manual"), None, 1e-6).k
        ko = oracle.tune_interval(a, b, ob, None, 1e-6).k
        assert kg == ko


@pytest.mark.parametrize("kind,m,s", [("gaussian", 160, 1), ("srht", 160, 1), ("countsketch", 160, 1),
                                      ("sjlt", 160, 4), ("gaussian", 24, 1), ("countsketch", 30, 1)])
def test_derive_rho_families_dense(rp, ctx, oracle, kind, m, s):
    n, d = 1500, 48  # m = 24/30 < d: the wide (SA SA^T) branch
    a = oracle.random_dense(n, d, 4) / np.sqrt(np.arange(1, d + 1))
    lo, hi = 1e-3, 1e2
    got = rp.derive_rho(rp.SketchSpec(kind, m, n, s, 9), a, lo, hi, ctx=ctx)
    ref = oracle.derive_rho(oracle.SketchSpec(kind, m, n, s, 9), a, lo, hi)
    _check(rp, oracle, got, ref, lo, hi)
    assert got[1]["lanczos_steps"] >= 1


def test_derive_rho_csr_and_identity(rp, ctx, oracle):
    rng = np.random.default_rng(2)
    dense = np.where(rng.random((2000, 60)) < 0.2, rng.standard_normal((2000, 60)), 0.0)
    c = oracle.Csr.from_dense(dense)
    gc = rp.Csr(c.rows, c.cols, c.offsets, c.indices, c.values)
    got = rp.derive_rho(rp.SketchSpec("countsketch", 200, 2000, 1, 1), gc, 1e-2, 1e2, ctx=ctx)
    ref = oracle.derive_rho(oracle.SketchSpec("countsketch", 200, 2000, 1, 1), c, 1e-2, 1e2)
    _check(rp, oracle, got, ref, 1e-2, 1e2)
    b, info = rp.derive_rho(rp.SketchSpec("identity", 2000, 2000, 1, 0), gc, 1e-2, 1e2, ctx=ctx)
    assert (b.rho1, b.rho2, b.provenance, info) == (1.0, 1.0, "identity", {})
    with pytest.raises(ValueError):
        rp.derive_rho(rp.SketchSpec("countsketch", 200, 2000, 1, 1), gc, 1e2, 1e-2, ctx=ctx)
    with pytest.raises(ValueError):  # spec.n != A.rows
        rp.derive_rho(rp.SketchSpec("countsketch", 200, 1999, 1, 1), gc, 1e-2, 1e2, ctx=ctx)


def test_derive_rho_c1_full_and_path(rp, ctx, oracle):
    """C1 at full size (4096 x 256, Gaussian m = 512): the derived envelope,
    then the whole path run with it on both sides (the CLI flow
    resolve_rho -> run_solver, ridgepath_main.cpp:281-290, 345-388)."""
    w = workloads.c1()
    lo, hi = w.lambda_min, w.lambda_max
    sk = w.sketch
    got = rp.derive_rho(rp.SketchSpec(sk["kind"], sk["m"], sk["n"], 1, 0), w.a, lo, hi, ctx=ctx)
    ref = oracle.derive_rho(oracle.SketchSpec(sk["kind"], sk["m"], sk["n"], 1, 0), w.a, lo, hi)
    _check(rp, oracle, got, ref, lo, hi)
    print(f"\nC1 derive_rho: d_e {got[1]['effective_dimension']:.4f} rho ({got[0].rho1:.6f}, {got[0].rho2:.6f}) "
          f"Lanczos steps {got[1]['lanczos_steps']}")
    grid = oracle.log_grid(lo, hi, 25)
    path = rp.ihs_bin_path(w.a, w.b, rp.PathConfig(lo, hi, grid, 1e-6), rp.SketchSpec("gaussian", sk["m"], sk["n"], 1, 0),
                           rp.RhoBounds(got[0].rho1, got[0].rho2, got[0].provenance), ctx=ctx)
    want = oracle.ihs_bin_path(w.a, w.b, oracle.PathConfig(lo, hi, grid, 1e-6, None),
                               oracle.SketchSpec("gaussian", sk["m"], sk["n"], 1, 0), ref[0])
    worst = max(oracle.rel_error(p.solution, q.solution) for p, q in zip(path.points, want.points))
    assert worst < 1e-8


def test_derive_rho_c2_scaled_srht(rp, ctx, oracle):
    w = workloads.c2(scale=1 / 8)
    sk = w.sketch
    lo, hi = w.lambda_min, w.lambda_max
    got = rp.derive_rho(rp.SketchSpec("srht", sk["m"], sk["n"], 1, 0), w.a, lo, hi, ctx=ctx)
    ref = oracle.derive_rho(oracle.SketchSpec("srht", sk["m"], sk["n"], 1, 0), w.a, lo, hi)
    _check(rp, oracle, got, ref, lo, hi)
