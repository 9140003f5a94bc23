"""Device draw contract vs the reference's own rng.hpp (golden fixtures) and the
oracle: every integer draw bit-exact; Gaussian entries reported as an exact-
match rate with the mismatches bounded (glibc log/sin/cos are not correctly
rounded)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_u64_stream_and_jump_ahead(rp, ctx, golden, oracle):
    assert np.array_equal(rp.draw_u64(0, 2048, ctx=ctx), golden["u64_seed0"])
    assert np.array_equal(rp.draw_u64(12345, 1024, skip=1_000_003, ctx=ctx), golden["u64_seed12345_skip1000003"])
    # segment boundaries (65536-word segments) and odd offsets
    for seed, skip, count in ((7, 65530, 20), (8, 311, 200000), (9, 2**20 + 1, 1000)):
        assert np.array_equal(rp.draw_u64(seed, count, skip=skip, ctx=ctx), oracle.fill_u64(seed, count, skip=skip))
    assert rp.draw_u64(1, 0, ctx=ctx).shape == (0,)


def test_uniform01_sign_uniform_index(rp, ctx, golden, oracle):
    assert np.array_equal(rp.draw_uniform01(0, 1024, ctx=ctx), golden["uniform01_seed0"])
    assert np.array_equal(rp.draw_sign(3, 1024, ctx=ctx), golden["sign_seed3"])
    assert np.array_equal(rp.draw_uniform_index(4, 1000, 512, ctx=ctx), golden["uindex_seed4_bound1000"])
    # rejection-heavy bound: exercises the sequential fallback (rng.hpp:32-37)
    assert np.array_equal(rp.draw_uniform_index(3, (1 << 63) + 1, 512, ctx=ctx), golden["uindex_seed3_bound2p63p1"])
    assert np.array_equal(rp.draw_uniform_index(11, 7, 70000, ctx=ctx), oracle.fill_uniform_index(11, 7, 70000))


def test_countsketch_and_sjlt_draws_bit_exact(rp, ctx, golden, oracle):
    h, s = rp.count_draws(rp.SketchSpec("countsketch", 8192, 4096, 1, 0), ctx=ctx)
    assert np.array_equal(h[0], golden["count_m8192_seed0_h"]) and np.array_equal(s[0], golden["count_m8192_seed0_sign"])
    h, s = rp.count_draws(rp.SketchSpec("sjlt", 12, 64, 3, 6), ctx=ctx)
    assert np.array_equal(h.reshape(-1), golden["sjlt_m12_s3_n64_seed6_h"])
    assert np.array_equal(s.reshape(-1), golden["sjlt_m12_s3_n64_seed6_sign"])
    for spec in (("countsketch", 1000, 100003, 1, 5), ("sjlt", 60, 50000, 4, 6)):
        hg, sg = rp.count_draws(rp.SketchSpec(*spec), ctx=ctx)
        ho, so = oracle.count_draws(oracle.SketchSpec(*spec))
        assert np.array_equal(hg, ho) and np.array_equal(sg, so)


def test_srht_draws_bit_exact(rp, ctx, golden, oracle):
    signs, rows = rp.srht_draws(rp.SketchSpec("srht", 2048, 65536, 1, 0), ctx=ctx)
    assert np.array_equal(np.packbits(signs > 0), golden["srht_n65536_m2048_seed0_signbits"])
    assert np.array_equal(rows, golden["srht_n65536_m2048_seed0_rows"])
    signs, rows = rp.srht_draws(rp.SketchSpec("srht", 4, 13, 1, 77), ctx=ctx)
    assert np.array_equal(signs, golden["srht_n13_m4_seed77_signs"]) and np.array_equal(rows, golden["srht_n13_m4_seed77_rows"])
    for m, n, seed in ((1, 1, 3), (5000, 70000, 9), (16, 16, 2)):
        sg, rg = rp.srht_draws(rp.SketchSpec("srht", m, n, 1, seed), ctx=ctx)
        so, ro = oracle.srht_draws(oracle.SketchSpec("srht", m, n, 1, seed))
        assert np.array_equal(sg, so) and np.array_equal(rg, ro)


def _gauss_report(got, want):
    exact = float(np.mean(got == want))
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    return exact, float(rel.max())


def test_gaussian_entries(rp, ctx, golden, oracle):
    """Box-Muller entries bit-exact: the device runs glibc's own log/sin/cos
    (glibc_libm.cuh) on the extracted tables, so every entry equals the
    reference's std::log/std::sin/std::cos result (rng.hpp:43-55)."""
    got = rp.draw_normals(0, 8192, ctx=ctx)
    exact, rel = _gauss_report(got, golden["normals_seed0"])
    print(f"normals: exact-match {exact:.4f}, max rel {rel:.2e}")
    assert exact == 1.0
    w = rp.gaussian_window(0, 512, 4096, 0, 2, 0, 4096, ctx=ctx)
    assert np.array_equal(w, golden["c1_S_rows01"])
    # odd n: rows start mid Box-Muller pair (cached sin half, rng.hpp:44-47)
    w = rp.gaussian_window(9, 7, 33, 0, 7, 0, 33, ctx=ctx)
    assert np.array_equal(w, golden["gauss_m7_n33_seed9"])
    # an interior window, odd offsets
    full = oracle.gaussian_sketch_matrix(oracle.SketchSpec("gaussian", 40, 1001, 1, 5))
    w = rp.gaussian_window(5, 40, 1001, 3, 30, 17, 900, ctx=ctx)
    assert np.array_equal(w, full[3:33, 17:917])


def test_gaussian_entries_many(rp, ctx, oracle):
    """2^22 consecutive normals vs the oracle's glibc Box-Muller: bit-exact."""
    n = 1 << 22
    got = rp.draw_normals(11, n, ctx=ctx)
    want = oracle.fill_normals(11, n)
    assert np.array_equal(got, want), f"{np.count_nonzero(got != want)} of {n} differ"
