"""RP_HOST_STREAM: the operator upload runs in column chunks on a copy stream
and the path consumes them as they land (sketch columns, A^T b rows, Gram
block rows).  The result must match the device-resident path to rounding (the
Gram matrix is formed by block rows instead of one SYRK) and the oracle to the
parity bar; generic readers wait for the upload."""
import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


def _run(rp, ctx, a, b, cfg, spec, rho, stream):
    n, d = a.shape
    K = b.shape[1]
    T = len(cfg.lambdas)
    a_host = torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory()  # column-major A
    b_host = torch.from_numpy(np.ascontiguousarray(b.T)).pin_memory()
    x = torch.empty(T * K * d, dtype=torch.float64).pin_memory()
    rp.set_dense_rows_host(ctx, n, 0, n, d, a_host.data_ptr(), n, stream=stream)
    rp.path_raw(ctx, b_host.data_ptr(), K, cfg, spec, rho, x.data_ptr(), rp.RP_HOST)
    ctx._op_key = None
    return x.numpy().reshape(T, K, d).copy(), a_host


@pytest.mark.parametrize("kind,K,mode", [("srht", 1, -1), ("srht", 2, 0), ("countsketch", 1, 1), ("sjlt", 1, -1),
                                         ("identity", 1, 1), ("gaussian", 1, -1), ("gaussian", 2, 1)])
def test_streamed_upload_matches_resident_path(rp, ctx, oracle, kind, K, mode):
    w = workloads.c2(scale=1 / 16)
    n, d = w.a.shape
    m = n if kind == "identity" else (4 * d if kind == "gaussian" else 16 * d)  # (Gaussian: S stays resident)
    s = 4 if kind == "sjlt" else 1
    b = np.asfortranarray(np.concatenate([w.b] + [w.b * (k + 2) - 0.5 for k in range(K - 1)], axis=1))
    grid = rp.log_grid(w.lambda_min, w.lambda_max, 40)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    spec = rp.SketchSpec(kind, m, n, s, 3)
    rho = rp.RhoBounds.manual(*workloads.mp_envelope(d, m)) if kind != "identity" else rp.RhoBounds.identity()
    ctx.set_option("gram_mode", mode)
    ctx.set_option("upload_chunk_bytes", n * 8 * 24)  # 24-column chunks: 3 chunks for d = 64
    try:
        xs, keep = _run(rp, ctx, w.a, b, cfg, spec, rho, True)
        xr, _ = _run(rp, ctx, w.a, b, cfg, spec, rho, False)
    finally:
        ctx.set_option("gram_mode", -1)
        ctx.set_option("upload_chunk_bytes", 32 << 20)
    for t in range(len(grid)):
        for k in range(K):
            assert oracle.rel_error(xs[t, k], xr[t, k]) < 1e-11


def test_streamed_upload_c2_scaled_parity(rp, ctx, oracle):
    """The C2 configuration at 1/8 scale (as tests/test_gpu_path.py) through the
    streamed upload: x(lambda) within the 1e-8 parity bar of the oracle."""
    w = workloads.c2(scale=1 / 8)
    n, d = w.a.shape
    sk = w.sketch
    grid = rp.log_grid(w.lambda_min, w.lambda_max, w.T)[::10]
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    ctx.set_option("upload_chunk_bytes", n * 8 * 40)  # 40-column chunks: 4 chunks for d = 128
    try:
        xs, keep = _run(rp, ctx, w.a, w.b, cfg, rp.SketchSpec("srht", sk["m"], n, 1, sk["seed"]),
                        rp.RhoBounds.manual(*w.rho), True)
    finally:
        ctx.set_option("upload_chunk_bytes", 32 << 20)
    ref = oracle.ihs_bin_path(w.a, w.b, oracle.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None),
                              oracle.SketchSpec("srht", sk["m"], n, 1, sk["seed"]), oracle.RhoBounds.manual(*w.rho))
    worst = max(oracle.rel_error(xs[t, 0], p.solution[:, 0]) for t, p in enumerate(ref.points))
    assert worst < 1e-8


def test_streamed_upload_generic_readers_wait(rp, ctx, oracle):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3000, 700))
    a_host = torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory()
    ctx.set_option("upload_chunk_bytes", 3000 * 8 * 100)
    rp.set_dense_rows_host(ctx, 3000, 0, 3000, 700, a_host.data_ptr(), 3000, stream=True)
    ctx._op_key = ("stream", a_host.data_ptr())
    y = rng.standard_normal(3000)
    out = np.empty(700)
    ctx.check(rp.lib().rp_apply_transpose(ctx.handle, rp._ptr(y), 1, rp._ptr(out), rp.RP_HOST))
    assert oracle.rel_error(out, a.T @ y) < 1e-13
    # replacing a still-uploading operator is safe
    rp.set_dense_rows_host(ctx, 3000, 0, 3000, 700, a_host.data_ptr(), 3000, stream=True)
    b2 = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((700, 3000)))).pin_memory()
    rp.set_dense_rows_host(ctx, 3000, 0, 3000, 700, b2.data_ptr(), 3000, stream=True)
    ctx.check(rp.lib().rp_apply_transpose(ctx.handle, rp._ptr(y), 1, rp._ptr(out), rp.RP_HOST))
    assert oracle.rel_error(out, b2.numpy() @ y) < 1e-13
    ctx.set_option("upload_chunk_bytes", 32 << 20)
    ctx._op_key = None


def test_streamed_upload_pageable_and_column_shard(rp, ctx, oracle):
    """RP_HOST_STREAM from pageable memory (the copies degrade to synchronous
    ones) and for a column-sharded (dual-route) operator (no chunked consumer:
    the first reader waits for the whole upload) give the resident results."""
    w = workloads.c2(scale=1 / 16)
    n, d = w.a.shape
    grid = rp.log_grid(w.lambda_min, w.lambda_max, 20)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    spec = rp.SketchSpec("srht", 4 * d, n, 1, 3)
    rho = rp.RhoBounds.manual(*workloads.mp_envelope(d, 4 * d))
    ctx.set_option("upload_chunk_bytes", n * 8 * 24)
    try:
        xr, _ = _run(rp, ctx, w.a, w.b, cfg, spec, rho, False)
        a_cm = np.ascontiguousarray(w.a.T)  # pageable, column-major A
        b_cm = np.ascontiguousarray(w.b[:, 0])
        x = np.empty(len(grid) * d)
        ctx.check(rp.lib().rp_set_dense_rows(ctx.handle, n, 0, n, d, rp._ptr(a_cm), n, rp.RP_HOST_STREAM))
        rp.path_raw(ctx, b_cm.ctypes.data, 1, cfg, spec, rho, x.ctypes.data, rp.RP_HOST)
        ctx._op_key = None
        for t in range(len(grid)):
            assert oracle.rel_error(x[t * d:(t + 1) * d], xr[t, 0]) < 1e-11
        # dual route on a column-sharded streamed operator (one rank holds every column)
        a2 = np.ascontiguousarray(w.a[:, :40].T)  # A' = first 40 columns (n x 40), column-major
        sk = rp.SketchSpec("countsketch", 16, 40, 1, 5)  # sketch of A'^T (40 rows)
        outs = []
        for where in (rp.RP_HOST, rp.RP_HOST_STREAM):
            ctx.check(rp.lib().rp_set_dense_cols(ctx.handle, n, 40, 0, 40, rp._ptr(a2), n, where))
            sa = np.empty(16 * n)
            ctx.check(rp.lib().rp_sketch_apply(ctx.handle, rp.ctypes.byref(sk.c()), 1, rp._ptr(sa), rp.RP_HOST))
            outs.append(sa)
        ctx._op_key = None
        assert np.array_equal(outs[0], outs[1])
    finally:
        ctx.set_option("upload_chunk_bytes", 32 << 20)


def test_streamed_gaussian_blocks_of_several_chunks(rp, ctx, oracle):
    """Gaussian sketch through the streamed upload: S is drawn once and applied
    to blocks of several upload chunks (at least 128 columns wide); d = 300 with
    50-column chunks gives blocks of 150 columns.  Against the oracle."""
    rng = np.random.default_rng(11)
    n, d, m = 2048, 300, 600
    a = np.asfortranarray(rng.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1)))
    b = np.asfortranarray((a @ rng.standard_normal(d) + 0.1 * rng.standard_normal(n)).reshape(n, 1))
    grid = rp.log_grid(1e-2, 1e1, 12)
    rho = workloads.mp_envelope(d, m)
    cfg = rp.PathConfig(1e-2, 1e1, grid, 1e-6)
    ctx.set_option("upload_chunk_bytes", n * 8 * 50)
    try:
        xs, keep = _run(rp, ctx, a, b, cfg, rp.SketchSpec("gaussian", m, n, 1, 5), rp.RhoBounds.manual(*rho), True)
    finally:
        ctx.set_option("upload_chunk_bytes", 32 << 20)
    ref = oracle.ihs_bin_path(a, b, oracle.PathConfig(1e-2, 1e1, grid, 1e-6, None),
                              oracle.SketchSpec("gaussian", m, n, 1, 5), oracle.RhoBounds.manual(*rho))
    worst = max(oracle.rel_error(xs[t, 0], p.solution[:, 0]) for t, p in enumerate(ref.points))
    assert worst < 1e-8
