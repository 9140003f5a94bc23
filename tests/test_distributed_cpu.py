"""Multi-rank path on CPU (gloo, world_size 2).

The device library shards the primal operator by rows (rp_set_dense_rows): each
rank sketches its rows (Gaussian: columns [row0, row1) of S, i.e. MT stream
offsets r*n + row0; CountSketch: the global draw stream, local rows; SRHT: the
local rows zero-padded), forms its partial Gram matrix and linear term, and
all-reduces SA, G = A^T A and c = A^T b; the intervals are then split
round-robin and the composed x(lambda) summed (ridgepath.cpp run_path).  This
test runs exactly that decomposition with the oracle's CPU kernels under a
real 2-rank gloo process group and checks it against the unsharded oracle
path, so the sharding and reduction logic is covered without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _sharded_path(kind, rank, world):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import ridgepath_oracle as o

    import workloads

    w = workloads.c1(scale=0.25)
    a, b = w.a, w.b
    n, d = a.shape
    m = w.sketch["m"] if kind != "srht" else 96
    r0, r1 = rank * n // world, (rank + 1) * n // world
    a_loc, b_loc = a[r0:r1], b[r0:r1]
    spec = o.SketchSpec(kind, m, n, 1, 3)
    # 1) partial sketch of the local rows
    if kind == "gaussian":
        s_win = np.empty((m, r1 - r0))
        o._load().or_gaussian_window(3, m, n, 0, m, r0, r1 - r0, o._ptr(s_win))
        sa = s_win @ a_loc
    elif kind == "countsketch":
        h, sg = o.count_draws(spec)
        sa = np.zeros((m, d))
        for j in range(r0, r1):
            sa[h[0, j]] += sg[0, j] * a[j]
    else:  # srht: local rows zero-padded (the transform is linear)
        a_pad = np.zeros_like(a)
        a_pad[r0:r1] = a_loc
        sa = o.sketch_apply(spec, a_pad)
    sa = _allreduce(sa)
    # 2) linear term and Gram matrix partials
    c = _allreduce(a_loc.T @ b_loc)
    G = _allreduce(a_loc.T @ a_loc)
    # 3) intervals round-robin, x summed
    grid = w.lambdas(o.log_grid)
    cfg = o.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    rho = o.RhoBounds.manual(*workloads.mp_envelope(d, m))
    plans = o.plan_intervals(cfg, rho, None)
    pre = o.Preconditioner.build(sa, plans[0].params.lambda0)
    x = np.zeros((len(grid), d, 1))
    for li, plan in enumerate(plans):
        if li % world != rank:
            continue
        p = pre.reshift(plan.params.lambda0)
        basis = o.build_interval_basis_matrix(a, c, p, plan, gram=lambda W: G @ W)
        for lam in plan.grid:
            x[grid.index(lam)] = o.compose_horner(basis, basis.tau * lam)
    x = _allreduce(x)
    # unsharded reference
    ref = o.ihs_bin_path(a, b, cfg, spec, rho)
    return max(o.rel_error(x[t], ref.points[t].solution) for t in range(len(grid))), o.rel_error(
        sa, o.sketch_apply(spec, a))


def _worker(rank, world, port, kind, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, _sharded_path(kind, rank, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["gaussian", "countsketch", "srht"])
def test_row_sharded_path_world2(kind):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (x_err, sa_err) in res.items():
        assert sa_err < 1e-13, f"rank {rank}: summed partial sketches differ ({sa_err:.2e})"
        assert x_err < 1e-8, f"rank {rank}: sharded path differs from the unsharded oracle ({x_err:.2e})"
