"""The NCCL code path on one GPU: a one-rank communicator (rp_comm_init with
world = 1 and an id) routes every all-reduce of the path, the sketch, the
Gram matrix, the losses and the baselines through ncclAllReduce.  A one-rank
sum is the identity, so results must equal the communicator-free run bit for
bit; this exercises NCCL loading (dlopen), communicator set-up and the stream
semantics of the collectives on hardware."""
import numpy as np
import pytest

try:  # torch's bundled libnccl must be the process's NCCL: a system libnccl loaded first (by the library's
    import torch  # noqa: F401  dlopen) makes a later `import torch` fail on its newer symbols
except Exception:  # pragma: no cover
    torch = None

import workloads

pytestmark = pytest.mark.gpu


def _runs(rp, ctx, w, K=1):
    a = w.a
    if isinstance(a, dict):
        a = rp.Csr(a["rows"], a["cols"], a["offsets"], a["indices"], a["values"])
    grid = rp.log_grid(w.lambda_min, w.lambda_max, 30)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    sk = w.sketch
    spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    path = rp.ihs_bin_path(a, w.b, cfg, spec, rho, ctx=ctx)
    cg = rp.warm_cg_path(a, w.b[:, 0], rp.PathConfig(w.lambda_min, w.lambda_max, grid[-5:], 1e-8), ctx=ctx)
    der = rp.derive_rho(spec, a, w.lambda_min, w.lambda_max, ctx=ctx)
    return path, cg, der


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_one_rank_nccl_matches_local(rp, oracle, name):
    w = workloads.get(name, scale=1.0 if name == "c1" else 1 / 1024)
    plain = rp.Context(0)
    want = _runs(rp, plain, w)
    comm = rp.Context(0)
    rp.comm_init(comm, 0, 1, rp.comm_unique_id())
    got = _runs(rp, comm, w)
    for p, q in zip(got[0].points, want[0].points):
        assert np.array_equal(p.solution, q.solution) and p.train_loss == q.train_loss
    for p, q in zip(got[1].points, want[1].points):
        assert np.array_equal(p.solution, q.solution) and p.iterations == q.iterations
    assert got[2][0] == want[2][0]


def test_concurrent_contexts(rp, oracle):
    """Two contexts on one GPU driven from two host threads, their kernels
    running concurrently (no device lock since the stage-release fix), give
    the bits of sequential runs."""
    import threading

    w = workloads.get("c1")
    grid = rp.log_grid(w.lambda_min, w.lambda_max, 30)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    sk = w.sketch
    spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    want = rp.ihs_bin_path(w.a, w.b, cfg, spec, rho, ctx=rp.Context(0))
    ctxs = [rp.Context(0), rp.Context(0)]
    got = [None, None]

    def run(i):
        for _ in range(6):
            got[i] = rp.ihs_bin_path(w.a, w.b, cfg, spec, rho, ctx=ctxs[i])
            for p, q in zip(got[i].points, want.points):
                assert np.array_equal(p.solution, q.solution)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for res in got:
        for p, q in zip(res.points, want.points):
            assert np.array_equal(p.solution, q.solution)


def test_kernel_smem_limits_survive_other_threads(rp, ctx, oracle):
    """A kernel's dynamic shared-memory limit is per function and device, shared
    by every thread: a thread launching the fused column pass with a small
    operator must not lower the limit a larger operator's launch in another
    thread needs (regression: a per-thread cache of the limit let exactly that
    happen and the large launch failed with "invalid argument")."""
    import threading

    rng = np.random.default_rng(5)
    big = rng.standard_normal((4096, 1024))
    small = rng.standard_normal((4096, 64))

    def colpass(a, c):
        y = np.random.default_rng(a.shape[1]).standard_normal(a.shape[0])
        got = rp.apply_transpose(a, y, ctx=c)
        assert np.allclose(got, a.T @ y, rtol=1e-12, atol=1e-9)

    colpass(big, ctx)  # raises the limit (main thread)
    t = threading.Thread(target=colpass, args=(small, rp.Context(0)))  # another thread, smaller need
    t.start()
    t.join()
    colpass(big, ctx)  # still launches
