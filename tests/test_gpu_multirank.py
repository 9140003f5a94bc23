"""The library's multi-rank path, run for real with 2 and 3 ranks.

Each rank is a process with its own context holding its shard (rows, CSR
rows, or the dual's columns) and a host-side communicator over gloo
(rp_comm_init_host): the product's shard arithmetic, all-reduces, interval
split, per-generation Gram all-reduce (pass mode), Woodbury with shards,
dual recovery on column shards and divergence agreement all execute.  The
ranks share the one GPU and take turns on it (tests/multirank_worker.py), so
no kernel of one rank waits on, or time-slices with, another's.

Bars: x(lambda) within 1e-10 (relative l2, every lambda) of the same path on
the whole operator in one process -- the ranks only change summation order --
and within 1e-8 of the oracle (north_star); the sharded train losses within
1e-10 of the unsharded ones.  With NCCL and >= 2 visible GPUs the same
decomposition runs through ncclAllReduce (test_nccl_two_gpus, skipped on a
one-GPU box).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import multirank_cases as mc  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [c[0] for c in mc.cases()]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(world, tmp, extra_env=None):
    port = _free_port()
    lock = os.path.join(tmp, "gpu.token")
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   **(extra_env or {}))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"), tmp, lock],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        out, _ = p.communicate(timeout=900)
        logs.append(out)
        assert p.returncode == 0, out[-3000:]
    return [dict(np.load(os.path.join(tmp, f"rank{r}.npz"))) for r in range(world)]


@pytest.fixture(scope="module", params=[2, 3])
def ranks(request, tmp_path_factory):
    world = request.param
    tmp = str(tmp_path_factory.mktemp(f"world{world}"))
    return world, _spawn(world, tmp)


@pytest.fixture(scope="module")
def single(rp, oracle):
    """Unsharded device run (one context, no communicator) and the oracle, per case."""
    out = {}
    for name, w, route, opts in mc.cases():
        ctx = rp.Context(0)
        for k, v in opts.items():
            ctx.set_option(k, v)
        b = mc.b_matrix(w)
        lam = mc.grid(w, rp.log_grid)
        sk = w.sketch
        cfg = rp.PathConfig(w.lambda_min, w.lambda_max, lam, w.epsilon)
        spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
        ocfg = oracle.PathConfig(w.lambda_min, w.lambda_max, lam, w.epsilon, None)
        ospec = oracle.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
        if isinstance(w.a, dict):
            ga = rp.Csr(w.a["rows"], w.a["cols"], w.a["offsets"], w.a["indices"], w.a["values"])
            oa = oracle.Csr(w.a["rows"], w.a["cols"], w.a["offsets"], w.a["indices"], w.a["values"])
        else:
            ga = oa = w.a
        if route == "rows":
            got = rp.ihs_bin_path(ga, b, cfg, spec, rp.RhoBounds.manual(*w.rho), ctx=ctx)
            ref = oracle.ihs_bin_path(oa, b, ocfg, ospec, oracle.RhoBounds.manual(*w.rho))
        else:
            got = rp.dual_path(ga, b, cfg, spec, rp.RhoBounds.manual(*w.rho), ctx=ctx)
            ref = oracle.dual_path(oa, b, ocfg, ospec, oracle.RhoBounds.manual(*w.rho))
        out[name] = (got, ref, route)
    return out


def _rel(x, ref):
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300)


@pytest.mark.parametrize("case", CASES)
def test_sharded_path_matches_single_and_oracle(ranks, single, oracle, case):
    world, res = ranks
    got1, ref, route = single[case]
    T = len(got1.points)
    dim_full, K = got1.points[0].solution.shape
    if route == "rows":
        # every rank returns the whole x(lambda) (replicated state / all-reduced composition)
        for r in range(world):
            x = res[r][case + ":x"].reshape(T, K, dim_full).transpose(0, 2, 1)
            worst1 = max(_rel(x[t], got1.points[t].solution) for t in range(T))
            worst0 = max(_rel(x[t], ref.points[t].solution) for t in range(T))
            assert worst1 <= 1e-10, (case, world, r, worst1)
            assert worst0 <= 1e-8, (case, world, r, worst0)
        loss1 = np.array([p.train_loss for p in got1.points])
        for r in range(world):
            assert np.max(np.abs(res[r][case + ":loss"] - loss1) / np.abs(loss1)) <= 1e-10
    else:
        # dual: rank r recovers v = A^T z on its own columns; stitch them
        parts = []
        for r in range(world):
            c0, c1 = res[r][case + ":split"]
            parts.append((c0, res[r][case + ":x"].reshape(T, K, c1 - c0).transpose(0, 2, 1)))
        x = np.concatenate([p for _, p in sorted(parts, key=lambda q: q[0])], axis=1)
        worst1 = max(_rel(x[t], got1.points[t].solution) for t in range(T))
        worst0 = max(_rel(x[t], ref.points[t].solution) for t in range(T))
        assert worst1 <= 1e-10, (case, world, worst1)
        assert worst0 <= 1e-8, (case, world, worst0)
    for r in range(world):
        assert res[r][case + ":collectives"][0] > 0, "the host communicator was never called"
    if case == "c1_gauss_matrix":
        assert res[0][case + ":gram_mode"][0] == 1  # Gram-matrix mode: intervals split over the ranks
    if case == "c1_gauss_pass":
        assert res[0][case + ":gram_mode"][0] == 0  # pass mode: one all-reduce per generation


def test_host_comm_failure_maps_to_enccl(rp):
    ctx = rp.Context(0)

    def bad(*_):
        raise RuntimeError("transport down")

    rp.comm_init_host(ctx, 0, 2, bad, bad)
    n, d = 64, 8
    a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, d)))
    rp.set_dense_rows_host(ctx, 2 * n, 0, n, d, a.ctypes.data, n)
    y = np.ones(n)
    out = np.empty(d)
    st = rp.lib().rp_apply_transpose(ctx.handle, rp._ptr(y), 1, rp._ptr(out), rp.RP_HOST)
    assert st == 6  # RP_ENCCL
    assert "host allreduce" in rp.lib().rp_last_error(ctx.handle).decode()


def test_nccl_two_gpus(tmp_path):
    """Real NCCL between two GPUs (skipped when fewer are visible)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs; the multi-rank path is covered above through the host communicator")
    world = 2
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                                       "--warmup", "1", "--config", "c1", "--no-cpu-baseline", "--check"],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    for p in procs:
        out, _ = p.communicate(timeout=900)
        assert p.returncode == 0, out[-3000:]
