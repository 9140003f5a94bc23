#!/usr/bin/env python
"""bench.py -- IHS-BIN ridge-path time on the BASELINE configs, 1..8 B200.

One "step" = one full ridge path (sketch + factor + every interval basis + all
T compositions; path_solver.cpp:147-190, the metric's setup + sum of point
seconds) over one BASELINE config, with the operator, b and x resident in HBM
(`value`).  `e2e` repeats the step through the public C ABI with host buffers:
pinned A (or the CSR arrays) and b copied in, x copied out, every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]

Default config: C2 (65536 x 1024 dense, SRHT m = 2048, T = 1000) at N = 1,
the config the metric is quoted on; C3 (1M x 2048 dense, Gaussian m = 4096,
T = 1000, 16 GB, row-sharded) for N > 1 -- SURVEY 8(e) keeps C2 on one GPU.
With --gpus N > 1 and no WORLD_SIZE in the environment the script relaunches
itself under torchrun (one process per GPU).  Ranks: row shards of A (C1-C4)
or column shards (C5, dual route), NCCL all-reduces inside the library, the
time is the max over ranks.  `--impl reference` times the CPU restatement of
the reference (oracle/; the reference itself needs Eigen, absent here) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "ridge-path time (sketch+basis+T lambda solves)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default: c2 at 1 GPU, c3 at more)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-1thread", type=int, default=-1,
                    help="also time the 1-thread CPU baseline (default: on for c1-c3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--check", action="store_true", help="c1 only: x(lambda) vs the oracle, every rank")
    ap.add_argument("--dump-gemm", default=None, help="write the per-launch GEMM profile of a step (JSON)")
    ap.add_argument("--path-only", action="store_true",
                    help="only the timed steps (no roofline / pass / e2e / CPU legs): for ncu launch lists")
    a = ap.parse_args()
    if a.config is None:
        a.config = "c2" if a.gpus == 1 else "c3"
    a.config = a.config.lower()
    if a.cpu_1thread < 0:
        a.cpu_1thread = 1 if a.config in ("c1", "c2", "c3") else 0
    return a


def relaunch_under_torchrun(args):
    """--gpus N > 1 without a launcher: one process per GPU via torchrun."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (CPU restatement of the reference) on a bounded
# sample of the workload, extrapolated
# ---------------------------------------------------------------------------

# rows of the sketched operator in the CPU sample (d, m unchanged); None = all
CPU_ROWS = {"c1": None, "c2": None, "c3": 16384, "c4": 65536, "c5": 8192}
CPU_ROWS_1THREAD = {"c1": None, "c2": 8192, "c3": 8192, "c4": 32768, "c5": 4096}
FULL_ROWS = {"c1": 4096, "c2": 65536, "c3": 1048576, "c4": 4194304, "c5": 131072}


def _threads(n):
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(limits=n)
    except Exception:  # pragma: no cover
        import contextlib

        return contextlib.nullcontext()


def cpu_model(name, threads=None):
    """Times the reference algorithm (oracle/ridgepath_oracle.py, which
    restates path_solver.cpp / preconditioner.cpp / sketch.cpp) on the host.

    C1: the whole path.  Otherwise on `rows` rows of the sketched operator
    (same d, m, distributions): the linear term and the sketch (linear in the
    row count, scaled to the full n), the thin SVD of SA (m x d, independent
    of n), and one interval basis with its compositions -- its Gram products
    are timed inside (linear in n, scaled) and the rest (preconditioner
    applies, updates) is n-independent; the total is
    t_setup + L * K * t_interval + T * K * t_compose, since the reference runs
    every interval and every right-hand-side column separately
    (path_solver.cpp:122-123, 168-186).  For C4 (and C5 at one thread) the
    SVD of the full m x d SA is timed on m/4 rows and scaled by 16 (O(m^2 d)),
    and for C4/C5 the interval
    runs with a synthetic rank-m preconditioner of the full shape (the path's
    work does not depend on its values)."""
    from oracle import ridgepath_oracle as o

    threads = threads or (os.cpu_count() or 1)
    rows = (CPU_ROWS_1THREAD if threads == 1 else CPU_ROWS)[name]
    with _threads(threads):
        w = workloads.get(name, n_rows=rows) if name != "c5" else workloads.c5(n_rows=rows)
        sk = w.sketch
        spec = o.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
        grid = w.lambdas(o.log_grid)
        cfg = o.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
        rho = o.RhoBounds.manual(*w.rho)
        if isinstance(w.a, dict):
            a = o.Csr(w.a["rows"], w.a["cols"], w.a["offsets"], w.a["indices"], w.a["values"])
        else:
            a = w.a
        b = np.asarray(w.b).reshape(w.b.shape[0], -1)
        K = b.shape[1]
        if name == "c1":
            t0 = time.perf_counter()
            o.ihs_bin_path(a, b, cfg, spec, rho)
            t = time.perf_counter() - t0
            return t, threads, f"the whole C1 path (oracle port, {threads} thread(s))"
        op = o.transpose(a) if w.dual else a
        n_s = o._rows(op)
        n_full = FULL_ROWS[name]
        scale = n_full / n_s
        t0 = time.perf_counter()
        c = b[:, :1].copy() if w.dual else o.apply_transpose(op, b[:, :1])
        sa = o.sketch_apply(spec, op)
        t_lin = time.perf_counter() - t0
        m, dim = sa.shape
        # (the zero-initialised m x d output is n-independent: timed once, not scaled)
        tz = time.perf_counter()
        np.zeros((m, dim)).fill(0.0)
        t_zero = min(time.perf_counter() - tz, t_lin)
        t_lin -= t_zero
        plans = o.plan_intervals(cfg, rho, None)
        plan = plans[0]
        synthetic = name in ("c4", "c5")
        t1 = time.perf_counter()
        if synthetic:
            ms = m if (name == "c5" and threads > 1) else max(16, m // 4)
            o.thin_svd(sa[:ms])
            t_svd = (time.perf_counter() - t1) * (m / ms) ** 2
            rng = np.random.default_rng(1)
            vt = rng.standard_normal((m, dim)) / np.sqrt(dim)
            sig = np.linspace(2.0, 0.5, m)
            pre = o.Preconditioner(vt, sig, plan.params.lambda0, m, dim, False)
        else:
            svd = o.thin_svd(sa)
            t_svd = time.perf_counter() - t1
            pre = o.Preconditioner.build_from_svd(svd, m, dim, plan.params.lambda0)
        gram_t = [0.0]

        def gram(wv):
            tg = time.perf_counter()
            r = o.gram_apply(op, wv)
            gram_t[0] += time.perf_counter() - tg
            return r

        t2 = time.perf_counter()
        p = pre.reshift(plan.params.lambda0)
        tau = plan.params.alpha * (1e-12 if synthetic else 1.0)  # (synthetic P: keep the recursion finite)
        with np.errstate(all="ignore"):
            tilde = o.ihs_basis_core(op, c[:, 0], p, tau, plan.params.k, gram=gram)
        t_int_sample = time.perf_counter() - t2
        basis = o.BinomialBasis([tilde[:, [j]] for j in range(plan.params.k)], tau)
        t3 = time.perf_counter()
        for lam in plan.grid:
            o.compose_horner(basis, tau * lam)
        t_comp = (time.perf_counter() - t3) / max(len(plan.grid), 1)
        t_int = (t_int_sample - gram_t[0]) + gram_t[0] * scale
        L = len(plans)
        total = t_lin * scale + t_zero + t_svd + L * K * t_int + len(grid) * K * t_comp
    sample = (f"oracle port, {threads} thread(s): {n_s} of {n_full} operator rows (d={dim}, m={m}); "
              f"A^T b + sketch {t_lin:.2f}s x{scale:g}, SVD {t_svd:.2f}s"
              f"{(' (on %d of %d rows, x%g)' % (ms, m, (m / ms) ** 2)) if synthetic and ms < m else ''}, interval 0 basis {t_int_sample:.2f}s of which Gram "
              f"{gram_t[0]:.2f}s x{scale:g}{', synthetic rank-m preconditioner' if synthetic else ''}; "
              f"extrapolated to {L} intervals x K={K} and T={len(grid)} compositions")
    return total, threads, sample


def run_reference(args):
    vals = []
    sample = cores = None
    for i in range(args.warmup + args.steps):
        total, cores, sample = cpu_model(args.config)
        if i >= args.warmup:
            vals.append(total)
    v = statistics.mean(vals)
    w = workloads_desc(args.config)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": w, "parallelism": "host CPU (numpy/OpenBLAS + C oracle)"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workloads_desc(name):
    if name in ("c1", "c2"):
        w = workloads.get(name)
        return workloads._desc(w.name, w.meta["n"], w.meta["d"], w, "dense")
    fixed = {
        "c3": ("C3", 1048576, 2048, workloads.Workload("C3", None, None, dict(kind="gaussian", m=4096, n=1048576,
                                                                                s=1, seed=0), 1e-3, 1e2, 1000,
                                                      workloads.mp_envelope(2048, 4096)), "dense"),
        "c4": ("C4", 4194304, 65536, workloads.Workload("C4", None, None, dict(kind="countsketch", m=8192,
                                                                                 n=4194304, s=1, seed=0),
                                                       1e-2, 1e2, 500, (1.0, 1e-5)), "CSR 16 nnz/row"),
        "c5": ("C5", 16384, 131072, workloads.Workload("C5", None, None, dict(kind="gaussian", m=4096, n=131072,
                                                                                s=1, seed=0), 1e-3, 1e1, 200,
                                                      (1.0, 1e-5), dual=True), "dense, dual (A^T sketched), K=16"),
    }[name]
    return workloads._desc(fixed[0], fixed[1], fixed[2], fixed[3], fixed[4])


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------


def measure_dgemm_peak(torch):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e12


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("hbm_gbs", 6449.1)), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6449.1, "fallback (SURVEY 8d measured copy bandwidth)"


class Arm:
    """One rank's operator/b/x and the library calls of a step."""

    def __init__(self, rp, torch, ctx, dw, dev):
        self.rp, self.torch, self.ctx, self.w, self.dev = rp, torch, ctx, dw, dev
        self.grid = rp.log_grid(dw.lambda_min, dw.lambda_max, dw.T)
        sk = dw.sketch
        self.cfg = rp.PathConfig(dw.lambda_min, dw.lambda_max, self.grid, dw.epsilon)
        self.spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
        self.rho = rp.RhoBounds.manual(*dw.rho)
        self.dual = dw.route == "cols"
        self.x_rows = dw.local if self.dual else dw.d
        self.x = torch.empty((dw.T * dw.K * self.x_rows,), dtype=torch.float64, device=dev)
        self.set_device()

    def set_device(self):
        rp, w = self.rp, self.w
        if w.sparse:
            off, cols, vals = w.csr
            self.ctx.check(rp.lib().rp_set_csr_rows(self.ctx.handle, w.n, w.lo, w.local, w.d, rp._P(off.data_ptr()),
                                                    rp._P(cols.data_ptr()), rp._P(vals.data_ptr()), rp.RP_DEVICE))
        elif self.dual:
            rp.set_dense_cols_device(self.ctx, w.n, w.d, w.lo, w.local, w.a_t.data_ptr(), w.n)
        else:
            rp.set_dense_rows_device(self.ctx, w.n, w.lo, w.local, w.d, w.a_t.data_ptr(), w.local)
        self.ctx._op_key = None

    def step(self):
        return self.rp.path_raw(self.ctx, self.w.b.data_ptr(), self.w.K, self.cfg, self.spec, self.rho,
                                self.x.data_ptr(), self.rp.RP_DEVICE, dual=self.dual)

    # -- end to end through the public API with host buffers -------------------
    def e2e_setup(self):
        torch, w = self.torch, self.w
        self.b_host = torch.empty(tuple(w.b.shape), dtype=torch.float64, pin_memory=True).copy_(w.b)
        self.x_host = torch.empty(self.x.numel(), dtype=torch.float64, pin_memory=True)
        if w.sparse:
            self.csr_host = [t.cpu().numpy() for t in w.csr]
            h2d = sum(a.nbytes for a in self.csr_host)
        else:
            self.a_host = torch.empty(tuple(w.a_t.shape), dtype=torch.float64, pin_memory=True).copy_(w.a_t)
            h2d = self.a_host.numel() * 8
        return h2d + self.b_host.numel() * 8, self.x_host.numel() * 8

    def e2e_step(self):
        rp, w = self.rp, self.w
        if w.sparse:
            off, cols, vals = self.csr_host
            rp.set_csr_rows(self.ctx, w.n, w.lo, rp.Csr(w.local, w.d, off, cols, vals))
        elif self.dual:
            self.ctx.check(rp.lib().rp_set_dense_cols(self.ctx.handle, w.n, w.d, w.lo, w.local,
                                                      rp._P(self.a_host.data_ptr()), w.n, rp.RP_HOST_STREAM))
        else:
            rp.set_dense_rows_host(self.ctx, w.n, w.lo, w.local, w.d, self.a_host.data_ptr(), w.local, stream=True)
        rp.path_raw(self.ctx, self.b_host.data_ptr(), w.K, self.cfg, self.spec, self.rho, self.x_host.data_ptr(),
                    rp.RP_HOST, dual=self.dual)


def check_c1(rp, arm):
    """--check: the whole C1 x(lambda) against the oracle (every rank holds it)."""
    from oracle import ridgepath_oracle as o

    w = workloads.c1()
    grid = w.lambdas(o.log_grid)
    ref = o.ihs_bin_path(w.a, w.b, o.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None),
                         o.SketchSpec("gaussian", 512, 4096, 1, 0), o.RhoBounds.manual(*w.rho))
    x = arm.x.view(len(grid), -1).cpu().numpy()
    worst = max(o.rel_error(x[t], ref.points[t].solution[:, 0]) for t in range(len(grid)))
    assert worst <= 1e-8, f"--check: x(lambda) rel err {worst:.3e}"
    return worst


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2210_12212_b200 import ridgepath as rp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def allreduce_t(t):
        dist.all_reduce(t)

    dw = workloads.device_workload(args.config, rank, world, dev, allreduce=allreduce_t)
    torch.cuda.synchronize(dev)
    ctx = rp.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [rp.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        rp.comm_init(ctx, rank, world, uid[0])
    arm = Arm(rp, torch, ctx, dw, dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def maxover(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        arm.step()
    torch.cuda.synchronize(dev)
    barrier()
    check = check_c1(rp, arm) if args.check else None
    clocks = ClockSampler(local)
    if not os.environ.get("BENCH_NO_CLOCKS"):
        clocks.start()
    launches0 = rp.launch_count()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(dev)
    barrier()
    e0.record(stream)
    tms = []
    for _ in range(args.steps):
        tms.append(arm.step())
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    launches = rp.launch_count() - launches0
    clk = clocks.stop()
    value = maxover(e0.elapsed_time(e1) * 1e-3 / args.steps)
    phases = {k: statistics.mean(getattr(tm, k) for tm in tms)
              for k in ("sketch_seconds", "linear_seconds", "gram_seconds", "precond_seconds", "basis_seconds",
                        "eval_seconds", "total_seconds")}
    gram_mode = tms[-1].gram_mode
    if args.path_only:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
                              "config": {"workload": dw.desc}, "phases_s": phases,
                              "gpu_launches": int(launches)}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # Roofline of the dominant kernel family (the FP64 DMMA GEMMs: sketch,
    # SYRK, factor, preconditioner applies, Gram products): the same steps
    # again with every GEMM bracketed by CUDA events on the step's stream
    # (the side-stream Gram overlap is switched off there, so each launch is
    # timed alone).
    ctx.set_option("gram_overlap", 0)
    arm.step()  # (untimed: the serialized schedule's first step sizes the main stream's split-K workspace)
    ctx.set_option("profile", 1)
    prof = [arm.step() for _ in range(max(1, min(args.steps, 2)))]
    ctx.set_option("gram_overlap", 1)
    ctx.set_option("profile", 0)
    l_sec, l_flops, l_bytes = rp.last_gemm_profile(ctx)  # per launch, last profiled step
    if args.dump_gemm and rank == 0:
        with open(args.dump_gemm, "w") as f:
            json.dump({"seconds": list(map(float, l_sec)), "flops": list(map(float, l_flops)),
                       "bytes": list(map(float, l_bytes))}, f)
    g_s = sum(p.gemm_seconds for p in prof)
    g_f = sum(p.gemm_flops for p in prof)
    g_calls = sum(p.gemm_calls for p in prof)
    tot_s = sum(p.total_seconds for p in prof)
    peak = measure_dgemm_peak(torch)
    achieved = g_f / g_s / 1e12 if g_s > 0 else 0.0
    hbm, hbm_src = hbm_peak()
    # DRAM traffic per launch of a representative GEMM from the committed ncu
    # --set full capture (C2 top launch), beside its algorithmic operand bytes
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_gemm_top.json")) as f:
            rec = json.load(f)
        traffic = float(rec["dram_bytes"])
        traffic_note = rec["note"]
    except Exception:
        try:
            with open(os.path.join(ROOT, "profiles", "r01_ncu_gemm_tma.json")) as f:
                rec = json.load(f)[0]
            traffic = 1e6 * (float(rec["dram__bytes_read.sum"].split()[0]) +
                             float(rec["dram__bytes_write.sum"].split()[0]))
            traffic_note = ("bytes per launch of %s (ncu --set full, profiles/r01_ncu_gemm_tma.json, the C2 Gram "
                            "product 1024 x 2016 x 1024 at split 4); algorithmic operand bytes of that launch "
                            "8*(1024*1024 + 1024*2016 + 4*1024*2016) = 90 MB" % rec["kernel"][:60])
        except Exception:
            pass
    bound_t = sum(max(fl / (peak * 1e12), by / (hbm * 1e9)) for fl, by in zip(l_flops, l_bytes)) if peak else 0.0
    n_hbm = sum(1 for fl, by in zip(l_flops, l_bytes) if peak and by / (hbm * 1e9) > fl / (peak * 1e12))
    binding = {"frac": bound_t / float(sum(l_sec)) if len(l_sec) else None, "launches": int(len(l_sec)),
               "hbm_bound_launches": int(n_hbm), "hbm_peak_gbs": hbm,
               "note": "sum over the GEMM launches of one step of max(flops/tensor peak, operand bytes/HBM peak) "
                       "divided by their summed device time"}
    roofline = {"bound": "tensor",
                "kernel": "dgemm_tma_kernel / dgemm_kernel (FP64 DMMA m8n8k4, TMA-fed; all GEMMs of the path)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                "traffic": traffic, "traffic_note": traffic_note,
                "share_of_step": g_s / tot_s if tot_s else None,
                "gemm_launches_per_step": g_calls / len(prof), "gemm_flops_per_step": g_f / len(prof),
                "binding_roof": binding,
                "peak_source": "cuBLAS DGEMM 8192^3 (torch.matmul fp64) measured in this run; MEASURED_PEAKS.json "
                               "has no FP64 figure; DMMA issue peak measured 37.1 TFLOP/s (profiles/fp64_peaks_r01.txt)"}

    # HBM-bound single passes over A (north_star: the fused Gram-matvec
    # A^T (A W) against the HBM roofline), device-timed by the library.
    passes = {}
    if world == 1 and dw.route == "rows" and not dw.sparse:
        widths = [("gram_fused_w1", 1), ("gram_fused_w2", 2), ("gram_fused_w4", 4), ("gram_fused_w8", 8),
                  ("atb_w1", 1)]
        for name, wcols in widths:
            fn = rp.apply_transpose_raw if name.startswith("atb") else rp.gram_apply_raw
            rows_in = dw.local if fn is rp.apply_transpose_raw else dw.d
            xin = torch.randn(rows_in * wcols, dtype=torch.float64, device=dev)
            xout = torch.empty(dw.d * wcols, dtype=torch.float64, device=dev)
            for _ in range(2):
                fn(ctx, xin.data_ptr(), wcols, xout.data_ptr())
            ctx.set_option("profile", 1)
            dev_t = []
            for _ in range(10):
                fn(ctx, xin.data_ptr(), wcols, xout.data_ptr())
                dev_t.append(rp.last_device_seconds(ctx))
            ctx.set_option("profile", 0)
            t = statistics.median(dev_t)
            byts = 8.0 * dw.local * dw.d
            passes[name] = {"seconds": t, "algorithmic_bytes": byts, "achieved_gbs": byts / t / 1e9,
                            "frac_hbm": byts / t / 1e9 / hbm, "timing": "median of 10 calls, CUDA events"}
    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        h2d, d2h = arm.e2e_setup()
        arm.e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            arm.e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        e2e = {"value": maxover((time.perf_counter() - t0) / args.steps), "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}
        arm.set_device()

    cpu = cpu1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        total, cores, sample = cpu_model(args.config)
        cpu = {"value": total, "unit": "s", "cores": cores, "kind": "port", "sample": sample}
        if args.cpu_1thread:
            total, cores, sample = cpu_model(args.config, threads=1)
            cpu1 = {"value": total, "unit": "s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        par = "single GPU" if world == 1 else (
            f"column-sharded x{world} (dual), NCCL all-reduce" if dw.route == "cols"
            else f"row-sharded x{world}, NCCL all-reduce" + (", intervals split" if gram_mode == 1 else ""))
        a_bytes = (dw.csr[0].numel() * 8 + dw.csr[1].numel() * 12) if dw.sparse else dw.n * dw.d * 8
        line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": dw.desc,
                           "l2": "inputs larger than L2 (operator %d MB > 126 MB L2)" % (a_bytes // 2 ** 20)
                           if a_bytes > 126 * 2 ** 20 else "operator L2-resident (no flush: the path re-reads it)",
                           "gram_mode": "gram-matrix" if gram_mode == 1 else "pass",
                           "parallelism": par, "phases_s": phases},
                "roofline": roofline, "hbm_passes": passes or None, "cpu_baseline": cpu,
                "cpu_baseline_1thread": cpu1, "e2e": e2e, "clocks": clk, "gpu_launches": int(launches)}
        if check is not None:
            line["check"] = {"max_rel_err_vs_oracle": check}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        run_reference(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
