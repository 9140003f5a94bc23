#!/usr/bin/env python
"""bench.py -- IHS-BIN ridge-path time on BASELINE config C2, 1..8 B200.

One "step" = one full ridge path (sketch + factor + every interval basis + all
T compositions) over the synthetic C2 workload (65536 x 1024 dense,
A = U diag(0.99^j) V^T, SRHT m = 2048, T = 1000 lambdas in [1e-4, 1e3]), with
A, b and x resident in HBM (`value`).  `e2e` repeats the step through the
public API with host buffers (pinned A and b copied in, x copied out).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Under torchrun each rank drives one GPU (row-sharded A, NCCL all-reduce of
the sketch / Gram matrix / linear term, intervals split across ranks); the
time is the max over ranks.  `--impl reference` times the CPU restatement of
the reference (oracle/, the reference itself needs Eigen which this image
lacks) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload_desc(w):
    m = w.meta
    return (f"{w.name}: {m['n']}x{m['d']} dense, {w.sketch['kind']} m={w.sketch['m']}, T={w.T} log-spaced "
            f"[{w.lambda_min:g},{w.lambda_max:g}], eps={w.epsilon:g}, L=auto, rho=({w.rho[0]:.4g},{w.rho[1]:.4g})")


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
# CPU baseline: the oracle (CPU restatement of the reference) on a bounded sample
# ---------------------------------------------------------------------------


def cpu_sample(w, interval_subset=(0,)):
    """Times the reference algorithm on the host: full sketch + SVD + plan + the
    linear term, then `interval_subset` interval bases and their compositions;
    extrapolates t = t_setup + L * t_interval + T * t_compose (each interval is
    independent in the reference, path_solver.cpp:168-186)."""
    from oracle import ridgepath_oracle as o

    a = w.a
    spec = o.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    grid = w.lambdas(o.log_grid)
    cfg = o.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    rho = o.RhoBounds.manual(*w.rho)
    t0 = time.perf_counter()
    c = o.apply_transpose(a, w.b)
    sa = o.sketch_apply(spec, a)
    svd = o.thin_svd(sa)
    plans = o.plan_intervals(cfg, rho, None)
    pre = o.Preconditioner.build_from_svd(svd, sa.shape[0], sa.shape[1], plans[0].params.lambda0)
    t_setup = time.perf_counter() - t0
    t_int, t_comp, n_comp = 0.0, 0.0, 0
    for idx in interval_subset:
        plan = plans[idx]
        t1 = time.perf_counter()
        p = pre.reshift(plan.params.lambda0)
        basis = o.build_interval_basis_matrix(a, c, p, plan)
        t_int += time.perf_counter() - t1
        for lam in plan.grid:
            t2 = time.perf_counter()
            o.compose_horner(basis, basis.tau * lam)
            t_comp += time.perf_counter() - t2
            n_comp += 1
    L = len(plans)
    per_int = t_int / len(interval_subset)
    per_comp = t_comp / max(n_comp, 1)
    total = t_setup + L * per_int + len(grid) * per_comp
    try:
        from threadpoolctl import threadpool_info

        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count() or 1
    sample = (f"full sketch+SVD+plan+A^T b ({t_setup:.2f}s) + {len(interval_subset)} of {L} interval bases "
              f"({per_int:.2f}s each) + {n_comp} composes; extrapolated to {L} intervals and T={len(grid)}")
    return total, cores, sample


def run_reference(args, w):
    vals = []
    for i in range(args.warmup + args.steps):
        total, cores, sample = cpu_sample(w)
        if i >= args.warmup:
            vals.append(total)
    v = statistics.mean(vals)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_desc(w), "parallelism": "host CPU (numpy/OpenBLAS + C oracle)"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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


def run_ours(args, w):
    import torch
    import torch.distributed as dist

    from paper_2210_12212_b200 import ridgepath as rp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, d = w.meta["n"], w.meta["d"]
    K = w.b.shape[1]
    # A (column-major) and b on the device; every rank holds the same data.
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).to(dev)  # (d, n) row-major == A column-major
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).to(dev)  # (K, n) == b column-major
    r0 = (rank * n) // world
    r1 = ((rank + 1) * n) // world
    nl = r1 - r0
    b_loc = b_dev[:, r0:r1].contiguous()  # (K, nl) == b_local column-major
    grid = w.lambdas(rp.log_grid)
    T = len(grid)
    x_dev = torch.empty((T * K * d,), dtype=torch.float64, device=dev)
    ctx = rp.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [rp.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        rp.comm_init(ctx, rank, world, uid[0])
    rp.set_dense_rows_device(ctx, n, r0, nl, d, a_dev.data_ptr() + 8 * r0, n)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)

    def step():
        return rp.path_raw(ctx, b_loc.data_ptr(), K, cfg, spec, rho, x_dev.data_ptr(), rp.RP_DEVICE)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    barrier()
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
        tms.append(step())
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    launches = rp.launch_count() - launches0
    clk = clocks.stop()
    step_s = e0.elapsed_time(e1) * 1e-3 / args.steps
    t = torch.tensor([step_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = float(t.item())
    phases = {k: statistics.mean(getattr(tm, k) for tm in tms)
              for k in ("sketch_seconds", "linear_seconds", "gram_seconds", "precond_seconds", "basis_seconds",
                        "eval_seconds", "total_seconds")}
    if os.environ.get("BENCH_VERBOSE"):
        for tm in tms:
            print(json.dumps(tm.as_dict()), file=sys.stderr)
    gram_mode = tms[-1].gram_mode

    # Roofline of the dominant kernel family (FP64 DMMA GEMM): the same steps
    # again with every GEMM bracketed by CUDA events on the step's stream.
    # (profiled steps keep every GEMM on one stream, so each launch is timed
    # alone: the side-stream Gram overlap of the timed steps is switched off)
    ctx.set_option("profile", 1)
    ctx.set_option("gram_overlap", 0)
    prof = [step() for _ in range(max(1, min(args.steps, 3)))]
    ctx.set_option("gram_overlap", 1)
    ctx.set_option("profile", 0)
    l_sec, l_flops, l_bytes = rp.last_gemm_profile(ctx)  # per launch, last profiled step
    g_s = sum(p.gemm_seconds for p in prof)
    g_f = sum(p.gemm_flops for p in prof)
    g_calls = sum(p.gemm_calls for p in prof)
    tot_s = sum(p.total_seconds for p in prof)
    peak = measure_dgemm_peak(torch)
    achieved = g_f / g_s / 1e12 if g_s > 0 else 0.0
    # DRAM traffic per launch of the representative top GEMM (the Gram product
    # at the last generation, 1024 x 2016 x 1024) from the committed ncu
    # --set full capture, beside that launch's algorithmic operand bytes.
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_gemm_tma.json")) as f:
            rec = json.load(f)[0]
        mb = float(rec["dram__bytes_read.sum"].split()[0]) + float(rec["dram__bytes_write.sum"].split()[0])
        traffic = mb * 1e6
        traffic_note = ("bytes per launch of %s (ncu, profiles/r01_ncu_gemm_tma.json); algorithmic "
                        "operand bytes of that launch 8*(1024*1024 + 1024*2016 + 4*1024*2016) = 90 MB "
                        "(split-K partials included)" % rec["kernel"][:60])
    except Exception:
        pass
    # Per-launch binding roof: the recursion's early generations are skinny
    # (N = g+1 columns) and HBM-bound, the late ones DMMA-bound, so each
    # launch is held to max(flops / tensor peak, bytes / HBM peak).
    hbm_peak = 6449.1
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f).get("hbm_gbs", hbm_peak))
    except Exception:
        pass
    bound_t = sum(max(fl / (peak * 1e12), by / (hbm_peak * 1e9)) for fl, by in zip(l_flops, l_bytes)) if peak else 0.0
    n_hbm = sum(1 for fl, by in zip(l_flops, l_bytes) if peak and by / (hbm_peak * 1e9) > fl / (peak * 1e12))
    binding = {"frac": bound_t / float(sum(l_sec)) if len(l_sec) else None, "launches": int(len(l_sec)),
               "hbm_bound_launches": int(n_hbm), "hbm_peak_gbs": hbm_peak,
               "note": "sum over the GEMM launches of one step of max(flops/tensor peak, operand bytes/HBM peak) "
                       "divided by their summed device time"}
    roofline = {"bound": "tensor", "kernel": "dgemm_tma_kernel / dgemm_kernel (FP64 DMMA m8n8k4, TMA-fed; all GEMMs of the path)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                "traffic": traffic, "traffic_note": traffic_note, "share_of_step": g_s / tot_s if tot_s else None,
                "gemm_launches_per_step": g_calls / len(prof),
                "gemm_flops_per_step": g_f / len(prof),
                "binding_roof": binding,
                "peak_source": "cuBLAS DGEMM 8192^3 (torch.matmul fp64) measured in this run; "
                               "MEASURED_PEAKS.json has no FP64 figure; DMMA issue peak measured 37.1 TFLOP/s "
                               "(profiles/fp64_peaks_r01.txt)"}

    # HBM-bound single passes over A (north_star: the fused Gram-matvec pass
    # A^T (A w) against the HBM roofline), timed with CUDA events on the stream.
    passes = {}
    if world == 1:
        hbm = 6449.1
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                hbm = float(json.load(f).get("hbm_gbs", hbm))
        except Exception:
            pass
        for name, fn, wcols in (("gram_fused_w1", rp.gram_apply_raw, 1), ("gram_fused_w4", rp.gram_apply_raw, 4),
                                ("atb_w1", rp.apply_transpose_raw, 1)):
            rows_in = d if fn is rp.gram_apply_raw else nl
            xin = torch.randn(rows_in * wcols, dtype=torch.float64, device=dev)
            xout = torch.empty(d * wcols, dtype=torch.float64, device=dev)
            for _ in range(2):
                fn(ctx, xin.data_ptr(), wcols, xout.data_ptr())
            torch.cuda.synchronize(dev)
            reps = 10
            # device time of the pass itself (events recorded by the library
            # around its kernels on the call's stream; each C-ABI call
            # synchronizes, so a host-side bracket would add the round trip)
            ctx.set_option("profile", 1)
            dev_t = []
            for _ in range(reps):
                fn(ctx, xin.data_ptr(), wcols, xout.data_ptr())
                dev_t.append(rp.last_device_seconds(ctx))
            ctx.set_option("profile", 0)
            t = statistics.median(dev_t)
            byts = 8.0 * nl * d
            passes[name] = {"seconds": t, "algorithmic_bytes": byts, "achieved_gbs": byts / t / 1e9,
                            "frac_hbm": byts / t / 1e9 / hbm, "timing": "median of 10 calls, CUDA events"}
            if name == "gram_fused_w4":
                passes[name]["note"] = ("4 columns: 8 FP64 FMAs + 2 shared-memory reads per element of A on 17 "
                                        "warps per SM; issue-bound, not HBM-bound (ncu: profiles/r01_ncu_colpass.json)")

    # e2e through the public API with host buffers: pinned A and b copied in,
    # x copied out, every step.
    e2e = None
    if not args.no_e2e:
        a_host = torch.from_numpy(np.ascontiguousarray(w.a.T)).pin_memory()
        b_host = torch.from_numpy(np.ascontiguousarray(b_loc.cpu().numpy())).pin_memory()
        x_host = torch.empty((T * K * d,), dtype=torch.float64).pin_memory()

        def e2e_step():
            rp.set_dense_rows_host(ctx, n, r0, nl, d, a_host.data_ptr() + 8 * r0, n, stream=True)
            rp.path_raw(ctx, b_host.data_ptr(), K, cfg, spec, rho, x_host.data_ptr(), rp.RP_HOST)

        e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(te.item()), "unit": "s", "h2d_bytes_per_step": int(nl * d * 8 + nl * K * 8),
               "d2h_bytes_per_step": int(T * K * d * 8)}
        # restore the device operator
        rp.set_dense_rows_device(ctx, n, r0, nl, d, a_dev.data_ptr() + 8 * r0, n)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        total, cores, sample = cpu_sample(w)
        cpu = {"value": total, "unit": "s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_desc(w),
                           "l2": "inputs larger than L2 (A = %d MB > 126 MB L2)" % (n * d * 8 // 2**20),
                           "gram_mode": "gram-matrix" if gram_mode == 1 else "pass",
                           "parallelism": f"row-sharded x{world}, NCCL all-reduce, intervals split" if world > 1
                           else "single GPU",
                           "phases_s": phases},
                "roofline": roofline, "hbm_passes": passes or None, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk,
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        w = workloads.get(args.config)
        run_reference(args, w)
        return
    w = workloads.get(args.config)
    run_ours(args, w)


if __name__ == "__main__":
    main()
