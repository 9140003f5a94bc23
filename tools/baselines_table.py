"""In-framework solver comparison on one BASELINE config (the paper's Table 1
shape): IHS-BIN path vs the reference's baselines (direct, warm IHS, warm CG),
all on the device, same data, same grid.

    python tools/baselines_table.py [config] [T]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else None
    w = workloads.get(name)
    ctx = rp.Context(0)
    grid = w.lambdas(rp.log_grid)
    if T:
        grid = rp.log_grid(w.lambda_min, w.lambda_max, T)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    sk = w.sketch
    spec = rp.SketchSpec(sk["kind"], sk["m"], sk["n"], sk["s"], sk["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    b = w.b[:, 0]
    ctx.set_operator(w.a)
    rows = {}
    ref = None
    for solver in ("ihs-bin", "direct", "svd", "warm-ihs", "warm-cg"):
        t0 = time.perf_counter()
        if solver == "ihs-bin":
            r = rp.ihs_bin_path(w.a, b, cfg, spec, rho, ctx=ctx)
        elif solver == "direct":
            r = rp.direct_path(w.a, b, cfg, ctx=ctx)
        elif solver == "svd":
            r = rp.svd_path(w.a, b, cfg, ctx=ctx)
        elif solver == "warm-ihs":
            r = rp.warm_ihs_path(w.a, b, cfg, spec, rho, ctx=ctx)
        else:
            r = rp.warm_cg_path(w.a, b, cfg, ctx=ctx)
        wall = time.perf_counter() - t0
        X = np.stack([p.solution[:, 0] for p in r.points], axis=1)
        if ref is None and solver == "direct":
            ref = X
        rows[solver] = dict(total_seconds=r.total_seconds, wall_seconds=wall,
                            iterations=int(sum(p.iterations for p in r.points)), X=X)
        print(f"{solver:9s} total {r.total_seconds:9.4f} s  wall {wall:9.4f} s  "
              f"iterations {rows[solver]['iterations']}", flush=True)
    out = {}
    for k, v in rows.items():
        err = float(np.max(np.linalg.norm(v["X"] - ref, axis=0) / np.linalg.norm(ref, axis=0)))
        out[k] = dict(total_seconds=v["total_seconds"], wall_seconds=v["wall_seconds"], iterations=v["iterations"],
                      max_rel_err_vs_direct=err)
        print(f"{k:9s} max rel err vs direct {err:.3e}")
    print(json.dumps(dict(config=name, T=len(grid), solvers=out)))


if __name__ == "__main__":
    main()
