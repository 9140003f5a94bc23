"""C4 (sparse CSR, CountSketch, Woodbury) path timing at a chosen row scale.

    python tools/c4_profile.py [row_scale] [reps]

row_scale shrinks n only (d = 65536 and m = 8192 stay at BASELINE size), so
the preconditioner shapes are the real ones and the Gram passes scale with
nnz.  Prints the path's phase timings; run under ncu for the launch list.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    t0 = time.time()
    w = workloads.c4()
    n = int(w.meta["n"] * scale)
    off = w.a["offsets"][: n + 1]
    nnz = int(off[-1])
    a = rp.Csr(n, w.a["cols"], off, w.a["indices"][:nnz], w.a["values"][:nnz])
    b = w.b[:n]
    print(f"data {time.time()-t0:.1f}s  n={n} d={w.meta['d']} nnz={nnz}", flush=True)
    ctx = rp.Context(0)
    for kv in filter(None, os.environ.get("RP_OPTS", "").split(",")):  # e.g. RP_OPTS=gram_overlap_tma=1
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    grid = rp.log_grid(w.lambda_min, w.lambda_max, w.T)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon)
    spec = rp.SketchSpec("countsketch", w.sketch["m"], n, 1, 0)
    rho = rp.RhoBounds.manual(*w.rho)
    for _ in range(reps):
        path = rp.ihs_bin_path(a, b, cfg, spec, rho, ctx=ctx)
        t = path.timings
        print("path %.1f ms: " % (t["total_seconds"] * 1e3)
              + " ".join(f"{k[:-8]} {v*1e3:.1f}" for k, v in t.items() if k.endswith("_seconds")), flush=True)
    x = np.stack([p.solution[:, 0] for p in path.points])
    print("finite", bool(np.isfinite(x).all()), "norm", float(np.linalg.norm(x)))


if __name__ == "__main__":
    main()
