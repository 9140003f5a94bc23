"""Fused Gram pass z = A^T (A W) on the C2 operator (65536 x 1024), W = 1..8:
device time (library CUDA events, median of 10) against the HBM roof, and
the result against torch (cuBLAS) in float64.

    RP_GRAM_DMMA_MIN=k python tools/gram_pass_bench.py [n] [d]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    hbm = 6549.1
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    g = torch.Generator(device="cuda").manual_seed(1)
    at = torch.randn(d, n, generator=g, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx = rp.Context(0)
    rp.set_dense_rows_device(ctx, n, 0, n, d, at.data_ptr(), n)
    only = int(os.environ.get("RP_GRAM_W_ONLY", "0"))
    for W in ([only] if only else range(1, 9)):
        w = torch.randn(W, d, generator=g, dtype=torch.float64, device="cuda")
        z = torch.empty(W, d, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):
            rp.gram_apply_raw(ctx, w.data_ptr(), W, z.data_ptr())
        ctx.set_option("profile", 1)
        ts = []
        for _ in range(10):
            rp.gram_apply_raw(ctx, w.data_ptr(), W, z.data_ptr())
            ts.append(rp.last_device_seconds(ctx))
        ctx.set_option("profile", 0)
        ref = (at @ (at.T @ w.T)).T
        err = float((z - ref).norm() / ref.norm())
        t = statistics.median(ts)
        gbs = 8.0 * n * d / t / 1e9
        print(json.dumps({"n": n, "d": d, "W": W, "dmma_min": os.environ.get("RP_GRAM_DMMA_MIN", "2"),
                          "us": round(t * 1e6, 1), "gbs": round(gbs, 1), "frac_hbm": round(gbs / hbm, 3),
                          "rel_err": err}), flush=True)


if __name__ == "__main__":
    main()
