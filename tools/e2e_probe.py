"""e2e (host A in, host x out) timing of the bench workload for several
upload modes: synchronous RP_HOST and RP_HOST_STREAM at several chunk sizes.

    python tools/e2e_probe.py [config]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = workloads.get(name)
    n, d = w.a.shape
    K = w.b.shape[1]
    ctx = rp.Context(0)
    grid = w.lambdas(rp.log_grid)
    T = len(grid)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    a_host = torch.from_numpy(np.ascontiguousarray(w.a.T)).pin_memory()
    b_host = torch.from_numpy(np.ascontiguousarray(w.b.T)).pin_memory()
    x_host = torch.empty((T * K * d,), dtype=torch.float64).pin_memory()
    for mode, chunk in (("sync", 0), ("stream", 512 << 20), ("stream", 128 << 20), ("stream", 64 << 20),
                        ("stream", 32 << 20), ("stream", 16 << 20), ("sync", 0)):
        if chunk:
            ctx.set_option("upload_chunk_bytes", chunk)
        ts, tu, tp = [], [], []
        for it in range(6):
            t0 = time.perf_counter()
            rp.set_dense_rows_host(ctx, n, 0, n, d, a_host.data_ptr(), n, stream=(mode == "stream"))
            t1 = time.perf_counter()
            tm = rp.path_raw(ctx, b_host.data_ptr(), K, cfg, spec, rho, x_host.data_ptr(), rp.RP_HOST)
            t2 = time.perf_counter()
            if it >= 1:
                ts.append(t2 - t0)
                tu.append(t1 - t0)
                tp.append(tm.total_seconds)
        print(f"{mode:6s} chunk {chunk >> 20:4d} MiB: e2e {1e3*np.median(ts):7.2f} ms  (set {1e3*np.median(tu):6.2f} ms, "
              f"path device {1e3*np.median(tp):6.2f} ms, sketch {1e3*tm.sketch_seconds:6.2f} gram {1e3*tm.gram_seconds:5.2f})",
              flush=True)


if __name__ == "__main__":
    main()
