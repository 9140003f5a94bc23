"""Two contexts running the C2 path concurrently from two host threads (each
on its own stream) vs the sequential result: a probe for cross-stream
interference in the kernels.

    python tools/concurrency_probe.py [reps]
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    w = workloads.get("c2")
    n, d = w.a.shape
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).cuda()
    torch.cuda.synchronize()
    grid = w.lambdas(rp.log_grid)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    ctxs = [rp.Context(0), rp.Context(0)]
    xs = [torch.empty(len(grid) * d, dtype=torch.float64, device="cuda") for _ in ctxs]
    for c in ctxs:
        rp.set_dense_rows_device(c, n, 0, n, d, a_dev.data_ptr(), n)

    def run(i):
        rp.path_raw(ctxs[i], b_dev.data_ptr(), 1, cfg, spec, rho, xs[i].data_ptr())

    run(0)
    ref = xs[0].cpu().numpy().copy()
    for r in range(reps):
        ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for i in range(2):
            x = xs[i].cpu().numpy().reshape(len(grid), d)
            err = np.max(np.linalg.norm(x - ref.reshape(len(grid), d), axis=1) / np.linalg.norm(ref.reshape(len(grid), d), axis=1))
            print(f"rep {r} ctx {i}: max rel diff vs sequential {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
