"""Compare the C2 path under different stream/launch options against a
conservative run (no side stream, no high-priority sketch) -- a race probe.

    python tools/race_probe.py [opt=val ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    w = workloads.get("c2")
    n, d = w.a.shape
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).cuda()
    torch.cuda.synchronize()
    grid = w.lambdas(rp.log_grid)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)

    def run(opts, reps=3):
        ctx = rp.Context(0)
        for k, v in opts.items():
            ctx.set_option(k, v)
        rp.set_dense_rows_device(ctx, n, 0, n, d, a_dev.data_ptr(), n)
        xs = []
        for _ in range(reps):
            x = torch.empty(len(grid) * d, dtype=torch.float64, device="cuda")
            rp.path_raw(ctx, b_dev.data_ptr(), 1, cfg, spec, rho, x.data_ptr())
            xs.append(x.view(len(grid), d).cpu().numpy())
        return xs

    ref = run({"gram_overlap": 0}, 1)[0]
    for arg in sys.argv[1:] or ["default"]:
        opts = {}
        if arg != "default":
            for kv in arg.split(","):
                k, v = kv.split("=")
                opts[k] = int(v)
        for i, x in enumerate(run(opts)):
            err = np.max(np.linalg.norm(x - ref, axis=1) / np.linalg.norm(ref, axis=1))
            print(f"{arg:30s} rep {i}: max rel diff vs conservative {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
