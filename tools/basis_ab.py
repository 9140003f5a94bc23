"""A/B of recursion variants on the C2 bench workload: path time with the
preconditioner update fused into the GEMM epilogue vs split GEMM + kernel."""
import json
import subprocess
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    w = workloads.get("c2")
    n, d = w.a.shape
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).cuda()
    ctx = rp.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    rp.set_dense_rows_device(ctx, n, 0, n, d, a_dev.data_ptr(), n)
    grid = w.lambdas(rp.log_grid)
    x = torch.empty(len(grid) * d, dtype=torch.float64, device="cuda")
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    out = {}
    for opt in sys.argv[1:]:
        key, val = opt.split("=")
        ctx.set_option(key, int(val))
        ts = []
        for _ in range(5):
            tm = rp.path_raw(ctx, b_dev.data_ptr(), 1, cfg, spec, rho, x.data_ptr())
            ts.append((tm.total_seconds, tm.basis_seconds, tm.precond_seconds))
        ts = sorted(ts)[1:4]
        out[opt] = {"total_ms": round(1e3 * np.mean([t[0] for t in ts]), 3),
                    "basis_ms": round(1e3 * np.mean([t[1] for t in ts]), 3),
                    "precond_ms": round(1e3 * np.mean([t[2] for t in ts]), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
