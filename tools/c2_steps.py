"""Run K device-resident path steps of a bench workload (for ncu launch lists).

    python tools/c2_steps.py [config] [steps]
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
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = workloads.get(name)
    n, d = w.a.shape
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).cuda()
    ctx = rp.Context(0)
    for kv in filter(None, os.environ.get("RP_OPTS", "").split(",")):  # e.g. RP_OPTS=gram_overlap_tma=1
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    rp.set_dense_rows_device(ctx, n, 0, n, d, a_dev.data_ptr(), n)
    grid = w.lambdas(rp.log_grid)
    K = w.b.shape[1]
    x = torch.empty(len(grid) * d * K, dtype=torch.float64, device="cuda")
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    for _ in range(steps):
        tm = rp.path_raw(ctx, b_dev.data_ptr(), K, cfg, spec, rho, x.data_ptr(), rp.RP_DEVICE)
        print(f"path {tm.total_seconds*1e3:.2f} ms", {k: round(v * 1e3, 3) for k, v in tm.as_dict().items()
                                                      if k.endswith("_seconds")}, flush=True)


if __name__ == "__main__":
    main()
