"""Run-to-run determinism of the path on one config: x(lambda) of repeated
calls compared bitwise, for several option sets.

    python tools/determinism_probe.py [config] [reps] [opt=val,...] ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    sets = sys.argv[3:] or ["default"]
    dw = workloads.device_workload(name)
    torch.cuda.synchronize()
    ref = None
    for label in sets:
        ctx = rp.Context(0)
        opts = {} if label == "default" else {k: int(v) for k, v in (kv.split("=") for kv in label.split(","))}
        for k, v in opts.items():
            ctx.set_option(k, v)
        arm = bench.Arm(rp, torch, ctx, dw, torch.device("cuda"))
        xs = []
        for _ in range(reps):
            arm.step()
            xs.append(arm.x.clone())
        if ref is None:
            ref = xs[0]
        diffs = [float((x - ref).norm() / ref.norm()) for x in xs]
        same = [bool(torch.equal(x, xs[0])) for x in xs]
        print(f"{name} [{label}]: bitwise equal to its first run: {same}; rel diff vs reference run: "
              + ", ".join(f"{d:.2e}" for d in diffs), flush=True)
        del arm, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
