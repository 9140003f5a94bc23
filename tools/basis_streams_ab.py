"""A/B of the two-stream basis recursion (option basis_streams 1 vs 2): path
time (CUDA events, device-resident data) and bitwise equality of x(lambda).

    python tools/basis_streams_ab.py [config] [reps]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    dw = workloads.device_workload(name)
    torch.cuda.synchronize()
    ctx = rp.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    arm = bench.Arm(rp, torch, ctx, dw, torch.device("cuda"))
    xs = {}
    for mode in (1, 2, 1, 2):
        ctx.set_option("basis_streams", mode)
        for _ in range(3):
            arm.step()
        ts, basis = [], []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(stream)
            tm = arm.step()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            basis.append(tm.basis_seconds * 1e3)
        xs[mode] = arm.x.clone()
        print(f"{name} basis_streams={mode}: path {statistics.median(ts):.3f} ms (min {min(ts):.3f}), "
              f"basis phase {statistics.median(basis):.3f} ms", flush=True)
    same = torch.equal(xs[1], xs[2])
    err = float((xs[1] - xs[2]).norm() / xs[1].norm())
    print(f"{name}: x(lambda) bitwise equal across modes: {same} (rel diff {err:.2e})")


if __name__ == "__main__":
    main()
