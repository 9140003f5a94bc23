"""A/B of context options on one config's path (CUDA events around each call,
device-resident data), with x(lambda) compared to the first option set.

    python tools/option_ab.py config reps "opt=v,opt=v" "opt=v" ...   ("default" = no options)
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
    name, reps = sys.argv[1], int(sys.argv[2])
    dw = workloads.device_workload(name)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ref = None
    for rnd in range(2):
        for label in sys.argv[3:]:
            ctx = rp.Context(0)
            ctx.set_stream(stream.cuda_stream)
            if label != "default":
                for kv in label.split(","):
                    k, v = kv.split("=")
                    ctx.set_option(k, int(v))
            arm = bench.Arm(rp, torch, ctx, dw, torch.device("cuda"))
            for _ in range(3):
                arm.step()
            ts, ph = [], []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(stream)
                tm = arm.step()
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
                ph.append((tm.sketch_seconds, tm.precond_seconds, tm.basis_seconds))
            if ref is None:
                ref = arm.x.clone()
            err = float((arm.x - ref).norm() / ref.norm())
            med = [statistics.median(p[i] for p in ph) * 1e3 for i in range(3)]
            print(f"{name} [{label}] round {rnd}: path {statistics.median(ts):.3f} ms (min {min(ts):.3f}); sketch "
                  f"{med[0]:.3f} precond {med[1]:.3f} basis {med[2]:.3f}; x vs first set {err:.1e}", flush=True)
            del arm, ctx


if __name__ == "__main__":
    main()
