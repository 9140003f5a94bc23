"""Stress test for concurrency races: the C2 path many times under an option
set, every x(lambda) compared bitwise with one fully serialized run
(gram_overlap = 0).

    python tools/race_stress.py config reps "opt=v,..." ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def run_set(dw, label, reps, ref):
    ctx = rp.Context(0)
    if label != "default":
        for kv in label.split(","):
            k, v = kv.split("=")
            ctx.set_option(k, int(v))
    arm = bench.Arm(rp, torch, ctx, dw, torch.device("cuda"))
    bad = []
    for i in range(reps):
        arm.step()
        if ref is None:
            return arm.x.clone()
        if not torch.equal(arm.x, ref):
            bad.append((i, float((arm.x - ref).norm() / ref.norm())))
    print(f"{dw.name} [{label}]: {len(bad)}/{reps} runs differ from the serialized reference "
          + (str([f'{i}:{e:.1e}' for i, e in bad[:8]]) if bad else ""), flush=True)
    return None


def main():
    name, reps = sys.argv[1], int(sys.argv[2])
    dw = workloads.device_workload(name)
    torch.cuda.synchronize()
    ref = run_set(dw, "gram_overlap=0", 1, None)
    for label in sys.argv[3:]:
        run_set(dw, label, reps, ref)


if __name__ == "__main__":
    main()
