"""Device time of the fused Gram pass z = A^T (A w) and of A^T y on the C2 operator.

    python tools/colpass_probe.py
"""
import os
import statistics
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
    torch.cuda.synchronize()
    ctx = rp.Context(0)
    rp.set_dense_rows_device(ctx, n, 0, n, d, a_dev.data_ptr(), n)
    for name, fn, cols in (("gram_w1", rp.gram_apply_raw, 1), ("gram_w2", rp.gram_apply_raw, 2),
                           ("gram_w4", rp.gram_apply_raw, 4), ("atb_w1", rp.apply_transpose_raw, 1)):
        rows_in = d if fn is rp.gram_apply_raw else n
        xin = torch.randn(rows_in * cols, dtype=torch.float64, device="cuda")
        xout = torch.empty(d * cols, dtype=torch.float64, device="cuda")
        for _ in range(3):
            fn(ctx, xin.data_ptr(), cols, xout.data_ptr())
        ctx.set_option("profile", 1)
        ts = []
        for _ in range(15):
            fn(ctx, xin.data_ptr(), cols, xout.data_ptr())
            ts.append(rp.last_device_seconds(ctx))
        ctx.set_option("profile", 0)
        t = statistics.median(ts)
        print(f"{name}: {t*1e6:7.1f} us  {8.0*n*d/t/1e9:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
