"""Times the HBM-bound narrow passes (fused Gram z = A^T(A w), x = A^T y) on a
C2-shaped operator (65536 x 1024, column-major, 512 MB) with CUDA events, and
checks them against torch fp64.  Small enough to run under ncu.

usage: python tools/hbm_probe.py [reps]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n, d = 65536, 1024
    g = torch.Generator(device="cuda").manual_seed(0)
    at = torch.randn(d, n, generator=g, dtype=torch.float64, device="cuda")  # A column-major
    ctx = rp.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # events below bracket the library's launches
    ctx.check(rp.lib().rp_set_dense(ctx.handle, n, d, rp._P(at.data_ptr()), n, rp.RP_DEVICE))
    out = {}
    byts = 8.0 * n * d
    for name, k, fn in (("gram_fused_w1", 1, rp.gram_apply_raw), ("gram_fused_w2", 2, rp.gram_apply_raw),
                        ("gram_fused_w4", 4, rp.gram_apply_raw), ("gram_fused_w8", 8, rp.gram_apply_raw),
                        ("atv_w1", 1, rp.apply_transpose_raw), ("atv_w4", 4, rp.apply_transpose_raw)):
        rows = d if fn is rp.gram_apply_raw else n
        x = torch.randn(k, rows, generator=g, dtype=torch.float64, device="cuda")
        z = torch.empty(k, d, dtype=torch.float64, device="cuda")
        fn(ctx, x.data_ptr(), k, z.data_ptr())
        torch.cuda.synchronize()
        ref = (at @ (at.T @ x.T)).T if fn is rp.gram_apply_raw else (at @ x.T).T
        err = float((z - ref).norm() / ref.norm())
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn(ctx, x.data_ptr(), k, z.data_ptr())
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / reps * 1e-3  # per call, host round trip included
        ctx.set_option("profile", 1)
        dt = []
        for _ in range(reps):
            fn(ctx, x.data_ptr(), k, z.data_ptr())
            dt.append(rp.last_device_seconds(ctx))
        ctx.set_option("profile", 0)
        td = sorted(dt)[len(dt) // 2]  # device time of the pass (median)
        out[name] = {"us_call": round(t * 1e6, 1), "us_device": round(td * 1e6, 1),
                     "GBs_device": round(byts / td / 1e9, 1), "rel_err": err}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
