import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2210_12212_b200 import ridgepath as rp
for (n, d, K) in ((64*148, 1024, 2), (8192, 1024, 4), (65536, 1024, 8), (65537, 1000, 2), (1000, 3000, 1)):
    g = torch.Generator(device="cuda").manual_seed(0)
    at = torch.randn(d, n, generator=g, dtype=torch.float64, device="cuda")
    ctx = rp.Context(0)
    ctx.check(rp.lib().rp_set_dense(ctx.handle, n, d, rp._P(at.data_ptr()), n, rp.RP_DEVICE))
    y = torch.randn(K, n, generator=g, dtype=torch.float64, device="cuda")
    x = torch.empty(K, d, dtype=torch.float64, device="cuda")
    rp.apply_transpose_raw(ctx, y.data_ptr(), K, x.data_ptr()); torch.cuda.synchronize()
    ref = (at @ y.T).T
    err = ((x - ref).abs() / ref.abs().max()).cpu().numpy()
    print("ATV", n, d, K, "max err per k", err.max(axis=1), "bad cols k0:", np.nonzero(err[0] > 1e-12)[0][:20], "k1:", np.nonzero(err[-1] > 1e-12)[0][:40])
    r = (x / ref).cpu().numpy()
    print("  ratio sample k0", r[0][:8], "k1", r[-1][:8])
