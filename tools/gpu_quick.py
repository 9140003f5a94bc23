"""Quick GPU bring-up check of every building block against the oracle."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle import ridgepath_oracle as o  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def rel(a, b):
    return o.rel_error(a, b)


def step(name, fn):
    t0 = time.time()
    try:
        r = fn()
        print(f"[ok] {name}: {r}  ({time.time()-t0:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


ctx = rp.default_context()
g = np.load("tests/golden/ref_draws.npz")

step("u64", lambda: bool(np.array_equal(rp.draw_u64(0, 2048), g["u64_seed0"])))
step("u64 skip", lambda: bool(np.array_equal(rp.draw_u64(12345, 1024, skip=1_000_003), g["u64_seed12345_skip1000003"])))
step("uniform01", lambda: bool(np.array_equal(rp.draw_uniform01(0, 1024), g["uniform01_seed0"])))
step("sign", lambda: bool(np.array_equal(rp.draw_sign(3, 1024), g["sign_seed3"])))
step("uindex rej", lambda: bool(np.array_equal(rp.draw_uniform_index(3, (1 << 63) + 1, 512), g["uindex_seed3_bound2p63p1"])))
step("uindex", lambda: bool(np.array_equal(rp.draw_uniform_index(4, 1000, 512), g["uindex_seed4_bound1000"])))
step("normals match rate", lambda: float(np.mean(rp.draw_normals(0, 8192) == g["normals_seed0"])))
step("normals maxrel", lambda: float(np.max(np.abs(rp.draw_normals(0, 8192) - g["normals_seed0"]) / np.abs(g["normals_seed0"]))))
step("gauss window", lambda: float(np.mean(rp.gaussian_window(0, 512, 4096, 0, 2, 0, 4096) == g["c1_S_rows01"])))
step("gauss odd", lambda: float(np.mean(rp.gaussian_window(9, 7, 33, 0, 7, 0, 33) == g["gauss_m7_n33_seed9"])))
step("count draws", lambda: (lambda hs: bool(np.array_equal(hs[0][0], g["count_m8192_seed0_h"]) and np.array_equal(hs[1][0], g["count_m8192_seed0_sign"])))(rp.count_draws(rp.SketchSpec("countsketch", 8192, 4096, 1, 0))))
step("sjlt draws", lambda: (lambda hs: bool(np.array_equal(hs[0].reshape(-1), g["sjlt_m12_s3_n64_seed6_h"]) and np.array_equal(hs[1].reshape(-1), g["sjlt_m12_s3_n64_seed6_sign"])))(rp.count_draws(rp.SketchSpec("sjlt", 12, 64, 3, 6))))
step("srht draws", lambda: (lambda sr: bool(np.array_equal(np.packbits(sr[0] > 0), g["srht_n65536_m2048_seed0_signbits"]) and np.array_equal(sr[1], g["srht_n65536_m2048_seed0_rows"])))(rp.srht_draws(rp.SketchSpec("srht", 2048, 65536, 1, 0))))

rng = np.random.default_rng(0)
A = rng.standard_normal((300, 37))
X = rng.standard_normal((37, 5))
step("apply", lambda: rel(rp.apply(A, X), A @ X))
step("apply_t", lambda: rel(rp.apply_transpose(A, rng.standard_normal((300, 3))), None) if False else rel(rp.apply_transpose(A, A @ X), A.T @ (A @ X)))
step("gram", lambda: rel(rp.gram_apply(A, X), A.T @ (A @ X)))
Ab = rng.standard_normal((1000, 260))
Xb = rng.standard_normal((260, 130))
step("gram big", lambda: rel(rp.gram_apply(Ab, Xb), Ab.T @ (Ab @ Xb)))
csr = o.Csr.from_dense(np.where(rng.random((120, 37)) < 0.2, rng.standard_normal((120, 37)), 0.0))
C = rp.Csr(csr.rows, csr.cols, csr.offsets, csr.indices, csr.values)
step("csr apply", lambda: rel(rp.apply(C, X), csr.to_dense() @ X))
step("csr gram", lambda: rel(rp.gram_apply(C, X), o.gram_apply(csr, X)))

for kind, m, s in [("gaussian", 12, 1), ("countsketch", 12, 1), ("sjlt", 12, 3), ("srht", 12, 1), ("identity", 64, 1)]:
    Ad = o.random_dense(64, 9, 7)
    sp = o.SketchSpec(kind, m, 64, s, 4)
    ref = o.sketch_apply(sp, Ad)
    got = rp.sketch_apply(rp.SketchSpec(kind, m, 64, s, 4), Ad).product
    step(f"sketch {kind} dense", lambda: (rel(got, ref), bool(np.array_equal(got, ref))))

Acsr = o.Csr.from_dense(np.where(rng.random((64, 9)) < 0.3, rng.standard_normal((64, 9)), 0.0))
for kind, m, s in [("gaussian", 12, 1), ("countsketch", 12, 1), ("sjlt", 12, 3), ("srht", 12, 1), ("identity", 64, 1)]:
    sp = o.SketchSpec(kind, m, 64, s, 5)
    ref = o.sketch_apply(sp, Acsr)
    got = rp.sketch_apply(rp.SketchSpec(kind, m, 64, s, 5), rp.Csr(64, 9, Acsr.offsets, Acsr.indices, Acsr.values)).product
    step(f"sketch {kind} csr", lambda: (rel(got, ref), bool(np.array_equal(got, ref))))

# C2-shaped SRHT, bitwise
A2 = rng.standard_normal((65536, 8))
step("srht C2 shape bitwise", lambda: bool(np.array_equal(rp.sketch_apply(rp.SketchSpec("srht", 2048, 65536, 1, 0), A2).product, o.sketch_apply(o.SketchSpec("srht", 2048, 65536, 1, 0), A2))))

SA = rng.standard_normal((20, 9))
for lam in (0.5, 3.0):
    P = rp.Preconditioner.build(SA, lam)
    v = rng.standard_normal(9)
    step(f"precond tall {lam}", lambda: rel(P.apply(v), o.dense_preconditioner_oracle(SA, lam) @ v))
SW = rng.standard_normal((8, 20))
P = rp.Preconditioner.build(SW, 0.5)
v = rng.standard_normal(20)
step("precond wide", lambda: rel(P.apply(v), o.dense_preconditioner_oracle(SW, 0.5) @ v))
step("precond reshift", lambda: rel(P.reshift(3.7).apply(v), o.dense_preconditioner_oracle(SW, 3.7) @ v))

# scalar KAT ihs basis
a1 = np.array([[1.0]])
P1 = rp.Preconditioner.build(np.array([[1.0]]), 1.0)
step("scalar basis", lambda: [t[0, 0] for t in rp.ihs_basis(a1, np.ones(1), P1, 1.0, 2).terms])

# small path vs oracle
n, d = 400, 20
Ad = o.random_dense(n, d, 3)
b = o.fill_normals(5, n)
cfg = o.PathConfig(1e-2, 1e2, o.log_grid(1e-2, 1e2, 30), 1e-6, None)
spec = o.SketchSpec("gaussian", 60, n, 1, 11)
rho = o.RhoBounds.manual((1 + (d / 60) ** 0.5) ** 2, (1 - (d / 60) ** 0.5) ** 2)
ref = o.ihs_bin_path(Ad, b, cfg, spec, rho)
for mode in (0, 1):
    ctx.set_option("gram_mode", mode)
    got = rp.ihs_bin_path(Ad, b, rp.PathConfig(cfg.lambda_min, cfg.lambda_max, cfg.lambdas, 1e-6),
                          rp.SketchSpec("gaussian", 60, n, 1, 11), rp.RhoBounds.manual(rho.rho1, rho.rho2))
    step(f"path gaussian mode {mode}", lambda: max(rel(gp.solution[:, 0], rp_.solution[:, 0]) for gp, rp_ in zip(got.points, ref.points)))
ctx.set_option("gram_mode", -1)
# dual
nd, dd = 30, 80
Adu = o.random_dense(nd, dd, 8)
bd = o.fill_normals(9, nd)
cfgd = o.PathConfig(1.0, 50.0, o.log_grid(1.0, 50.0, 6), 1e-10, None)
refd = o.dual_path(Adu, bd, cfgd, o.SketchSpec("identity", dd, dd, 1, 0), o.RhoBounds.identity())
gotd = rp.dual_path(Adu, bd, rp.PathConfig(1.0, 50.0, cfgd.lambdas, 1e-10), rp.SketchSpec("identity", dd, dd, 1, 0), rp.RhoBounds.identity())
step("dual path", lambda: max(rel(gp.solution[:, 0], rp_.solution[:, 0]) for gp, rp_ in zip(gotd.points, refd.points)))
print("launches", rp.launch_count())
