"""Which set-up product goes wrong under stream priorities?  Runs the C2 path
conservatively (no side stream) and then with the given options, dumping the
sketch SA, the linear term c, the Gram matrix G and the first preconditioner
inverse (RP_DUMP_DIR) of every run, and reports bitwise mismatches per object
plus the x(lambda) error.

    python tools/race_hunt.py [reps] [opt=val,...]
"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2210_12212_b200 import ridgepath as rp  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    opts = {}
    if len(sys.argv) > 2 and sys.argv[2] != "default":
        for kv in sys.argv[2].split(","):
            k, v = kv.split("=")
            opts[k] = int(v)
    w = workloads.get("c2")
    n, d = w.a.shape
    a_dev = torch.from_numpy(np.ascontiguousarray(w.a.T)).cuda()
    b_dev = torch.from_numpy(np.ascontiguousarray(w.b.T)).cuda()
    torch.cuda.synchronize()
    grid = w.lambdas(rp.log_grid)
    cfg = rp.PathConfig(w.lambda_min, w.lambda_max, grid, w.epsilon, None)
    spec = rp.SketchSpec(w.sketch["kind"], w.sketch["m"], w.sketch["n"], w.sketch["s"], w.sketch["seed"])
    rho = rp.RhoBounds.manual(*w.rho)
    tmp = tempfile.mkdtemp()

    def run(o, tag):
        ctx = rp.Context(0)
        for k, v in o.items():
            ctx.set_option(k, v)
        rp.set_dense_rows_device(ctx, n, 0, n, d, a_dev.data_ptr(), n)
        out = os.path.join(tmp, tag)
        os.makedirs(out, exist_ok=True)
        os.environ["RP_DUMP_DIR"] = out
        x = torch.empty(len(grid) * d, dtype=torch.float64, device="cuda")
        rp.path_raw(ctx, b_dev.data_ptr(), 1, cfg, spec, rho, x.data_ptr())
        del os.environ["RP_DUMP_DIR"]
        objs = {}
        for name in ("sa", "c", "gram", "inv0"):
            p = os.path.join(out, name + ".bin")
            if os.path.exists(p):
                objs[name] = np.fromfile(p, dtype=np.float64)
        return x.view(len(grid), d).cpu().numpy(), objs

    ref_x, ref_o = run({"gram_overlap": 0}, "ref")
    label = ",".join(f"{k}={v}" for k, v in opts.items()) or "default"
    env = " ".join(f"{k}={os.environ[k]}" for k in ("RP_LEAK_ALLOC", "RP_GEMM_TMA", "RP_GEMM_PDL",
                                                       "CUDA_MODULE_LOADING", "RP_FACTOR_PRIORITIES")
                   if k in os.environ)
    for i in range(reps):
        x, o = run(opts, f"rep{i}")
        err = np.max(np.linalg.norm(x - ref_x, axis=1) / np.linalg.norm(ref_x, axis=1))
        parts = []
        for name, v in ref_o.items():
            g = o.get(name)
            if g is None:
                parts.append(f"{name}=absent")
                continue
            bad = np.count_nonzero(g.view(np.uint64) != v.view(np.uint64))
            rel = np.max(np.abs(g - v)) / max(np.max(np.abs(v)), 1e-300)
            parts.append(f"{name}: {bad} words differ (max rel {rel:.1e})")
            if name == "gram" and bad:
                dd = int(round(np.sqrt(v.size)))
                m = (g.view(np.uint64) != v.view(np.uint64)).reshape(dd, dd).T  # [row, col]
                rows, cols = np.nonzero(m)
                low = rows >= cols
                tiles = {}
                for r, c in zip(rows[low], cols[low]):
                    tiles[(r // 64, c // 32)] = tiles.get((r // 64, c // 32), 0) + 1
                hist = np.bincount(np.minimum(np.array(list(tiles.values())), 2048) // 256)
                t0 = sorted(tiles)[:4]
                parts.append(f"gram lower mismatches in {len(tiles)} 64x32 tiles, per-tile count/256 hist {hist.tolist()}, "
                             f"first tiles {t0}, rows {rows.min()}..{rows.max()} cols {cols.min()}..{cols.max()}")
                dv = (g - v).reshape(dd, dd).T
                r0, c0 = rows[low][0], cols[low][0]
                parts.append(f"example G[{r0},{c0}] ref {v.reshape(dd, dd).T[r0, c0]:.6e} got {dv[r0, c0] + v.reshape(dd, dd).T[r0, c0]:.6e}")
        print(f"[{label} {env}] rep {i}: x err {err:.3e}; " + "; ".join(parts), flush=True)


if __name__ == "__main__":
    main()
