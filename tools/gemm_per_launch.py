"""Per-launch table of the recursion's GEMMs of one path step: shape, tile,
seconds, TFLOP/s and the launch's binding floor max(flops / DGEMM peak,
operand bytes / HBM peak) -- from bench.py --dump-gemm joined with RP_GEMM_LOG.

    python tools/gemm_per_launch.py gemm_prof.json gemm.log [dgemm_peak_tflops] [hbm_gbs]
"""
import json
import sys


def main(prof_path, log_path, peak=35.4, hbm=6549.0):
    prof = json.load(open(prof_path))
    log = [ln.split() for ln in open(log_path) if ln.strip()]
    n = len(prof["seconds"])
    log = log[-n:]
    tot = {}
    print("   m     n     k batch split tile epi      us   TF/s  floor_us  frac")
    for sec, fl, by, g in zip(prof["seconds"], prof["flops"], prof["bytes"], log):
        m, nn, k, batch, split, tile, epi = (int(g[0]), int(g[1]), int(g[2]), int(g[4]), int(g[6]), int(g[8]),
                                             int(g[16]))
        floor = max(fl / (peak * 1e12), by / (hbm * 1e9))
        key = "P" if epi == 2 else ("G" if (k == m and batch == 1) else "other")
        t = tot.setdefault(key, [0.0, 0.0])
        t[0] += sec
        t[1] += floor
        if key != "other":
            print(f"{m:5d} {nn:5d} {k:5d} {batch:5d} {split:5d} {tile:4d} {epi:3d} {sec*1e6:7.1f} {fl/sec/1e12:6.2f} "
                  f"{floor*1e6:8.1f} {floor/sec:5.2f}")
    for key, (s, f) in tot.items():
        print(f"## {key}: {s*1e3:.3f} ms, floor {f*1e3:.3f} ms, frac {f/s:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *[float(x) for x in sys.argv[3:5]])
