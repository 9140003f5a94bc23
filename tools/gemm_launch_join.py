"""Join an ncu launch list (gpu__time_duration per launch, in launch order)
with the library's RP_GEMM_LOG (one line per dgemm call: shape, batch, split,
tile) and report time / TF/s per GEMM class.

    python tools/gemm_launch_join.py launches.csv gemm.log [steps]
"""
import collections
import csv
import re
import sys


def main(csv_path, log_path, steps=1):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    launches = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            try:
                launches.append((r[ki], float(r[vi].replace(",", ""))))
            except ValueError:
                pass
    gemms = [ln.split() for ln in open(log_path) if ln.strip()]
    # dgemm kernels in launch order, paired with the log lines in call order
    gk = [(n, t) for n, t in launches if "dgemm" in n and "splitk" not in n]
    reduce_t = [t for n, t in launches if "splitk_reduce" in n]
    print(f"{len(gk)} dgemm launches, {len(gemms)} logged calls, {len(reduce_t)} split-K reductions "
          f"({sum(reduce_t) / 1e3 / steps:.3f} ms/step)")
    n = min(len(gk), len(gemms))
    cls = collections.defaultdict(lambda: [0, 0.0, 0.0])
    off = len(gk) - n  # align on the last calls (the profiled steps)
    for (name, t), g in zip(gk[off:], gemms[len(gemms) - n:]):
        m, nn, k = int(g[0]), int(g[1]), int(g[2])
        batch, split, tile, epi = int(g[4]), int(g[6]), int(g[8]), int(g[16])
        fl = 2.0 * m * nn * k * batch
        key = f"m{m} k{k} batch{batch} epi{epi} n{'<=64' if nn <= 64 else '>64'}"
        c = cls[key]
        c[0] += 1
        c[1] += t
        c[2] += fl
    tot = sum(v[1] for v in cls.values())
    for key, (cnt, t, fl) in sorted(cls.items(), key=lambda kv: -kv[1][1]):
        print(f"{t / 1e3 / steps:8.3f} ms/step {100 * t / tot:5.1f}%  n={cnt // steps:4d}  "
              f"{fl / (t * 1e-9) / 1e12:6.2f} TF/s  {key}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
