"""Per-class GEMM efficiency of one path step from the library's own
profile (bench.py --dump-gemm: CUDA-event seconds, flops, operand bytes per
launch, GEMMs serialized on one stream) joined with RP_GEMM_LOG (shapes).

    python tools/gemm_profile_classes.py gemm_prof.json gemm.log [dgemm_peak_tflops] [hbm_gbs]
"""
import collections
import json
import sys


def classify(g):
    m, n, k, batch, split, tile, epi = (int(g[0]), int(g[1]), int(g[2]), int(g[4]), int(g[6]), int(g[8]),
                                        int(g[16]))
    lower = int(g[18])
    if lower:
        return f"SYRK m{m} k{k} batch{batch}"
    if epi == 2:
        return "recursion P GEMM (batched, update epilogue)"
    if epi == 1:
        return "recursion Gram GEMM (fused argument epilogue)"
    if m == n and batch > 1:
        return f"factor m{m} k{k} batch{batch}"
    if k == m and batch == 1 and n > 0:
        return f"m{m} k{k} n-varying split{split} (recursion Gram GEMM, partials)"
    return f"m{m} k{k} batch{batch}"


def main(prof_path, log_path, peak=35.4, hbm=6549.0):
    prof = json.load(open(prof_path))
    log = [ln.split() for ln in open(log_path) if ln.strip()]
    n = len(prof["seconds"])
    log = log[-n:]
    cls = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for sec, fl, by, g in zip(prof["seconds"], prof["flops"], prof["bytes"], log):
        c = cls[classify(g)]
        c[0] += 1
        c[1] += sec
        c[2] += fl
        c[3] += max(fl / (peak * 1e12), by / (hbm * 1e9))
    tot = sum(v[1] for v in cls.values())
    print(f"{n} GEMM launches, {tot * 1e3:.3f} ms of GEMM time in one step (serialized)")
    print(f"{'ms':>8} {'share':>6} {'n':>4} {'TF/s':>6} {'frac':>5} {'binding':>7}  class")
    for key, (cnt, sec, fl, bound) in sorted(cls.items(), key=lambda kv: -kv[1][1]):
        print(f"{sec * 1e3:8.3f} {100 * sec / tot:5.1f}% {cnt:4d} {fl / sec / 1e12:6.2f} {fl / sec / 1e12 / peak:5.2f} "
              f"{bound / sec:7.2f}  {key}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], float(a[3]) if len(a) > 3 else 35.4, float(a[4]) if len(a) > 4 else 6549.0)
