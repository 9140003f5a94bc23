"""Regenerate tests/golden/ref_draws.npz from the REFERENCE's own rng.hpp.

Run in the build container (needs /root/reference for `make -C oracle ref`):
    python tests/golden/make_golden.py
The library oracle/_ref/libref_rng.so is compiled from
/root/reference/proj/core/include/ridgepath/rng.hpp by oracle/Makefile; the
draw loops in oracle/ref_rng_harness.cpp restate sketch.cpp's consumption
order.  The fixtures pin both oracle/rp_oracle.c (CPU tests) and the device
draw kernels (GPU tests) without needing /root/reference at run time.
"""
import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "libref_rng.so")


def lib():
    if not os.path.exists(REF):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    L = ctypes.CDLL(REF)
    P, u64, i64, dbl, cint = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    L.ref_fill_u64.argtypes = [u64, u64, i64, P]
    L.ref_fill_uniform01.argtypes = [u64, i64, P]
    L.ref_fill_uniform_index.argtypes = [u64, u64, i64, P]
    L.ref_fill_sign.argtypes = [u64, i64, P]
    L.ref_fill_normals.argtypes = [u64, i64, dbl, P]
    L.ref_count_draws.argtypes = [u64, i64, i64, cint, dbl, P, P]
    L.ref_srht_draws.argtypes = [u64, i64, i64, P, P]
    return L


def p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def main():
    L = lib()
    out = {}
    u = np.empty(2048, np.uint64); L.ref_fill_u64(0, 0, 2048, p(u)); out["u64_seed0"] = u
    u = np.empty(1024, np.uint64); L.ref_fill_u64(12345, 1_000_003, 1024, p(u)); out["u64_seed12345_skip1000003"] = u
    u = np.empty(1, np.uint64); L.ref_fill_u64(5489, 9999, 1, p(u)); out["u64_default_10000th"] = u
    f = np.empty(1024, np.float64); L.ref_fill_uniform01(0, 1024, p(f)); out["uniform01_seed0"] = f
    f = np.empty(1024, np.float64); L.ref_fill_sign(3, 1024, p(f)); out["sign_seed3"] = f
    b = (1 << 63) + 1  # rejection probability ~1/2 per draw
    u = np.empty(512, np.uint64); L.ref_fill_uniform_index(3, b, 512, p(u)); out["uindex_seed3_bound2p63p1"] = u
    u = np.empty(512, np.uint64); L.ref_fill_uniform_index(4, 1000, 512, p(u)); out["uindex_seed4_bound1000"] = u
    f = np.empty(8192, np.float64); L.ref_fill_normals(0, 8192, 1.0, p(f)); out["normals_seed0"] = f
    # C1 Gaussian sketch (m=512, n=4096, seed 0): rows 0-1 and row 511, entry = scale * normal
    m, n = 512, 4096
    full = np.empty(m * n, np.float64); L.ref_fill_normals(0, m * n, 1.0 / np.sqrt(m), p(full))
    S = full.reshape(m, n)
    out["c1_S_rows01"] = S[:2].copy()
    out["c1_S_row511"] = S[511].copy()
    # odd n: rows start mid Box-Muller pair
    m2, n2 = 7, 33
    f = np.empty(m2 * n2, np.float64); L.ref_fill_normals(9, m2 * n2, 1.0 / np.sqrt(m2), p(f))
    out["gauss_m7_n33_seed9"] = f.reshape(m2, n2)
    # CountSketch C4 shape (m=8192), first 4096 rows, seed 0
    h = np.empty(4096, np.int64); s = np.empty(4096, np.float64)
    L.ref_count_draws(0, 4096, 8192, 1, 1.0, p(h), p(s)); out["count_m8192_seed0_h"] = h; out["count_m8192_seed0_sign"] = s
    # SJLT m=12 s=3 n=64 seed 6 (reference test_sketch.cpp:80)
    h = np.empty(3 * 64, np.int64); s = np.empty(3 * 64, np.float64)
    L.ref_count_draws(6, 64, 4, 3, 1.0 / np.sqrt(3.0), p(h), p(s)); out["sjlt_m12_s3_n64_seed6_h"] = h; out["sjlt_m12_s3_n64_seed6_sign"] = s
    # SRHT C2 shape: n=65536, m=2048, seed 0
    sg = np.empty(65536, np.float64); rows = np.empty(2048, np.int64)
    L.ref_srht_draws(0, 65536, 2048, p(sg), p(rows))
    out["srht_n65536_m2048_seed0_signbits"] = np.packbits(sg > 0)
    out["srht_n65536_m2048_seed0_rows"] = rows
    sg = np.empty(13, np.float64); rows = np.empty(4, np.int64)
    L.ref_srht_draws(77, 13, 4, p(sg), p(rows)); out["srht_n13_m4_seed77_signs"] = sg; out["srht_n13_m4_seed77_rows"] = rows
    np.savez_compressed(os.path.join(HERE, "ref_draws.npz"), **out)
    print("wrote", os.path.join(HERE, "ref_draws.npz"), {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
