// Bit-exact device (and host) versions of the glibc libm functions the
// reference's Box-Muller uses: log, sin, cos on doubles (rng.hpp:43-55).
//
// The reference computes r = sqrt(-2 log u1), r cos(2 pi u2), r sin(2 pi u2)
// with glibc, whose log (optimized-routines, e_log.c) and sin/cos (IBM,
// s_sin.c) are not correctly rounded.  To draw the *same* Gaussian entries the
// device runs those algorithms operation for operation, including every fused
// multiply-add of glibc's x86-64 FMA build (the variant the dynamic loader
// selects on AVX2/FMA hosts), on the tables extracted from the host libm
// (tools/gen_libm_tables.py -> glibc_tables.h).  Only the argument ranges
// Box-Muller produces are implemented: log on (0, 1], sin/cos on (0, 2 pi].
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>

#include "glibc_tables.h"

#if defined(__CUDACC__)
#define RPB_HD __host__ __device__ __forceinline__
#else
#define RPB_HD inline
#endif

namespace rpb {
namespace glibc {

#if RP_GLIBC_EXACT

// Exact-rounding primitives: no contraction, explicit fusion.
RPB_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
RPB_HD double mul_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
RPB_HD double add_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
RPB_HD double sub_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  volatile double r = a - b;
  return r;
#endif
}
RPB_HD uint64_t bits_(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
RPB_HD double dbl_(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}
RPB_HD double copysign_(double mag, double sgn) {
  return dbl_((bits_(mag) & 0x7fffffffffffffffULL) | (bits_(sgn) & 0x8000000000000000ULL));
}
RPB_HD double fabs_(double x) { return dbl_(bits_(x) & 0x7fffffffffffffffULL); }

// Tables: the device reads a global copy, the host the static arrays.  (This
// header is included by one device translation unit, draws.cu.)
#if defined(__CUDACC__)
__device__ double d_log_head[18] = RP_GLIBC_LOG_HEAD;
__device__ double d_log_tab[256] = RP_GLIBC_LOG_TAB;
__device__ double d_sincos_tab[440] = RP_GLIBC_SINCOS_TAB;
#endif

RPB_HD const double* log_head() {
#if defined(__CUDA_ARCH__)
  return d_log_head;
#else
  return kLogHead;
#endif
}
RPB_HD const double* log_tab() {
#if defined(__CUDA_ARCH__)
  return d_log_tab;
#else
  return kLogTab;
#endif
}
RPB_HD const double* sincos_tab() {
#if defined(__CUDA_ARCH__)
  return d_sincos_tab;
#else
  return kSinCosTab;
#endif
}

// ---- log: e_log.c (optimized-routines), FMA build ---------------------------
// x in (0, 1] (normal): the table path and the |x - 1| < 0x1.09p-4 path.
RPB_HD double log(double x) {
  const double* H = log_head();
  const double Ln2hi = H[0], Ln2lo = H[1];
  const double* A = H + 2;  // poly[5]
  const double* B = H + 7;  // poly1[11]
  const uint64_t ix = bits_(x);
  if (ix - 0x3fee000000000000ULL <= 0x308ffffffffffULL) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = sub_(x, 1.0);
    const double r2 = mul_(r, r);
    const double r3 = mul_(r, r2);
    double p1 = fma_(r, B[2], B[1]);
    double p4 = fma_(r, B[5], B[4]);
    double p7 = fma_(r, B[8], B[7]);
    p1 = fma_(r2, B[3], p1);
    p4 = fma_(r2, B[6], p4);
    p7 = fma_(r2, B[9], p7);
    p7 = fma_(r3, B[10], p7);
    p4 = fma_(p7, r3, p4);
    const double p = fma_(p4, r3, p1);
    const double w = fma_(r, 0x1p27, r);     // r + r*2^27
    const double rhi = fma_(-0x1p27, r, w);  // (r + w) - w
    const double rlo = sub_(r, rhi);
    const double rh2 = mul_(rhi, rhi);
    const double hi = fma_(rh2, B[0], r);
    double lo = fma_(rh2, B[0], sub_(r, hi));
    lo = fma_(mul_(B[0], rlo), add_(r, rhi), lo);
    return add_(hi, fma_(p, r3, lo));
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ULL);
  const double invc = log_tab()[2 * i], logc = log_tab()[2 * i + 1];
  const double z = dbl_(iz);
  const double kd = static_cast<double>(k);
  const double w = fma_(kd, Ln2hi, logc);
  const double r = fma_(z, invc, -1.0);
  const double p12 = fma_(r, A[2], A[1]);
  const double hi = add_(r, w);
  const double r2 = mul_(r, r);
  double lo = add_(sub_(w, hi), r);
  lo = fma_(kd, Ln2lo, lo);
  const double rr2 = mul_(r, r2);
  const double p34 = fma_(r, A[4], A[3]);
  lo = fma_(r2, A[0], lo);
  const double p = fma_(p34, r2, p12);
  return add_(fma_(rr2, p, lo), hi);
}

// ---- sin / cos: s_sin.c (IBM), FMA build -------------------------------------

struct SinCos {
  double sn, ssn, cs, ccs;
};

RPB_HD SinCos lookup(double u) {
  const int k = static_cast<int>(static_cast<uint32_t>(bits_(u)) << 2);
  const double* t = sincos_tab();
  return SinCos{t[k], t[k + 1], t[k + 2], t[k + 3]};
}

// TAYLOR_SIN(xx, a, da)
RPB_HD double taylor_sin(double a, double da) {
  const double xx = mul_(a, a);
  double p = fma_(xx, k_s5, k_s4);
  p = fma_(xx, p, k_s3);
  p = fma_(xx, p, k_s2);
  p = fma_(xx, p, k_s1);
  const double t = fma_(p, a, -mul_(da, 0.5));  // vfmsub: P*a - 0.5*da
  return add_(a, fma_(xx, t, da));
}

// do_sin(x, dx): |x| >= 0.126 part (the Taylor branch is taylor_sin)
RPB_HD double do_sin_main(double x, double dx) {
  if (!(x > 0.0)) dx = -dx;
  const double ax = fabs_(x);
  const double u = add_(ax, k_big);
  const double xr = sub_(ax, sub_(u, k_big));
  const SinCos t = lookup(u);
  const double xx = mul_(xr, xr);
  const double s = add_(xr, fma_(mul_(xr, xx), fma_(xx, k_sn5, k_sn3), dx));
  const double c = fma_(xr, dx, mul_(xx, fma_(xx, fma_(xx, k_cs6, k_cs4), k_cs2)));
  const double cor = fma_(s, t.cs, fma_(-c, t.sn, fma_(s, t.ccs, t.ssn)));
  return copysign_(add_(t.sn, cor), x);
}

RPB_HD double do_sin(double x, double dx) {
  if (fabs_(x) < 0.126) return taylor_sin(x, dx);
  return do_sin_main(x, dx);
}

// do_cos(x, dx)
RPB_HD double do_cos(double x, double dx) {
  if (x < 0.0) dx = -dx;
  const double ax = fabs_(x);
  const double u = add_(ax, k_big);
  const double xr = add_(sub_(ax, sub_(u, k_big)), dx);
  const SinCos t = lookup(u);
  const double xx = mul_(xr, xr);
  const double s = fma_(mul_(xr, xx), fma_(xx, k_sn5, k_sn3), xr);
  const double c = mul_(xx, fma_(xx, fma_(xx, k_cs6, k_cs4), k_cs2));
  const double cor = fma_(-s, t.sn, fma_(-c, t.cs, fma_(-s, t.ssn, t.ccs)));
  return add_(t.cs, cor);
}

// reduce_sincos: x in [2.426265, 105414350)
RPB_HD int reduce(double x, double& a, double& da) {
  const double t = fma_(x, k_hpinv, k_toint);
  const double xn = sub_(t, k_toint);
  const int n = static_cast<int>(static_cast<uint32_t>(bits_(t)) & 3u);
  const double y = fma_(-xn, k_mp2, fma_(-xn, k_mp1, x));
  const double t2 = fma_(-xn, k_pp3, y);
  const double db = fma_(-k_pp3, xn, sub_(y, t2));
  const double b = fma_(-xn, k_pp4, t2);
  const double db2 = fma_(-xn, k_pp4, sub_(t2, b));
  a = b;
  da = add_(db, db2);
  return n;
}

RPB_HD double do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

// sin(x) for 0 < x <= 2 pi (plus tiny x)
RPB_HD double sin(double x) {
  const uint32_t k = static_cast<uint32_t>(bits_(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0);
  if (k < 0x400368fdu) {
    const double t = sub_(k_hp0, fabs_(x));
    return copysign_(do_cos(t, k_hp1), x);
  }
  double a, da;
  const int n = reduce(x, a, da);
  return do_sincos(a, da, n);
}

// cos(x) for 0 < x <= 2 pi (plus tiny x)
RPB_HD double cos(double x) {
  const uint32_t k = static_cast<uint32_t>(bits_(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = sub_(k_hp0, fabs_(x));
    const double a = add_(y, k_hp1);
    const double da = add_(sub_(y, a), k_hp1);
    return do_sin(a, da);
  }
  double a, da;
  const int n = reduce(x, a, da);
  return do_sincos(a, da, n + 1);
}

#endif  // RP_GLIBC_EXACT

}  // namespace glibc
}  // namespace rpb
