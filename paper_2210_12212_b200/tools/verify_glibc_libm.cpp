// Host check of csrc/glibc_libm.cuh against the running glibc: the Box-Muller
// arguments u1 = ((w >> 11) + 1) 2^-53 and theta = 2 pi u2 (rng.hpp:26-28,
// 43-55) over N pseudo-random words plus the interval edges.  Exit 1 on any
// bit difference.   usage: verify_glibc_libm [N]
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include "glibc_libm.cuh"

static uint64_t bits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }

int main(int argc, char** argv) {
#if !RP_GLIBC_EXACT
  std::printf("RP_GLIBC_EXACT=0: nothing to verify\n");
  return 0;
#else
  const long long n = argc > 1 ? std::atoll(argv[1]) : 10000000LL;
  std::mt19937_64 g(12345);
  long long bad_log = 0, bad_sin = 0, bad_cos = 0;
  const double two_pi = 6.283185307179586476925286766559;
  auto check = [&](double u) {
    volatile double vu = u;
    const double l = std::log(vu), th = two_pi * u;
    volatile double vth = th;
    const double s = std::sin(vth), c = std::cos(vth);
    if (bits(l) != bits(rpb::glibc::log(u))) {
      if (bad_log++ < 5) std::printf("log  %a: glibc %a ours %a\n", u, l, rpb::glibc::log(u));
    }
    if (bits(s) != bits(rpb::glibc::sin(th))) {
      if (bad_sin++ < 5) std::printf("sin  %a: glibc %a ours %a\n", th, s, rpb::glibc::sin(th));
    }
    if (bits(c) != bits(rpb::glibc::cos(th))) {
      if (bad_cos++ < 5) std::printf("cos  %a: glibc %a ours %a\n", th, c, rpb::glibc::cos(th));
    }
  };
  for (uint64_t k = 1; k < 100000; ++k) {  // both ends of (0, 1]
    check(static_cast<double>(k) * 0x1.0p-53);
    check(static_cast<double>((1ULL << 53) + 1 - k) * 0x1.0p-53);
  }
  for (long long i = 0; i < n; ++i) check(static_cast<double>((g() >> 11) + 1) * 0x1.0p-53);
  // log's near-1 window and sin/cos range switches, densely
  for (double lo : {0.9375, 1.0 - 1e-3, 0.126 / two_pi, 0.855469 / two_pi, 2.426265 / two_pi, 0.25, 0.5, 0.75}) {
    double u = lo;
    for (int i = 0; i < 200000 && u <= 1.0; ++i) { check(u); u = std::nextafter(u, 2.0); }
  }
  std::printf("checked %lld + edges: log mismatches %lld, sin %lld, cos %lld\n", n, bad_log, bad_sin, bad_cos);
  return (bad_log || bad_sin || bad_cos) ? 1 : 0;
#endif
}
