// Host GF(2)[x] arithmetic for std::mt19937_64 jump-ahead (see mt19937.h).
#include <wmmintrin.h>
#include <smmintrin.h>

#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

#include "common.h"
#include "mt19937.h"

namespace rpb {
namespace mt {
namespace {

inline uint64_t temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

inline uint64_t next_word(uint64_t x0, uint64_t x1, uint64_t xm) {
  const uint64_t y = (x0 & kUpper) | (x1 & kLower);
  return xm ^ (y >> 1) ^ ((y & 1ULL) ? kMatrixA : 0ULL);
}

// ---- bit-vector polynomials ------------------------------------------------

int degree(const Poly& a) {
  for (int64_t w = static_cast<int64_t>(a.size()) - 1; w >= 0; --w)
    if (a[w]) return static_cast<int>(w * 64 + 63 - __builtin_clzll(a[w]));
  return -1;
}

void trim(Poly& a) {
  while (!a.empty() && a.back() == 0) a.pop_back();
}

bool get_bit(const Poly& a, int64_t i) {
  const size_t w = static_cast<size_t>(i >> 6);
  return w < a.size() && ((a[w] >> (i & 63)) & 1ULL);
}

void xor_shifted(Poly& dst, const Poly& src, int64_t shift) {
  // dst ^= src << shift
  const int64_t ws = shift >> 6, bs = shift & 63;
  const size_t need = src.size() + static_cast<size_t>(ws) + 1;
  if (dst.size() < need) dst.resize(need, 0);
  if (bs == 0) {
    for (size_t i = 0; i < src.size(); ++i) dst[i + ws] ^= src[i];
  } else {
    uint64_t carry = 0;
    for (size_t i = 0; i < src.size(); ++i) {
      dst[i + ws] ^= (src[i] << bs) | carry;
      carry = src[i] >> (64 - bs);
    }
    dst[src.size() + ws] ^= carry;
  }
}

Poly shr(const Poly& a, int64_t shift) {
  const int64_t ws = shift >> 6, bs = shift & 63;
  if (static_cast<int64_t>(a.size()) <= ws) return {};
  Poly r(a.size() - ws, 0);
  for (size_t i = 0; i < r.size(); ++i) {
    uint64_t lo = a[i + ws] >> bs;
    uint64_t hi = (bs && i + ws + 1 < a.size()) ? (a[i + ws + 1] << (64 - bs)) : 0;
    r[i] = lo | hi;
  }
  trim(r);
  return r;
}

Poly clmul(const Poly& a, const Poly& b) {
  if (a.empty() || b.empty()) return {};
  Poly r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    if (!a[i]) continue;
    const __m128i av = _mm_cvtsi64_si128(static_cast<long long>(a[i]));
    for (size_t j = 0; j < b.size(); ++j) {
      const __m128i p = _mm_clmulepi64_si128(av, _mm_cvtsi64_si128(static_cast<long long>(b[j])), 0);
      r[i + j] ^= static_cast<uint64_t>(_mm_cvtsi128_si64(p));
      r[i + j + 1] ^= static_cast<uint64_t>(_mm_extract_epi64(p, 1));
    }
  }
  trim(r);
  return r;
}

struct Tables {
  Poly phi;                // degree kDeg
  Poly mu;                 // floor(x^(2 kDeg) / phi)
  std::vector<Poly> pow2;  // x^(2^i) mod phi, i < 64
  std::map<uint64_t, Poly> cache;
  double init_ms = 0.0;
};

Tables* g_tables = nullptr;
std::once_flag g_once;
std::mutex g_cache_mu;

// Barrett reduction mod phi for deg(a) < 2 kDeg.
Poly reduce(const Poly& a) {
  const Tables& t = *g_tables;
  if (degree(a) < kDeg) return a;
  Poly q = shr(clmul(shr(a, kDeg), t.mu), kDeg);
  Poly r = a;
  Poly qp = clmul(q, t.phi);
  if (r.size() < qp.size()) r.resize(qp.size(), 0);
  for (size_t i = 0; i < qp.size(); ++i) r[i] ^= qp[i];
  trim(r);
  if (degree(r) >= kDeg) throw std::logic_error("mt: Barrett reduction failed");
  return r;
}

Poly mulmod(const Poly& a, const Poly& b) { return reduce(clmul(a, b)); }

// Berlekamp-Massey over GF(2) on bit 63 of the tempered outputs of seed 5489.
Poly berlekamp_massey() {
  const int64_t len = 2 * kDeg + 64;
  std::vector<uint8_t> s(static_cast<size_t>(len));
  {
    std::vector<uint64_t> out(static_cast<size_t>(len));
    host_outputs(5489, 0, len, out.data());
    for (int64_t i = 0; i < len; ++i) s[i] = static_cast<uint8_t>(out[i] >> 63);
  }
  const size_t W = kPolyWords + 2;
  Poly C(W, 0), B(W, 0), win(W, 0);
  C[0] = 1;
  B[0] = 1;
  int64_t L = 0, m = 1;
  for (int64_t n = 0; n < len; ++n) {
    // d = s_n + sum_{i=1..L} c_i s_{n-i}; win bit (i-1) = s_{n-i}
    uint64_t par = 0;
    for (size_t w = 0; w < W; ++w) {
      const uint64_t cshift = (C[w] >> 1) | (w + 1 < W ? (C[w + 1] << 63) : 0);
      par ^= static_cast<uint64_t>(__builtin_popcountll(cshift & win[w]));
    }
    const int d = (s[n] ^ static_cast<int>(par & 1));
    if (d) {
      if (2 * L <= n) {
        Poly T = C;
        xor_shifted(C, B, m);
        C.resize(W);
        L = n + 1 - L;
        B = T;
        m = 1;
      } else {
        xor_shifted(C, B, m);
        C.resize(W);
        ++m;
      }
    } else {
      ++m;
    }
    // shift the window: win = (win << 1) | s_n
    uint64_t carry = s[n];
    for (size_t w = 0; w < W; ++w) {
      const uint64_t nc = win[w] >> 63;
      win[w] = (win[w] << 1) | carry;
      carry = nc;
    }
  }
  if (L != kDeg) throw std::logic_error("mt: Berlekamp-Massey degree mismatch");
  // phi(x) = x^L C(1/x): coefficient of x^(L-i) is c_i.
  Poly phi(kPolyWords + 1, 0);
  for (int64_t i = 0; i <= L; ++i)
    if (get_bit(C, i)) phi[(L - i) >> 6] |= 1ULL << ((L - i) & 63);
  trim(phi);
  return phi;
}

void build_tables() {
  const auto t0 = std::chrono::steady_clock::now();
  g_tables = new Tables();
  Tables& t = *g_tables;
  t.phi = berlekamp_massey();
  // mu = floor(x^(2 deg) / phi) by long division.
  {
    Poly rem(static_cast<size_t>((2 * kDeg) / 64 + 2), 0);
    rem[(2 * kDeg) >> 6] |= 1ULL << ((2 * kDeg) & 63);
    Poly q(static_cast<size_t>(kDeg / 64 + 2), 0);
    for (int64_t i = 2 * kDeg; i >= kDeg; --i) {
      if (get_bit(rem, i)) {
        xor_shifted(rem, t.phi, i - kDeg);
        q[(i - kDeg) >> 6] |= 1ULL << ((i - kDeg) & 63);
      }
    }
    trim(q);
    t.mu = q;
  }
  t.pow2.resize(64);
  t.pow2[0] = Poly{2ULL};  // x
  for (int i = 1; i < 64; ++i) t.pow2[i] = mulmod(t.pow2[i - 1], t.pow2[i - 1]);
  // Self-check: a jump by 1003 outputs must equal direct generation.
  {
    uint64_t w0[kN], w1[kN];
    seed_window(20240607ULL, w0);
    Poly p = Poly{1ULL};
    const uint64_t e = 1003;
    for (int i = 0; i < 64; ++i)
      if ((e >> i) & 1ULL) p = mulmod(p, t.pow2[i]);
    host_jump(w0, p, w1);
    // outputs from the jumped window must equal outputs 1003.. of the stream
    uint64_t direct[8];
    host_outputs(20240607ULL, e, 8, direct);
    uint64_t win[2 * kN];
    std::memcpy(win, w1, sizeof(w1));
    for (int k = 0; k < 8; ++k) {
      win[kN + k] = next_word(win[k], win[k + 1], win[k + kM]);
      if (temper(win[kN + k]) != direct[k]) throw std::logic_error("mt: jump self-check failed");
    }
  }
  t.init_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void seed_window(uint64_t seed, uint64_t out[kN]) {
  out[0] = seed;
  for (int i = 1; i < kN; ++i)
    out[i] = 6364136223846793005ULL * (out[i - 1] ^ (out[i - 1] >> 62)) + static_cast<uint64_t>(i);
}

void host_outputs(uint64_t seed, uint64_t skip, int64_t count, uint64_t* out) {
  uint64_t mtw[kN];
  seed_window(seed, mtw);
  int idx = kN;
  auto next = [&]() -> uint64_t {
    if (idx >= kN) {
      for (int i = 0; i < kN; ++i) mtw[i] = next_word(mtw[i], mtw[(i + 1) % kN], mtw[(i + kM) % kN]);
      idx = 0;
    }
    return temper(mtw[idx++]);
  };
  for (uint64_t i = 0; i < skip; ++i) next();
  for (int64_t i = 0; i < count; ++i) out[i] = next();
}

void host_jump(const uint64_t in[kN], const Poly& p, uint64_t out[kN]) {
  const int dp = degree(p);
  std::vector<uint64_t> x(static_cast<size_t>(std::max(dp, 0) + kN + 1));
  std::memcpy(x.data(), in, sizeof(uint64_t) * kN);
  for (size_t k = 0; k + kN < x.size(); ++k) x[k + kN] = next_word(x[k], x[k + 1], x[k + kM]);
  for (int w = 0; w < kN; ++w) out[w] = 0;
  for (int i = 0; i <= dp; ++i)
    if (get_bit(p, i))
      for (int w = 0; w < kN; ++w) out[w] ^= x[static_cast<size_t>(i + w)];
}

double init_tables() {
  bool first = false;
  std::call_once(g_once, [&] {
    build_tables();
    first = true;
  });
  return first ? g_tables->init_ms : 0.0;
}

Poly xpow(uint64_t e) {
  init_tables();
  std::lock_guard<std::mutex> lock(g_cache_mu);
  auto it = g_tables->cache.find(e);
  if (it != g_tables->cache.end()) return it->second;
  Poly p{1ULL};
  for (int i = 0; i < 64; ++i)
    if ((e >> i) & 1ULL) p = mulmod(p, g_tables->pow2[i]);
  if (g_tables->cache.size() > 4096) g_tables->cache.clear();
  return g_tables->cache.emplace(e, std::move(p)).first->second;
}

}  // namespace mt
}  // namespace rpb
