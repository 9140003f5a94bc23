// derive_rho's spectral sums and the envelope formulas; see spectrum.h.
#include "spectrum.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "common.h"
#include "factor.h"
#include "gemm_f64.h"
#include "vecops.h"

namespace rpb {

// ---- host scalar formulas (spectrum.cpp:87-169, same operation order) ----------

double effective_dimension(const double* sigma, int64_t count, double lambda0) {
  require(count > 0, "effective_dimension: empty spectrum");
  require(lambda0 >= 0.0, "effective_dimension: negative shift");
  double fro = 0.0, top = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double s = sigma[i];
    require(s >= 0.0, "effective_dimension: negative singular value");
    if (s == 0.0) continue;
    const double dii_sq = s * s / (s * s + lambda0);
    fro += dii_sq;
    top = std::max(top, dii_sq);
  }
  require(top > 0.0, "effective_dimension: all-zero spectrum");
  return fro / top;
}

static void validate_bounds(const RhoResult& r) {  // RhoBounds::validate, spectrum.cpp:71-76
  require(r.rho2 > 0.0, "rho bounds: rho2 must be positive");
  require(r.rho1 >= r.rho2, "rho bounds: rho1 must be >= rho2");
}

RhoResult rho_gaussian(double rho, double eta, double dnorm_sq, std::optional<int64_t> m) {
  require(rho > 0.0 && rho < 1.0, "rho_gaussian: rho not in (0,1)");
  const double eta_cap = (1.0 - std::sqrt(rho)) * (1.0 - std::sqrt(rho)) / 4.0;
  require(eta > 0.0 && eta < eta_cap, "rho_gaussian: eta outside (0, (1-sqrt(rho))^2/4)");
  require(dnorm_sq > 0.0 && dnorm_sq <= 1.0, "rho_gaussian: ||D||^2 must lie in (0,1]");
  const double sq_eta = std::sqrt(eta);
  const double c_eta = std::pow((1.0 + sq_eta) / (1.0 - sq_eta), 2.0);
  const double up = (1.0 + std::sqrt(rho)) * (1.0 + sq_eta);
  const double down = 1.0 - std::sqrt(c_eta * rho);
  RhoResult out;
  out.rho1 = 1.0 - dnorm_sq + dnorm_sq * up * up;
  out.rho2 = 1.0 - dnorm_sq + dnorm_sq * down * down;
  out.provenance = 0;
  validate_bounds(out);
  if (m) out.success_probability = 1.0 - 16.0 * std::exp(-eta * eta * rho * static_cast<double>(*m) / 2.0);
  return out;
}

RhoResult rho_srht(double rho, double dnorm_sq, std::optional<std::pair<int64_t, double>> n_and_de) {
  require(rho > 0.0 && rho < 1.0, "rho_srht: rho not in (0,1)");
  require(dnorm_sq > 0.0, "rho_srht: ||D||^2 must be positive");
  require(dnorm_sq * rho < 1.0, "rho_srht: ||D||^2 * rho must be below 1");
  RhoResult out;
  out.rho1 = 1.0 + dnorm_sq * rho;
  out.rho2 = 1.0 - dnorm_sq * rho;
  out.provenance = 2;
  if (n_and_de) {
    const int64_t n = n_and_de->first;
    const double de = n_and_de->second;
    require(n >= 1 && de >= 1.0, "rho_srht: bad (n, d_e)");
    const double c = 16.0 / 3.0 * std::pow(1.0 + std::sqrt(8.0 * std::log(de * static_cast<double>(n)) / de), 2.0);
    out.recommended_m = static_cast<int64_t>(std::ceil(c * de * std::log(de) / rho));
  }
  return out;
}

RhoResult rho_sjlt(double eps, std::optional<std::tuple<double, double, double>> alpha_delta_de) {
  require(eps > 0.0 && eps < 0.5, "rho_sjlt: eps not in (0, 1/2)");
  RhoResult out;
  out.rho1 = 1.0 + eps;
  out.rho2 = 1.0 - eps;
  out.provenance = 1;
  if (alpha_delta_de) {
    const auto [alpha, delta, de] = *alpha_delta_de;
    require(alpha > 2.0, "rho_sjlt: alpha must exceed 2");
    require(delta > 0.0 && delta < 0.5, "rho_sjlt: delta not in (0, 1/2)");
    require(de >= 1.0, "rho_sjlt: d_e must be >= 1");
    const double log_alpha = std::log(de / delta) / std::log(alpha);
    out.recommended_s = static_cast<int>(std::ceil(log_alpha / eps));
    out.recommended_m = static_cast<int64_t>(std::ceil(alpha * de * log_alpha / (eps * eps)));
  }
  return out;
}

RhoResult envelope_from_spectrum(int kind, int64_t m_rows, int64_t n_rows, const SketchedSpectrum& sp,
                                 double lambda0, double* de_out, double* dnorm_sq_out) {
  // effective_dimension(svd.sigma, lambda0) = ||D||_F^2 / max_i D_ii^2
  const double top = sp.sigma_max_sq;
  require(top > 0.0, "effective_dimension: all-zero spectrum");
  const double de = sp.sum_dii_sq / (top / (top + lambda0));
  const double dnorm_sq = top / (top + lambda0);
  const double m = static_cast<double>(m_rows);
  if (de_out) *de_out = de;
  if (dnorm_sq_out) *dnorm_sq_out = dnorm_sq;
  RhoResult bounds;  // identity
  switch (kind) {
    case 0: {  // Gaussian
      const double rho = std::min(0.95, de / m);
      const double eta = 0.5 * (1.0 - std::sqrt(rho)) * (1.0 - std::sqrt(rho)) / 4.0;
      bounds = rho_gaussian(rho, eta, dnorm_sq, m_rows);
      break;
    }
    case 3: {  // SRHT
      const double c =
          16.0 / 3.0 * std::pow(1.0 + std::sqrt(8.0 * std::log(de * static_cast<double>(n_rows)) / de), 2.0);
      double rho = c * de * std::max(1.0, std::log(de)) / m;
      rho = std::min(rho, 0.95 / std::max(dnorm_sq, 1e-12));
      rho = std::clamp(rho, 1e-6, 0.95);
      bounds = rho_srht(rho, dnorm_sq, std::nullopt);
      break;
    }
    case 1:    // CountSketch (the single-block SJLT)
    case 2: {  // SJLT
      const double alpha = 4.0, delta = 0.1;
      const double log_term = std::log(std::max(de / delta, 1.5)) / std::log(alpha);
      double eps = std::sqrt(alpha * de * log_term / m);
      eps = std::clamp(eps, 1e-6, 0.49);
      bounds = rho_sjlt(eps, std::make_tuple(alpha, delta, de));
      break;
    }
    default:
      break;
  }
  return bounds;
}

// ---- device spectral sums ------------------------------------------------------

namespace {

// v_out = w / sqrt(nrm2); also stores beta = sqrt(nrm2).
__global__ void normalize_kernel(const double* __restrict__ w, int64_t n, const double* __restrict__ nrm2,
                                 double* __restrict__ v_out, double* __restrict__ beta) {
  const double b = sqrt(*nrm2);
  if (blockIdx.x == 0 && threadIdx.x == 0) *beta = b;
  const double inv = b > 0.0 ? 1.0 / b : 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v_out[i] = w[i] * inv;
}

// Deterministic start vector (splitmix64 signs scaled to unit norm).
__global__ void start_kernel(double* __restrict__ v, int64_t n) {
  const double s = 1.0 / sqrt(static_cast<double>(n));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t z = static_cast<uint64_t>(i) + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    v[i] = (z >> 63) ? s : -s;
  }
}

unsigned blocks_for(int64_t work) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 16)));
}

// Largest eigenvalue of the symmetric tridiagonal (a[0..k), b[0..k-1)) by
// Sturm-sequence bisection to adjacent doubles.
double tridiag_top(const std::vector<double>& a, const std::vector<double>& b) {
  const size_t k = a.size();
  double lo = a[0], hi = a[0];
  for (size_t i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto below = [&](double x) {  // eigenvalues < x
    int cnt = 0;
    double q = a[0] - x;
    if (q < 0) ++cnt;
    for (size_t i = 1; i < k; ++i) {
      if (q == 0.0) q = std::numeric_limits<double>::min();
      q = a[i] - x - b[i - 1] * b[i - 1] / q;
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  for (int it = 0; it < 2000; ++it) {
    const double mid = lo + 0.5 * (hi - lo);
    if (mid <= lo || mid >= hi) break;
    if (below(mid) == static_cast<int>(k)) hi = mid;
    else lo = mid;
  }
  return hi;
}

}  // namespace

SketchedSpectrum sketched_spectrum(const double* sa, int64_t m, int64_t d, double lambda0, cudaStream_t s) {
  require(m >= 1 && d >= 1, "derive_rho: empty sketch");
  require(lambda0 > 0.0, "derive_rho: lambda0 must be positive");
  const bool wide = m < d;
  const int64_t N = wide ? m : d;
  SketchedSpectrum out;
  // H = SA^T SA (d x d) or SA SA^T (m x m): the same non-zero spectrum, sigma(SA)^2
  DBuf<double> H(static_cast<size_t>(N * N), s);
  {
    GemmArgs g;
    g.opa = wide ? Op::N : Op::T;
    g.opb = wide ? Op::T : Op::N;
    g.m = N;
    g.n = N;
    g.k = wide ? d : m;
    g.a = sa;
    g.lda = m;
    g.b = sa;
    g.ldb = m;
    g.c = H.get();
    g.ldc = N;
    g.lower_only = true;
    g.mirror = true;
    dgemm(g, s);
  }
  DBuf<double> part(kDotParts, s), scal(4, s);
  // ||D||_F^2 = tr(H (H + l0 I)^{-1}) = <H, (H + l0 I)^{-1}>_F  (both symmetric)
  {
    DBuf<double> l0(1, s), hs(static_cast<size_t>(N * N), s), inv(static_cast<size_t>(N * N), s);
    RP_CUDA(cudaMemcpyAsync(l0.get(), &lambda0, sizeof(double), cudaMemcpyHostToDevice, s));
    shifted_copies(H.get(), N, l0.get(), 1, hs.get(), s);
    spd_inverse_batched(hs.get(), N, N, N * N, 1, inv.get(), N, N * N, s);
    vec_dot(H.get(), inv.get(), N * N, part.get(), scal.get(), s);
    RP_CUDA(cudaMemcpyAsync(&out.sum_dii_sq, scal.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
  // s_max^2 = lambda_max(H): Lanczos with full (twice-applied) reorthogonalization.
  const int64_t kcap = std::min<int64_t>(N, 400);
  DBuf<double> V(static_cast<size_t>(N * (kcap + 1)), s), w(static_cast<size_t>(N), s), c(static_cast<size_t>(kcap + 1), s);
  start_kernel<<<blocks_for(N), 256, 0, s>>>(V.get(), N);
  RP_LAUNCH_CHECK();
  std::vector<double> alpha, beta;
  double theta = 0.0, prev = -1.0;
  int still = 0;
  for (int64_t j = 0; j < kcap; ++j) {
    double* vj = V.get() + j * N;
    GemmArgs mv;  // w = H v_j
    mv.m = N;
    mv.n = 1;
    mv.k = N;
    mv.a = H.get();
    mv.lda = N;
    mv.b = vj;
    mv.ldb = N;
    mv.c = w.get();
    mv.ldc = N;
    dgemm(mv, s);
    for (int pass = 0; pass < 2; ++pass) {
      GemmArgs pc;  // c = V_{0..j}^T w
      pc.opa = Op::T;
      pc.m = j + 1;
      pc.n = 1;
      pc.k = N;
      pc.a = V.get();
      pc.lda = N;
      pc.b = w.get();
      pc.ldb = N;
      pc.c = c.get();
      pc.ldc = j + 1;
      dgemm(pc, s);
      if (pass == 0) {  // alpha_j = v_j^T H v_j
        double aj = 0.0;
        RP_CUDA(cudaMemcpyAsync(&aj, c.get() + j, sizeof(double), cudaMemcpyDeviceToHost, s));
        RP_CUDA(cudaStreamSynchronize(s));
        alpha.push_back(aj);
      }
      GemmArgs up;  // w -= V_{0..j} c
      up.m = N;
      up.n = 1;
      up.k = j + 1;
      up.alpha = -1.0;
      up.beta = 1.0;
      up.a = V.get();
      up.lda = N;
      up.b = c.get();
      up.ldb = j + 1;
      up.c = w.get();
      up.ldc = N;
      dgemm(up, s);
    }
    vec_dot(w.get(), w.get(), N, part.get(), scal.get(), s);
    normalize_kernel<<<blocks_for(N), 256, 0, s>>>(w.get(), N, scal.get(), V.get() + (j + 1) * N, scal.get() + 1);
    RP_LAUNCH_CHECK();
    double bj = 0.0;
    RP_CUDA(cudaMemcpyAsync(&bj, scal.get() + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    theta = tridiag_top(alpha, beta);
    out.lanczos_steps = static_cast<int>(j + 1);
    // converged: the top Ritz value (non-decreasing in j) has stopped moving,
    // or the Krylov space is invariant
    if (std::fabs(theta - prev) <= 4.0 * std::numeric_limits<double>::epsilon() * std::fabs(theta)) {
      if (++still >= 3) break;
    } else {
      still = 0;
    }
    prev = theta;
    if (bj <= 1e-15 * std::max(std::fabs(theta), std::numeric_limits<double>::min()) * static_cast<double>(N)) break;
    beta.push_back(bj);
  }
  out.sigma_max_sq = std::max(theta, 0.0);
  return out;
}

}  // namespace rpb
