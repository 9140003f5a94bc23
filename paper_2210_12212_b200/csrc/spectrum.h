// The CLI's plug-in envelope (derive_rho, ref/proj/tools/ridgepath_main.cpp:218-279)
// and the envelope formulas it feeds (ref/proj/core/src/spectrum.cpp:87-169).
//
// The reference takes a thin SVD of SA only to read two spectral sums:
//   ||D||_F^2 = sum_i s_i^2 / (s_i^2 + l0)  = tr(H (H + l0 I)^{-1})
//   s_max^2   = lambda_max(H),             H = SA^T SA (m >= d) or SA SA^T (m < d).
// Here the first is the Frobenius inner product of H with the shifted inverse
// (the batched SPD inverse of factor.cu) and the second comes from Lanczos
// with full reorthogonalization on H; no SVD is formed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <optional>
#include <tuple>
#include <utility>

namespace rpb {

struct RhoResult {
  double rho1 = 1.0, rho2 = 1.0;
  int provenance = 3;  // RhoProvenance: 0 Gaussian, 1 Sjlt, 2 Srht, 3 Identity, 4 Manual
  std::optional<double> success_probability;
  std::optional<int64_t> recommended_m;
  std::optional<int> recommended_s;
};

// spectrum.cpp:87-103 (host, bit-identical restatement).
double effective_dimension(const double* sigma, int64_t count, double lambda0);
// spectrum.cpp:105-128 / 130-148 / 150-169.
RhoResult rho_gaussian(double rho, double eta, double dnorm_sq, std::optional<int64_t> m);
RhoResult rho_srht(double rho, double dnorm_sq, std::optional<std::pair<int64_t, double>> n_and_de);
RhoResult rho_sjlt(double eps, std::optional<std::tuple<double, double, double>> alpha_delta_de);

struct SketchedSpectrum {
  double sum_dii_sq = 0.0;   // ||D||_F^2 at l0
  double sigma_max_sq = 0.0; // s_max(SA)^2
  int lanczos_steps = 0;
};

// Spectral sums of the m x d sketch SA (column-major, on the device).
SketchedSpectrum sketched_spectrum(const double* sa, int64_t m, int64_t d, double lambda0, cudaStream_t s);

// derive_rho's family switch (ridgepath_main.cpp:226-272) from the spectral
// sums; kind follows rp_sketch_kind.  Returns the envelope; de / dnorm_sq out.
RhoResult envelope_from_spectrum(int kind, int64_t m, int64_t n, const SketchedSpectrum& sp, double lambda0,
                                 double* de_out, double* dnorm_sq_out);

}  // namespace rpb
