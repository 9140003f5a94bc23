// Sketch application S * M on the device (sketch.cpp:83-248).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.h"

#include "operator.h"

namespace rpb {

enum SketchKind : int { kGaussian = 0, kCountSketch = 1, kSjlt = 2, kSrht = 3, kIdentity = 4 };

struct SketchSpecC {
  int kind = kIdentity;
  int64_t m = 0;
  int64_t n = 0;
  int s = 1;
  uint64_t seed = 0;
};

// SketchSpec::validate (sketch.cpp:202-212).
void validate_spec(const SketchSpecC& spec);

// d_sa (m x D, column-major, ld = m) = S[:, local rows] * M_local.  For a
// single rank this is the reference's sketch_apply; for several ranks the
// partials sum to it (the caller all-reduces).
void sketch_apply(const SketchSpecC& spec, const OpView& op, double* d_sa, cudaStream_t stream);

// The per-spec part of CountSketch / SJLT / SRHT (draws, SRHT target tables),
// computed once and applied to any column block of the operator: applying a
// plan to columns [c0, c1) of M gives columns [c0, c1) of S M, bit for bit.
struct SketchPlan {
  SketchSpecC spec;
  bool sparse = false;
  // CountSketch / SJLT
  int blocks = 1;
  int64_t rpb = 0;
  DBuf<int32_t> h;
  DBuf<double> sg;
  // SRHT
  int64_t npad = 1;
  int P = 0;
  std::vector<int> widths;
  bool two_pass = false;
  DBuf<double> signs;
  std::vector<int64_t> tpos;
  std::vector<int32_t> meta;
  DBuf<int64_t> d_tpos;
  DBuf<int32_t> d_meta;
  // Gaussian (dense operators): the local columns of S, drawn once -- row r of
  // S at gauss_s + r * n_loc (column-major n_loc x m) -- so that column blocks
  // of the operator can be sketched as they arrive (streamed uploads).
  DBuf<double> gauss_s;
  int64_t gauss_rows = 0;
};
void sketch_plan(const SketchSpecC& spec, const OpView& op, SketchPlan& plan, cudaStream_t stream);
void sketch_apply_planned(const SketchPlan& plan, const OpView& op, double* d_sa, cudaStream_t stream);

// Column-major densification of the local rows of M (n_loc x D).
void densify(const OpView& op, double* d_out, int64_t ld_out, cudaStream_t stream);

}  // namespace rpb
