// The data operator M the path runs on (A for the primal route, A^T for the
// dual route, path_solver.cpp:289-351), resident in HBM and row-sharded:
// this rank holds rows [row0, row0 + n_loc) of the N x D operator.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_f64.h"

namespace rpb {

struct OpView {
  int64_t n_global = 0;  // N (rows of M over all ranks) == SketchSpec::n
  int64_t row0 = 0;      // first local row
  int64_t n_loc = 0;     // local rows
  int64_t d = 0;         // D (columns of M)
  bool sparse = false;

  // Dense storage.  !trans: M(i, j) = a[i + j*ld] (column-major M, the
  // Eigen::MatrixXd layout).  trans: M(i, j) = a[j + i*ld] (the buffer is the
  // column-major D x n_loc matrix M^T, i.e. the dual route's A stored as-is).
  const double* a = nullptr;
  int64_t ld = 0;
  bool trans = false;

  // CSR of the local rows (row-local indices) and its CSC mirror.
  const int64_t* csr_off = nullptr;  // n_loc + 1
  const int32_t* csr_col = nullptr;  // nnz
  const double* csr_val = nullptr;   // nnz
  const int64_t* csc_off = nullptr;  // d + 1
  const int32_t* csc_row = nullptr;  // nnz (row-local), ascending within a column
  const double* csc_val = nullptr;   // nnz
  int64_t nnz = 0;

  // Dense helpers: op(X) for GEMMs where M is the left operand.
  Op op_m() const { return trans ? Op::T : Op::N; }
  Op op_mt() const { return trans ? Op::N : Op::T; }
  // Pointer to local row r (dense).
  const double* row_ptr(int64_t r) const { return trans ? a + r * ld : a + r; }
};

}  // namespace rpb
