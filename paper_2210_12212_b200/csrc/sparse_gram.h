// Sparse Gram product Y = M^T (M W) for a CSR operator, L2-blocked
// (reference: gram_apply for CsrMatrix = apply then apply_transpose,
// ref/proj/core/src/matrix.cpp:140-172).
//
// The operator's local rows are cut into panels of `panel_rows` rows and the
// right-hand columns into chunks of <= 128.  Per (chunk, panel):
//   pass 1  Y_p = M_p W_c            (warp per row, gathers rows of the
//                                     row-major W_c, which stays in L2)
//   pass 2  Z  = Z + M_p^T Y_p       (warp per column through the panel's own
//                                     CSC, gathers rows of Y_p from L2)
// so the n x cols intermediate M W never reaches HBM.  Pass 2 continues each
// column's running sum across panels in ascending row order, which is exactly
// the order of the reference's apply_transpose (out.row(c) += v * x.row(r),
// rows ascending): the result is bit-identical to the unblocked two-pass
// product and independent of the panel and chunk sizes.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"

namespace rpb {

// CSC of every row panel of a CSR matrix (n local rows, d columns): entries of
// panel p, column j are [off[p*d + j], off[p*d + j + 1]), rows ascending.
struct PanelCsc {
  int64_t n = 0, d = 0, nnz = 0, panel_rows = 0, panels = 0;
  DBuf<int64_t> off;  // panels * d + 1
  DBuf<int32_t> row;  // nnz, local row index
  DBuf<double> val;   // nnz
  bool matches(int64_t n_, int64_t d_, int64_t nnz_, int64_t pr) const {
    return panels > 0 && n == n_ && d == d_ && nnz == nnz_ && panel_rows == pr;
  }
};

// Non-owning view of a panel CSC.  The operator's plain CSC (d + 1 offsets,
// rows ascending per column) is the one-panel case.
struct PanelView {
  int64_t n = 0, d = 0, panel_rows = 0, panels = 0;
  const int64_t* off = nullptr;
  const int32_t* row = nullptr;
  const double* val = nullptr;
};
inline PanelView view_of(const PanelCsc& pc) {
  return PanelView{pc.n, pc.d, pc.panel_rows, pc.panels, pc.off.get(), pc.row.get(), pc.val.get()};
}
inline PanelView single_panel(int64_t n, int64_t d, const int64_t* csc_off, const int32_t* csc_row,
                              const double* csc_val) {
  return PanelView{n, d, n > 0 ? n : 1, 1, csc_off, csc_row, csc_val};
}

// Build the panel CSC on the device (stable radix sort of (panel, column) keys).
void build_panel_csc(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, int64_t n, int64_t d,
                     int64_t nnz, int64_t panel_rows, PanelCsc& out, cudaStream_t s);

// Y (d x cols, column-major, ld ldy) = M^T (M W), W (d x cols, column-major, ld ldw).
// l2_persist: mark the running sums Z (d x chunk) as persisting in L2 for the
// duration of the product (stream access-policy window), so the panels'
// Y_p gathers do not evict them.
// CsrMatrix invariants on the device (matrix.cpp:22-50): column indices in
// [0, d), strictly increasing within a row, finite values; writes the int32
// column indices.  *d_flag (initialized to INT64_MAX by the caller) receives
// min over violating entries p of 4 p + code (1 = range, 2 = order, 3 = value):
// the violation a row-major scan meets first.
void csr_validate_convert(const int64_t* d_off, const int64_t* d_col64, const double* d_val, int64_t n, int64_t d,
                          int32_t* d_col32, long long* d_flag, cudaStream_t s);

void sparse_gram(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, const PanelView& pc,
                 const double* W, int64_t ldw, int64_t cols, double* Y, int64_t ldy, int64_t chunk, cudaStream_t s,
                 bool l2_persist = false, int blocks_per_sm = 0);

}  // namespace rpb
