// L2-blocked sparse Gram product, see sparse_gram.h.
#include "sparse_gram.h"

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "basis.h"

namespace rpb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

unsigned grid_for(int64_t work, int threads = 256) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), 148 * 32)));
}

// ---- panel CSC build ------------------------------------------------------------

// keys[e] = panel(row(e)) * d + col[e]; idx[e] = e; rows[e] = row(e).
template <class Key>
__global__ void expand_keys_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ col, int64_t n,
                                   int64_t d, int64_t panel_rows, Key* __restrict__ keys, int32_t* __restrict__ idx,
                                   int32_t* __restrict__ rows) {
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    const Key pk = static_cast<Key>(r / panel_rows) * static_cast<Key>(d);
    for (int64_t e = off[r] + lane; e < off[r + 1]; e += 32) {
      keys[e] = pk + static_cast<Key>(col[e]);
      idx[e] = static_cast<int32_t>(e);
      rows[e] = static_cast<int32_t>(r);
    }
  }
}

template <class Key>
__global__ void gather_sorted_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ rows,
                                     const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ prow,
                                     double* __restrict__ pval) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nnz;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t e = perm[q];
    prow[q] = rows[e];
    pval[q] = val[e];
  }
}

// off[k] = first position with key >= k (k = 0 .. nkeys).
template <class Key>
__global__ void key_offsets_kernel(const Key* __restrict__ keys, int64_t nnz, int64_t nkeys, int64_t* __restrict__ off) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k <= nkeys;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(keys[mid]) < k) lo = mid + 1;
      else hi = mid;
    }
    off[k] = lo;
  }
}

template <class Key>
void build_impl(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, int64_t n, int64_t d,
                int64_t nnz, int64_t panel_rows, PanelCsc& out, cudaStream_t s) {
  const int64_t nkeys = out.panels * d;
  DBuf<Key> k_in(static_cast<size_t>(nnz), s), k_out(static_cast<size_t>(nnz), s);
  DBuf<int32_t> i_in(static_cast<size_t>(nnz), s), i_out(static_cast<size_t>(nnz), s), rows(static_cast<size_t>(nnz), s);
  expand_keys_kernel<Key><<<grid_for(n * 32), 256, 0, s>>>(csr_off, csr_col, n, d, panel_rows, k_in.get(), i_in.get(),
                                                          rows.get());
  RP_LAUNCH_CHECK();
  int end_bit = 1;
  while (end_bit < static_cast<int>(8 * sizeof(Key)) && (int64_t{1} << end_bit) <= nkeys) ++end_bit;
  size_t tmp_bytes = 0;
  RP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in.get(), k_out.get(), i_in.get(), i_out.get(),
                                          static_cast<int>(nnz), 0, end_bit, s));
  DBuf<unsigned char> tmp(std::max<size_t>(tmp_bytes, 1), s);
  // (LSD radix sort is stable: equal keys keep ascending entry = ascending row order)
  RP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, k_in.get(), k_out.get(), i_in.get(), i_out.get(),
                                          static_cast<int>(nnz), 0, end_bit, s));
  gather_sorted_kernel<Key><<<grid_for(nnz), 256, 0, s>>>(i_out.get(), rows.get(), csr_val, nnz, out.row.get(),
                                                         out.val.get());
  RP_LAUNCH_CHECK();
  key_offsets_kernel<Key><<<grid_for(nkeys + 1), 256, 0, s>>>(k_out.get(), nnz, nkeys, out.off.get());
  RP_LAUNCH_CHECK();
}

// ---- ingest ---------------------------------------------------------------------

__global__ void csr_validate_kernel(const int64_t* __restrict__ off, const int64_t* __restrict__ col,
                                    const double* __restrict__ val, int64_t n, int64_t d, int32_t* __restrict__ c32,
                                    long long* __restrict__ flag) {
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t p0 = off[r], p1 = off[r + 1];
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int64_t c = col[p];
      int code = 0;
      if (c < 0 || c >= d) code = 1;
      else if (p > p0 && !(col[p - 1] < c)) code = 2;
      else if (!isfinite(val[p])) code = 3;
      if (code) atomicMin(flag, static_cast<long long>(4 * p + code));
      c32[p] = static_cast<int32_t>(c);
    }
  }
}

// ---- the two passes ---------------------------------------------------------------

// Yp (rows x cc, row-major) = M[row0 : row0 + rows] * Wr (d x cc, row-major).
// Warp per row; the row's entries are loaded cooperatively and broadcast.
template <int CPL>
__global__ void __launch_bounds__(256) pass1_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                                    const double* __restrict__ val, int64_t row0, int64_t rows,
                                                    const double* __restrict__ wr, int cc, double* __restrict__ yp) {
  // (the passes of a chunk are chained by programmatic dependent launch: the next pass's blocks take the
  // slots this one's tail frees, and wait here until the previous grid -- whose Yp / Z they touch -- is done)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const int64_t p0 = off[row0 + r], p1 = off[row0 + r + 1];
    double acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
    for (int64_t base = p0; base < p1; base += 32) {
      const int cnt = static_cast<int>(p1 - base < 32 ? p1 - base : 32);
      int mc = 0;
      double mv = 0.0;
      if (lane < cnt) {
        mc = __ldcs(col + base + lane);
        mv = __ldcs(val + base + lane);
      }
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const int cj = __shfl_sync(kFull, mc, t);
        const double v = __shfl_sync(kFull, mv, t);
        const double* w = wr + static_cast<int64_t>(cj) * cc;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int c = lane + 32 * q;
          if (c < cc) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, w[c]));
        }
      }
    }
    double* y = yp + r * cc;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      if (c < cc) y[c] = acc[q];
    }
  }
}

// Z (d x cc, row-major) = (first ? 0 : Z) + M_p^T Yp, panel p = rows [row0, row0 + panel_rows).
// Warp per column; entries in ascending row order continue the column's running sum.
template <int CPL>
__global__ void __launch_bounds__(256) pass2_kernel(const int64_t* __restrict__ poff, const int32_t* __restrict__ prow,
                                                    const double* __restrict__ pval, int64_t d, int64_t row0,
                                                    const double* __restrict__ yp, int cc, double* __restrict__ z,
                                                    int first) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp; j < d; j += nwarps) {
    const int64_t e0 = poff[j], e1 = poff[j + 1];
    double* zr = z + j * cc;
    double acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      // (Z only streams through: read once and written once per panel -- evict-first
      // loads / stores keep it from displacing the gathered Yp and W rows in L2)
      acc[q] = (!first && c < cc) ? __ldcs(zr + c) : 0.0;
    }
    for (int64_t base = e0; base < e1; base += 32) {
      const int cnt = static_cast<int>(e1 - base < 32 ? e1 - base : 32);
      int mr = 0;
      double mv = 0.0;
      if (lane < cnt) {
        mr = __ldcs(prow + base + lane);
        mv = __ldcs(pval + base + lane);
      }
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const int ri = __shfl_sync(kFull, mr, t);
        const double v = __shfl_sync(kFull, mv, t);
        const double* y = yp + (static_cast<int64_t>(ri) - row0) * cc;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int c = lane + 32 * q;
          if (c < cc) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, y[c]));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = lane + 32 * q;
      if (c < cc) __stcs(zr + c, acc[q]);
    }
  }
}

// blocks_per_sm > 0: the passes run as that many 256-thread blocks per SM, leaving the rest of every SM to
// another stream's kernels (the two-stream basis recursion: these gather-bound passes beside the other
// interval group's tensor-bound GEMMs).
template <int CPL>
void run_chunk(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, const PanelView& pc,
               const double* wr, int cc, double* yp, double* z, cudaStream_t s, int blocks_per_sm) {
  // (a grid of 148 x blocks_per_sm blocks lands that many blocks on every SM; the passes walk their rows /
  // columns with grid-stride loops.  Registers and shared memory stay free for the other stream's CTAs.)
  const int pad = 0;
  const unsigned cap = blocks_per_sm > 0 ? 148u * static_cast<unsigned>(blocks_per_sm) : 148u * 32u;
  for (int64_t p = 0; p < pc.panels; ++p) {
    const int64_t row0 = p * pc.panel_rows;
    const int64_t rows = std::min(pc.panel_rows, pc.n - row0);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = pad;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(std::min(grid_for(rows * 32), cap));
    RP_CUDA(cudaLaunchKernelEx(&cfg, pass1_kernel<CPL>, csr_off, csr_col, csr_val, row0, rows, wr, cc, yp));
    RP_LAUNCH_CHECK();
    cfg.gridDim = dim3(std::min(grid_for(pc.d * 32), cap));
    const int64_t* poff = pc.off + p * pc.d;
    const int first = p == 0 ? 1 : 0;
    RP_CUDA(cudaLaunchKernelEx(&cfg, pass2_kernel<CPL>, poff, pc.row, pc.val, pc.d, row0,
                               static_cast<const double*>(yp), cc, z, first));
    RP_LAUNCH_CHECK();
  }
}

}  // namespace

void csr_validate_convert(const int64_t* d_off, const int64_t* d_col64, const double* d_val, int64_t n, int64_t d,
                          int32_t* d_col32, long long* d_flag, cudaStream_t s) {
  if (n <= 0) return;
  csr_validate_kernel<<<grid_for(n * 32), 256, 0, s>>>(d_off, d_col64, d_val, n, d, d_col32, d_flag);
  RP_LAUNCH_CHECK();
}

void build_panel_csc(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, int64_t n, int64_t d,
                     int64_t nnz, int64_t panel_rows, PanelCsc& out, cudaStream_t s) {
  require(panel_rows > 0, "panel csc: panel rows must be positive");
  require(nnz < (int64_t{1} << 31) && n < (int64_t{1} << 31), "panel csc: more than 2^31 entries");
  out.n = n;
  out.d = d;
  out.nnz = nnz;
  out.panel_rows = panel_rows;
  out.panels = std::max<int64_t>(1, ceil_div(n, panel_rows));
  out.off.alloc(static_cast<size_t>(out.panels * d + 1), s);
  out.row.alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)), s);
  out.val.alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)), s);
  if (nnz == 0) {
    RP_CUDA(cudaMemsetAsync(out.off.get(), 0, sizeof(int64_t) * (out.panels * d + 1), s));
    return;
  }
  if (out.panels * d < (int64_t{1} << 32))
    build_impl<uint32_t>(csr_off, csr_col, csr_val, n, d, nnz, panel_rows, out, s);
  else
    build_impl<uint64_t>(csr_off, csr_col, csr_val, n, d, nnz, panel_rows, out, s);
}

void sparse_gram(const int64_t* csr_off, const int32_t* csr_col, const double* csr_val, const PanelView& pc,
                 const double* W, int64_t ldw, int64_t cols, double* Y, int64_t ldy, int64_t chunk, cudaStream_t s,
                 bool l2_persist, int blocks_per_sm) {
  if (cols <= 0 || pc.d <= 0) return;
  chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, 128));
  const int64_t cmax = std::min(chunk, cols);
  DBuf<double> wr(static_cast<size_t>(pc.d * cmax), s), z(static_cast<size_t>(pc.d * cmax), s);
  DBuf<double> yp(static_cast<size_t>(std::max<int64_t>(1, std::min(pc.panel_rows, pc.n)) * cmax), s);
  struct Persist {
    cudaStream_t s = nullptr;
    ~Persist() {
      if (!s) return;
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.num_bytes = 0;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
      cudaCtxResetPersistingL2Cache();
    }
  } persist;
  if (l2_persist && pc.panels > 1) {
    int dev = 0, max_window = 0, max_persist = 0;
    RP_CUDA(cudaGetDevice(&dev));
    RP_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    RP_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    const size_t zbytes = static_cast<size_t>(pc.d * cmax) * sizeof(double);
    RP_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(zbytes, max_persist)));
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = z.get();
    v.accessPolicyWindow.num_bytes = std::min<size_t>(zbytes, static_cast<size_t>(max_window));
    v.accessPolicyWindow.hitRatio = std::min(1.0f, static_cast<float>(max_persist) / static_cast<float>(zbytes));
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    RP_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
    persist.s = s;
  }
  for (int64_t c0 = 0; c0 < cols; c0 += chunk) {
    const int cc = static_cast<int>(std::min(chunk, cols - c0));
    transpose(W + c0 * ldw, pc.d, cc, ldw, wr.get(), cc, s);  // row-major W chunk
    if (pc.n == 0) {
      fill(z.get(), pc.d * cc, 0.0, s);
    } else if (cc <= 32) {
      run_chunk<1>(csr_off, csr_col, csr_val, pc, wr.get(), cc, yp.get(), z.get(), s, blocks_per_sm);
    } else if (cc <= 64) {
      run_chunk<2>(csr_off, csr_col, csr_val, pc, wr.get(), cc, yp.get(), z.get(), s, blocks_per_sm);
    } else if (cc <= 96) {
      run_chunk<3>(csr_off, csr_col, csr_val, pc, wr.get(), cc, yp.get(), z.get(), s, blocks_per_sm);
    } else {
      run_chunk<4>(csr_off, csr_col, csr_val, pc, wr.get(), cc, yp.get(), z.get(), s, blocks_per_sm);
    }
    transpose(z.get(), cc, pc.d, cc, Y + c0 * ldy, ldy, s);  // back to column-major
  }
}

}  // namespace rpb
