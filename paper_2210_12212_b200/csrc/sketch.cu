// Sketch families on the device.
//
//   Gaussian     sketch.cpp:83-109   S generated slab by slab from the MT
//                                    stream (draws.cu) and multiplied on the
//                                    FP64 tensor cores (gemm_f64.cu).
//   CountSketch  sketch.cpp:114-136  per output column, rows accumulated in
//   / SJLT                           ascending order -- the reference's own
//                                    summation order, so SA is bit-exact.
//   SRHT         sketch.cpp:25-48,   Walsh-Hadamard butterflies in shared
//                138-173             memory, stride n_pad/2 first (descending),
//                                    the reference's order: SA is bit-exact.
//   Identity     sketch.cpp:229-231  densifying copy.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.h"
#include "draws.h"
#include "gemm_f64.h"
#include "sketch.h"

namespace rpb {

void validate_spec(const SketchSpecC& spec) {
  require(spec.kind >= 0 && spec.kind <= 4, "unknown sketch kind");
  require(spec.n >= 1, "sketch: n must be positive");
  require(spec.m >= 1, "sketch: m must be positive");
  if (spec.kind == kSjlt) {
    require(spec.s >= 1, "sjlt: sparsity must be >= 1");
    require(spec.m % spec.s == 0, "sjlt: sparsity must divide m");
  }
  if (spec.kind == kIdentity) require(spec.m == spec.n, "identity sketch: m must equal n");
}

namespace {

// ---- densify / identity ------------------------------------------------------

__global__ void densify_dense(const double* __restrict__ a, int64_t ld, bool trans, int64_t n, int64_t d,
                              double* __restrict__ out, int64_t ldo) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < n * d;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    out[i + j * ldo] = trans ? a[j + i * ld] : a[i + j * ld];
  }
}

__global__ void zero_fill(double* __restrict__ out, int64_t rows, int64_t cols, int64_t ld) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < rows * cols;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    out[i + j * ld] = 0.0;
  }
}

__global__ void densify_csr(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                            const double* __restrict__ val, int64_t n, double* __restrict__ out, int64_t ldo) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t p = off[r]; p < off[r + 1]; ++p) out[r + static_cast<int64_t>(col[p]) * ldo] = val[p];
}

unsigned grid_for(int64_t work, int threads = 256) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), 148 * 16)));
}

// ---- CountSketch / SJLT -------------------------------------------------------

// One thread per (output column c, block b).  Rows are visited in ascending
// order, so every SA entry receives its terms in the reference's order
// (sketch.cpp:125-134); the product sgn * value is rounded before the add,
// exactly as `out(...) += sgn * value`.
__global__ void count_dense(const double* __restrict__ a, int64_t ld, bool trans, int64_t n_loc, int64_t row0,
                            int64_t n_glob, int64_t d, int blocks, int64_t rpb, const int32_t* __restrict__ h,
                            const double* __restrict__ sgn, double* __restrict__ sa, int64_t m) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= d * blocks) return;
  const int64_t c = t % d;
  const int b = static_cast<int>(t / d);
  double* col = sa + c * m + static_cast<int64_t>(b) * rpb;
  const int32_t* hb = h + static_cast<int64_t>(b) * n_glob + row0;
  const double* sb = sgn + static_cast<int64_t>(b) * n_glob + row0;
  for (int64_t j = 0; j < n_loc; ++j) {
    const double v = trans ? a[c + j * ld] : a[j + c * ld];
    double* dst = col + hb[j];
    *dst = __dadd_rn(*dst, __dmul_rn(sb[j], v));
  }
}

__global__ void count_csc(const int64_t* __restrict__ coff, const int32_t* __restrict__ crow,
                          const double* __restrict__ cval, int64_t row0, int64_t n_glob, int64_t d, int blocks,
                          int64_t rpb, const int32_t* __restrict__ h, const double* __restrict__ sgn,
                          double* __restrict__ sa, int64_t m) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= d * blocks) return;
  const int64_t c = t % d;
  const int b = static_cast<int>(t / d);
  double* col = sa + c * m + static_cast<int64_t>(b) * rpb;
  const int32_t* hb = h + static_cast<int64_t>(b) * n_glob + row0;
  const double* sb = sgn + static_cast<int64_t>(b) * n_glob + row0;
  for (int64_t p = coff[c]; p < coff[c + 1]; ++p) {
    const int32_t j = crow[p];
    double* dst = col + hb[j];
    *dst = __dadd_rn(*dst, __dmul_rn(sb[j], cval[p]));
  }
}

// ---- SRHT ------------------------------------------------------------------------

__global__ void srht_scatter_csc(const int64_t* __restrict__ coff, const int32_t* __restrict__ crow,
                                 const double* __restrict__ cval, int64_t row0, int64_t d,
                                 const double* __restrict__ signs, double* __restrict__ x, int64_t npad) {
  const int64_t c = blockIdx.x;
  if (c >= d) return;
  for (int64_t p = coff[c] + threadIdx.x; p < coff[c + 1]; p += blockDim.x) {
    const int64_t i = row0 + crow[p];
    x[i + c * npad] = signs[i] * cval[p];
  }
}

// One pass of butterflies over index bits [lo, lo + B): for every column and
// every fixed value of the other bits, an S = 2^B point transform with the
// largest stride first (the reference's descending recursion, sketch.cpp:25-48).
// Tile = S x W elements (W consecutive low indices).  from_op: the first pass
// reads the operator directly (x[i] = sign[i] * M(i - row0, c), zero padding,
// sketch.cpp:160-162); to_sa: the last pass (lo = 0, W = 1) writes only the
// sampled rows, scaled, into SA (sketch.cpp:168-170).
struct FwhtArgs {
  double* x;  // scratch, npad x d
  int64_t npad, d;
  int lo, logW, logG;
  bool from_op;
  const double* a;
  int64_t lda, n_loc, row0;
  bool trans;
  const double* signs;
  bool to_sa;
  const int64_t* tpos;  // target positions sorted ascending
  const int32_t* tslot;
  const int32_t* boff;  // per S-block offsets into tpos (npad/S + 1)
  double scale;
  double* sa;
  int64_t m;
};

template <int B>
__global__ void __launch_bounds__(256) fwht_pass(FwhtArgs f) {
  constexpr int S = 1 << B;
  extern __shared__ double tile[];  // lo > 0: [S][W];  lo == 0: [G][S] (G consecutive groups)
  const int W = 1 << f.logW;
  const int G = f.lo == 0 ? (1 << f.logG) : 1;
  const int64_t groups_per_col = f.npad >> (B + f.logW + (f.lo == 0 ? f.logG : 0));
  const int64_t c = blockIdx.x / groups_per_col;
  const int64_t gidx = blockIdx.x - c * groups_per_col;
  int64_t base;
  if (f.lo == 0) {
    base = gidx << (B + f.logG);
  } else {
    const int64_t wblocks = int64_t{1} << (f.lo - f.logW);
    const int64_t hi_part = gidx >> (f.lo - f.logW);
    const int64_t l0 = (gidx & (wblocks - 1)) << f.logW;
    base = (hi_part << (B + f.lo)) + l0;
  }
  const int total = (S << f.logW) * G;
  double* col = f.x + c * f.npad;
  // element e of the tile -> global index (contiguous when lo == 0)
  auto gindex = [&](int e) -> int64_t {
    if (f.lo == 0) return base + e;
    const int t = e >> f.logW, l = e & (W - 1);
    return base + (static_cast<int64_t>(t) << f.lo) + l;
  };
  if (f.from_op) {
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int64_t i = gindex(e);
      const int64_t li = i - f.row0;
      double v = 0.0;
      if (li >= 0 && li < f.n_loc) v = f.signs[i] * (f.trans ? f.a[c + li * f.lda] : f.a[li + c * f.lda]);
      tile[e] = v;
    }
  } else {
    for (int e = threadIdx.x; e < total; e += blockDim.x) tile[e] = col[gindex(e)];
  }
  __syncthreads();
#pragma unroll 1
  for (int lh = B - 1; lh >= 0; --lh) {
    const int h = 1 << lh;
    for (int e = threadIdx.x; e < (total >> 1); e += blockDim.x) {
      double* pa;
      int step;
      if (f.lo == 0) {  // e -> (group, pair within group)
        const int grp = e >> (B - 1), pp = e & ((S >> 1) - 1);
        pa = tile + (grp << B) + ((pp >> lh) << (lh + 1)) + (pp & (h - 1));
        step = h;
      } else {
        const int pair = e >> f.logW, l = e & (W - 1);
        const int t = ((pair >> lh) << (lh + 1)) + (pair & (h - 1));
        pa = tile + (t << f.logW) + l;
        step = h << f.logW;
      }
      double* pb = pa + step;
      const double a = *pa, b = *pb;
      *pa = a + b;
      *pb = a - b;
    }
    __syncthreads();
  }
  if (f.to_sa) {  // lo == 0: blocks [base + g*S, base + (g+1)*S)
    const int64_t blk0 = base >> B;
    for (int k = f.boff[blk0] + threadIdx.x; k < f.boff[blk0 + G]; k += blockDim.x)
      f.sa[f.tslot[k] + c * f.m] = tile[f.tpos[k] - base] * f.scale;
  } else {
    for (int e = threadIdx.x; e < total; e += blockDim.x) col[gindex(e)] = tile[e];
  }
}

// ---- two-pass SRHT transform -------------------------------------------------
//
// n_pad = 2^QB * CH (CH <= 8192).  Pass 1 (fwht_top_kernel): the QB largest
// strides -- one thread per row offset r < CH keeps the 2^QB elements
// r + CH j in registers (sign multiply and zero padding fused into the load,
// coalesced 8 KB segments per j).  Pass 2 (fwht_chunk_kernel): one CTA per
// (column, CH-row chunk) does the remaining log2(CH) strides -- the four
// largest in registers, the rest in shared memory -- and writes only the
// sampled rows to SA.  Strides run largest first, the reference's order
// (sketch.cpp:25-48), so every entry is bit-identical to the reference.
constexpr int kFwhtChunkThreads = 512;
constexpr int64_t kFwhtMaxChunk = 8192;

__device__ __forceinline__ double signed_op_value(const FwhtArgs& f, int64_t c, int64_t i) {
  const int64_t li = i - f.row0;
  if (li < 0 || li >= f.n_loc) return 0.0;
  return f.signs[i] * (f.trans ? f.a[c + li * f.lda] : f.a[li + c * f.lda]);
}

template <int QB>
__global__ void __launch_bounds__(256) fwht_top_kernel(FwhtArgs f, int64_t ch) {
  constexpr int J = 1 << QB;
  const int64_t per_col = ch;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < per_col * f.d;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / per_col, r = idx - c * per_col;
    double v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = signed_op_value(f, c, r + ch * j);
#pragma unroll
    for (int kk = J / 2; kk >= 1; kk >>= 1)
#pragma unroll
      for (int j = 0; j < J; ++j)
        if ((j & kk) == 0) {
          const double a = v[j], b = v[j + kk];
          v[j] = a + b;
          v[j + kk] = a - b;
        }
    double* col = f.x + c * f.npad;
#pragma unroll
    for (int j = 0; j < J; ++j) col[r + ch * j] = v[j];
  }
}

// from_x: the chunk comes from the pass-1 scratch; else straight from the
// operator (n_pad <= CH: the whole transform is local).
__global__ void __launch_bounds__(kFwhtChunkThreads) fwht_chunk_kernel(FwhtArgs f, int64_t ch, bool from_x) {
  extern __shared__ __align__(16) double xs[];  // ch doubles
  constexpr int kT = kFwhtChunkThreads;
  const int ch32 = static_cast<int>(ch);
  const int64_t chunks = f.npad / ch;
  const int64_t c = blockIdx.x / chunks, q = blockIdx.x - c * chunks;
  const int64_t chunk0 = q * ch;
  const int t = threadIdx.x;
  const int nj = ch32 >= kT ? ch32 / kT : 0;
  if (nj >= 1) {
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nj) {
        const int64_t i = chunk0 + t + static_cast<int64_t>(kT) * j;
        v[j] = from_x ? f.x[c * f.npad + i] : signed_op_value(f, c, i);
      }
#pragma unroll
    for (int kk = 8; kk >= 1; kk >>= 1)
      if (kk < nj)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < nj && (j & kk) == 0) {
            const double a = v[j], b = v[j + kk];
            v[j] = a + b;
            v[j + kk] = a - b;
          }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nj) xs[t + kT * j] = v[j];
  } else {
    for (int e = t; e < ch32; e += kT) xs[e] = from_x ? f.x[c * f.npad + chunk0 + e] : signed_op_value(f, c, chunk0 + e);
  }
  __syncthreads();
  int lh = 0;
  const int local = nj >= 1 ? kT : ch32;  // strides below this are still to do
  while ((2 << lh) <= local) ++lh;
  for (--lh; lh >= 0; --lh) {
    const int h = 1 << lh;
#pragma unroll 4
    for (int e = t; e < (ch32 >> 1); e += kT) {
      const int i0 = ((e >> lh) << (lh + 1)) + (e & (h - 1));
      const double a = xs[i0], b = xs[i0 + h];
      xs[i0] = a + b;
      xs[i0 + h] = a - b;
    }
    __syncthreads();
  }
  for (int k = f.boff[q] + t; k < f.boff[q + 1]; k += kT) f.sa[f.tslot[k] + c * f.m] = xs[f.tpos[k] - chunk0] * f.scale;
}

// CH = 8192 specialisation: the 13 local strides as three register passes
// (bits 12-9, 8-5, 4-0), each a 16- or 32-point transform held by one thread,
// with one shared-memory round trip between passes (padded layout i + i/32:
// every access conflict-free) instead of one per stride.
__device__ __forceinline__ int fpad(int i) { return i + (i >> 5); }

template <int N>
__device__ __forceinline__ void fwht_regs(double (&v)[N]) {  // strides N/2 ... 1 over the register index
#pragma unroll
  for (int kk = N / 2; kk >= 1; kk >>= 1)
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((j & kk) == 0) {
        const double a = v[j], b = v[j + kk];
        v[j] = a + b;
        v[j + kk] = a - b;
      }
}

__global__ void __launch_bounds__(kFwhtChunkThreads) fwht_chunk8192_kernel(FwhtArgs f, bool from_x) {
  extern __shared__ __align__(16) double xs[];  // fpad(8192) doubles
  constexpr int CH = 8192;
  const int64_t chunks = f.npad / CH;
  const int64_t c = blockIdx.x / chunks, q = blockIdx.x - c * chunks;
  const int64_t chunk0 = q * CH;
  const int t = threadIdx.x;
  {  // pass A: bits 12-9 (strides 4096 .. 512); thread t = bits 8-0
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t i = chunk0 + t + 512 * j;
      v[j] = from_x ? f.x[c * f.npad + i] : signed_op_value(f, c, i);
    }
    fwht_regs<16>(v);
#pragma unroll
    for (int j = 0; j < 16; ++j) xs[fpad(t + 512 * j)] = v[j];
  }
  __syncthreads();
  {  // pass B: bits 8-5 (strides 256 .. 32); thread t = (bits 12-9, bits 4-0)
    const int hi = t >> 5, lo = t & 31;
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = xs[fpad((hi << 9) | (j << 5) | lo)];
    fwht_regs<16>(v);
#pragma unroll
    for (int j = 0; j < 16; ++j) xs[fpad((hi << 9) | (j << 5) | lo)] = v[j];
  }
  __syncthreads();
  if (t < 256) {  // pass C: bits 4-0 (strides 16 .. 1); thread t = bits 12-5
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = xs[fpad((t << 5) | j)];
    fwht_regs<32>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) xs[fpad((t << 5) | j)] = v[j];
  }
  __syncthreads();
  for (int k = f.boff[q] + t; k < f.boff[q + 1]; k += kFwhtChunkThreads)
    f.sa[f.tslot[k] + c * f.m] = xs[fpad(static_cast<int>(f.tpos[k] - chunk0))] * f.scale;
}

// Dense operators with n_pad <= 2^5 * 8192 take the two-pass path.
bool fwht2_ok(const FwhtArgs& f) { return f.npad >= 2 && f.npad <= 32 * kFwhtMaxChunk; }
int64_t fwht2_chunk(int64_t npad) { return std::min<int64_t>(npad, kFwhtMaxChunk); }

void launch_fwht2(FwhtArgs f, cudaStream_t stream) {
  const int64_t ch = fwht2_chunk(f.npad);
  int qb = 0;
  while ((ch << qb) < f.npad) ++qb;
  if (qb > 0) {
    const int64_t work = ch * f.d;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(work, 256), 148 * 16));
    switch (qb) {
      case 1: fwht_top_kernel<1><<<blocks, 256, 0, stream>>>(f, ch); break;
      case 2: fwht_top_kernel<2><<<blocks, 256, 0, stream>>>(f, ch); break;
      case 3: fwht_top_kernel<3><<<blocks, 256, 0, stream>>>(f, ch); break;
      case 4: fwht_top_kernel<4><<<blocks, 256, 0, stream>>>(f, ch); break;
      default: fwht_top_kernel<5><<<blocks, 256, 0, stream>>>(f, ch); break;
    }
    RP_LAUNCH_CHECK();
  }
  if (ch == 8192) {
    const size_t smem = static_cast<size_t>(8192 + 8192 / 32) * sizeof(double);
    ensure_dynamic_smem(fwht_chunk8192_kernel, smem);
    fwht_chunk8192_kernel<<<static_cast<unsigned>(f.d * (f.npad / ch)), kFwhtChunkThreads, smem, stream>>>(f, qb > 0);
    RP_LAUNCH_CHECK();
    return;
  }
  const size_t smem = static_cast<size_t>(ch) * sizeof(double);
  ensure_dynamic_smem(fwht_chunk_kernel, smem);
  fwht_chunk_kernel<<<static_cast<unsigned>(f.d * (f.npad / ch)), kFwhtChunkThreads, smem, stream>>>(f, ch, qb > 0);
  RP_LAUNCH_CHECK();
}

void launch_fwht(FwhtArgs f, int bits, cudaStream_t stream) {
  const int S = 1 << bits;
  int logW = 0;
  while (logW < f.lo && (S << (logW + 1)) <= 4096) ++logW;
  int logG = 0;  // lo == 0: consecutive groups per CTA
  if (f.lo == 0)
    while ((S << (logG + 1)) <= 4096 && (int64_t{S} << (logG + 1)) <= f.npad) ++logG;
  f.logW = logW;
  f.logG = logG;
  const int64_t blocks = f.d * (f.npad >> (bits + logW + logG));
  const int smem = (S << (logW + logG)) * 8;
  auto go = [&](auto kern) {
    ensure_dynamic_smem(kern, smem);
    kern<<<static_cast<unsigned>(blocks), 256, smem, stream>>>(f);
    RP_LAUNCH_CHECK();
  };
  switch (bits) {
    case 0: go(fwht_pass<0>); break;
    case 1: go(fwht_pass<1>); break;
    case 2: go(fwht_pass<2>); break;
    case 3: go(fwht_pass<3>); break;
    case 4: go(fwht_pass<4>); break;
    case 5: go(fwht_pass<5>); break;
    case 6: go(fwht_pass<6>); break;
    case 7: go(fwht_pass<7>); break;
    case 8: go(fwht_pass<8>); break;
    default: throw InvalidArgument("fwht: pass width out of range");
  }
}

__global__ void transpose_rm_to_cm(const double* __restrict__ in, int64_t rows, int64_t cols,
                                   double* __restrict__ out) {
  // in: rows x cols row-major; out: rows x cols column-major
  __shared__ double tile[32][33];
  const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[r + c * rows] = tile[threadIdx.x][i];
  }
}

// SA[:, c] += S_slab[:, j] * v over the CSC entries (j in the slab) of column c.
__global__ void gauss_csc_accum(const int64_t* __restrict__ coff, const int32_t* __restrict__ crow,
                                const double* __restrict__ cval, int64_t j0, int64_t J,
                                const double* __restrict__ s_cm, int64_t m, double* __restrict__ sa, int64_t c0) {
  const int64_t c = blockIdx.y + c0;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = sa[r + c * m];
    for (int64_t p = coff[c]; p < coff[c + 1]; ++p) {
      const int64_t j = crow[p] - j0;
      if (j < 0 || j >= J) continue;
      acc = __dadd_rn(acc, __dmul_rn(s_cm[r + j * m], cval[p]));
    }
    sa[r + c * m] = acc;
  }
}

}  // namespace

void densify(const OpView& op, double* d_out, int64_t ld_out, cudaStream_t stream) {
  if (!op.sparse) {
    densify_dense<<<grid_for(op.n_loc * op.d), 256, 0, stream>>>(op.a, op.ld, op.trans, op.n_loc, op.d, d_out,
                                                                  ld_out);
    RP_LAUNCH_CHECK();
  } else {
    zero_fill<<<grid_for(op.n_loc * op.d), 256, 0, stream>>>(d_out, op.n_loc, op.d, ld_out);
    RP_LAUNCH_CHECK();
    densify_csr<<<grid_for(op.n_loc), 256, 0, stream>>>(op.csr_off, op.csr_col, op.csr_val, op.n_loc, d_out,
                                                         ld_out);
    RP_LAUNCH_CHECK();
  }
}

void sketch_apply(const SketchSpecC& spec, const OpView& op, double* d_sa, cudaStream_t stream) {
  validate_spec(spec);
  require(op.n_global == spec.n, "sketch_apply: spec.n must match A.rows");
  const int64_t m = spec.m, d = op.d;
  switch (spec.kind) {
    case kIdentity: {
      zero_fill<<<grid_for(m * d), 256, 0, stream>>>(d_sa, m, d, m);
      RP_LAUNCH_CHECK();
      densify(op, d_sa + op.row0, m, stream);
      return;
    }
    case kGaussian: {
      const double scale = 1.0 / std::sqrt(static_cast<double>(m));
      // S slab budget: 1 GiB of doubles.
      const int64_t J = std::max<int64_t>(
          2, std::min<int64_t>(op.n_loc, ((int64_t{1} << 27) / std::max<int64_t>(m, 1)) & ~int64_t{1}));
      // One slab holding whole rows of an unsharded operator: S is the stream
      // [0, m n) itself (row r = normals r n .. r n + n - 1, sketch.cpp:86-95).
      const bool one_stream = op.row0 == 0 && op.n_loc == spec.n && J >= op.n_loc;
      DBuf<uint64_t> states(one_stream ? 1 : static_cast<size_t>(m) * 312, stream);
      DBuf<int64_t> cursor(one_stream ? 1 : static_cast<size_t>(m), stream);
      GaussRows g;
      g.d_states = states.get();
      g.d_cursor = cursor.get();
      if (!one_stream) gauss_rows_init(spec.seed, m, op.row0, spec.n, g, stream);
      DBuf<double> slab(static_cast<size_t>(m * J), stream);
      DBuf<double> slab_cm;
      if (op.sparse) {
        slab_cm.alloc(static_cast<size_t>(m * J), stream);
        zero_fill<<<grid_for(m * d), 256, 0, stream>>>(d_sa, m, d, m);
        RP_LAUNCH_CHECK();
      }
      // Several slabs of a dense operator: slab j + 1 is drawn on a second
      // stream (FP64 SIMT + integer work) while the DMMA GEMM consumes slab j;
      // two slab buffers, events both ways.  (C3: 32 slabs, 1.8 ms of normals
      // beside each 16 ms GEMM.)
      const bool two_buf = !op.sparse && !one_stream && op.n_loc > J;
      DBuf<double> slab_b;
      cudaStream_t gs = stream;
      std::vector<cudaEvent_t> evs;
      auto new_event = [&]() {
        cudaEvent_t e;
        RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        return e;
      };
      cudaEvent_t gemm_done[2] = {nullptr, nullptr};
      if (two_buf) {
        slab_b.alloc(static_cast<size_t>(m * J), stream);
        RP_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
        cudaEvent_t start = new_event();  // (the row states and both buffers exist in `stream` order)
        RP_CUDA(cudaEventRecord(start, stream));
        RP_CUDA(cudaStreamWaitEvent(gs, start, 0));
      }
      int64_t slab_index = 0;
      for (int64_t j0 = 0; j0 < op.n_loc; j0 += J, ++slab_index) {
        const int64_t Jc = std::min(J, op.n_loc - j0);
        double* const buf = (two_buf && (slab_index & 1)) ? slab_b.get() : slab.get();
        if (one_stream) {
          draw_gauss_stream(spec.seed, 0, m * Jc, scale, buf, stream);
        } else {
          if (two_buf && gemm_done[slab_index & 1]) RP_CUDA(cudaStreamWaitEvent(gs, gemm_done[slab_index & 1], 0));
          gauss_rows_next(g, Jc, scale, buf, Jc, gs);
          if (two_buf) {
            cudaEvent_t drawn = new_event();
            RP_CUDA(cudaEventRecord(drawn, gs));
            RP_CUDA(cudaStreamWaitEvent(stream, drawn, 0));
          }
        }
        if (!op.sparse) {
          GemmArgs ga;
          ga.opa = Op::T;  // slab is row-major m x Jc == column-major Jc x m
          ga.opb = op.trans ? Op::T : Op::N;
          ga.m = m;
          ga.n = d;
          ga.k = Jc;
          ga.a = buf;
          ga.lda = Jc;
          ga.b = op.trans ? op.a + j0 * op.ld : op.a + j0;
          ga.ldb = op.ld;
          ga.c = d_sa;
          ga.ldc = m;
          ga.beta = j0 == 0 ? 0.0 : 1.0;
          dgemm(ga, stream);
          if (two_buf) {
            gemm_done[slab_index & 1] = new_event();
            RP_CUDA(cudaEventRecord(gemm_done[slab_index & 1], stream));
          }
        } else {
          dim3 tg(static_cast<unsigned>(ceil_div(Jc, 32)), static_cast<unsigned>(ceil_div(m, 32)));
          transpose_rm_to_cm<<<tg, dim3(32, 8), 0, stream>>>(slab.get(), m, Jc, slab_cm.get());
          RP_LAUNCH_CHECK();
          for (int64_t c0 = 0; c0 < d; c0 += 65535) {  // (grid.y <= 65535)
            dim3 ag(static_cast<unsigned>(ceil_div(m, 256)), static_cast<unsigned>(std::min<int64_t>(65535, d - c0)));
            gauss_csc_accum<<<ag, 256, 0, stream>>>(op.csc_off, op.csc_row, op.csc_val, j0, Jc, slab_cm.get(), m,
                                                    d_sa, c0);
            RP_LAUNCH_CHECK();
          }
        }
      }
      for (cudaEvent_t e : evs) RP_CUDA(cudaEventDestroy(e));  // (released once complete)
      if (two_buf) RP_CUDA(cudaStreamDestroy(gs));  // (every draw was awaited by its GEMM on `stream`)
      return;
    }
    case kCountSketch:
    case kSjlt:
    case kSrht: {
      SketchPlan plan;
      sketch_plan(spec, op, plan, stream);
      sketch_apply_planned(plan, op, d_sa, stream);
      return;
    }
  }
}

void sketch_plan(const SketchSpecC& spec, const OpView& op, SketchPlan& plan, cudaStream_t stream) {
  validate_spec(spec);
  plan.spec = spec;
  plan.sparse = op.sparse;
  const int64_t m = spec.m;
  if (spec.kind == kCountSketch || spec.kind == kSjlt) {
    plan.blocks = spec.kind == kSjlt ? spec.s : 1;
    const double entry = spec.kind == kSjlt ? 1.0 / std::sqrt(static_cast<double>(spec.s)) : 1.0;
    plan.rpb = m / plan.blocks;
    plan.h.alloc(static_cast<size_t>(spec.n * plan.blocks), stream);
    plan.sg.alloc(static_cast<size_t>(spec.n * plan.blocks), stream);
    draw_count(spec.seed, spec.n, plan.rpb, plan.blocks, entry, plan.h.get(), plan.sg.get(), stream);
    return;
  }
  if (spec.kind == kGaussian) {
    require(!op.sparse, "sketch plan: the Gaussian plan needs a dense operator");
    const double scale = 1.0 / std::sqrt(static_cast<double>(m));
    plan.gauss_rows = op.n_loc;
    plan.gauss_s.alloc(static_cast<size_t>(m * op.n_loc), stream);
    if (op.row0 == 0 && op.n_loc == spec.n) {
      // unsharded: S is the normal stream [0, m n) itself (sketch.cpp:86-95)
      draw_gauss_stream(spec.seed, 0, m * op.n_loc, scale, plan.gauss_s.get(), stream);
    } else {
      DBuf<uint64_t> states(static_cast<size_t>(m) * 312, stream);
      DBuf<int64_t> cursor(static_cast<size_t>(m), stream);
      GaussRows g;
      g.d_states = states.get();
      g.d_cursor = cursor.get();
      gauss_rows_init(spec.seed, m, op.row0, spec.n, g, stream);
      gauss_rows_next(g, op.n_loc, scale, plan.gauss_s.get(), op.n_loc, stream);
      RP_CUDA(cudaStreamSynchronize(stream));  // (states / cursor are released with this frame)
    }
    return;
  }
  require(spec.kind == kSrht, "sketch plan: only Gaussian / CountSketch / SJLT / SRHT are planned");
  int64_t npad = 1;
  int P = 0;
  while (npad < spec.n) {
    npad <<= 1;
    ++P;
  }
  plan.npad = npad;
  plan.P = P;
  plan.signs.alloc(static_cast<size_t>(spec.n), stream);
  DBuf<int64_t> rows(static_cast<size_t>(m), stream);
  draw_srht(spec.seed, spec.n, m, plan.signs.get(), rows.get(), stream);
  // Pass plan: descending bit ranges of at most 8 bits, balanced (a
  // single 0-bit pass when n_pad = 1).
  {
    const int passes = std::max(1, (P + 7) / 8);
    int rem = P;
    for (int i = 0; i < passes; ++i) {
      const int w = (rem + (passes - i) - 1) / (passes - i);
      plan.widths.push_back(w);
      rem -= w;
    }
  }
  FwhtArgs probe{};
  probe.npad = npad;
  plan.two_pass = !op.sparse && fwht2_ok(probe);
  // (two-pass path: targets bucketed per CH-row chunk)
  const int last_bits = plan.two_pass ? [&] {
    int lb = 0;
    while ((int64_t{1} << lb) < fwht2_chunk(npad)) ++lb;
    return lb;
  }() : plan.widths.back();
  // Targets sorted by position, bucketed per block of the last pass.
  std::vector<int64_t> hrows(static_cast<size_t>(m));
  RP_CUDA(cudaMemcpyAsync(hrows.data(), rows.get(), sizeof(int64_t) * m, cudaMemcpyDeviceToHost, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  std::vector<std::pair<int64_t, int32_t>> tg(static_cast<size_t>(m));
  for (int64_t r = 0; r < m; ++r) tg[r] = {hrows[r], static_cast<int32_t>(r)};
  std::sort(tg.begin(), tg.end());
  const int64_t nblk = npad >> last_bits;
  plan.tpos.assign(static_cast<size_t>(m), 0);
  plan.meta.assign(static_cast<size_t>(m + nblk + 1), 0);
  for (int64_t r = 0; r < m; ++r) {
    plan.tpos[r] = tg[r].first;
    plan.meta[r] = tg[r].second;
  }
  {
    int64_t k = 0;
    for (int64_t b = 0; b <= nblk; ++b) {
      while (k < m && (plan.tpos[k] >> last_bits) < b) ++k;
      plan.meta[m + b] = static_cast<int32_t>(k);
    }
  }
  plan.d_tpos.alloc(static_cast<size_t>(m), stream);
  plan.d_meta.alloc(plan.meta.size(), stream);
  // (the plan keeps the host tables alive until it is destroyed)
  RP_CUDA(cudaMemcpyAsync(plan.d_tpos.get(), plan.tpos.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, stream));
  RP_CUDA(cudaMemcpyAsync(plan.d_meta.get(), plan.meta.data(), sizeof(int32_t) * plan.meta.size(),
                          cudaMemcpyHostToDevice, stream));
}

void sketch_apply_planned(const SketchPlan& plan, const OpView& op, double* d_sa, cudaStream_t stream) {
  const SketchSpecC& spec = plan.spec;
  require(op.n_global == spec.n, "sketch_apply: spec.n must match A.rows");
  require(op.sparse == plan.sparse, "sketch plan: operator kind changed");
  const int64_t m = spec.m, d = op.d;
  if (spec.kind == kCountSketch || spec.kind == kSjlt) {
    zero_fill<<<grid_for(m * d), 256, 0, stream>>>(d_sa, m, d, m);
    RP_LAUNCH_CHECK();
    const int64_t threads = d * plan.blocks;
    if (!op.sparse) {
      count_dense<<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, stream>>>(
          op.a, op.ld, op.trans, op.n_loc, op.row0, spec.n, d, plan.blocks, plan.rpb, plan.h.get(), plan.sg.get(),
          d_sa, m);
    } else {
      count_csc<<<static_cast<unsigned>(ceil_div(threads, 128)), 128, 0, stream>>>(
          op.csc_off, op.csc_row, op.csc_val, op.row0, spec.n, d, plan.blocks, plan.rpb, plan.h.get(),
          plan.sg.get(), d_sa, m);
    }
    RP_LAUNCH_CHECK();
    return;
  }
  if (spec.kind == kGaussian) {
    require(!op.sparse && op.n_loc == plan.gauss_rows, "sketch plan: operator changed");
    GemmArgs ga;  // SA[:, block] = S_local (m x n_loc) * M_local[:, block]
    ga.opa = Op::T;
    ga.opb = op.trans ? Op::T : Op::N;
    ga.m = m;
    ga.n = d;
    ga.k = op.n_loc;
    ga.a = plan.gauss_s.get();
    ga.lda = op.n_loc;
    ga.b = op.a;
    ga.ldb = op.ld;
    ga.c = d_sa;
    ga.ldc = m;
    dgemm(ga, stream);
    return;
  }
  const int64_t npad = plan.npad;
  DBuf<double> x;  // pass scratch (not needed when one chunk holds the whole transform)
  if (!plan.two_pass || npad > fwht2_chunk(npad)) x.alloc(static_cast<size_t>(npad * d), stream);
  FwhtArgs f{};
  f.x = x.get();
  f.npad = npad;
  f.d = d;
  f.signs = plan.signs.get();
  f.a = op.a;
  f.lda = op.ld;
  f.n_loc = op.n_loc;
  f.row0 = op.row0;
  f.trans = op.trans;
  f.tpos = plan.d_tpos.get();
  f.tslot = plan.d_meta.get();
  f.boff = plan.d_meta.get() + m;
  f.scale = 1.0 / std::sqrt(static_cast<double>(m));
  f.sa = d_sa;
  f.m = m;
  const bool first_from_op = !op.sparse;
  if (plan.two_pass) {
    launch_fwht2(f, stream);
    return;
  }
  if (op.sparse) {
    zero_fill<<<grid_for(npad * d), 256, 0, stream>>>(x.get(), npad, d, npad);
    RP_LAUNCH_CHECK();
    srht_scatter_csc<<<static_cast<unsigned>(d), 128, 0, stream>>>(op.csc_off, op.csc_row, op.csc_val, op.row0, d,
                                                                   plan.signs.get(), x.get(), npad);
    RP_LAUNCH_CHECK();
  }
  int hi = plan.P;
  for (size_t i = 0; i < plan.widths.size(); ++i) {
    const int bits = plan.widths[i];
    f.lo = hi - bits;
    f.from_op = (i == 0) && first_from_op;
    f.to_sa = (i + 1 == plan.widths.size());
    launch_fwht(f, bits, stream);
    hi -= bits;
  }
}

}  // namespace rpb
