// Jump-ahead and draw kernels: the reference's draw contract on the device.
//
//   SeededRng            rng.hpp:17-55
//   Gaussian draw order  sketch.cpp:94-95 (row-major S, scale * normal())
//   CountSketch / SJLT   sketch.cpp:119-124 (per block, per row: index, sign)
//   SRHT                 sketch.cpp:62-79 (signs, then partial Fisher-Yates)
//
// Fast paths assume no rejection in uniform_index (probability ~bound/2^64
// per draw) and flag any rejection on the device; a flagged stream is redone
// by a sequential single-block consumer, so the results are exact either way.
#include <algorithm>
#include <cmath>
#include <map>
#include <vector>

#include "common.h"
#include "draws.h"
#include "mt_device.cuh"
#include "glibc_libm.cuh"

namespace rpb {
namespace mt {
namespace {

constexpr int kGenThreads = 160;  // 156 generator lanes rounded up to 5 warps
constexpr int kJumpThreads = 320;
constexpr int kSeqWords = kDeg + kN;  // X_0 .. X_{deg+311}

// dst[job] = poly[job](T) src[job]  (window jump).  `parts` CTAs share a job:
// each generates the word sequence X_0.. from the source window into shared
// memory (up to the last coefficient it owns) and XORs X_{i+w} over its slice
// of the set coefficients i of p into dst (zeroed beforehand) -- a jump costs
// ~deg/parts sequence-window XORs per CTA instead of deg.
__global__ void __launch_bounds__(kJumpThreads) jump_kernel(const uint64_t* __restrict__ src_base,
                                                            const int* __restrict__ src_idx,
                                                            uint64_t* __restrict__ dst_base,
                                                            const int* __restrict__ dst_idx,
                                                            const uint64_t* __restrict__ polys,
                                                            const int* __restrict__ poly_idx,
                                                            const int* __restrict__ poly_deg, int parts) {
  extern __shared__ uint64_t X[];
  const int job = blockIdx.x / parts;
  const int part = blockIdx.x - job * parts;
  const uint64_t* src = src_base + static_cast<int64_t>(src_idx[job]) * kN;
  uint64_t* dst = dst_base + static_cast<int64_t>(dst_idx[job]) * kN;
  const uint64_t* p = polys + static_cast<int64_t>(poly_idx[job]) * kPolyWords;
  const int deg = poly_deg[poly_idx[job]];
  const int words = deg / 64 + 1;
  const int per = (words + parts - 1) / parts;
  const int w0 = part * per;
  const int w1 = min(words, w0 + per);
  if (w0 >= w1) return;
  const int t = threadIdx.x;
  for (int i = t; i < kN; i += blockDim.x) X[i] = src[i];
  __syncthreads();
  const int need = min(deg, w1 * 64 - 1) + kN;  // words X_0 .. X_{last coefficient + 311}
  for (int base = kN; base < need; base += kM) {
    const int k = base + t;
    if (t < kM && k < need) X[k] = d_twist(X[k - kN], X[k - kN + 1], X[k - kM]);
    __syncthreads();
  }
  if (t < kN) {
    uint64_t acc = 0;
    for (int wi = w0; wi < w1; ++wi) {
      uint64_t bits = p[wi];
      while (bits) {
        const int b = __ffsll(static_cast<long long>(bits)) - 1;
        bits &= bits - 1;
        acc ^= X[wi * 64 + b + t];
      }
    }
    if (parts == 1)
      dst[t] = acc;
    else
      atomicXor(reinterpret_cast<unsigned long long*>(dst + t), static_cast<unsigned long long>(acc));
  }
}

int poly_degree(const Poly& a) {
  for (int64_t w = static_cast<int64_t>(a.size()) - 1; w >= 0; --w)
    if (a[w]) return static_cast<int>(w * 64 + 63 - __builtin_clzll(a[w]));
  return -1;
}

struct JumpJob {
  int src, dst;
  uint64_t diff;
};

// Runs one batch of jobs; src/dst index into `states` (row r at r*312), with
// index -1 meaning the seed window buffer.
void run_jobs(const std::vector<JumpJob>& jobs, uint64_t* d_states, const uint64_t* d_seed,
              cudaStream_t stream) {
  if (jobs.empty()) return;
  std::map<uint64_t, int> pidx;
  std::vector<uint64_t> polys;
  std::vector<int> degs;
  std::vector<int> hs(jobs.size()), hd(jobs.size()), hp(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i) {
    auto it = pidx.find(jobs[i].diff);
    if (it == pidx.end()) {
      Poly p = xpow(jobs[i].diff);
      const int id = static_cast<int>(degs.size());
      it = pidx.emplace(jobs[i].diff, id).first;
      polys.resize(polys.size() + kPolyWords, 0);
      std::copy(p.begin(), p.end(), polys.end() - kPolyWords);
      degs.push_back(std::max(poly_degree(p), 0));
    }
    hs[i] = jobs[i].src;
    hd[i] = jobs[i].dst;
    hp[i] = it->second;
  }
  // Source rows are rebased so that the seed buffer is row 0 of a virtual
  // array: we pass two base pointers through one kernel by copying the seed
  // window into a scratch row when needed.
  const bool uses_seed = std::any_of(jobs.begin(), jobs.end(), [](const JumpJob& j) { return j.src < 0; });
  DBuf<uint64_t> scratch;
  const uint64_t* src_base = d_states;
  if (uses_seed) {
    // all jobs in a batch read either the seed or states, never both
    src_base = d_seed;
    for (auto& s : hs) s = 0;
  }
  DBuf<int> d_meta(jobs.size() * 3 + degs.size(), stream);
  DBuf<uint64_t> d_polys(polys.size(), stream);
  std::vector<int> meta;
  meta.insert(meta.end(), hs.begin(), hs.end());
  meta.insert(meta.end(), hd.begin(), hd.end());
  meta.insert(meta.end(), hp.begin(), hp.end());
  meta.insert(meta.end(), degs.begin(), degs.end());
  RP_CUDA(cudaMemcpyAsync(d_meta.get(), meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
  RP_CUDA(cudaMemcpyAsync(d_polys.get(), polys.data(), polys.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                          stream));
  const int smem = kSeqWords * 8;
  ensure_dynamic_smem(jump_kernel, smem);
  const int n = static_cast<int>(jobs.size());
  const int parts = std::max(1, std::min(16, 296 / n));
  jump_kernel<<<n * parts, kJumpThreads, smem, stream>>>(src_base, d_meta.get(), d_states, d_meta.get() + n,
                                                         d_polys.get(), d_meta.get() + 2 * n, d_meta.get() + 3 * n,
                                                         parts);
  RP_LAUNCH_CHECK();
  // Host vectors above must outlive the async copies: synchronize cheaply via
  // the stream before they go out of scope.
  RP_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace

int states_at(uint64_t seed, const std::vector<uint64_t>& offsets, uint64_t* d_states, cudaStream_t stream) {
  init_tables();
  const int64_t R = static_cast<int64_t>(offsets.size());
  if (R == 0) return 0;
  for (int64_t r = 1; r < R; ++r)
    require(offsets[r] >= offsets[r - (int64_t{1} << (63 - __builtin_clzll(static_cast<uint64_t>(r))))],
            "mt: offsets must be non-decreasing along the doubling schedule");
  // every row is produced by exactly one job; multi-CTA jobs XOR into zeros
  RP_CUDA(cudaMemsetAsync(d_states, 0, sizeof(uint64_t) * kN * static_cast<size_t>(R), stream));
  uint64_t seedw[kN];
  seed_window(seed, seedw);
  DBuf<uint64_t> d_seed(kN, stream);
  RP_CUDA(cudaMemcpyAsync(d_seed.get(), seedw, sizeof(seedw), cudaMemcpyHostToDevice, stream));
  int launches = 0;
  run_jobs({JumpJob{-1, 0, offsets[0]}}, d_states, d_seed.get(), stream);
  ++launches;
  for (int64_t lvl = 1; lvl < R; lvl <<= 1) {
    std::vector<JumpJob> jobs;
    for (int64_t r = lvl; r < std::min<int64_t>(2 * lvl, R); ++r)
      jobs.push_back(JumpJob{static_cast<int>(r - lvl), static_cast<int>(r), offsets[r] - offsets[r - lvl]});
    run_jobs(jobs, d_states, d_seed.get(), stream);
    ++launches;
  }
  return launches;
}

}  // namespace mt

namespace {

using mt::BlockGen;
using mt::d_temper;
using mt::d_uniform01;
using mt::kGenThreads;
using mt::kN;

__device__ __forceinline__ uint64_t reject_limit(uint64_t n) { return n * (~0ULL / n); }

// Segment s covers outputs [s*seg, min((s+1)*seg, count)).
__global__ void __launch_bounds__(kGenThreads) words_kernel(const uint64_t* __restrict__ states, int64_t seg,
                                                            int64_t count, int mode, void* out) {
  __shared__ uint64_t sm[2 * kN];
  BlockGen g;
  g.init(sm);
  g.load(states + static_cast<int64_t>(blockIdx.x) * kN);
  const int64_t start = static_cast<int64_t>(blockIdx.x) * seg;
  const int64_t len = min(seg, count - start);
  for (int64_t done = 0; done < len; done += kN) {
    g.step();
    for (int i = threadIdx.x; i < kN; i += blockDim.x) {
      if (done + i >= len) break;
      const uint64_t w = d_temper(g.cur[i]);
      const int64_t pos = start + done + i;
      if (mode == 0)
        static_cast<uint64_t*>(out)[pos] = w;
      else if (mode == 1)
        static_cast<double*>(out)[pos] = d_uniform01(w);
      else
        static_cast<double*>(out)[pos] = (w >> 63) ? 1.0 : -1.0;
    }
  }
}

// uniform_index fast path: draw i consumes word i; flags any rejection.
__global__ void __launch_bounds__(kGenThreads) uindex_kernel(const uint64_t* __restrict__ states, int64_t seg,
                                                             int64_t count, uint64_t bound, uint64_t* out,
                                                             int* flag) {
  __shared__ uint64_t sm[2 * kN];
  BlockGen g;
  g.init(sm);
  g.load(states + static_cast<int64_t>(blockIdx.x) * kN);
  const uint64_t limit = reject_limit(bound);
  const int64_t start = static_cast<int64_t>(blockIdx.x) * seg;
  const int64_t len = min(seg, count - start);
  for (int64_t done = 0; done < len; done += kN) {
    g.step();
    for (int i = threadIdx.x; i < kN; i += blockDim.x) {
      if (done + i >= len) break;
      const uint64_t w = d_temper(g.cur[i]);
      if (w >= limit) atomicOr(flag, 1);
      out[start + done + i] = w % bound;
    }
  }
}

// CountSketch/SJLT fast path: stream position 2*(b*n + j) is the index word of
// row j in block b, the next word its sign.
__global__ void __launch_bounds__(kGenThreads) count_kernel(const uint64_t* __restrict__ states, int64_t seg_rows,
                                                            int64_t total_rows, uint64_t rpb, double entry,
                                                            int32_t* h, double* sgn, int* flag) {
  __shared__ uint64_t sm[2 * kN];
  BlockGen g;
  g.init(sm);
  g.load(states + static_cast<int64_t>(blockIdx.x) * kN);
  const uint64_t limit = reject_limit(rpb);
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * seg_rows;
  const int64_t rows = min(seg_rows, total_rows - row0);
  constexpr int kPairs = kN / 2;
  for (int64_t done = 0; done < rows; done += kPairs) {
    g.step();
    const int t = threadIdx.x;
    if (t < kPairs && done + t < rows) {
      const uint64_t wh = d_temper(g.cur[2 * t]);
      const uint64_t ws = d_temper(g.cur[2 * t + 1]);
      if (wh >= limit) atomicOr(flag, 1);
      const int64_t r = row0 + done + t;
      h[r] = static_cast<int32_t>(wh % rpb);
      sgn[r] = ((ws >> 63) ? 1.0 : -1.0) * entry;
    }
  }
}

// Sequential consumers (exact rejection semantics).  Thread 0 consumes the
// words of each 312-word step in order; the block generates.
// kind 0: uniform_index stream.  kind 1: count draws.
__global__ void __launch_bounds__(kGenThreads) sequential_kernel(const uint64_t* __restrict__ state0, int kind,
                                                                 int64_t count, uint64_t bound, int64_t n,
                                                                 int blocks, double entry, uint64_t* out_idx,
                                                                 int32_t* h, double* sgn) {
  __shared__ uint64_t sm[2 * kN];
  __shared__ int done_flag;
  BlockGen g;
  g.init(sm);
  g.load(state0);
  if (threadIdx.x == 0) done_flag = 0;
  __syncthreads();
  const uint64_t limit = reject_limit(bound);
  int64_t i = 0;          // draws produced (kind 0) / rows produced over all blocks (kind 1)
  bool want_sign = false;  // kind 1: next word is the sign
  int64_t hcur = 0;
  const int64_t total = kind == 0 ? count : n * blocks;
  while (true) {
    g.step();
    if (threadIdx.x == 0) {
      for (int k = 0; k < kN && i < total; ++k) {
        const uint64_t w = d_temper(g.cur[k]);
        if (kind == 0) {
          if (w < limit) out_idx[i++] = w % bound;
        } else if (!want_sign) {
          if (w < limit) {
            hcur = static_cast<int64_t>(w % bound);
            want_sign = true;
          }
        } else {
          h[i] = static_cast<int32_t>(hcur);
          sgn[i] = ((w >> 63) ? 1.0 : -1.0) * entry;
          ++i;
          want_sign = false;
        }
      }
      if (i >= total) done_flag = 1;
    }
    __syncthreads();
    if (done_flag) break;
  }
}

// SRHT partial Fisher-Yates (sketch.cpp:70-77) from the window at offset n.
// The permutation pool is the identity except at touched slots, kept in an
// open-addressing map (shared memory when it fits, global otherwise).
template <int CAP>
__device__ __forceinline__ int64_t* map_slot(int64_t* keys, int64_t key) {
  uint64_t hsh = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ULL;
  int idx = static_cast<int>(hsh >> 40) & (CAP - 1);
  while (keys[idx] != -1 && keys[idx] != key) idx = (idx + 1) & (CAP - 1);
  return keys + idx;
}

template <int CAP, bool SMEM>
__global__ void __launch_bounds__(kGenThreads) srht_fy_kernel(const uint64_t* __restrict__ state_n, int64_t m,
                                                              int64_t npad, int64_t* rows, int64_t* gkeys,
                                                              int64_t* gvals) {
  __shared__ uint64_t sm[2 * kN];
  __shared__ int done_flag;
  extern __shared__ int64_t dyn[];
  int64_t* keys = SMEM ? dyn : gkeys;
  int64_t* vals = SMEM ? dyn + CAP : gvals;
  for (int64_t i = threadIdx.x; i < CAP; i += blockDim.x) keys[i] = -1;
  BlockGen g;
  g.init(sm);
  g.load(state_n);
  if (threadIdx.x == 0) done_flag = 0;
  __syncthreads();
  int64_t i = 0;
  while (true) {
    g.step();
    if (threadIdx.x == 0) {
      for (int k = 0; k < kN && i < m; ++k) {
        const uint64_t w = d_temper(g.cur[k]);
        const uint64_t bound = static_cast<uint64_t>(npad - i);
        if (w >= reject_limit(bound)) continue;
        const int64_t j = i + static_cast<int64_t>(w % bound);
        int64_t* si = map_slot<CAP>(keys, i);
        const int64_t vi = (*si == i) ? vals[si - keys] : i;
        int64_t* sj = map_slot<CAP>(keys, j);
        const int64_t vj = (*sj == j) ? vals[sj - keys] : j;
        // swap(pool[i], pool[j]); rows[i] = pool[i]
        *si = i;
        vals[si - keys] = vj;
        sj = map_slot<CAP>(keys, j);
        *sj = j;
        vals[sj - keys] = vi;
        rows[i] = vj;
        ++i;
      }
      if (i >= m) done_flag = 1;
    }
    __syncthreads();
    if (done_flag) break;
  }
}

// SRHT fast path: words[0..n) are the signs, words[n + i] the Fisher-Yates
// draw of pick i when no rejection occurs (flagged otherwise).  The divisions
// run in parallel; only the swaps stay sequential.
__global__ void srht_prep_kernel(const uint64_t* __restrict__ words, int64_t n, int64_t m, int64_t npad,
                                 double* __restrict__ signs, int64_t* __restrict__ jv, int* flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n + m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t w = words[i];
    if (i < n) {
      signs[i] = (w >> 63) ? 1.0 : -1.0;
    } else {
      const int64_t p = i - n;
      const uint64_t bound = static_cast<uint64_t>(npad - p);
      if (w >= reject_limit(bound)) atomicOr(flag, 1);
      jv[p] = p + static_cast<int64_t>(w % bound);
    }
  }
}

// npad <= 65536: the whole pool as uint16 in shared memory (2 loads + 2 stores
// per pick instead of hash probes).
__global__ void srht_swap_small_kernel(const int64_t* __restrict__ jv, int64_t m, int64_t npad, int64_t* rows) {
  extern __shared__ uint16_t pool16[];
  for (int64_t i = threadIdx.x; i < npad; i += blockDim.x) pool16[i] = static_cast<uint16_t>(i);
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t j = jv[i];
    const uint16_t vi = pool16[i], vj = pool16[j];
    pool16[i] = vj;
    pool16[j] = vi;
    rows[i] = vj;
  }
}

template <int CAP, bool SMEM>
__global__ void srht_swap_kernel(const int64_t* __restrict__ jv, int64_t m, int64_t* rows, int64_t* gkeys,
                                 int64_t* gvals) {
  extern __shared__ int64_t dyn2[];
  int64_t* keys = SMEM ? dyn2 : gkeys;
  int64_t* vals = SMEM ? dyn2 + CAP : gvals;
  for (int64_t i = threadIdx.x; i < CAP; i += blockDim.x) keys[i] = -1;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t j = jv[i];
    int64_t* si = map_slot<CAP>(keys, i);
    const int64_t vi = (*si == i) ? vals[si - keys] : i;
    int64_t* sj = map_slot<CAP>(keys, j);
    const int64_t vj = (*sj == j) ? vals[sj - keys] : j;
    *si = i;
    vals[si - keys] = vj;
    sj = map_slot<CAP>(keys, j);
    *sj = j;
    vals[sj - keys] = vi;
    rows[i] = vj;
  }
}

std::vector<uint64_t> progression(uint64_t first, uint64_t stride, int64_t count) {
  std::vector<uint64_t> o(static_cast<size_t>(count));
  for (int64_t r = 0; r < count; ++r) o[r] = first + static_cast<uint64_t>(r) * stride;
  return o;
}

constexpr int64_t kSegWords = 1 << 16;

// Segment length: one sequential block for short streams (no jump at all),
// otherwise enough segments to fill the machine twice over.
int64_t seg_words(int64_t count) {
  if (count <= (int64_t{1} << 17)) return std::max<int64_t>(count, 2);
  return std::max<int64_t>(kSegWords, (ceil_div(count, 296) + 1) & ~int64_t{1});
}

}  // namespace

void draw_words(uint64_t seed, uint64_t skip, int64_t count, WordMode mode, void* d_out, cudaStream_t stream) {
  if (count <= 0) return;
  const int64_t seg = seg_words(count);
  const int64_t segs = ceil_div(count, seg);
  DBuf<uint64_t> st(static_cast<size_t>(segs) * kN, stream);
  mt::states_at(seed, progression(skip, seg, segs), st.get(), stream);
  words_kernel<<<static_cast<unsigned>(segs), kGenThreads, 0, stream>>>(st.get(), seg, count,
                                                                         static_cast<int>(mode), d_out);
  RP_LAUNCH_CHECK();
}

void draw_uniform_index(uint64_t seed, uint64_t bound, int64_t count, uint64_t* d_out, cudaStream_t stream) {
  require(bound >= 1, "uniform_index: bound must be positive");
  if (count <= 0) return;
  const int64_t seg = seg_words(count);
  const int64_t segs = ceil_div(count, seg);
  DBuf<uint64_t> st(static_cast<size_t>(segs) * kN, stream);
  DBuf<int> flag(1, stream);
  RP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), stream));
  mt::states_at(seed, progression(0, seg, segs), st.get(), stream);
  uindex_kernel<<<static_cast<unsigned>(segs), kGenThreads, 0, stream>>>(st.get(), seg, count, bound, d_out,
                                                                          flag.get());
  RP_LAUNCH_CHECK();
  int hflag = 0;
  RP_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  if (hflag) {
    sequential_kernel<<<1, kGenThreads, 0, stream>>>(st.get(), 0, count, bound, 0, 0, 0.0, d_out, nullptr, nullptr);
    RP_LAUNCH_CHECK();
  }
}

void gauss_rows_init(uint64_t seed, int64_t rows, int64_t first, int64_t stride, GaussRows& g, cudaStream_t stream) {
  require(rows >= 1, "gaussian rows: need at least one row");
  // Row r starts at normal index c_r = first + r*stride; its window sits at the
  // pair-aligned u64 offset 2*floor(c_r/2).  For odd stride the parity of c_r
  // alternates, so offsets differ by stride +- 1 at doubling level 0 and by
  // an even multiple of stride above -- states_at handles any such schedule.
  std::vector<uint64_t> off(static_cast<size_t>(rows));
  std::vector<int64_t> cur(static_cast<size_t>(rows));
  for (int64_t r = 0; r < rows; ++r) {
    cur[r] = first + r * stride;
    off[r] = static_cast<uint64_t>(cur[r] & ~int64_t{1});
  }
  mt::states_at(seed, off, g.d_states, stream);
  RP_CUDA(cudaMemcpyAsync(g.d_cursor, cur.data(), cur.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  g.rows = rows;
}

namespace {

// Box-Muller exactly as SeededRng::normal (rng.hpp:43-55): u1, u2 from two
// consecutive words, r = sqrt(-2 log u1), cos first, sin second.
// log / sin / cos are glibc's own algorithms and tables (glibc_libm.cuh), so
// the entries equal the reference's bit for bit; without the extracted tables
// (RP_GLIBC_EXACT 0) CUDA's libm is used and entries agree to ~1 ulp.
__device__ __forceinline__ void box_muller(uint64_t w1, uint64_t w2, double& c, double& s) {
  const double u1 = d_uniform01(w1);
  const double u2 = d_uniform01(w2);
  const double two_pi = 6.283185307179586476925286766559;
  const double th = __dmul_rn(two_pi, u2);
#if RP_GLIBC_EXACT
  const double r = __dsqrt_rn(__dmul_rn(-2.0, glibc::log(u1)));
  const double cv = glibc::cos(th), sv = glibc::sin(th);
#else
  const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
  double sv, cv;
  sincos(th, &sv, &cv);
#endif
  c = __dmul_rn(r, cv);
  s = __dmul_rn(r, sv);
}

__global__ void __launch_bounds__(kGenThreads) gauss_rows_kernel(uint64_t* __restrict__ states,
                                                                 int64_t* __restrict__ cursor, int64_t J,
                                                                 double scale, double* __restrict__ out,
                                                                 int64_t ld) {
  __shared__ uint64_t sm[2 * kN];
  const int64_t r = blockIdx.x;
  BlockGen g;
  g.init(sm);
  g.load(states + r * kN);
  const int64_t c0 = cursor[r];
  const int first = static_cast<int>(c0 & 1);  // skip the cos half of the first pair
  const int64_t words_needed = 2 * ((J + first + 1) / 2);
  double* row = out + r * ld;
  constexpr int kPairs = kN / 2;
  int64_t base = 0;
  for (; base < words_needed; base += kN) {
    g.step();
    const int t = threadIdx.x;
    if (t < kPairs) {
      const int64_t p = base / 2 + t;  // pair index within the segment
      double cv, sv;
      box_muller(d_temper(g.cur[2 * t]), d_temper(g.cur[2 * t + 1]), cv, sv);
      const int64_t s0 = 2 * p - first;
      if (s0 >= 0 && s0 < J) row[s0] = __dmul_rn(scale, cv);
      if (s0 + 1 >= 0 && s0 + 1 < J) row[s0 + 1] = __dmul_rn(scale, sv);
    }
  }
  // Advance the window to the pair-aligned offset of the new cursor.
  const int64_t c1 = c0 + J;
  const int64_t P = (c1 & ~int64_t{1}) - (c0 & ~int64_t{1});  // words consumed
  const int64_t last_base = base - kN;
  g.save(states + r * kN, static_cast<int>(P - last_base));
  if (threadIdx.x == 0) cursor[r] = c1;
}

}  // namespace

namespace {
// Normals [first, first + count) of the normal() stream (first even), times
// scale, contiguous: segment s starts at pair-aligned word first + s*seg.
__global__ void __launch_bounds__(kGenThreads) gauss_stream_kernel(const uint64_t* __restrict__ states, int64_t seg,
                                                                   int64_t count, double scale,
                                                                   double* __restrict__ out) {
  __shared__ uint64_t sm[2 * kN];
  BlockGen g;
  g.init(sm);
  g.load(states + static_cast<int64_t>(blockIdx.x) * kN);
  const int64_t start = static_cast<int64_t>(blockIdx.x) * seg;
  const int64_t len = min(seg, count - start);
  constexpr int kPairs = kN / 2;
  for (int64_t done = 0; done < len; done += kN) {
    g.step();
    const int t = threadIdx.x;
    if (t < kPairs) {
      double cv, sv;
      box_muller(d_temper(g.cur[2 * t]), d_temper(g.cur[2 * t + 1]), cv, sv);
      const int64_t q = done + 2 * t;
      if (q < len) out[start + q] = __dmul_rn(scale, cv);
      if (q + 1 < len) out[start + q + 1] = __dmul_rn(scale, sv);
    }
  }
}
}  // namespace

void draw_gauss_stream(uint64_t seed, int64_t first, int64_t count, double scale, double* d_out, cudaStream_t stream) {
  require(first % 2 == 0, "gaussian stream: the first normal must start a pair");
  if (count <= 0) return;
  const int64_t seg = seg_words(count);  // (even: pairs never straddle segments)
  const int64_t segs = ceil_div(count, seg);
  DBuf<uint64_t> st(static_cast<size_t>(segs) * kN, stream);
  mt::states_at(seed, progression(static_cast<uint64_t>(first), seg, segs), st.get(), stream);
  gauss_stream_kernel<<<static_cast<unsigned>(segs), kGenThreads, 0, stream>>>(st.get(), seg, count, scale, d_out);
  RP_LAUNCH_CHECK();
}

void gauss_rows_next(GaussRows& g, int64_t J, double scale, double* d_out, int64_t ld, cudaStream_t stream) {
  if (J <= 0) return;
  gauss_rows_kernel<<<static_cast<unsigned>(g.rows), kGenThreads, 0, stream>>>(g.d_states, g.d_cursor, J, scale,
                                                                                d_out, ld);
  RP_LAUNCH_CHECK();
}

void draw_count(uint64_t seed, int64_t n, int64_t rows_per_block, int blocks, double entry, int32_t* d_h,
                double* d_sgn, cudaStream_t stream) {
  require(rows_per_block >= 1 && blocks >= 1, "count draws: bad block shape");
  const int64_t total_rows = n * blocks;
  if (total_rows == 0) return;
  const int64_t seg_rows = kSegWords / 2;
  const int64_t segs = ceil_div(total_rows, seg_rows);
  DBuf<uint64_t> st(static_cast<size_t>(segs) * kN, stream);
  DBuf<int> flag(1, stream);
  RP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), stream));
  mt::states_at(seed, progression(0, 2 * seg_rows, segs), st.get(), stream);
  count_kernel<<<static_cast<unsigned>(segs), kGenThreads, 0, stream>>>(
      st.get(), seg_rows, total_rows, static_cast<uint64_t>(rows_per_block), entry, d_h, d_sgn, flag.get());
  RP_LAUNCH_CHECK();
  int hflag = 0;
  RP_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  if (hflag) {
    sequential_kernel<<<1, kGenThreads, 0, stream>>>(st.get(), 1, 0, static_cast<uint64_t>(rows_per_block), n,
                                                     blocks, entry, nullptr, d_h, d_sgn);
    RP_LAUNCH_CHECK();
  }
}

void draw_srht(uint64_t seed, int64_t n, int64_t m, double* d_signs, int64_t* d_rows, cudaStream_t stream) {
  int64_t npad = 1;
  while (npad < n) npad <<= 1;
  require(m <= npad, "srht: m must not exceed the padded size");
  // map capacity: power of two >= 4m (at most 2m distinct keys are touched)
  int64_t cap = 1024;
  while (cap < 4 * m) cap <<= 1;
  require(cap <= (int64_t{1} << 22), "srht: m too large for the Fisher-Yates map");
  const bool in_smem = cap <= 8192;
  DBuf<int64_t> keys(in_smem ? 1 : static_cast<size_t>(cap), stream), vals(in_smem ? 1 : static_cast<size_t>(cap), stream);
  // Fast path: all n + m words at once, divisions in parallel.
  DBuf<uint64_t> words(static_cast<size_t>(n + m), stream);
  DBuf<int64_t> jv(static_cast<size_t>(m), stream);
  DBuf<int> flag(1, stream);
  RP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), stream));
  draw_words(seed, 0, n + m, WordMode::Raw, words.get(), stream);
  srht_prep_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n + m, 256), 148 * 8)), 256, 0, stream>>>(
      words.get(), n, m, npad, d_signs, jv.get(), flag.get());
  RP_LAUNCH_CHECK();
  int hflag = 0;
  RP_CUDA(cudaMemcpyAsync(&hflag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  if (!hflag && npad <= 65536) {
    const int bytes = static_cast<int>(npad * sizeof(uint16_t));
    ensure_dynamic_smem(srht_swap_small_kernel, bytes);
    srht_swap_small_kernel<<<1, 256, bytes, stream>>>(jv.get(), m, npad, d_rows);
    RP_LAUNCH_CHECK();
    RP_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  auto go = [&](auto seq_kern, auto swap_kern, bool smem) {
    const int bytes = smem ? static_cast<int>(2 * cap * sizeof(int64_t)) : 0;
    if (!hflag) {
      if (smem) ensure_dynamic_smem(swap_kern, bytes);
      swap_kern<<<1, 256, bytes, stream>>>(jv.get(), m, d_rows, keys.get(), vals.get());
    } else {  // a rejection somewhere: exact sequential consumer from offset n
      DBuf<uint64_t> st(kN, stream);
      mt::states_at(seed, {static_cast<uint64_t>(n)}, st.get(), stream);
      if (smem) ensure_dynamic_smem(seq_kern, bytes);
      seq_kern<<<1, kGenThreads, bytes, stream>>>(st.get(), m, npad, d_rows, keys.get(), vals.get());
      RP_CUDA(cudaStreamSynchronize(stream));
    }
    RP_LAUNCH_CHECK();
  };
#define RP_FY(C, SM) go(srht_fy_kernel<C, SM>, srht_swap_kernel<C, SM>, SM)
  switch (cap) {
    case 1024: RP_FY(1024, true); break;
    case 2048: RP_FY(2048, true); break;
    case 4096: RP_FY(4096, true); break;
    case 8192: RP_FY(8192, true); break;
    case 16384: RP_FY(16384, false); break;
    case 32768: RP_FY(32768, false); break;
    case 65536: RP_FY(65536, false); break;
    case 131072: RP_FY(131072, false); break;
    case 262144: RP_FY(262144, false); break;
    case 524288: RP_FY(524288, false); break;
    case 1048576: RP_FY(1048576, false); break;
    case 2097152: RP_FY(2097152, false); break;
    default: RP_FY(4194304, false); break;
  }
#undef RP_FY
  RP_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace rpb
