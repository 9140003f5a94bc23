// Shared definitions for the ridgepath B200 library (CUDA + host C++).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace rpb {

// Error categories map 1:1 onto rp_status (include/ridgepath_b200.h) and onto
// the reference's exception types (path_solver.hpp:18-27, std::invalid_argument,
// std::runtime_error from thin_svd, matrix.cpp:227-228).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct BasisDiverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FactorFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// ParseError (data_io.hpp): message "line L, column C: ...", 1-based position.
struct ParseFailure : std::runtime_error {
  ParseFailure(const std::string& msg, int64_t l, int64_t c) : std::runtime_error(msg), line(l), column(c) {}
  int64_t line, column;
};
struct NcclFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool cond, const char* msg) {
  if (!cond) throw InvalidArgument(msg);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                      std::to_string(line));
}

#define RP_CUDA(x) ::rpb::cuda_check((x), #x, __FILE__, __LINE__)
// Every kernel launch of the library goes through RP_LAUNCH_CHECK, which also
// counts it (the bench reports the count as gpu_launches).
inline std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}
#define RP_LAUNCH_CHECK()                                                              \
  do {                                                                                 \
    ::rpb::launch_counter().fetch_add(1, std::memory_order_relaxed);                  \
    ::rpb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);         \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }


// Raises a kernel's dynamic shared-memory limit on the current device to at
// least `bytes`, never lowering it: the attribute is per function and device,
// shared by every thread and context, so a caller needing less must not
// undercut another's launch (a lowered limit fails that launch with "invalid
// argument").
inline void ensure_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> limits;
  int dev = 0;
  RP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = limits[{func, dev}];
  if (bytes > cur) {
    RP_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    cur = bytes;
  }
}
template <class F>
void ensure_dynamic_smem(F* func, size_t bytes) {
  ensure_dynamic_smem(reinterpret_cast<const void*>(func), bytes);
}

}  // namespace rpb

namespace rpb {

// Stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync).
template <class T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t s) {
    release();
    s_ = s;
    n_ = n;
    if (n) {
      void* p = nullptr;
      const cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), s);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw CudaFailure(std::string("device allocation of ") + std::to_string(n * sizeof(T)) +
                          " bytes failed: " + cudaGetErrorString(e));
      }
      p_ = static_cast<T*>(p);
    }
  }
  void release() {
    if (p_) {
      cudaFreeAsync(p_, s_);
    }
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  cudaStream_t stream() const { return s_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

}  // namespace rpb
