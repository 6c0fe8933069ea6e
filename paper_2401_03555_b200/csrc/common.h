// Shared host-side plumbing of libimpact_b200: status/last-error handling,
// CUDA checks, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/impact_b200.h"

namespace imp {

void set_error(const char* fmt, ...);

struct Failure {
  int status;
};

[[noreturn]] inline void fail(int status, const char* msg) {
  set_error("%s", msg);
  throw Failure{status};
}

#define IMP_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      ::imp::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),   \
                       __FILE__, __LINE__, cudaGetErrorString(e_));          \
      throw ::imp::Failure{e_ == cudaErrorMemoryAllocation ? IMP_E_NOMEM      \
                                                           : IMP_E_CUDA};    \
    }                                                                        \
  } while (0)

#define IMP_REQUIRE(cond, ...)                                               \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ::imp::set_error(__VA_ARGS__);                                         \
      throw ::imp::Failure{IMP_E_ARG};                                       \
    }                                                                        \
  } while (0)

// Run a body translating Failure / std exceptions into status codes.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return IMP_OK;
  } catch (const Failure& f) {
    return f.status;
  } catch (const std::exception& e) {
    set_error("internal error: %s", e.what());
    return IMP_E_CUDA;
  }
}

// Device memory comes from the device's stream-ordered pool with the
// release threshold lifted, so the multi-GB CSR of one build is reused by
// the next instead of being unmapped and remapped (cudaFree / cudaMalloc of
// 4-10 GB cost 0.1-3 s of host time per build).  Allocation and release stay
// synchronous, like cudaMalloc / cudaFree: the buffer is ready on return,
// and it is released only after the device is idle.
void* pool_alloc(size_t bytes);
void pool_free(void* p);

// Owning device buffer; movable, not copyable.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n) { o.ptr = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); ptr = o.ptr; n = o.n; o.ptr = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) ptr = static_cast<T*>(pool_alloc(count * sizeof(T)));
  }
  void release() {
    if (ptr) pool_free(ptr);
    ptr = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

}  // namespace imp

// Device-resident abstraction shard.  CSR over the t columns; the target
// and avoid masses ride along as per-row vectors (virtual columns n_s and
// n_s+1 of the reference's stacked bounds, synthesis.py:79-83).
struct imp_imdp {
  int device = 0;
  int32_t n_s = 0, n_u = 1, n_w = 1;
  int32_t k_begin = 0, k_count = 0;
  int64_t n_rows = 0;
  int64_t nnz = 0;
  int32_t max_row = 0;
  imp::DevBuf<int64_t> row_ptr;  // n_rows + 1
  imp::DevBuf<int32_t> col;      // nnz
  imp::DevBuf<double> lo, hi;    // nnz   (t_min, t_max of stored entries)
  imp::DevBuf<double> r_min, r_max, a_min, a_max;  // n_rows
  imp::DevBuf<double> slack;     // n_rows: max(0, 1 - sum(lower))
  imp::DevBuf<double> hd;        // nnz: hi - lo (heads, for the sweep passes
                                 // that read no lower bounds)
  // working set cached by host-driven (sharded) iterations
  void* sweep_cache = nullptr;
  int64_t sweep_cache_rows = -1;
  void (*free_cache)(void*) = nullptr;
  ~imp_imdp() {
    if (sweep_cache && free_cache) free_cache(sweep_cache);
  }
};

namespace imp {
void finalize_imdp(imp_imdp* h, cudaStream_t s);  // slack + max_row
// Kernel launches issued by this library (graph replays count every node):
// our own kernels, and CUB primitive calls (sort / scan) separately.
void count_launches(unsigned long long mine, unsigned long long cub);

// out[i] = in[0] + ... + in[i-1] (exclusive scan of int64, out[0] = 0),
// in-place allowed; our own block-scan kernels (no CUB): the CSR row
// offsets of a build, the text offsets of an export.  Returns launches.
int device_exclusive_scan(const int64_t* in, int64_t* out, int64_t n,
                          cudaStream_t s);
}
