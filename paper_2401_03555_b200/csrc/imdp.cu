// Abstraction handles: import / export / validate / free, error plumbing,
// device facts and the FP64 roofline microbenchmark.
#include <algorithm>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"

namespace imp {

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_mine{0}, g_cub{0};

// --- exclusive scan of int64 (block tiles, then the tile sums) ------------
namespace {
constexpr int SCAN_THREADS = 1024, SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) >= d) v += y;
  }
  return v;
}

// per tile: exclusive scan of the tile into out, the tile total into sums
__global__ void __launch_bounds__(SCAN_THREADS)
    k_scan_tiles(const int64_t* in, int64_t* out, int64_t* sums, int64_t n) {
  __shared__ int64_t warp_tot[SCAN_THREADS / 32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE +
                       (int64_t)threadIdx.x * SCAN_PER;
  int64_t v[SCAN_PER], run = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    run += v[k];
  }
  const int64_t incl = warp_incl_scan(run);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int64_t t = warp_incl_scan(warp_tot[lane]);
    warp_tot[lane] = t;
  }
  __syncthreads();
  int64_t off = incl - run + (warp > 0 ? warp_tot[warp - 1] : 0);
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    const int64_t x = v[k];
    if (base + k < n) out[base + k] = off;
    off += x;
  }
  if (threadIdx.x == SCAN_THREADS - 1) sums[blockIdx.x] = off;
}

__global__ void k_scan_add(int64_t* out, const int64_t* offs, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += offs[i / SCAN_TILE];
}
}  // namespace

int device_exclusive_scan(const int64_t* in, int64_t* out, int64_t n,
                          cudaStream_t s) {
  if (n <= 0) return 0;
  const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  DevBuf<int64_t> sums(tiles);
  k_scan_tiles<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, sums.ptr, n);
  IMP_CUDA(cudaGetLastError());
  int launches = 1;
  if (tiles > 1) {
    launches += device_exclusive_scan(sums.ptr, sums.ptr, tiles, s);
    k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, sums.ptr, n);
    IMP_CUDA(cudaGetLastError());
    ++launches;
  }
  count_launches(tiles > 1 ? 2 : 1, 0);   // this level's kernels
  return launches;
}

void count_launches(unsigned long long mine, unsigned long long cub) {
  g_mine += mine;
  g_cub += cub;
}

void set_error(const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void* pool_alloc(size_t bytes) {
  static std::mutex mu;
  static bool ready[64] = {};
  int dev = 0;
  IMP_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && !ready[dev]) {
      cudaMemPool_t pool;
      IMP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t keep = ~0ull;   // never hand freed blocks back to the OS
      IMP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold,
                                       &keep));
      ready[dev] = true;
    }
  }
  void* p = nullptr;
  IMP_CUDA(cudaMallocAsync(&p, bytes, cudaStreamLegacy));
  IMP_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  return p;
}

void pool_free(void* p) {
  // cudaFree's implicit device synchronisation: the library's streams are
  // non-blocking, so the buffer may still be in use by any of them
  cudaDeviceSynchronize();
  cudaFreeAsync(p, cudaStreamLegacy);
  cudaStreamSynchronize(cudaStreamLegacy);
}

namespace {

// Imdp.validate (reference abstraction.py:121-137) over the CSR shard.
// Writes the first offending row (global min) into *bad.
__global__ void k_validate(const int64_t* row_ptr, const double* lo,
                           const double* hi, const double* r_min,
                           const double* r_max, const double* a_min,
                           const double* a_max, int64_t n_rows, double tol,
                           unsigned long long* bad_interval,
                           unsigned long long* bad_sum) {
  const int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < n_rows; r += nw) {
    int64_t b = row_ptr[r], e = row_ptr[r + 1];
    double s0 = 0.0, s1 = 0.0;
    bool badi = false;
    for (int64_t q = b + lane; q < e; q += 32) {
      double l = lo[q], u = hi[q];
      badi |= (l < 0.0) | (u > 1.0) | (l > u);
      s0 += l;
      s1 += u;
    }
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_down_sync(0xffffffffu, s0, o);
      s1 += __shfl_down_sync(0xffffffffu, s1, o);
    }
    badi = __any_sync(0xffffffffu, badi);
    if (lane == 0) {
      double rl = r_min[r], rh = r_max[r], al = a_min[r], ah = a_max[r];
      badi |= (rl < 0.0) | (rh > 1.0) | (rl > rh) | (al < 0.0) | (ah > 1.0) |
              (al > ah);
      if (badi) atomicMin(bad_interval, (unsigned long long)r);
      double smin = s0 + rl + al, smax = s1 + rh + ah;
      if (smin > 1.0 + tol || smax < 1.0 - tol)
        atomicMin(bad_sum, (unsigned long long)r);
    }
  }
}

__global__ void k_dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9,
         a3 = a0 + 3e-9, a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9,
         a7 = a0 + 7e-9;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c);
      a3 = fma(a3, m, c); a4 = fma(a4, m, c); a5 = fma(a5, m, c);
      a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.0) out[0] = s;
}

}  // namespace
}  // namespace imp

using namespace imp;

extern "C" size_t imp_last_error(char* buf, size_t len) {
  const std::string& m = g_last_error;
  if (buf && len) {
    size_t n = std::min(len - 1, m.size());
    memcpy(buf, m.data(), n);
    buf[n] = 0;
  }
  return m.size();
}

extern "C" const char* imp_version(void) { return "impact_b200 0.1.0 sm_100a"; }

extern "C" void imp_launch_count(unsigned long long* mine,
                                 unsigned long long* cub) {
  if (mine) *mine = g_mine.load();
  if (cub) *cub = g_cub.load();
}

extern "C" int imp_device_query(int device, int* sm_count, int* cc_major,
                                int* cc_minor) {
  return guarded([&] {
    int v = 0;
    IMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    if (sm_count) *sm_count = v;
    IMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device));
    if (cc_major) *cc_major = v;
    IMP_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device));
    if (cc_minor) *cc_minor = v;
  });
}

extern "C" int imp_imdp_import(int device, int32_t n_s, int32_t n_u,
                               int32_t n_w, int32_t k_begin, int64_t n_rows,
                               const int64_t* row_ptr, const int32_t* col,
                               const double* t_lo, const double* t_hi,
                               const double* r_min, const double* r_max,
                               const double* a_min, const double* a_max,
                               imp_imdp** out) {
  imp_imdp* h = nullptr;
  int st = guarded([&] {
    IMP_REQUIRE(out && row_ptr && r_min && r_max && a_min && a_max,
                "null argument");
    IMP_REQUIRE(n_s > 0 && n_u > 0 && n_w > 0 && n_rows >= 0, "bad sizes");
    IMP_REQUIRE(n_rows % ((int64_t)n_u * n_w) == 0,
                "n_rows must be a multiple of n_u*n_w");
    IMP_REQUIRE(row_ptr[0] == 0, "row_ptr[0] must be 0");
    const int64_t nnz = row_ptr[n_rows];
    IMP_REQUIRE(nnz >= 0 && (nnz == 0 || (col && t_lo && t_hi)),
                "missing CSR arrays");
    IMP_CUDA(cudaSetDevice(device));
    h = new imp_imdp();
    h->device = device;
    h->n_s = n_s;
    h->n_u = n_u;
    h->n_w = n_w;
    h->k_begin = k_begin;
    h->k_count = (int32_t)(n_rows / ((int64_t)n_u * n_w));
    IMP_REQUIRE(k_begin >= 0 && k_begin + h->k_count <= n_s,
                "shard outside the safe-state range");
    h->n_rows = n_rows;
    h->nnz = nnz;
    h->row_ptr.alloc(n_rows + 1);
    h->col.alloc(std::max<int64_t>(nnz, 1));
    h->lo.alloc(std::max<int64_t>(nnz, 1));
    h->hi.alloc(std::max<int64_t>(nnz, 1));
    for (auto* b : {&h->r_min, &h->r_max, &h->a_min, &h->a_max})
      b->alloc(std::max<int64_t>(n_rows, 1));
    IMP_CUDA(cudaMemcpy(h->row_ptr.ptr, row_ptr, sizeof(int64_t) * (n_rows + 1),
                        cudaMemcpyHostToDevice));
    if (nnz) {
      for (int64_t q = 0; q < nnz; ++q)
        IMP_REQUIRE(col[q] >= 0 && col[q] < n_s, "column %d out of range",
                    (int)col[q]);
      IMP_CUDA(cudaMemcpy(h->col.ptr, col, sizeof(int32_t) * nnz,
                          cudaMemcpyHostToDevice));
      IMP_CUDA(cudaMemcpy(h->lo.ptr, t_lo, sizeof(double) * nnz,
                          cudaMemcpyHostToDevice));
      IMP_CUDA(cudaMemcpy(h->hi.ptr, t_hi, sizeof(double) * nnz,
                          cudaMemcpyHostToDevice));
    }
    const double* src[4] = {r_min, r_max, a_min, a_max};
    DevBuf<double>* dst[4] = {&h->r_min, &h->r_max, &h->a_min, &h->a_max};
    for (int q = 0; q < 4; ++q)
      if (n_rows)
        IMP_CUDA(cudaMemcpy(dst[q]->ptr, src[q], sizeof(double) * n_rows,
                            cudaMemcpyHostToDevice));
    finalize_imdp(h, 0);
    *out = h;
  });
  if (st != IMP_OK) delete h;
  return st;
}

extern "C" int imp_imdp_info_get(const imp_imdp* h, imp_imdp_info* o) {
  return guarded([&] {
    IMP_REQUIRE(h && o, "null argument");
    o->n_rows = h->n_rows;
    o->row_begin = (int64_t)h->k_begin * h->n_u * h->n_w;
    o->nnz = h->nnz;
    o->n_s = h->n_s;
    o->n_u = h->n_u;
    o->n_w = h->n_w;
    o->k_begin = h->k_begin;
    o->k_count = h->k_count;
    o->max_row = h->max_row;
    o->device = h->device;
  });
}

extern "C" int imp_imdp_export(const imp_imdp* h, int64_t* row_ptr,
                               int32_t* col, double* t_lo, double* t_hi,
                               double* r_min, double* r_max, double* a_min,
                               double* a_max) {
  return guarded([&] {
    IMP_REQUIRE(h, "null handle");
    IMP_CUDA(cudaSetDevice(h->device));
    auto d2h = [](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) IMP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    d2h(row_ptr, h->row_ptr.ptr, sizeof(int64_t) * (h->n_rows + 1));
    d2h(col, h->col.ptr, sizeof(int32_t) * h->nnz);
    d2h(t_lo, h->lo.ptr, sizeof(double) * h->nnz);
    d2h(t_hi, h->hi.ptr, sizeof(double) * h->nnz);
    d2h(r_min, h->r_min.ptr, sizeof(double) * h->n_rows);
    d2h(r_max, h->r_max.ptr, sizeof(double) * h->n_rows);
    d2h(a_min, h->a_min.ptr, sizeof(double) * h->n_rows);
    d2h(a_max, h->a_max.ptr, sizeof(double) * h->n_rows);
  });
}

extern "C" int imp_imdp_validate(const imp_imdp* h, double tol) {
  return guarded([&] {
    IMP_REQUIRE(h, "null handle");
    IMP_CUDA(cudaSetDevice(h->device));
    if (h->n_rows == 0) return;
    DevBuf<unsigned long long> bad(2);
    IMP_CUDA(cudaMemset(bad.ptr, 0xff, 2 * sizeof(unsigned long long)));
    int sms = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    int blocks = (int)std::min<int64_t>((h->n_rows * 32 + 255) / 256,
                                        (int64_t)std::max(sms, 1) * 64);
    k_validate<<<blocks, 256>>>(h->row_ptr.ptr, h->lo.ptr, h->hi.ptr,
                                h->r_min.ptr, h->r_max.ptr, h->a_min.ptr,
                                h->a_max.ptr, h->n_rows, tol, bad.ptr,
                                bad.ptr + 1);
    IMP_CUDA(cudaGetLastError());
    unsigned long long hb[2];
    IMP_CUDA(cudaMemcpy(hb, bad.ptr, sizeof(hb), cudaMemcpyDeviceToHost));
    const long long row0 = (long long)h->k_begin * h->n_u * h->n_w;
    if (hb[0] != ~0ull) {
      set_error("bounds violate 0<=min<=max<=1 (row %lld)", row0 + (long long)hb[0]);
      throw Failure{IMP_E_ABSTRACTION};
    }
    if (hb[1] != ~0ull) {
      set_error("row %lld sum invariant violated; inconsistent noise model",
                row0 + (long long)hb[1]);
      throw Failure{IMP_E_ABSTRACTION};
    }
  });
}

extern "C" void imp_imdp_free(imp_imdp* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  delete h;
}

extern "C" int imp_fp64_peak(int device, double* gflops) {
  return guarded([&] {
    IMP_REQUIRE(gflops, "null argument");
    IMP_CUDA(cudaSetDevice(device));
    int sms = 0;   // queried below
    IMP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DevBuf<double> o(1);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    k_dfma_peak<<<blocks, threads>>>(o.ptr, 64);  // warm-up
    IMP_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    IMP_CUDA(cudaEventCreate(&e0));
    IMP_CUDA(cudaEventCreate(&e1));
    IMP_CUDA(cudaEventRecord(e0));
    k_dfma_peak<<<blocks, threads>>>(o.ptr, iters);
    IMP_CUDA(cudaEventRecord(e1));
    IMP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    *gflops = flops / (ms * 1e-3) / 1e9;
  });
}
