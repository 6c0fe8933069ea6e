// Device -> text export in the reference's file formats.
//
// Reference: pkg/src/impact/fileio.py
//   save_matrix  :94-101   "imdpmat 1 R C" then R lines of C reals
//   save_vector  :118-123  "imdpvec 1 N" then N lines of one real
//   _fmt         :36-41    format(x, ".17g"), fields joined by one space
// The abstraction lives on the device as a cutoff-sparse CSR (common.h), so
// the dense t_min / t_max text -- zeros included -- is rendered by the GPU
// straight from it, a block of rows per call, and only the finished bytes
// cross PCIe.  Every value is formatted by fmt17.h (exact, checked against
// Python's own format).
//
// Layout of one dense row's line (n fields, each followed by ' ' or '\n'):
// a field is "0" unless the column is stored, so the byte offset of field j
// is 2*j + sum over stored columns c < j of (len(c) - 1).
//   k_row_len   one CTA per row: formatted lengths of the stored values,
//               CTA scan -> per-entry extra offsets (scratch) and the line
//               length; a CUB scan over the block's rows gives line offsets
//   k_row_text  one CTA per row: stored values at their offsets, zero runs
//               by binary search of the entry whose extra prefix applies

#include <algorithm>
#include <vector>

#include "common.h"
#include "fmt17.h"

namespace imp {
namespace {

constexpr int XT = 256;   // threads per row CTA

// Exclusive CTA scan of one int per thread (values of a 256-chunk).
__device__ int cta_exclusive_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  int before = 0, tot = 0;
  for (int w = 0; w < XT / 32; ++w) {
    const int t = warp_tot[w];
    if (w < warp) before += t;
    tot += t;
  }
  *total = tot;
  return before + inc - v;
}

struct TextArgs {
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  int64_t row0;        // first row of the block (handle-local)
  int n_cols;
  int* extra;          // (block nnz) per stored entry: sum of (len-1) before it
  int64_t* line_len;   // (rows + 1) line lengths -> exclusive offsets
  const int64_t* line_off;
  char* out;
};

__global__ void __launch_bounds__(XT) k_row_len(TextArgs a) {
  __shared__ int warp_tot[XT / 32];
  const int64_t r = a.row0 + blockIdx.x;
  const int64_t b = a.row_ptr[r], e = a.row_ptr[r + 1];
  const int64_t base = a.row_ptr[a.row0];
  int carry = 0;
  char buf[IMP_FMT17_MAX];
  for (int64_t q0 = b; q0 < e; q0 += XT) {
    const int64_t q = q0 + threadIdx.x;
    const int len = q < e ? imp_fmt17(a.val[q], buf) : 1;
    int tot;
    const int before = cta_exclusive_scan(len - 1, warp_tot, &tot);
    if (q < e) a.extra[q - base] = carry + before;
    carry += tot;
  }
  if (threadIdx.x == 0) a.line_len[blockIdx.x] = 2 * (int64_t)a.n_cols + carry;
}

__global__ void __launch_bounds__(XT) k_row_text(TextArgs a) {
  const int64_t r = a.row0 + blockIdx.x;
  const int64_t b = a.row_ptr[r], e = a.row_ptr[r + 1];
  const int64_t base = a.row_ptr[a.row0];
  const int m = (int)(e - b);
  char* line = a.out + a.line_off[blockIdx.x];
  const int n = a.n_cols;
  // stored fields
  for (int q = threadIdx.x; q < m; q += XT) {
    const int c = a.col[b + q];
    char buf[IMP_FMT17_MAX];
    const int len = imp_fmt17(a.val[b + q], buf);
    char* p = line + 2 * (int64_t)c + a.extra[b - base + q];
    for (int i = 0; i < len; ++i) p[i] = buf[i];
    p[len] = c == n - 1 ? '\n' : ' ';
  }
  // zero fields: extra prefix = that of the first stored column > j, i.e.
  // extra[k] + len_k - 1 of the last stored column < j (or 0)
  for (int j = threadIdx.x; j < n; j += XT) {
    int lo = 0, hi = m;   // first stored index with col >= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (a.col[b + mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo < m && a.col[b + lo] == j) continue;   // stored
    int ex;
    if (lo == m) {
      // after the last stored entry: the row's total extra
      ex = (int)(a.line_len[blockIdx.x + 1] - a.line_off[blockIdx.x]) - 2 * n;
    } else {
      ex = a.extra[b - base + lo];
    }
    char* p = line + 2 * (int64_t)j + ex;
    p[0] = '0';
    p[1] = j == n - 1 ? '\n' : ' ';
  }
}

// fields of a dense host matrix / vector (cols per line)
__global__ void k_vec_len(const double* x, int64_t n, int64_t* len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  char buf[IMP_FMT17_MAX];
  len[i] = imp_fmt17(x[i], buf) + 1;
}

__global__ void k_vec_text(const double* x, int64_t n, int64_t cols,
                           const int64_t* off, char* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  char* p = out + off[i];
  const int len = imp_fmt17(x[i], p);
  p[len] = (i + 1) % cols == 0 ? '\n' : ' ';
}

// exclusive scan of len[0..n) in place into off[0..n]; returns the total
int64_t scan_lengths(const int64_t* len, int64_t* off, int64_t n,
                     cudaStream_t s) {
  // off[0..n] = exclusive scan of len[0..n) with off[n] the total: scan
  // n + 1 values, the last one a zero appended behind a copy of len
  DevBuf<int64_t> ext(n + 1);
  if (n > 0)
    IMP_CUDA(cudaMemcpyAsync(ext.ptr, len, sizeof(int64_t) * n,
                             cudaMemcpyDeviceToDevice, s));
  IMP_CUDA(cudaMemsetAsync(ext.ptr + n, 0, sizeof(int64_t), s));
  device_exclusive_scan(ext.ptr, off, n + 1, s);
  int64_t total = 0;
  IMP_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
  IMP_CUDA(cudaStreamSynchronize(s));
  return total;
}

}  // namespace
}  // namespace imp

using namespace imp;

extern "C" int imp_export_text_rows(const imp_imdp* h, int32_t which,
                                    int64_t row_begin, int64_t row_end,
                                    char* buf, int64_t cap,
                                    int64_t* out_len) {
  return guarded([&] {
    IMP_REQUIRE(h && out_len && (which == 0 || which == 1), "bad argument");
    IMP_REQUIRE(0 <= row_begin && row_begin <= row_end &&
                row_end <= h->n_rows, "row range outside the handle");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = 0;
    const int64_t rows = row_end - row_begin;
    *out_len = 0;
    if (rows == 0) return;
    int64_t rp[2];
    IMP_CUDA(cudaMemcpy(rp, h->row_ptr.ptr + row_begin, sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(rp + 1, h->row_ptr.ptr + row_end, sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
    const int64_t nnz = rp[1] - rp[0];
    DevBuf<int> extra(std::max<int64_t>(nnz, 1));
    DevBuf<int64_t> len(rows + 1), off(rows + 1);
    TextArgs a{};
    a.row_ptr = h->row_ptr.ptr;
    a.col = h->col.ptr;
    a.val = which ? h->hi.ptr : h->lo.ptr;
    a.row0 = row_begin;
    a.n_cols = h->n_s;
    a.extra = extra.ptr;
    a.line_len = len.ptr;
    k_row_len<<<(unsigned)rows, XT, 0, s>>>(a);
    IMP_CUDA(cudaGetLastError());
    const int64_t total = scan_lengths(len.ptr, off.ptr, rows, s);
    *out_len = total;
    if (!buf) return;   // size query
    IMP_REQUIRE(cap >= total, "buffer of %lld bytes, need %lld",
                (long long)cap, (long long)total);
    DevBuf<char> text(std::max<int64_t>(total, 1));
    a.line_len = off.ptr;   // k_row_text reads offsets[r + 1] as line end
    a.line_off = off.ptr;
    a.out = text.ptr;
    k_row_text<<<(unsigned)rows, XT, 0, s>>>(a);
    IMP_CUDA(cudaGetLastError());
    IMP_CUDA(cudaMemcpy(buf, text.ptr, total, cudaMemcpyDeviceToHost));
    count_launches(2, 0);
  });
}

extern "C" int imp_format_values(const double* x, int64_t n, int64_t cols,
                                 int32_t device, char* buf, int64_t cap,
                                 int64_t* out_len) {
  return guarded([&] {
    IMP_REQUIRE((x || n == 0) && out_len && n >= 0 && cols >= 1 &&
                n % cols == 0, "bad argument");
    IMP_CUDA(cudaSetDevice(device));
    cudaStream_t s = 0;
    *out_len = 0;
    if (n == 0) return;
    DevBuf<double> dx(n);
    DevBuf<int64_t> len(n), off(n + 1);
    IMP_CUDA(cudaMemcpy(dx.ptr, x, sizeof(double) * n, cudaMemcpyHostToDevice));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    k_vec_len<<<blocks, 256, 0, s>>>(dx.ptr, n, len.ptr);
    IMP_CUDA(cudaGetLastError());
    const int64_t total = scan_lengths(len.ptr, off.ptr, n, s);
    *out_len = total;
    if (!buf) return;
    IMP_REQUIRE(cap >= total, "buffer of %lld bytes, need %lld",
                (long long)cap, (long long)total);
    DevBuf<char> text(total);
    k_vec_text<<<blocks, 256, 0, s>>>(dx.ptr, n, cols, off.ptr, text.ptr);
    IMP_CUDA(cudaGetLastError());
    IMP_CUDA(cudaMemcpy(buf, text.ptr, total, cudaMemcpyDeviceToHost));
    count_launches(2, 0);
  });
}
