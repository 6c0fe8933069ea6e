// Interval iteration on the B200: global stable order (K4), twin greedy-LP
// sweep over cutoff-sparse rows (K5), robust Bellman reduction, and the
// on-device termination logic of the reference's _run_phase.
//
// Reference semantics (pkg/src/impact/):
//   weight_order   feasible.py:53-58  stable argsort, desc for max, -0 == +0
//   RowsSolver     feasible.py:80-111 val = lower.w + min(cumsum(head[order]),
//                                     slack) . dw  (Abel form of the greedy fill)
//   bellman_step   synthesis.py:97-135 min/max over disturbances, first
//                                     arg-best input
//   _run_phase     synthesis.py:145-205 monotone / k0,k1 / bracket / gap /
//                                     stall fallback / horizon / cap
//   diagnose_convergence synthesis.py:321-361
//
// K5 uses the early-exit form of the greedy fill: with
// P = the largest global rank such that sum_{rank<P} head < slack, a row's
// value is  sum(l*w) + sum_{rank<P} head*w + (slack - C(<P)) * w_sorted[P].
// One streaming pass per row (pass A) verifies last sweep's crossing column
// with certified float sums and walks a captured rank window when the
// crossing moved a little; larger moves use an exact integer (2^-88 fixed
// point) bucketed search with shared-memory atomics.  The value is always
// built from the canonical per-lane float sums below P with a fixed team
// tree (k_sweep, below), so it depends only on a row's contents and the
// shared order -- never on the hint, the path taken, its position or its
// shard: bitwise-identical rows give bitwise-identical values.
#include <type_traits>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.h"

namespace imp {

constexpr unsigned FULL = 0xffffffffu;

// SM count of a device (grid sizing: persistent grids are a multiple of it)
inline int sm_count_of(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) !=
          cudaSuccess || v <= 0)
    v = 1;
  return v;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// Order-preserving map double -> uint64 (ascending), -0.0 folded onto +0.0
// so that the stable radix sort matches numpy's comparison sort.
__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Deterministic warp sum: xor butterfly.  Partners add the same two
// operands (a + b == b + a in IEEE), so after five steps every lane holds
// the bit-identical total, with no broadcast.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Packed value layout of the device-resident sharded loop: the value
// vectors of every rank's shard side by side, [rank][track][pw] (pw >= the
// largest shard), so one in-place all-gather of a rank's [V0' | V1'] chunk
// refreshes both full vectors.  sb = shard begins (world + 1).
struct Packed {
  const int64_t* sb;   // nullptr: plain layout v[t][p][c]
  int world;
  int64_t pw;
};

__device__ __forceinline__ int64_t vpos(const Packed& pk, int t, int64_t c) {
  if (!pk.sb) return c;
  int r = 0;
  for (int q = 1; q < pk.world; ++q) r += c >= pk.sb[q];
  return ((int64_t)r * 2 + t) * pk.pw + (c - pk.sb[r]);
}

// Control block of a phase loop living in device memory.  Kernels of an
// iteration read `done` and return immediately once the loop terminated, so
// a CUDA graph of G iterations can be replayed without host round trips.
struct Ctl {
  long long it;       // completed iterations
  int done;
  int status;         // imp_status
  int fallback;
  int has_prev;
  int cur;            // ping-pong buffer holding the current values
  int mode;           // IMP_MODE_*
  int frozen0, frozen1;
  long long k0, k1;   // -1 == None
  double prev_gap, gap, eps;
  long long horizon, max_iter;
  unsigned long long slot_d0, slot_d1, slot_gap;  // order_key-encoded maxima
  unsigned int slot_flags;                        // 1: monotone, 2: bracket
  // the gap at every 1000th iteration that continued (the reference logs
  // it, synthesis.py:204-205), first GAP_LOG of them
  int gap_log_n;
  double gap_log[256];
};
constexpr int GAP_LOG = 256;

// ---------------------------------------------------------------------------
// K4: global order of the (n_s + 2) weights of both tracks
// ---------------------------------------------------------------------------

struct OrderArgs {
  const double* v[2][2];    // [track][pingpong] values (n_s), or explicit
  const Ctl* ctl;           // selects pingpong; nullptr -> v[t][0]
  int n_s, n;               // n = n_s + 2
  double d1, d2;            // virtual-slot weights (reach: 1,0; safety: 0,1)
  int lp_max;
  uint64_t* keys[2];
  int* idx[2];
  double2* colw;            // (n) {w0, w1} by column
  Packed pk;                // sharded loop: packed value layout
};

__global__ void k_order_keys(OrderArgs a) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n) return;
  if (a.ctl && a.ctl->done) return;
  int pp = a.ctl ? a.ctl->cur : 0;
  double w[2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
    w[t] = c < a.n_s ? a.v[t][pp][vpos(a.pk, t, c)]
                     : (c == a.n_s ? a.d1 : a.d2);
  a.colw[c] = make_double2(w[0], w[1]);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    a.keys[t][c] = order_key(a.lp_max ? -w[t] : w[t]);
    a.idx[t][c] = c;
  }
}

struct RankArgs {
  const Ctl* ctl;
  int n;
  const int* perm[2];
  const double2* colw;
  int2* rank;               // (n) {rank0, rank1} by column
  unsigned* rank16;         // (n) packed rank0 | rank1 << 16 (n <= 65536)
  double* ws[2];            // (n + 1) weights in sorted order, ws[n] = 0
};

__global__ void k_ranks(RankArgs a) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > a.n) return;
  if (a.ctl && a.ctl->done) return;
  if (p == a.n) {
    a.ws[0][p] = 0.0;
    a.ws[1][p] = 0.0;
    return;
  }
  int c0 = a.perm[0][p], c1 = a.perm[1][p];
  a.rank[c0].x = p;
  a.rank[c1].y = p;
  a.ws[0][p] = a.colw[c0].x;
  a.ws[1][p] = a.colw[c1].y;
}

__global__ void k_pack_ranks(const Ctl* ctl, int n, const int2* rank,
                             unsigned* rank16) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (ctl && ctl->done) return;
  int2 r = rank[c];
  rank16[c] = (unsigned)r.x | ((unsigned)r.y << 16);
}

// ---------------------------------------------------------------------------
// K4 sort: the stable order of both tracks' keys (numpy's argsort(kind=
// "stable"), feasible.py:53-58).  Sorting the pairs (key, column) by key
// then column is a total order, so any correct sort is the stable sort.
// Tiles of SORT_TILE pairs are bitonic-sorted in shared memory (one CTA per
// tile and track), then merge passes of doubling width (merge path: each
// thread finds its split of the two runs by binary search and merges a
// fixed stretch of the output) until one run remains: 1 + ceil(log2(tiles))
// launches for both tracks (robot2d: 1; vehicle3d: 3; bas7d: 7).
// ---------------------------------------------------------------------------
constexpr int SORT_TILE = 2048;      // pairs per tile (1 024 threads, 2 each)
constexpr int MERGE_CHUNK = 2048;    // outputs per merge CTA
constexpr int MERGE_THREADS = 256;   // -> 8 outputs per thread

__device__ __forceinline__ bool pair_less(uint64_t ka, int ia, uint64_t kb,
                                          int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

struct SortArgs {
  const Ctl* ctl;
  int n;
  uint64_t* key_in[2];   // per track
  int* idx_in[2];
  uint64_t* key_out[2];
  int* idx_out[2];
  int width;             // merge: current run width
};

__global__ void __launch_bounds__(SORT_TILE / 2)
    k_sort_tiles(SortArgs a) {
  if (a.ctl && a.ctl->done) return;
  __shared__ uint64_t sk[SORT_TILE];
  __shared__ int si[SORT_TILE];
  const bool t1 = blockIdx.y != 0;   // track (selects, no local copies)
  const uint64_t* kin = t1 ? a.key_in[1] : a.key_in[0];
  const int* iin = t1 ? a.idx_in[1] : a.idx_in[0];
  uint64_t* kout = t1 ? a.key_out[1] : a.key_out[0];
  int* iout = t1 ? a.idx_out[1] : a.idx_out[0];
  const int base = blockIdx.x * SORT_TILE;
  for (int q = threadIdx.x; q < SORT_TILE; q += blockDim.x) {
    const int g = base + q;
    sk[q] = g < a.n ? kin[g] : ~0ull;
    si[q] = g < a.n ? iin[g] : INT_MAX;
  }
  __syncthreads();
  const int p = threadIdx.x;
  for (int k = 2; k <= SORT_TILE; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int i = (p / j) * 2 * j + (p % j);
      const int l = i + j;
      const bool up = (i & k) == 0;
      const uint64_t ki = sk[i], kl = sk[l];
      const int ii = si[i], il = si[l];
      if (pair_less(kl, il, ki, ii) == up) {
        sk[i] = kl; si[i] = il;
        sk[l] = ki; si[l] = ii;
      }
      __syncthreads();
    }
  }
  for (int q = threadIdx.x; q < SORT_TILE; q += blockDim.x) {
    const int g = base + q;
    if (g < a.n) {
      kout[g] = sk[q];
      iout[g] = si[q];
    }
  }
}

__global__ void __launch_bounds__(MERGE_THREADS) k_merge_pass(SortArgs a) {
  if (a.ctl && a.ctl->done) return;
  const bool t1 = blockIdx.y != 0;
  const int w = a.width;
  const int n = a.n;
  constexpr int PER = MERGE_CHUNK / MERGE_THREADS;
  const int o = blockIdx.x * MERGE_CHUNK + threadIdx.x * PER;  // output pos
  if (o >= n) return;
  const int pair0 = (o / (2 * w)) * 2 * w;
  const int a0 = pair0, a1 = min(pair0 + w, n);
  const int b0 = a1, b1 = min(pair0 + 2 * w, n);
  const uint64_t* K = t1 ? a.key_in[1] : a.key_in[0];
  const int* I = t1 ? a.idx_in[1] : a.idx_in[0];
  const int na = a1 - a0, nb = b1 - b0;
  const int diag = o - pair0;
  // merge path: the number i of A elements among the first diag outputs
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    const int i = (lo + hi) >> 1;
    const int j = diag - 1 - i;
    // A[i] comes before B[j] -> more A elements
    if (pair_less(K[a0 + i], I[a0 + i], K[b0 + j], I[b0 + j])) lo = i + 1;
    else hi = i;
  }
  int i = lo, j = diag - lo;
  uint64_t* KO = t1 ? a.key_out[1] : a.key_out[0];
  int* IO = t1 ? a.idx_out[1] : a.idx_out[0];
  const int end = min(o + PER, pair0 + na + nb);
  for (int q = o; q < end; ++q) {
    bool take_a;
    if (i >= na) take_a = false;
    else if (j >= nb) take_a = true;
    else take_a = pair_less(K[a0 + i], I[a0 + i], K[b0 + j], I[b0 + j]);
    if (take_a) { KO[q] = K[a0 + i]; IO[q] = I[a0 + i]; ++i; }
    else { KO[q] = K[b0 + j]; IO[q] = I[b0 + j]; ++j; }
  }
}

// perm[t] (column by rank) of keys[t] / idx[t] (idx = column on entry;
// keys and idx are clobbered).  Returns the number of launches.
int launch_sort(const Ctl* ctl, int n, uint64_t* const keys[2],
                int* const idx[2], uint64_t* const keys_tmp[2],
                int* const perm[2], cudaStream_t s) {
  if (n <= 0) return 0;
  const int tiles = (n + SORT_TILE - 1) / SORT_TILE;
  int passes = 0;
  while ((SORT_TILE << passes) < n) ++passes;
  // ping-pong so that the last pass writes (keys_tmp, perm)
  SortArgs A{};
  A.ctl = ctl;
  A.n = n;
  for (int t = 0; t < 2; ++t) {
    A.key_in[t] = keys[t];
    A.idx_in[t] = idx[t];
    A.key_out[t] = passes % 2 ? keys[t] : keys_tmp[t];
    A.idx_out[t] = passes % 2 ? idx[t] : perm[t];
  }
  k_sort_tiles<<<dim3(tiles, 2), SORT_TILE / 2, 0, s>>>(A);
  IMP_CUDA(cudaGetLastError());
  uint64_t* ck[2] = {A.key_out[0], A.key_out[1]};
  int* ci[2] = {A.idx_out[0], A.idx_out[1]};
  for (int p = 0; p < passes; ++p) {
    SortArgs M{};
    M.ctl = ctl;
    M.n = n;
    M.width = SORT_TILE << p;
    for (int t = 0; t < 2; ++t) {
      M.key_in[t] = ck[t];
      M.idx_in[t] = ci[t];
      M.key_out[t] = ck[t] == keys[t] ? keys_tmp[t] : keys[t];
      M.idx_out[t] = ci[t] == idx[t] ? perm[t] : idx[t];
      ck[t] = M.key_out[t];
      ci[t] = M.idx_out[t];
    }
    k_merge_pass<<<dim3((n + MERGE_CHUNK - 1) / MERGE_CHUNK, 2),
                   MERGE_THREADS, 0, s>>>(M);
    IMP_CUDA(cudaGetLastError());
  }
  return 1 + passes;
}

// ---------------------------------------------------------------------------
// K5: twin greedy-LP sweep
// ---------------------------------------------------------------------------

struct SweepArgs {
  const Ctl* ctl;
  const int64_t* row_ptr;
  const int32_t* col;
  const double* lo;
  const double* hi;
  const double* hd;         // hi - lo per stored entry (finalize_imdp)
  const double* r_min;
  const double* r_max;
  const double* a_min;
  const double* a_max;
  const double* slack;
  const double2* colw;
  const int2* rank;
  const unsigned* rank16;
  const double* ws0;
  const double* ws1;
  const int64_t* fixed;     // phase-2 policy (local states) or nullptr
  int64_t n_phase_rows;
  int n_u, n_w, n_s, n, nbits;
  // phase rows of this launch's class (a fixed function of the row's own
  // stored length m, so the kernel -- hence the summation tree -- a row
  // gets never depends on its shard or neighbours)
  const int* list;
  int64_t n_list;
  unsigned long long* miss_total;  // IMP_SWEEP_STATS: [rows off the hint,
                                   //  rows needing the bucketed search]
  int* hint;            // (2 * n_phase_rows) last sweep's crossing columns
  const int* perm0;     // columns by rank (hint publication)
  const int* perm1;
  double* out0;
  double* out1;
};

template <bool WIDE>
struct RankReg;
template <>
struct RankReg<false> {
  unsigned r;
  __device__ __forceinline__ int r0() const { return (int)(r & 0xffffu); }
  __device__ __forceinline__ int r1() const { return (int)(r >> 16); }
  __device__ __forceinline__ void load(const SweepArgs& a, int c) {
    r = __ldg(a.rank16 + c);
  }
  __device__ __forceinline__ void none() { r = 0xffffffffu; }
};
template <>
struct RankReg<true> {
  int x, y;
  __device__ __forceinline__ int r0() const { return x; }
  __device__ __forceinline__ int r1() const { return y; }
  __device__ __forceinline__ void load(const SweepArgs& a, int c) {
    int2 v = __ldg(a.rank + c);
    x = v.x;
    y = v.y;
  }
  __device__ __forceinline__ void none() { x = y = 0x7fffffff; }
};

__device__ __forceinline__ int64_t phase_row(const SweepArgs& a, int64_t t) {
  if (!a.fixed) return t;
  int64_t k = t / a.n_w, i = t - k * a.n_w;
  return (k * a.n_u + a.fixed[k]) * a.n_w + i;
}

// A row's value from its team-reduced sums (both K5 kernels use exactly
// this expression): lower mass + filled head below the crossing rank P +
// the partial fill of slot P.
__device__ __forceinline__ double row_value(double lw, double f, double s,
                                            double c, int p, int n,
                                            const double* ws) {
  const double x = p < n ? fma(s - c, __ldg(ws + p), f) : f;
  return lw + x;
}

// ---------------------------------------------------------------------------
// Exact crossing arithmetic.  Each head h = hi - lo in [0, 1] is rounded to
// the 2^-88 grid, h~ = RN(h * 2^88) / 2^88 (error <= 2^-89 per slot), and
// C(<q) = sum of h~ over the row's slots of rank < q is an exact integer
// multiple of 2^-88.  Integer sums do not depend on summation order, so the
// crossing P (largest q with C(<q) < slack) is one well-defined number
// however it is found: a verify pass at last sweep's crossing, or a
// bucketed search with shared-memory atomics.
// h~ is held as h~ * 2^88 = A * 2^44 + B (A = RN(h * 2^44) >= 0, B the
// signed remainder, |B| <= 2^43), obtained with two magic-number roundings
// in FP64 (no integer shifting).  Partial sums of A and of B over < 2^20
// slots stay below 2^64 / 2^63 in magnitude: plain 64-bit adds, no carries.
// ---------------------------------------------------------------------------

typedef unsigned __int128 u128;
constexpr int FIX_BITS = 88;

struct Fix {
  uint64_t a, b;   // b: two's-complement int64
};

__device__ __forceinline__ Fix to_fix(double h) {
  const double M1 = 384.0;       // 1.5 * 2^8: on [256, 512) the ulp is 2^-44
  const double M2 = 0x1.8p52;    // 1.5 * 2^52: ulp 1
  const double t = __dadd_rn(h, M1);            // 384 + RN(h, 2^-44)
  const double r = __dsub_rn(h, __dsub_rn(t, M1));  // exact, |r| <= 2^-45
  const double t2 = __fma_rn(r, 0x1p88, M2);    // M2 + RN(r * 2^88)
  return Fix{(uint64_t)(__double_as_longlong(t) - __double_as_longlong(M1)),
             (uint64_t)(__double_as_longlong(t2) - __double_as_longlong(M2))};
}

// Add h~ = {a, b} into a histogram bucket (two 64-bit words) with native
// 32-bit shared-memory atomics: 64-bit shared atomicAdd is a CAS spin loop
// on sm_100a.  The low words carry into the high words (detected from the
// returned old value), so each 64-bit word ends as the exact sum mod 2^64:
// a's sum stays below 2^64, b's is a two's-complement int64 -- the words
// the scan reads are bit-identical to 64-bit adds.
__device__ __forceinline__ void hist_add(unsigned long long* hb, Fix x) {
  unsigned* w = reinterpret_cast<unsigned*>(hb);
  const unsigned alo = (unsigned)x.a, ahi = (unsigned)(x.a >> 32);
  const unsigned blo = (unsigned)x.b, bhi = (unsigned)(x.b >> 32);
  const unsigned oa = atomicAdd(w, alo);
  const unsigned ob = atomicAdd(w + 2, blo);
  atomicAdd(w + 1, ahi + (oa + alo < oa ? 1u : 0u));
  atomicAdd(w + 3, bhi + (ob + blo < ob ? 1u : 0u));
}

__device__ __forceinline__ u128 fix_value(uint64_t a, uint64_t b) {
  return (u128)(((__int128)a << 44) + (__int128)(int64_t)b);
}

// ceil(s * 2^88): C < s  <=>  C * 2^88 < ceil(s * 2^88) for integer C * 2^88
__device__ __forceinline__ u128 fix_ceil(double s) {
  if (!(s > 0.0)) return 0;
  const uint64_t u = (uint64_t)__double_as_longlong(s);
  const int e = (int)((u >> 52) & 0x7ff);
  if (e == 0) return 1;
  const uint64_t M = (u & 0xfffffffffffffull) | (1ull << 52);
  const int sh = e - 1075 + FIX_BITS;
  if (sh >= 0) return (u128)M << sh;
  const int k = -sh;
  if (k >= 64) return 1;
  return (u128)((M >> k) + ((M & ((1ull << k) - 1)) != 0));
}


// Team sums.  Floats: per value a warp xor butterfly, then (CTA teams) warp
// partials through shared memory re-reduced by every warp -- a fixed tree,
// so a row's sums depend only on its contents and TEAM.  Integers: exact.
template <int TEAM, int K>
__device__ __forceinline__ void team_sum_f(double* v, double* part) {
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if constexpr (TEAM > 32) {
    constexpr int NW = TEAM / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) part[k * NW + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] = warp_sum(lane < NW ? part[k * NW + lane] : 0.0);
    __syncthreads();
  }
}

// Pass-A team sums of 6 doubles (the fixed tree of team_sum_f) in one
// exchange; CTA teams clear `clear` (the window buffer of the next row)
// between the two barriers, where no teammate can still be reading it
// (last row) or already writing it (next row).
template <int TEAM>
__device__ __forceinline__ void team_sum_pass_a(double* f, double* fpart,
                                                double* clear, int n_clear) {
#pragma unroll
  for (int k = 0; k < 6; ++k) f[k] = warp_sum(f[k]);
  if constexpr (TEAM > 32) {
    constexpr int NW = TEAM / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 6; ++k) fpart[k * NW + warp] = f[k];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n_clear; q += TEAM) clear[q] = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k)
      f[k] = warp_sum(lane < NW ? fpart[k * NW + lane] : 0.0);
    __syncthreads();
  } else {
    __syncwarp();
    for (int q = threadIdx.x & 31; q < n_clear; q += 32) clear[q] = 0.0;
    __syncwarp();
  }
}

// Exact sums.  Besides the crossing's C(<q) = sum h~, the filled part of
// the value, F(<q) = sum_{rank<q} h*w, is also summed exactly: each product
// is rounded to the 2^-88 grid once, (h w)~ (h, w in [0, 1]; error <= 2^-89
// per slot, < 2^-68 per row), and summed as an integer.  Integer sums do not
// depend on order, so F and C at any rank follow from F and C at another by
// adding or removing the slots in between -- a crossing that moved inside
// the captured window needs no second pass over the row, and the value
// lw + F(<P) + (s - C(<P)) w_sorted[P] is a pure function of (row, weights)
// whichever path found P.
__device__ __forceinline__ void fix_add(Fix& s, Fix x) { s.a += x.a; s.b += x.b; }
__device__ __forceinline__ void fix_sub(Fix& s, Fix x) { s.a -= x.a; s.b -= x.b; }
__device__ __forceinline__ u128 fixv(Fix x) { return fix_value(x.a, x.b); }

// deterministic double of an exact non-negative sum (two roundings)
__device__ __forceinline__ double fix_double(u128 v) {
  return fma((double)(uint64_t)(v >> 64), 0x1p-24,
             (double)(uint64_t)v * 0x1p-88);
}

__device__ __forceinline__ Fix warp_sum_fix(Fix x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x.a += __shfl_xor_sync(FULL, x.a, o);
    x.b += __shfl_xor_sync(FULL, x.b, o);
  }
  return x;
}

// Team sums of K exact values (any order: integers)
template <int TEAM, int K>
__device__ __forceinline__ void team_sum_fix(Fix* v, Fix* part) {
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum_fix(v[k]);
  if constexpr (TEAM > 32) {
    constexpr int NW = TEAM / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) part[k * NW + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k)
      v[k] = warp_sum_fix(lane < NW ? part[k * NW + lane] : Fix{0, 0});
    __syncthreads();
  }
}

// Warm-start hints, one int per (row, track): the crossing column of the
// last sweep (HINT_COL: none, P = n) with HINT_SEARCHED set if that sweep
// needed the bucketed search; negative: unknown (first sweep).
constexpr int HINT_COL = 0x1fffffff;       // value mask; also "P = n"
constexpr int HINT_RANKMODE = 0x20000000;  // value is last P (rank), not
                                           // the crossing column
constexpr int HINT_SEARCHED = 0x40000000;

// A row's crossing hint for this sweep: the rank, in this sweep's order, of
// last sweep's crossing column (column mode), or last sweep's crossing rank
// itself (rank mode: rows whose column order scrambles among near-equal
// values, e.g. dim14's symmetric states).  A row whose hint missed (it
// searched) switches mode for the next sweep.
template <bool WIDE>
__device__ __forceinline__ int hint_rank(const SweepArgs& a, int h, int track) {
  const int v = h & HINT_COL;
  if (v == HINT_COL) return a.n;
  if (h & HINT_RANKMODE) return v < a.n ? v : a.n;
  RankReg<WIDE> r;
  r.load(a, v);
  return track ? r.r1() : r.r0();
}

__device__ __forceinline__ int hint_encode(const SweepArgs& a, int old, int P,
                                           const int* perm, bool searched,
                                           bool adaptive) {
  const bool rank_mode =
      adaptive && (((old & HINT_RANKMODE) != 0) != searched);
  const int v = P >= a.n ? HINT_COL : (rank_mode ? P : __ldg(perm + P));
  return v | (rank_mode ? HINT_RANKMODE : 0) | (searched ? HINT_SEARCHED : 0);
}

// Buckets per search level: CTA teams 256, warp teams 32.
template <int TEAM>
struct K5Shape {
  static constexpr int NW = TEAM > 32 ? TEAM / 32 : 1;
#ifndef IMP_K5_LOGB_WARP
#define IMP_K5_LOGB_WARP 5
#endif
  static constexpr int LOGB = TEAM > 32 ? 8 : IMP_K5_LOGB_WARP;
  static constexpr int B = 1 << LOGB;
  // per team: float partials, integer partials, histogram [track][bucket]
  // {a, b}, search broadcast
  static constexpr int F_PART = 6 * NW;
  static constexpr int HIST = 2 * B * 2;
  // pass A captures {h, w} of the slots with rank in [g - W, g + W) per
  // track, so a crossing that moved by < W ranks is resolved exactly from
  // shared memory, with no further pass over the row
#ifndef IMP_K5_WWARP
#define IMP_K5_WWARP 32
#endif
#ifndef IMP_K5_WCTA
#define IMP_K5_WCTA 256
#endif
// 256-rank windows for every CTA class (vehicle3d 239 -> 256 phase-1
// sweeps/s, dim14 541 -> 641; the 128-thread class with a single buffer,
// see IMP_K5_WSINGLE.  profiles/r02/k5_window_ab.txt)
#ifndef IMP_K5_WCTA_BIG
#define IMP_K5_WCTA_BIG IMP_K5_WCTA
#endif
  static constexpr int W = TEAM > 32 ? (TEAM >= 256 ? IMP_K5_WCTA_BIG : IMP_K5_WCTA)
                                     : IMP_K5_WWARP;
  static constexpr int WIN = 2 * 2 * W;   // [track][slot] {h, w}
};

// Stream the row's slots in the canonical per-lane order -- entries
// q = tid, tid + TEAM, ... (U loads in flight), then the two virtual slots
// on team thread 0 -- calling f(l, h, w, rank) for each.  Heads come from
// the precomputed hd = hi - lo (bit-identical to forming it here); passes
// that need no lower bound (NEED_L false: search levels, the F pass) read
// 12 B per entry instead of 20 B, and get l = 0.
template <int TEAM, bool WIDE, bool NEED_L = true, class Fn>
__device__ __forceinline__ void for_slots(const SweepArgs& a, int tid,
                                          int64_t row, int64_t beg, int m,
                                          Fn&& f) {
#ifndef IMP_K5_U
#define IMP_K5_U 4
#endif
  constexpr int U = IMP_K5_U;
  const int32_t* colp = a.col + beg;
  const double* lop = a.lo + beg;
  const double* hdp = a.hd + beg;
  for (int q = tid; q < m; q += U * TEAM) {
    int c[U];
    double l[U], u[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int qq = q + k * TEAM;
      c[k] = -1;
      l[k] = u[k] = 0.0;
      if (qq < m) {
        c[k] = __ldg(colp + qq);
        if (NEED_L) l[k] = __ldg(lop + qq);
        u[k] = __ldg(hdp + qq);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (c[k] >= 0) {
        RankReg<WIDE> rk;
        rk.load(a, c[k]);
        f(l[k], u[k], __ldg(a.colw + c[k]), rk);
      }
    }
  }
  if (tid == 0) {   // virtual slots n_s (target) and n_s + 1 (avoid)
    const double lr = a.r_min[row], la = a.a_min[row];
    const double hr = a.r_max[row] - lr, ha = a.a_max[row] - la;
    RankReg<WIDE> rk;
    rk.load(a, a.n_s);
    f(lr, hr, __ldg(a.colw + a.n_s), rk);
    rk.load(a, a.n_s + 1);
    f(la, ha, __ldg(a.colw + a.n_s + 1), rk);
  }
}

// Team-uniform state of the bucketed search (shared memory).
struct SearchState {
  u128 cb[2];      // exact C(< lo) of the current range
  u128 C[2];       // result: C(<P)
  int lo[2], lg[2];  // current rank range [lo, lo + 2^lg)
  int P[2];        // result
  int pick[2];     // bucket chosen by the scan (-1: none)
  int act;         // bit o: track o still searching
};

// Levels of the exact search: each level is one pass over the row adding
// every in-range slot's h~ into its rank bucket (shared-memory atomics:
// exact, order-free), then one warp scans the buckets for the first whose
// inclusive cumulative sum reaches s; the range shrinks to that bucket.
// On return st.P / st.C hold P and C(<P) of every track searched.
template <int TEAM, bool WIDE>
__device__ __noinline__ void search_levels(const SweepArgs& a, int tid,
                                           int64_t row, int64_t beg, int m,
                                           double s, SearchState& st,
                                           unsigned long long* hist,
                                           bool prefilled) {
  using SH = K5Shape<TEAM>;
  auto team_sync = [] {
    if constexpr (TEAM == 32) __syncwarp();
    else __syncthreads();
  };
  const u128 S = fix_ceil(s);
  bool fill = !prefilled;   // level 1 may come filled from pass A
  while (st.act) {
    const int act = st.act;
    const int lo0 = st.lo[0], lo1 = st.lo[1];
    const int w0 = (act & 1) ? 1 << st.lg[0] : 0;
    const int w1 = (act & 2) ? 1 << st.lg[1] : 0;
    const int sh0 = max(0, st.lg[0] - SH::LOGB), sh1 = max(0, st.lg[1] - SH::LOGB);
    if (fill) {
    for (int q = tid; q < SH::HIST; q += TEAM) hist[q] = 0ull;
    team_sync();
    for_slots<TEAM, WIDE, false>(a, tid, row, beg, m,
        [&](double, double h, double2, const RankReg<WIDE>& rk) {
          const unsigned d0 = (unsigned)(rk.r0() - lo0);
          const unsigned d1 = (unsigned)(rk.r1() - lo1);
          const bool in0 = d0 < (unsigned)w0, in1 = d1 < (unsigned)w1;
          if (!(in0 || in1)) return;
          const Fix x = to_fix(h);
          if (in0) hist_add(hist + (d0 >> sh0) * 2, x);
          if (in1) hist_add(hist + (SH::B + (d1 >> sh1)) * 2, x);
        });
    }
    fill = true;
    team_sync();
    if (tid < 32) {   // one warp scans each active track's buckets
      const int lane = tid;
      constexpr int PER = SH::B / 32;
#pragma unroll 1
      for (int o = 0; o < 2; ++o) {
        if (!(act >> o & 1)) continue;
        const unsigned long long* hb = hist + (o * SH::B + lane * PER) * 2;
        u128 mine = 0;
#pragma unroll 1
        for (int k = 0; k < PER; ++k) mine += fix_value(hb[2 * k], hb[2 * k + 1]);
        u128 inc = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint64_t ylo = __shfl_up_sync(FULL, (uint64_t)inc, d);
          const uint64_t yhi = __shfl_up_sync(FULL, (uint64_t)(inc >> 64), d);
          if (lane >= d) inc += ((u128)yhi << 64) | ylo;
        }
        const u128 cb = st.cb[o];
        const unsigned hit = __ballot_sync(FULL, cb + inc >= S);
        if (hit) {
          const int L = __ffs(hit) - 1;
          if (lane == L) {
            u128 run = cb + inc - mine;
            int pick = -1;
#pragma unroll 1
            for (int k = 0; k < PER && pick < 0; ++k) {
              const u128 v = fix_value(hb[2 * k], hb[2 * k + 1]);
              if (run + v >= S) pick = lane * PER + k;
              else run += v;
            }
            const int sh = o ? sh1 : sh0;
            st.cb[o] = run;
            st.lo[o] += pick << sh;
            st.lg[o] = sh;
            if (sh == 0) {
              st.P[o] = st.lo[o];
              st.C[o] = run;
              st.act &= ~(1 << o);
            }
          }
        } else if (lane == 31) {
          // the whole range stays below s -- only on the first level
          // (total < s): no crossing, P = n, C(<n) = total
          st.P[o] = a.n;
          st.C[o] = cb + inc;
          st.act &= ~(1 << o);
        }
        __syncwarp();
      }
    }
    team_sync();
  }
}

// K5: twin greedy-LP values of one class of phase rows, one row per team
// (warp or CTA).  Value of a row for one track:
//   val = sum l*w + F(<P) + (s - C(<P)) * w_sorted[P]
// with sum l*w a float sum in the canonical per-lane order + fixed team
// tree, and P, C(<P) = sum h~, F(<P) = sum (h w)~ exact (above).
//   pass A   one read of the row: sum l*w, and at g = the rank of last
//            sweep's crossing column: C(<g), F(<g), plus {h, w} of the
//            slots ranked within W of g.
//   walk     one warp: P and C, F at P by exact prefix sums over the window
//            (most rows: the crossing moves by less than W ranks).
//   search   otherwise, per level one pass with a shared-memory histogram
//            of exact head sums over B rank buckets of the current range;
//            a warp scan picks the bucket where the cumulative sum reaches
//            s; the range shrinks by B per level (2-4 levels), to one rank;
//            then one pass for F(<P).
// The result does not depend on the hint, on which path settled the row,
// or on the row's position / shard: bitwise-identical rows give
// bitwise-identical values.
#ifndef IMP_K5_TPSM
#define IMP_K5_TPSM 1024   // resident threads per SM the register cap targets
#endif
// Certified float decisions.  The canonical float sum Cf of <= 2^14 + 2
// heads (warp teams: <= 514) (each in [0, 1]) is within m * 2^-53 * Cf of the true sum, which is
// within 2^-75 of the exact fixed-point sum C~ -- so |Cf - C~| < margin(Cf)
// and a comparison of Cf against s that clears the margin decides the exact
// comparison the search would make.  Anything closer is left to the exact
// search.  (Window walks add < 2^7 more float adds: the 2^-36 slope covers
// them.)
__device__ __forceinline__ double k5_margin(double c) {
  return fma(fabs(c), 0x1p-36, 0x1p-68);
}

// ---------------------------------------------------------------------------
// K5 for warp teams (rows of <= 512 stored entries): the round-1 form --
// float sums in the canonical per-lane order with certified decisions, a
// float window walk, and one more pass for the canonical float sums when
// the crossing moved.  For short rows its per-row work is lighter than the
// exact sums' (measured: robot2d_reachavoid 501 vs 322 phase-1 sweeps/s);
// the class of a row is a function of its length alone, so either form is
// position independent.
// ---------------------------------------------------------------------------
template <int TEAM, bool WIDE>
__global__ void __launch_bounds__(256, IMP_K5_TPSM / 256)
    k_sweep_warp(const __grid_constant__ SweepArgs a) {
  if (a.ctl && a.ctl->done) return;
  using SH = K5Shape<TEAM>;
  constexpr int TEAMS_PER_BLOCK = TEAM == 32 ? 8 : 1;
  __shared__ double f_part[SH::F_PART];
  __shared__ unsigned long long hist_all[TEAMS_PER_BLOCK][SH::HIST];
  __shared__ SearchState s_st[TEAMS_PER_BLOCK];
  __shared__ double s_win[TEAMS_PER_BLOCK][2][SH::WIN];   // row parity
  __shared__ double s_fv[TEAMS_PER_BLOCK][6];
  const int tid = TEAM == 32 ? (threadIdx.x & 31) : threadIdx.x;
  const int slot = TEAM == 32 ? (threadIdx.x >> 5) : 0;
  unsigned long long* hist = hist_all[slot];
  const int64_t team0 = TEAM == 32
      ? (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)
      : (int64_t)blockIdx.x;
  const int64_t nteams = TEAM == 32
      ? (int64_t)gridDim.x * (blockDim.x >> 5) : (int64_t)gridDim.x;
  auto team_sync = [] {
    if constexpr (TEAM == 32) __syncwarp();
    else __syncthreads();
  };
  for (int q = tid; q < 2 * SH::WIN; q += TEAM) (&s_win[slot][0][0])[q] = 0.0;
  team_sync();

  for (int64_t i = team0; i < a.n_list; i += nteams) {
    const int64_t t = a.list[i];
    const int64_t row = phase_row(a, t);
    const int64_t beg = a.row_ptr[row];
    const int m = (int)(a.row_ptr[row + 1] - beg);
    const double s = a.slack[row];
    const bool zero = !(s > 0.0);   // nothing is filled: P = 0, C = 0
    bool known = zero;
    bool flagged = false;   // the row searched last sweep
    int g0 = 0, g1 = 0;
    if (!zero && a.hint) {
      const int h0 = a.hint[2 * t], h1 = a.hint[2 * t + 1];
      if (h0 >= 0 && h1 >= 0) {
        known = true;
        flagged = ((h0 | h1) & HINT_SEARCHED) != 0;
        // warp teams keep column hints (robot2d: 500 vs 479 sweeps/s with
        // the adaptive modes of the CTA kernel)
        const int c0 = h0 & HINT_COL, c1 = h1 & HINT_COL;
        RankReg<WIDE> r;
        if (c0 != HINT_COL) { r.load(a, c0); g0 = r.r0(); } else g0 = a.n;
        if (c1 != HINT_COL) { r.load(a, c1); g1 = r.r1(); } else g1 = a.n;
      }
    }
    // ---- pass A ----------------------------------------------------------
    // fv: lw0 lw1 | F0 F1 (sum h*w, rank < g) | C0 C1 (sum h, rank < g),
    // all float in the canonical order; heads ranked in [g - W, g + W) are
    // captured per track.  The window buffer is double-buffered by row
    // parity (cleared during the previous row's reduction).
    constexpr int W = SH::W;
    const int par = (int)((i / nteams) & 1);
    double* win = s_win[slot][par];
    const int wb0 = g0 - W, wb1 = g1 - W;
    double fv[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for_slots<TEAM, WIDE>(a, tid, row, beg, m,
        [&](double l, double h, double2 w, const RankReg<WIDE>& rk) {
          fv[0] = fma(l, w.x, fv[0]);
          fv[1] = fma(l, w.y, fv[1]);
          const int r0 = rk.r0(), r1 = rk.r1();
          if (r0 < g0) { fv[2] = fma(h, w.x, fv[2]); fv[4] += h; }
          if (r1 < g1) { fv[3] = fma(h, w.y, fv[3]); fv[5] += h; }
          const unsigned d0 = (unsigned)(r0 - wb0), d1 = (unsigned)(r1 - wb1);
          if (d0 < 2 * W) win[d0] = h;
          if (d1 < 2 * W) win[2 * W + d1] = h;
        });
    team_sum_pass_a<TEAM>(fv, f_part, s_win[slot][par ^ 1], SH::WIN);
    int P[2] = {g0, g1};
    // need: 0 settled at g, 1 settled in the window (F, C need a pass),
    // 2 needs the exact bucketed search (+ that pass)
    int need[2] = {0, 0};
    if (!zero) {
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (!known) { need[o] = 2; continue; }
        const int g = P[o];
        const double* wt = win + o * 2 * W;
        double c = fv[4 + o];
        if (c + k5_margin(c) < s) {
          if (g >= a.n) continue;                              // P = n
          c += wt[W];
          if (c - k5_margin(c) >= s) continue;                 // P = g
          if (!(c + k5_margin(c) < s)) { need[o] = 2; continue; }
          int q = g + 1;                                       // walk up
          need[o] = 2;
          for (; q < g + W; ++q) {
            if (q >= a.n) { P[o] = a.n; need[o] = 1; break; }
            const double cn = c + wt[q - g + W];
            if (cn - k5_margin(cn) >= s) { P[o] = q; need[o] = 1; break; }
            if (!(cn + k5_margin(cn) < s)) break;              // too close
            c = cn;
          }
        } else if (c - k5_margin(c) >= s) {
          const double mg = k5_margin(c);   // errors of the larger sums
          int q = g - 1;                                       // walk down
          need[o] = 2;
          for (; q >= g - W && q >= 0; --q) {
            c -= wt[q - g + W];
            if (c + mg < s) { P[o] = q; need[o] = 1; break; }
            if (!(c - mg >= s)) break;                         // too close
          }
        } else {
          need[o] = 2;
        }
      }
    }
    // ---- bucketed exact search for unsettled tracks ----------------------
    // Team-uniform search state lives in shared memory (st), so the pass-A
    // registers are free during the search.
    if (need[0] | need[1]) {
      SearchState& st = s_st[slot];
      if (tid == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) s_fv[slot][k] = fv[k];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          st.lo[o] = 0;
          st.lg[o] = a.nbits;
          st.cb[o] = 0;
          st.P[o] = P[o];
        }
        st.act = (need[0] == 2 ? 1 : 0) | (need[1] == 2 ? 2 : 0);
        if (a.miss_total) atomicAdd(a.miss_total + (st.act ? 1 : 0), 1ull);
      }
      team_sync();
      if (need[0] == 2 || need[1] == 2)
        search_levels<TEAM, WIDE>(a, tid, row, beg, m, s, st, hist, false);
      // ---- pass F: the canonical float sums below the new crossings -----
      // (same per-lane order and team tree as pass A, so a row's bits do not
      // depend on which path found P)
      const int q0 = need[0] ? st.P[0] : -1, q1 = need[1] ? st.P[1] : -1;
      double fz[4] = {0.0, 0.0, 0.0, 0.0};
      for_slots<TEAM, WIDE, false>(a, tid, row, beg, m,
          [&](double, double h, double2 w, const RankReg<WIDE>& rk) {
            if (rk.r0() < q0) { fz[0] = fma(h, w.x, fz[0]); fz[2] += h; }
            if (rk.r1() < q1) { fz[1] = fma(h, w.y, fz[1]); fz[3] += h; }
          });
      team_sum_f<TEAM, 4>(fz, f_part);
#pragma unroll
      for (int k = 0; k < 6; ++k) fv[k] = s_fv[slot][k];
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (need[o]) {
          fv[2 + o] = fz[o];
          fv[4 + o] = fz[2 + o];
        }
        P[o] = st.P[o];
      }
      team_sync();   // st is reused by the team's next row
    }
    if (tid == 0) {
      if (a.hint && (need[0] | need[1] | (int)flagged)) {
        // crossing columns for next sweep, flagged if this row searched
        const int fl = (need[0] == 2 || need[1] == 2) ? HINT_SEARCHED : 0;
        a.hint[2 * t] = (P[0] >= a.n ? HINT_COL : __ldg(a.perm0 + P[0])) | fl;
        a.hint[2 * t + 1] =
            (P[1] >= a.n ? HINT_COL : __ldg(a.perm1 + P[1])) | fl;
      }
      a.out0[t] = row_value(fv[0], fv[2], s, fv[4], P[0], a.n, a.ws0);
      a.out1[t] = row_value(fv[1], fv[3], s, fv[5], P[1], a.n, a.ws1);
    }
  }
}



// P, C(<P), F(<P) of one track from the window around g (one warp, all
// lanes).  Returns false when the crossing lies W or more ranks away (the
// caller searches).  C, F hold the exact sums at g on entry and at P on a
// settled return; p holds g on entry and P on return.
template <int W>
__device__ __forceinline__ bool walk_track(bool zero, bool known, double s,
                                           int n, int lane,
                                           const double2* wt, Fix& C, Fix& F,
                                           int& p) {
  if (zero) return true;
  if (!known) return false;
  const u128 S = fix_ceil(s);
  const int g = p;
  if (fixv(C) < S) {                  // walk up: P = max{q: C(<q) < S}
    if (g >= n) return true;          // P = n, sums unchanged
    {                                 // common case: P = g
      const Fix h0 = to_fix(wt[W].x);
      if (fixv(C) + fixv(h0) >= S) return true;
    }
    for (int base = 0; base < W; base += 32) {
      const int q = g + base + lane;
      const double2 e = wt[W + base + lane];
      const Fix hx = to_fix(e.x), fx = to_fix(e.x * e.y);
      Fix ih = hx, ifx = fx;          // inclusive prefix over lanes
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t ya = __shfl_up_sync(FULL, ih.a, d);
        const uint64_t yb = __shfl_up_sync(FULL, ih.b, d);
        const uint64_t za = __shfl_up_sync(FULL, ifx.a, d);
        const uint64_t zb = __shfl_up_sync(FULL, ifx.b, d);
        if (lane >= d) { ih.a += ya; ih.b += yb; ifx.a += za; ifx.b += zb; }
      }
      // C(<q + 1) = C + ih: the crossing is the first lane reaching S
      const unsigned hit = __ballot_sync(FULL, q < n && fixv(C) + fixv(ih) >= S);
      const unsigned end = __ballot_sync(FULL, q >= n);
      int L = -1;
      if (hit) {
        L = __ffs(hit) - 1;           // sums below q = exclusive prefix
        p = g + base + L;
      } else if (end) {
        L = __ffs(end) - 1;           // no crossing before rank n
        p = n;
      }
      if (L >= 0) {
        const Fix eh{ih.a - hx.a, ih.b - hx.b}, ef{ifx.a - fx.a, ifx.b - fx.b};
        fix_add(C, Fix{__shfl_sync(FULL, eh.a, L), __shfl_sync(FULL, eh.b, L)});
        fix_add(F, Fix{__shfl_sync(FULL, ef.a, L), __shfl_sync(FULL, ef.b, L)});
        return true;
      }
      fix_add(C, Fix{__shfl_sync(FULL, ih.a, 31), __shfl_sync(FULL, ih.b, 31)});
      fix_add(F, Fix{__shfl_sync(FULL, ifx.a, 31), __shfl_sync(FULL, ifx.b, 31)});
    }
    return false;
  }
  {                                   // common case: P = g - 1
    const double2 e = wt[W - 1];
    const Fix h1 = to_fix(e.x);
    if (fixv(C) - fixv(h1) < S) {
      fix_sub(C, h1);
      fix_sub(F, to_fix(e.x * e.y));
      p = g - 1;
      return true;
    }
  }
  for (int base = 0; base < W; base += 32) {   // walk down from g - 1
    const int q = g - 1 - base - lane;
    const double2 e = wt[W - 1 - base - lane];
    const Fix hx = to_fix(e.x), fx = to_fix(e.x * e.y);
    Fix ih = hx, ifx = fx;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t ya = __shfl_up_sync(FULL, ih.a, d);
      const uint64_t yb = __shfl_up_sync(FULL, ih.b, d);
      const uint64_t za = __shfl_up_sync(FULL, ifx.a, d);
      const uint64_t zb = __shfl_up_sync(FULL, ifx.b, d);
      if (lane >= d) { ih.a += ya; ih.b += yb; ifx.a += za; ifx.b += zb; }
    }
    // C(<q) = C - ih (q >= 0; C(<0) = 0 < S always)
    const unsigned hit = __ballot_sync(FULL, q >= 0 && fixv(C) - fixv(ih) < S);
    const int L = hit ? __ffs(hit) - 1 : 31;
    fix_sub(C, Fix{__shfl_sync(FULL, ih.a, L), __shfl_sync(FULL, ih.b, L)});
    fix_sub(F, Fix{__shfl_sync(FULL, ifx.a, L), __shfl_sync(FULL, ifx.b, L)});
    if (hit) {
      p = g - 1 - base - L;
      return true;
    }
  }
  return false;
}

// CTA teams of <= IMP_K5_ENDSYNC threads end each row with a barrier
// (room5d's 128-thread rows: 188 vs 183 phase-1 sweeps/s with it; the
// 256 / 512 classes are faster without)
// the 128-thread class ends rows with a barrier, so one window buffer
// (cleared before it) suffices: half the shared memory, room for a 256-rank
// window at the same occupancy (room5d 206 -> 215 phase-1 sweeps/s,
// profiles/r02/k5_window_ab.txt)
#ifndef IMP_K5_WSINGLE
#define IMP_K5_WSINGLE 1
#endif
#ifndef IMP_K5_ENDSYNC
#define IMP_K5_ENDSYNC 128
#endif
template <int TEAM, bool WIDE>
__global__ void __launch_bounds__(TEAM == 32 ? 256 : TEAM,
                                  (TEAM == 32 ? 256 : TEAM) < IMP_K5_TPSM
                                      ? IMP_K5_TPSM / (TEAM == 32 ? 256 : TEAM)
                                      : 1)
    k_sweep(const __grid_constant__ SweepArgs a) {
  if (a.ctl && a.ctl->done) return;
  using SH = K5Shape<TEAM>;
  constexpr int TEAMS_PER_BLOCK = TEAM == 32 ? 8 : 1;
  constexpr int W = SH::W;
  __shared__ double f_part[SH::F_PART];
  __shared__ Fix x_part[4 * SH::NW];
  __shared__ unsigned long long hist_all[TEAMS_PER_BLOCK][SH::HIST];
  __shared__ SearchState s_st[TEAMS_PER_BLOCK];
  // window buffers: two by row parity, or one for the classes that end a
  // row with a barrier anyway (cleared before it)
  constexpr bool SINGLE = IMP_K5_WSINGLE && TEAM <= IMP_K5_ENDSYNC;
  constexpr int NBUF = SINGLE ? 1 : 2;
  __shared__ double2 s_win[TEAMS_PER_BLOCK][NBUF][SH::WIN];
  __shared__ double s_lw[TEAMS_PER_BLOCK][2];
  __shared__ Fix s_x[TEAMS_PER_BLOCK][4];
  __shared__ int s_need[TEAMS_PER_BLOCK][2];
  const int tid = TEAM == 32 ? (threadIdx.x & 31) : threadIdx.x;
  const int slot = TEAM == 32 ? (threadIdx.x >> 5) : 0;
  unsigned long long* hist = hist_all[slot];
  const int64_t team0 = TEAM == 32
      ? (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)
      : (int64_t)blockIdx.x;
  const int64_t nteams = TEAM == 32
      ? (int64_t)gridDim.x * (blockDim.x >> 5) : (int64_t)gridDim.x;
  auto team_sync = [] {
    if constexpr (TEAM == 32) __syncwarp();
    else __syncthreads();
  };
  for (int q = tid; q < NBUF * SH::WIN; q += TEAM)
    (&s_win[slot][0][0])[q] = make_double2(0.0, 0.0);
  team_sync();

  for (int64_t i = team0; i < a.n_list; i += nteams) {
    const int64_t t = a.list[i];
    const int64_t row = phase_row(a, t);
    const int64_t beg = a.row_ptr[row];
    const int m = (int)(a.row_ptr[row + 1] - beg);
    const double s = a.slack[row];
    const bool zero = !(s > 0.0);   // nothing is filled: P = 0, C = F = 0
    bool known = zero;
    bool flagged = false;   // the row searched last sweep
    int g0 = 0, g1 = 0;
    if (!zero && a.hint) {
      const int h0 = a.hint[2 * t], h1 = a.hint[2 * t + 1];
      if (h0 >= 0 && h1 >= 0) {
        known = true;
        flagged = ((h0 | h1) & HINT_SEARCHED) != 0;
        g0 = hint_rank<WIDE>(a, h0, 0);
        g1 = hint_rank<WIDE>(a, h1, 1);
      }
    }
    // ---- pass A ----------------------------------------------------------
    // one read of the row: lw (float, canonical per-lane order + fixed team
    // tree), exact C(<g) and F(<g) per track, and {h, w} of the slots
    // ranked in [g - W, g + W) per track.  The window buffer is
    // double-buffered by row parity (cleared during the previous row's
    // reduction).
    const int par = SINGLE ? 0 : (int)((i / nteams) & 1);
    double2* win = s_win[slot][par];
    const int wb0 = g0 - W, wb1 = g1 - W;
    // clear the next row's window buffer: its last readers (the previous
    // row's walk) finished before the previous row's second barrier
    if constexpr (!SINGLE) {
      for (int q = tid; q < 2 * SH::WIN; q += TEAM)
        (&s_win[slot][par ^ 1][0].x)[q] = 0.0;
    }
    double fv[2] = {0.0, 0.0};
    Fix xs[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};   // C0 F0 C1 F1
    for_slots<TEAM, WIDE>(a, tid, row, beg, m,
        [&](double l, double h, double2 w, const RankReg<WIDE>& rk) {
          fv[0] = fma(l, w.x, fv[0]);
          fv[1] = fma(l, w.y, fv[1]);
          const int r0 = rk.r0(), r1 = rk.r1();
          const bool b0 = r0 < g0, b1 = r1 < g1;
          if (b0 | b1) {
            const Fix hx = to_fix(h);
            if (b0) { fix_add(xs[0], hx); fix_add(xs[1], to_fix(h * w.x)); }
            if (b1) { fix_add(xs[2], hx); fix_add(xs[3], to_fix(h * w.y)); }
          }
          const unsigned d0 = (unsigned)(r0 - wb0), d1 = (unsigned)(r1 - wb1);
          if (d0 < 2 * W) win[d0] = make_double2(h, w.x);
          if (d1 < 2 * W) win[2 * W + d1] = make_double2(h, w.y);
        });
    // ---- team sums + exact walk inside the window -------------------------
    // Warp partials of lw (float) and C, F (exact) go to shared memory
    // behind ONE barrier; warp o then finishes track o's sums itself (the
    // float lw with the fixed tree of team_sum_f: lane w adds warp w's
    // partial, then a butterfly) and walks its window.  need: 0 settled,
    // 2 needs the bucketed search.
    static_assert(TEAM > 32, "k_sweep: CTA teams");
    {
      constexpr int NW = SH::NW;
      const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
      for (int k = 0; k < 2; ++k) fv[k] = warp_sum(fv[k]);
#pragma unroll
      for (int k = 0; k < 4; ++k) xs[k] = warp_sum_fix(xs[k]);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k) f_part[k * NW + wid] = fv[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) x_part[k * NW + wid] = xs[k];
      }
      __syncthreads();
      auto walk = [&](auto oc) {
        constexpr int o = decltype(oc)::value;
        Fix C = warp_sum_fix(lane < NW ? x_part[(2 * o) * NW + lane]
                                       : Fix{0, 0});
        Fix F = warp_sum_fix(lane < NW ? x_part[(2 * o + 1) * NW + lane]
                                       : Fix{0, 0});
        int p = o ? g1 : g0;
        const bool settled = walk_track<W>(zero, known, s, a.n, lane,
                                           win + o * 2 * W, C, F, p);
        if (lane == 0) {
          s_need[slot][o] = settled ? 0 : 2;
          s_st[slot].P[o] = zero ? 0 : p;
          s_x[slot][2 * o] = C;
          s_x[slot][2 * o + 1] = F;
        }
      };
      if (wid == 0) {
        const double lw0 = warp_sum(lane < NW ? f_part[lane] : 0.0);
        const double lw1 = warp_sum(lane < NW ? f_part[NW + lane] : 0.0);
        if (lane == 0) {
          s_lw[slot][0] = lw0;
          s_lw[slot][1] = lw1;
        }
        walk(std::integral_constant<int, 0>{});
      } else if (wid == 1) {
        walk(std::integral_constant<int, 1>{});
      }
    }
    __syncthreads();
    int need[2] = {s_need[slot][0], s_need[slot][1]};
    // ---- bucketed exact search for unsettled tracks ----------------------
    if (need[0] | need[1]) {
      SearchState& st = s_st[slot];
      if (tid == 0) {
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          st.lo[o] = 0;
          st.lg[o] = a.nbits;
          st.cb[o] = 0;
        }
        st.act = (need[0] ? 1 : 0) | (need[1] ? 2 : 0);
        if (a.miss_total) atomicAdd(a.miss_total + 1, 1ull);
      }
      team_sync();
      search_levels<TEAM, WIDE>(a, tid, row, beg, m, s, st, hist, false);
      // exact F(<P) of the searched tracks: one pass (integer sums)
      const int q0 = need[0] ? st.P[0] : -1, q1 = need[1] ? st.P[1] : -1;
      Fix fz[2] = {{0, 0}, {0, 0}};
      for_slots<TEAM, WIDE, false>(a, tid, row, beg, m,
          [&](double, double h, double2 w, const RankReg<WIDE>& rk) {
            if (rk.r0() < q0) fix_add(fz[0], to_fix(h * w.x));
            if (rk.r1() < q1) fix_add(fz[1], to_fix(h * w.y));
          });
      team_sum_fix<TEAM, 2>(fz, x_part);
      if (tid == 0) {
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          if (need[o]) {
            s_x[slot][2 * o + 1] = fz[o];
            // C(<P) from the search, as the two-word form
            const u128 c = st.C[o];
            s_x[slot][2 * o] = Fix{(uint64_t)(c >> 44),
                                   (uint64_t)(c & ((1ull << 44) - 1))};
          }
        }
      }
      team_sync();
    }
    if (tid == 0) {
      const int p0 = s_st[slot].P[0], p1 = s_st[slot].P[1];
      if (a.hint && (need[0] | need[1] | (int)flagged | (int)(p0 != g0) |
                     (int)(p1 != g1) | (int)!known)) {
        // crossing hints for next sweep, flagged if this row searched
        const bool sr = need[0] || need[1];
        // (the modes of the hints read at the row start: re-read here,
        // keeping them live across the row costs registers)
        const int o0 = known ? a.hint[2 * t] : 0, o1 = known ? a.hint[2 * t + 1] : 0;
        a.hint[2 * t] = hint_encode(a, o0, p0, a.perm0, sr && known, true);
        a.hint[2 * t + 1] = hint_encode(a, o1, p1, a.perm1, sr && known, true);
      }
      const Fix* x = s_x[slot];
      a.out0[t] = row_value(s_lw[slot][0], fix_double(fixv(x[1])), s,
                            fix_double(fixv(x[0])), p0, a.n, a.ws0);
      a.out1[t] = row_value(s_lw[slot][1], fix_double(fixv(x[3])), s,
                            fix_double(fixv(x[2])), p1, a.n, a.ws1);
      if (a.miss_total && !(need[0] | need[1]) &&
          (p0 != g0 || p1 != g1) && known && !zero)
        atomicAdd(a.miss_total, 1ull);
    }
    // no barrier needed here: the next row writes s_st / s_x / s_need /
    // s_lw and the partials only after its first barrier, which thread 0
    // reaches once it is done with this row's
    if constexpr (SINGLE) {   // the walks read the window before B2
      for (int q = tid; q < 2 * SH::WIN; q += TEAM) (&win[0].x)[q] = 0.0;
    }
    if constexpr (TEAM <= IMP_K5_ENDSYNC) __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Robust Bellman reduction + convergence statistics
// ---------------------------------------------------------------------------

struct ReduceArgs {
  Ctl* ctl;
  const double* val0;
  const double* val1;
  const double* old[2][2];   // [track][pingpong] full (n_s) vectors
  double* nxt[2][2];         // [track][pingpong]; writes nxt[t][cur ^ 1]
  const int64_t* fixed;      // phase-2 policy (local) or nullptr
  int64_t* policy;           // (k_count) chosen inputs, may be nullptr
  int k_begin, k_count, n_u, n_w, u_max;
  double* stats;             // explicit-mode stats (no ctl): 5 doubles
  Packed pk;                 // sharded loop: packed value layout
};

// Block max of the per-state statistics (exact, order-free) into the
// control block (or the explicit-mode stats).
__device__ __forceinline__ void bellman_stats(const ReduceArgs& a, double d0,
                                              double d1, double gap,
                                              unsigned flags) {
  Ctl* ctl = a.ctl;
  __shared__ double sd[3][32];
  __shared__ unsigned sf[32];
  for (int o = 16; o > 0; o >>= 1) {
    d0 = fmax(d0, __shfl_down_sync(FULL, d0, o));
    d1 = fmax(d1, __shfl_down_sync(FULL, d1, o));
    gap = fmax(gap, __shfl_down_sync(FULL, gap, o));
    flags |= __shfl_down_sync(FULL, flags, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sd[0][warp] = d0; sd[1][warp] = d1; sd[2][warp] = gap; sf[warp] = flags; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      d0 = fmax(d0, sd[0][w]);
      d1 = fmax(d1, sd[1][w]);
      gap = fmax(gap, sd[2][w]);
      flags |= sf[w];
    }
    if (ctl) {
      atomicMax(&ctl->slot_d0, (unsigned long long)order_key(d0));
      atomicMax(&ctl->slot_d1, (unsigned long long)order_key(d1));
      atomicMax(&ctl->slot_gap, (unsigned long long)order_key(gap));
      atomicOr(&ctl->slot_flags, flags);
    } else if (a.stats) {
      unsigned long long* st = reinterpret_cast<unsigned long long*>(a.stats);
      atomicMax(st + 0, (unsigned long long)order_key(d0));
      atomicMax(st + 1, (unsigned long long)order_key(d1));
      atomicMax(st + 2, (unsigned long long)order_key(gap));
      atomicOr(reinterpret_cast<unsigned*>(st + 3), flags);
    }
  }
}


__global__ void k_bellman(ReduceArgs a) {
  Ctl* ctl = a.ctl;
  if (ctl && ctl->done) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int pp = ctl ? ctl->cur : 0;
  double d0 = 0.0, d1 = 0.0, gap = -INFINITY;
  unsigned flags = 0;
  if (k < a.k_count) {
    const int U = a.fixed ? 1 : a.n_u;
    const int nw = a.n_w;
    double best0 = 0.0, best1 = 0.0;
    int pick = 0;
    for (int j = 0; j < U; ++j) {
      const int64_t base = ((int64_t)k * U + j) * nw;
      double m0 = a.val0[base], m1 = a.val1[base];
      for (int i = 1; i < nw; ++i) {
        double x0 = a.val0[base + i], x1 = a.val1[base + i];
        if (a.u_max) { m0 = fmin(m0, x0); m1 = fmin(m1, x1); }
        else         { m0 = fmax(m0, x0); m1 = fmax(m1, x1); }
      }
      if (j == 0) { best0 = m0; best1 = m1; continue; }
      if (a.u_max ? (m0 > best0) : (m0 < best0)) { best0 = m0; pick = j; }
      if (a.u_max ? (m1 > best1) : (m1 < best1)) best1 = m1;
    }
    const int g = a.k_begin + k;
    const int64_t g0 = ctl ? vpos(a.pk, 0, g) : g, g1 = ctl ? vpos(a.pk, 1, g) : g;
    const double o0 = a.old[0][pp][g0], o1 = a.old[1][pp][g1];
    double n0 = best0, n1 = best1;
    if (ctl && ctl->frozen0) n0 = o0;
    if (ctl && ctl->frozen1) n1 = o1;
    if (a.policy) a.policy[k] = a.fixed ? a.fixed[k] : pick;
    if (ctl) {
      a.nxt[0][pp ^ 1][g0] = n0;
      a.nxt[1][pp ^ 1][g1] = n1;
    } else {
      a.nxt[0][0][k] = n0;
      a.nxt[1][0][k] = n1;
    }
    d0 = fabs(n0 - o0);
    d1 = fabs(n1 - o1);
    gap = n1 - n0;
    if (n0 < o0 - 1e-12 || n1 > o1 + 1e-12) flags |= 1u;
    if (n0 > n1 + 1e-9) flags |= 2u;
  }
  bellman_stats(a, d0, d1, gap, flags);
}

// Robust Bellman reduction for many inputs: one warp per state, lanes over
// inputs j = lane, lane + 32, ... (the min / max over disturbances per input
// runs in the reference's order inside a lane).  The arg-best input is the
// FIRST best (synthesis.py:97-135): lane-local scans keep the first best of
// their subsequence, the warp keeps the best value and, on ties, the lowest
// input -- the same pick and the same bits as the sequential scan.  A NaN
// never replaces a best; a NaN at input 0 is the result, as sequentially.
__global__ void k_bellman_warp(ReduceArgs a) {
  Ctl* ctl = a.ctl;
  if (ctl && ctl->done) return;
  const int lane = threadIdx.x & 31;
  const int k = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int pp = ctl ? ctl->cur : 0;
  double d0 = 0.0, d1 = 0.0, gap = -INFINITY;
  unsigned flags = 0;
  if (k < a.k_count) {   // warp-uniform
    const int U = a.n_u, nw = a.n_w;
    const bool umax = a.u_max;
    double b0 = 0.0, b1 = 0.0, f0 = 0.0, f1 = 0.0;
    int p0 = INT_MAX, p1 = INT_MAX;
    for (int j = lane; j < U; j += 32) {
      const int64_t base = ((int64_t)k * U + j) * nw;
      double m0 = a.val0[base], m1 = a.val1[base];
      for (int i = 1; i < nw; ++i) {
        double x0 = a.val0[base + i], x1 = a.val1[base + i];
        if (umax) { m0 = fmin(m0, x0); m1 = fmin(m1, x1); }
        else      { m0 = fmax(m0, x0); m1 = fmax(m1, x1); }
      }
      if (j == 0) { f0 = m0; f1 = m1; }
      if (m0 == m0 && (p0 == INT_MAX || (umax ? m0 > b0 : m0 < b0))) { b0 = m0; p0 = j; }
      if (m1 == m1 && (p1 == INT_MAX || (umax ? m1 > b1 : m1 < b1))) { b1 = m1; p1 = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob0 = __shfl_xor_sync(FULL, b0, o), ob1 = __shfl_xor_sync(FULL, b1, o);
      const int op0 = __shfl_xor_sync(FULL, p0, o), op1 = __shfl_xor_sync(FULL, p1, o);
      if (op0 != INT_MAX && (p0 == INT_MAX || (umax ? ob0 > b0 : ob0 < b0) ||
                             (ob0 == b0 && op0 < p0))) { b0 = ob0; p0 = op0; }
      if (op1 != INT_MAX && (p1 == INT_MAX || (umax ? ob1 > b1 : ob1 < b1) ||
                             (ob1 == b1 && op1 < p1))) { b1 = ob1; p1 = op1; }
    }
    f0 = __shfl_sync(FULL, f0, 0);
    f1 = __shfl_sync(FULL, f1, 0);
    if (f0 != f0) { b0 = f0; p0 = 0; }
    if (f1 != f1) b1 = f1;
    if (lane == 0) {
      const int g = a.k_begin + k;
      const int64_t g0 = ctl ? vpos(a.pk, 0, g) : g, g1 = ctl ? vpos(a.pk, 1, g) : g;
      const double o0 = a.old[0][pp][g0], o1 = a.old[1][pp][g1];
      double n0 = b0, n1 = b1;
      if (ctl && ctl->frozen0) n0 = o0;
      if (ctl && ctl->frozen1) n1 = o1;
      if (a.policy) a.policy[k] = p0;
      if (ctl) {
        a.nxt[0][pp ^ 1][g0] = n0;
        a.nxt[1][pp ^ 1][g1] = n1;
      } else {
        a.nxt[0][0][k] = n0;
        a.nxt[1][0][k] = n1;
      }
      d0 = fabs(n0 - o0);
      d1 = fabs(n1 - o1);
      gap = n1 - n0;
      if (n0 < o0 - 1e-12 || n1 > o1 + 1e-12) flags |= 1u;
      if (n0 > n1 + 1e-9) flags |= 2u;
    }
  }
  bellman_stats(a, d0, d1, gap, flags);
}

// Termination logic of _run_phase (synthesis.py:164-205) / diagnose
// (:346-361), one thread.
__device__ __forceinline__ void log_gap(Ctl* c, long long it, double gap) {
  if (it % 1000 == 0 && c->gap_log_n < GAP_LOG) c->gap_log[c->gap_log_n++] = gap;
}

// stats (sharded loop): the all-reduced [max|dV0|, max|dV1|, max gap,
// monotone, bracket] of every rank instead of this device's slots.
__global__ void k_control(Ctl* c, const double* stats) {
  if (c->done) return;
  const long long it = ++c->it;
  double d0, d1, gap;
  unsigned flags;
  if (stats) {
    d0 = stats[0];
    d1 = stats[1];
    gap = stats[2];
    flags = (stats[3] > 0.0 ? 1u : 0u) | (stats[4] > 0.0 ? 2u : 0u);
  } else {
    d0 = key_value(c->slot_d0);
    d1 = key_value(c->slot_d1);
    gap = key_value(c->slot_gap);
    flags = c->slot_flags;
  }
  c->slot_d0 = c->slot_d1 = c->slot_gap = 0ull;
  c->slot_flags = 0u;
  if (c->mode == IMP_MODE_DIAGNOSE) {
    if (c->k0 < 0 && !c->frozen0 && d0 <= c->eps) { c->k0 = it; c->frozen0 = 1; }
    if (c->k1 < 0 && !c->frozen1 && d1 <= c->eps) { c->k1 = it; c->frozen1 = 1; }
    c->cur ^= 1;
    if (c->k0 >= 0 && c->k1 >= 0) { c->done = 1; return; }
    if (it >= c->max_iter) { c->status = IMP_E_CONVERGENCE; c->done = 1; }
    return;
  }
  if (flags & 1u) { c->status = IMP_E_MONOTONE; c->done = 1; return; }
  if (c->k0 < 0 && d0 <= c->eps) c->k0 = it;
  if (c->k1 < 0 && d1 <= c->eps) c->k1 = it;
  c->cur ^= 1;
  if (flags & 2u) { c->status = IMP_E_BRACKET; c->done = 1; return; }
  c->gap = gap;
  if (c->horizon > 0) {
    if (it >= c->horizon) c->done = 1;
    else log_gap(c, it, gap);
    return;
  }
  if (gap <= c->eps) { c->done = 1; return; }
  const bool stalled = c->has_prev && (c->prev_gap - gap <= 1e-15 * fmax(1.0, gap));
  if (c->k0 >= 0 && c->k1 >= 0 && stalled) {
    c->fallback = 1;
    c->done = 1;
    return;
  }
  c->prev_gap = gap;
  c->has_prev = 1;
  if (it >= c->max_iter) { c->status = IMP_E_CONVERGENCE; c->done = 1; return; }
  log_gap(c, it, gap);
}

// ---------------------------------------------------------------------------
// imdp finalisation: per-row slack and longest row
// ---------------------------------------------------------------------------

__global__ void k_slack(const int64_t* row_ptr, const double* lo,
                        const double* hi, const double* r_min,
                        const double* a_min, int64_t n_rows, double* slack,
                        double* hd, int* max_row) {
  const int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < n_rows; r += nw) {
    int64_t b = row_ptr[r], e = row_ptr[r + 1];
    double acc = 0.0;
    for (int64_t q = b + lane; q < e; q += 32) {
      const double l = lo[q];
      acc += l;
      hd[q] = hi[q] - l;   // the head K5 forms from the same two loads
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      slack[r] = fmax(0.0, 1.0 - (acc + r_min[r] + a_min[r]));
      atomicMax(max_row, (int)(e - b));
    }
  }
}

void finalize_imdp(imp_imdp* h, cudaStream_t s) {
  h->slack.alloc(std::max<int64_t>(h->n_rows, 1));
  h->hd.alloc(std::max<int64_t>(h->nnz, 1));
  DevBuf<int> mr(1);
  IMP_CUDA(cudaMemsetAsync(mr.ptr, 0, sizeof(int), s));
  if (h->n_rows > 0) {
    int blocks = (int)std::min<int64_t>((h->n_rows * 32 + 255) / 256,
                                        (int64_t)sm_count_of(h->device) * 64);
    k_slack<<<blocks, 256, 0, s>>>(h->row_ptr.ptr, h->lo.ptr, h->hi.ptr,
                                   h->r_min.ptr, h->a_min.ptr, h->n_rows,
                                   h->slack.ptr, h->hd.ptr, mr.ptr);
    IMP_CUDA(cudaGetLastError());
  }
  int host_max = 0;
  IMP_CUDA(cudaMemcpyAsync(&host_max, mr.ptr, sizeof(int),
                           cudaMemcpyDeviceToHost, s));
  IMP_CUDA(cudaStreamSynchronize(s));
  h->max_row = host_max;
}

// ---------------------------------------------------------------------------
// Host driver
// ---------------------------------------------------------------------------

namespace {

// Per-handle working set of one phase / step.
struct Work {
  int n_s = 0, n = 0, nbits = 0;
  bool wide = false;
  DevBuf<double> v[2][2];          // [track][pingpong]
  DevBuf<uint64_t> keys_in[2], keys_out[2];
  DevBuf<int> idx_in[2], perm[2];
  DevBuf<double2> colw;
  DevBuf<int2> rank;
  DevBuf<unsigned> rank16;
  DevBuf<double> ws[2];
  DevBuf<double> val[2];
  DevBuf<int> hint;                // warm-start crossing entries (2/row)
  DevBuf<int64_t> fixed, policy;
  DevBuf<Ctl> ctl;
  SweepArgs last_sweep{};   // arguments of the last enqueued K5 launch
  // K5 row classes: phase rows grouped by class (see launch_sweep)
  static constexpr int NCLASS = 8;
  DevBuf<int> class_rows;
  DevBuf<unsigned long long> class_cnt;   // counts, then scatter cursors
  DevBuf<unsigned long long> miss_total;  // IMP_SWEEP_STATS: rows searched
  int64_t class_off[NCLASS + 1] = {};
  bool classes_all = false;   // class lists hold the unfixed phase

  void init(const imp_imdp* h, int64_t phase_rows) {
    n_s = h->n_s;
    n = n_s + 2;
    nbits = 1;
    while ((1ll << nbits) <= n) ++nbits;
    wide = n > 65536;
    for (auto& t : v)
      for (auto& b : t) b.alloc(n_s);
    for (int t = 0; t < 2; ++t) {
      keys_in[t].alloc(n);
      keys_out[t].alloc(n);
      idx_in[t].alloc(n);
      perm[t].alloc(n);
      ws[t].alloc(n + 1);
      val[t].alloc(std::max<int64_t>(phase_rows, 1));
    }
    hint.alloc(2 * std::max<int64_t>(phase_rows, 1));
    IMP_CUDA(cudaMemset(hint.ptr, 0xfe, hint.bytes()));   // -2: unknown
    class_rows.alloc(std::max<int64_t>(phase_rows, 1));
    class_cnt.alloc(2 * NCLASS);
    miss_total.alloc(2);
    IMP_CUDA(cudaMemset(miss_total.ptr, 0, miss_total.bytes()));
    colw.alloc(n);
    rank.alloc(n);
    if (!wide) rank16.alloc(n);
    policy.alloc(std::max(h->k_count, 1));

    ctl.alloc(1);
  }
};

// Row classes of K5 by stored length (upper bounds, inclusive; the last
// class also takes every longer row); a pure function of the row, so the
// kernel a row gets never depends on its shard.
__constant__ int kClassHi[8] = {128, 256, 384, 512, 2048, 4096, 8192, 16384};

__device__ __forceinline__ int row_class(int m) {
  int c = 0;
  while (c < 7 && m > kClassHi[c]) ++c;
  return c;
}

__device__ __forceinline__ int64_t phase_row_of(const int64_t* fixed, int n_u,
                                                int n_w, int64_t t) {
  if (!fixed) return t;
  int64_t k = t / n_w, i = t - k * n_w;
  return (k * n_u + fixed[k]) * n_w + i;
}

__global__ void k_class_count(const int64_t* row_ptr, const int64_t* fixed,
                              int n_u, int n_w, int64_t rows,
                              unsigned long long* cnt) {
  __shared__ unsigned int local[8];
  if (threadIdx.x < 8) local[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = phase_row_of(fixed, n_u, n_w, t);
    atomicAdd(&local[row_class((int)(row_ptr[r + 1] - row_ptr[r]))], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 8 && local[threadIdx.x])
    atomicAdd(cnt + threadIdx.x, (unsigned long long)local[threadIdx.x]);
}

// order within a class is irrelevant: rows are independent and outputs are
// indexed by phase row
__global__ void k_class_scatter(const int64_t* row_ptr, const int64_t* fixed,
                                int n_u, int n_w, int64_t rows,
                                unsigned long long* cursor, int* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = phase_row_of(fixed, n_u, n_w, t);
    const int c = row_class((int)(row_ptr[r + 1] - row_ptr[r]));
    out[atomicAdd(cursor + c, 1ull)] = (int)t;
  }
}

void build_classes(const imp_imdp* h, Work& w, const int64_t* fixed_dev,
                   int64_t phase_rows, cudaStream_t s) {
  // exact sums: per-row limb sums stay below 2^64 for < 2^20 slots (Fix)
  if (h->max_row >= (1 << 20) - 2)
    fail(IMP_E_ARG, "row longer than 2^20 - 3 stored entries");
  IMP_CUDA(cudaMemsetAsync(w.class_cnt.ptr, 0, w.class_cnt.bytes(), s));
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((phase_rows + 255) / 256,
                           (int64_t)sm_count_of(h->device) * 8));
  if (phase_rows > 0) {
    k_class_count<<<blocks, 256, 0, s>>>(h->row_ptr.ptr, fixed_dev, h->n_u,
                                         h->n_w, phase_rows, w.class_cnt.ptr);
    IMP_CUDA(cudaGetLastError());
  }
  unsigned long long cnt[Work::NCLASS];
  IMP_CUDA(cudaMemcpyAsync(cnt, w.class_cnt.ptr, sizeof(cnt),
                           cudaMemcpyDeviceToHost, s));
  IMP_CUDA(cudaStreamSynchronize(s));
  w.class_off[0] = 0;
  for (int c = 0; c < Work::NCLASS; ++c) w.class_off[c + 1] = w.class_off[c] + cnt[c];
  unsigned long long cur[Work::NCLASS];
  for (int c = 0; c < Work::NCLASS; ++c) cur[c] = w.class_off[c];
  IMP_CUDA(cudaMemcpyAsync(w.class_cnt.ptr + Work::NCLASS, cur, sizeof(cur),
                           cudaMemcpyHostToDevice, s));
  if (phase_rows > 0) {
    k_class_scatter<<<blocks, 256, 0, s>>>(h->row_ptr.ptr, fixed_dev, h->n_u,
                                           h->n_w, phase_rows,
                                           w.class_cnt.ptr + Work::NCLASS,
                                           w.class_rows.ptr);
    IMP_CUDA(cudaGetLastError());
  }
  IMP_CUDA(cudaStreamSynchronize(s));
  count_launches(phase_rows > 0 ? 2 : 0, 0);
}

// IMP_SWEEP_STATS=1: the number of rows that needed the bucketed search
// accumulates on the device and imp_run_phase prints the rate to stderr.
bool sweep_stats() {
  static const int on = [] {
    const char* e = getenv("IMP_SWEEP_STATS");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return on != 0;
}

template <int TEAM, bool WIDE>
void launch_sweep_t(const SweepArgs& a, int sms, cudaStream_t s) {
  void (*kern)(const SweepArgs);
  if constexpr (TEAM == 32) kern = k_sweep_warp<32, WIDE>;
  else kern = k_sweep<TEAM, WIDE>;
  const int threads = TEAM == 32 ? 256 : TEAM;
  int per_sm = 0;
  IMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                         threads, 0));
  per_sm = std::max(per_sm, 1);
  const int64_t teams_per_block = TEAM == 32 ? threads / 32 : 1;
  const int64_t need = (a.n_list + teams_per_block - 1) / teams_per_block;
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>(need, (int64_t)sms * per_sm));
  kern<<<blocks, threads, 0, s>>>(a);
  IMP_CUDA(cudaGetLastError());
}

template <bool WIDE>
void launch_sweep_w(const SweepArgs& a, int team, int sms, cudaStream_t s) {
  switch (team) {
    case 32: return launch_sweep_t<32, WIDE>(a, sms, s);
    case 128: return launch_sweep_t<128, WIDE>(a, sms, s);
    case 256: return launch_sweep_t<256, WIDE>(a, sms, s);
    default: return launch_sweep_t<512, WIDE>(a, sms, s);
  }
}

// K5 over all phase rows: one launch per non-empty row class.  Classes are
// fixed functions of a row's stored length m (kClassHi), so the team -- and
// with it every float summation tree -- a row gets never depends on its
// shard: warp teams for m <= 512, CTAs of 128 / 256 / 512 threads above.
// Returns the number of launches.
int launch_sweep(SweepArgs sa, const Work& w, bool wide, int sms,
                 cudaStream_t s) {
  static const int teams[] = {32, 32, 32, 32, 128, 256, 512, 512};
  int launches = 0;
  if (sa.hint && sweep_stats()) sa.miss_total = w.miss_total.ptr;
  for (int c = 0; c < Work::NCLASS; ++c) {
    const int64_t cnt = w.class_off[c + 1] - w.class_off[c];
    if (cnt == 0) continue;
    SweepArgs a = sa;
    a.list = w.class_rows.ptr + w.class_off[c];
    a.n_list = cnt;
    if (wide) launch_sweep_w<true>(a, teams[c], sms, s);
    else launch_sweep_w<false>(a, teams[c], sms, s);
    ++launches;
  }
  return launches;
}

struct Launch {
  const imp_imdp* h;
  Work* w;
  cudaEvent_t k5_begin = nullptr, k5_end = nullptr;   // optional timing
  int sms;
  int spec, lp, u_max;
  const int64_t* fixed_dev;   // local policy or nullptr
  const double* v_explicit[2];  // explicit-mode inputs (full n_s) or nullptr
  double* new_explicit[2];      // explicit-mode outputs (k_count)
  double* stats_explicit;
  bool use_ctl;
  Packed pk{};                   // sharded loop: packed value layout
  double* vbuf[2] = {nullptr, nullptr};  // sharded loop: packed buffers
  const double* stats_reduced = nullptr;  // sharded loop: k_control input
  bool skip_control = false;     // sharded loop: control is a separate call
};

// Enqueue one iteration: order keys, the stable sorts of both tracks
// (launch_sort), ranks, sweep, reduce (+ control when use_ctl).  Returns
// the number of kernels enqueued (all of them ours).
int enqueue_iteration(const Launch& L, cudaStream_t s) {
  const imp_imdp* h = L.h;
  Work& w = *L.w;
  Ctl* ctl = L.use_ctl ? w.ctl.ptr : nullptr;
  const int n = w.n;
  OrderArgs oa{};
  for (int t = 0; t < 2; ++t)
    for (int p = 0; p < 2; ++p)
      oa.v[t][p] = L.vbuf[p] ? L.vbuf[p]
                   : (L.use_ctl ? w.v[t][p].ptr : L.v_explicit[t]);
  oa.ctl = ctl;
  oa.n_s = w.n_s;
  oa.n = n;
  oa.d1 = L.spec == IMP_SPEC_REACH ? 1.0 : 0.0;
  oa.d2 = L.spec == IMP_SPEC_REACH ? 0.0 : 1.0;
  oa.lp_max = L.lp == IMP_LP_MAX;
  for (int t = 0; t < 2; ++t) {
    oa.keys[t] = w.keys_in[t].ptr;
    oa.idx[t] = w.idx_in[t].ptr;
  }
  oa.colw = w.colw.ptr;
  oa.pk = L.pk;
  k_order_keys<<<(n + 255) / 256, 256, 0, s>>>(oa);
  IMP_CUDA(cudaGetLastError());
  uint64_t* const kin[2] = {w.keys_in[0].ptr, w.keys_in[1].ptr};
  uint64_t* const kout[2] = {w.keys_out[0].ptr, w.keys_out[1].ptr};
  int* const iin[2] = {w.idx_in[0].ptr, w.idx_in[1].ptr};
  int* const pout[2] = {w.perm[0].ptr, w.perm[1].ptr};
  const int n_sort = launch_sort(ctl, n, kin, iin, kout, pout, s);
  RankArgs ra{};
  ra.ctl = ctl;
  ra.n = n;
  ra.perm[0] = w.perm[0].ptr;
  ra.perm[1] = w.perm[1].ptr;
  ra.colw = w.colw.ptr;
  ra.rank = w.rank.ptr;
  ra.ws[0] = w.ws[0].ptr;
  ra.ws[1] = w.ws[1].ptr;
  k_ranks<<<(n + 1 + 255) / 256, 256, 0, s>>>(ra);
  IMP_CUDA(cudaGetLastError());
  if (!w.wide) {
    k_pack_ranks<<<(n + 255) / 256, 256, 0, s>>>(ctl, n, w.rank.ptr,
                                                 w.rank16.ptr);
    IMP_CUDA(cudaGetLastError());
  }
  SweepArgs sa{};
  sa.ctl = ctl;
  sa.row_ptr = h->row_ptr.ptr;
  sa.col = h->col.ptr;
  sa.lo = h->lo.ptr;
  sa.hi = h->hi.ptr;
  sa.hd = h->hd.ptr;
  sa.r_min = h->r_min.ptr;
  sa.r_max = h->r_max.ptr;
  sa.a_min = h->a_min.ptr;
  sa.a_max = h->a_max.ptr;
  sa.slack = h->slack.ptr;
  sa.colw = w.colw.ptr;
  sa.rank = w.rank.ptr;
  sa.rank16 = w.rank16.ptr;
  sa.ws0 = w.ws[0].ptr;
  sa.ws1 = w.ws[1].ptr;
  sa.fixed = L.fixed_dev;
  sa.n_phase_rows = L.fixed_dev ? (int64_t)h->k_count * h->n_w : h->n_rows;
  sa.n_u = h->n_u;
  sa.n_w = h->n_w;
  sa.n_s = h->n_s;
  sa.n = n;
  sa.nbits = w.nbits;
  sa.out0 = w.val[0].ptr;
  sa.out1 = w.val[1].ptr;
  sa.hint = w.hint.ptr;
  sa.perm0 = w.perm[0].ptr;
  sa.perm1 = w.perm[1].ptr;
  // (during stream capture, an External record is a real event-record
  // node -- a plain record only orders work inside the graph)
  if (L.k5_begin)
    IMP_CUDA(cudaEventRecordWithFlags(L.k5_begin, s, cudaEventRecordExternal));
  const int n_sweep = launch_sweep(sa, w, w.wide, L.sms, s);
  if (L.k5_end)
    IMP_CUDA(cudaEventRecordWithFlags(L.k5_end, s, cudaEventRecordExternal));
  w.last_sweep = sa;

  ReduceArgs rd{};
  rd.ctl = ctl;
  rd.val0 = w.val[0].ptr;
  rd.val1 = w.val[1].ptr;
  for (int t = 0; t < 2; ++t)
    for (int p = 0; p < 2; ++p) {
      rd.old[t][p] = L.vbuf[p] ? L.vbuf[p]
                     : (L.use_ctl ? w.v[t][p].ptr : L.v_explicit[t]);
      rd.nxt[t][p] = L.vbuf[p] ? L.vbuf[p]
                     : (L.use_ctl ? w.v[t][p].ptr : L.new_explicit[t]);
    }
  rd.fixed = L.fixed_dev;
  rd.policy = w.policy.ptr;
  rd.k_begin = L.use_ctl ? h->k_begin : h->k_begin;
  rd.k_count = h->k_count;
  rd.n_u = h->n_u;
  rd.n_w = h->n_w;
  rd.u_max = L.u_max;
  rd.stats = L.stats_explicit;
  rd.pk = L.pk;
  if (h->k_count > 0) {
    if (!rd.fixed && rd.n_u >= 16)
      k_bellman_warp<<<(int)(((int64_t)h->k_count * 32 + 255) / 256), 256, 0,
                       s>>>(rd);
    else
      k_bellman<<<(h->k_count + 255) / 256, 256, 0, s>>>(rd);
    IMP_CUDA(cudaGetLastError());
  }
  const bool control = ctl && !L.skip_control;
  if (control) {
    k_control<<<1, 1, 0, s>>>(ctl, L.stats_reduced);
    IMP_CUDA(cudaGetLastError());
  }
  return 2 + n_sort + n_sweep + (w.wide ? 0 : 1) + (h->k_count > 0 ? 1 : 0) +
         (control ? 1 : 0);
}

__global__ void k_fill(double* p, int64_t n, double v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

void fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n <= 0) return;
  k_fill<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, v);
  IMP_CUDA(cudaGetLastError());
}

}  // namespace

}  // namespace imp

using namespace imp;

extern "C" int imp_run_phase(imp_imdp* h, const imp_phase_desc* d,
                             imp_phase_out* out) {
  return guarded([&] {
    IMP_REQUIRE(h && d && out, "null argument");
    IMP_REQUIRE(h->k_begin == 0 && h->k_count == h->n_s,
                "imp_run_phase needs a single-shard handle; use "
                "imp_shard_sweep for sharded iteration");
    IMP_REQUIRE(d->eps > 0 || d->horizon > 0, "eps must be positive");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s;
    IMP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    const int64_t phase_rows = d->fixed_policy ? (int64_t)h->k_count * h->n_w
                                               : h->n_rows;
    Work w;
    w.init(h, phase_rows);
    if (d->fixed_policy) {
      w.fixed.alloc(h->k_count);
      IMP_CUDA(cudaMemcpyAsync(w.fixed.ptr, d->fixed_policy,
                               sizeof(int64_t) * h->k_count,
                               cudaMemcpyHostToDevice, s));
    }
    build_classes(h, w, d->fixed_policy ? w.fixed.ptr : nullptr, phase_rows, s);
    for (int p = 0; p < 2; ++p) {
      fill(w.v[0][p].ptr, h->n_s, 0.0, s);
      fill(w.v[1][p].ptr, h->n_s, 1.0, s);
    }
    Ctl c{};
    c.k0 = c.k1 = -1;
    c.mode = d->mode;
    c.eps = d->eps;
    c.horizon = d->horizon > 0 ? d->horizon : 0;
    c.max_iter = d->max_iterations > 0 ? d->max_iterations : (1ll << 62);
    IMP_CUDA(cudaMemcpyAsync(w.ctl.ptr, &c, sizeof(Ctl),
                             cudaMemcpyHostToDevice, s));

    Launch L{};
    L.h = h;
    L.w = &w;
    L.sms = sm_count_of(h->device);
    L.spec = d->spec;
    L.lp = d->lp;
    L.u_max = d->u_max;
    L.fixed_dev = d->fixed_policy ? w.fixed.ptr : nullptr;
    L.use_ctl = true;

    // Graph of G iterations; replay until the control block says done.
    const int G = 16;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    // K5 of every captured iteration between two events (event record
    // nodes), read after each replay: the live K5 time of the loop
    cudaEvent_t k5ev[2 * G];
    for (auto& e : k5ev) IMP_CUDA(cudaEventCreate(&e));
    struct EvGuard {
      cudaEvent_t* e;
      int n;
      ~EvGuard() { for (int q = 0; q < n; ++q) cudaEventDestroy(e[q]); }
    } evg{k5ev, 2 * G};
    IMP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int per_graph = 0;
    for (int g = 0; g < G; ++g) {
      L.k5_begin = k5ev[2 * g];
      L.k5_end = k5ev[2 * g + 1];
      per_graph += enqueue_iteration(L, s);
    }
    L.k5_begin = L.k5_end = nullptr;
    IMP_CUDA(cudaStreamEndCapture(s, &graph));
    IMP_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    struct GraphGuard {
      cudaGraph_t g;
      cudaGraphExec_t e;
      ~GraphGuard() { cudaGraphExecDestroy(e); cudaGraphDestroy(g); }
    } gg{graph, exec};

    cudaEvent_t e0, e1;
    IMP_CUDA(cudaEventCreate(&e0));
    IMP_CUDA(cudaEventCreate(&e1));
    IMP_CUDA(cudaEventRecord(e0, s));
    Ctl hc{};
    double ms_k5 = 0.0;
    long long it_before = 0;
    for (;;) {
      IMP_CUDA(cudaGraphLaunch(exec, s));
      count_launches(per_graph, 0);
      IMP_CUDA(cudaMemcpyAsync(&hc, w.ctl.ptr, sizeof(Ctl),
                               cudaMemcpyDeviceToHost, s));
      IMP_CUDA(cudaStreamSynchronize(s));
      // iterations of this replay that ran (later ones exit at once)
      const long long ran = std::min<long long>(G, hc.it - it_before);
      for (int g = 0; g < ran; ++g) {
        float t = 0.f;
        IMP_CUDA(cudaEventElapsedTime(&t, k5ev[2 * g], k5ev[2 * g + 1]));
        ms_k5 += t;
      }
      it_before = hc.it;
      if (hc.done) break;
    }
    IMP_CUDA(cudaEventRecord(e1, s));
    IMP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);

    if (sweep_stats()) {
      unsigned long long mt[2] = {0, 0};
      IMP_CUDA(cudaMemcpy(mt, w.miss_total.ptr, sizeof(mt),
                          cudaMemcpyDeviceToHost));
      const double sweeps = (double)hc.it * (double)phase_rows;
      fprintf(stderr, "[imp] phase: %lld iterations, %lld rows: crossing "
              "moved in %.2f%% of row sweeps, bucketed search in %.2f%%; "
              "%.3f ms/iteration\n", hc.it, (long long)phase_rows,
              sweeps > 0 ? 100.0 * mt[0] / sweeps : 0.0,
              sweeps > 0 ? 100.0 * mt[1] / sweeps : 0.0,
              hc.it ? ms / hc.it : 0.0);
    }
    const int cur = hc.cur;
    if (out->v0)
      IMP_CUDA(cudaMemcpy(out->v0, w.v[0][cur].ptr, sizeof(double) * h->n_s,
                          cudaMemcpyDeviceToHost));
    if (out->v1)
      IMP_CUDA(cudaMemcpy(out->v1, w.v[1][cur].ptr, sizeof(double) * h->n_s,
                          cudaMemcpyDeviceToHost));
    if (out->policy)
      IMP_CUDA(cudaMemcpy(out->policy, w.policy.ptr,
                          sizeof(int64_t) * h->k_count,
                          cudaMemcpyDeviceToHost));
    out->iterations = hc.it;
    out->k0 = hc.k0;
    out->k1 = hc.k1;
    out->fallback = hc.fallback;
    out->gap = hc.gap;
    if (out->gap_log) {
      const int nlog = std::min<int>(hc.gap_log_n, (int)out->gap_log_cap);
      std::copy(hc.gap_log, hc.gap_log + nlog, out->gap_log);
      out->gap_log_n = nlog;
    }
    out->ms_device = ms;
    out->sweeps = hc.it;
    out->ms_sweep = ms_k5;
    if (hc.status != IMP_OK) {
      if (hc.status == IMP_E_CONVERGENCE)
        set_error("gap %.17g above eps=%.17g after %lld iterations", hc.gap,
                  d->eps, hc.it);
      else if (hc.status == IMP_E_MONOTONE)
        set_error("value iterates lost monotonicity; abstraction bounds "
                  "inconsistent (iteration %lld)", hc.it);
      else
        set_error("interval iteration bracket violated (v0 > v1); "
                  "abstraction bounds inconsistent (iteration %lld)", hc.it);
      throw Failure{hc.status};
    }
  });
}

namespace imp {
namespace {
// Explicit-mode stats (order_key-encoded maxima + flag bits) -> plain
// doubles [max|dV0|, max|dV1|, max(V1'-V0'), monotone, bracket]; an empty
// shard reports -inf maxima (neutral under a max all-reduce).
__global__ void k_decode_stats(double* st) {
  unsigned long long* u = reinterpret_cast<unsigned long long*>(st);
  const unsigned flags = *reinterpret_cast<unsigned*>(u + 3);
  double v[3];
  for (int q = 0; q < 3; ++q) v[q] = u[q] ? key_value(u[q]) : -INFINITY;
  st[0] = v[0];
  st[1] = v[1];
  st[2] = v[2];
  st[3] = (flags & 1u) ? 1.0 : 0.0;
  st[4] = (flags & 2u) ? 1.0 : 0.0;
}

void free_work(void* p) { delete static_cast<Work*>(p); }

// Per-handle cached working set for host-driven iterations (sharded loop):
// reallocated only when the phase row count changes.
Work& cached_work(imp_imdp* h, int64_t phase_rows) {
  Work* w = static_cast<Work*>(h->sweep_cache);
  if (!w || h->sweep_cache_rows != phase_rows) {
    delete w;
    w = new Work();
    w->init(h, phase_rows);
    h->sweep_cache = w;
    h->sweep_cache_rows = phase_rows;
    h->free_cache = free_work;
  }
  return *w;
}

// Shared body of the explicit (host-driven) single iterations.
void explicit_step(imp_imdp* h, const double* v0, const double* v1, int spec,
                   int lp, int u_max, const int64_t* fixed_dev, double* new0,
                   double* new1, int64_t* policy_dev, double* stats,
                   cudaStream_t s) {
  const int64_t phase_rows = fixed_dev ? (int64_t)h->k_count * h->n_w
                                       : h->n_rows;
  Work& w = cached_work(h, phase_rows);
  // classes of the unfixed phase are a property of the handle; a fixed
  // policy's may change between calls
  if (fixed_dev || !w.classes_all) {
    build_classes(h, w, fixed_dev, phase_rows, s);
    w.classes_all = !fixed_dev;
  }
  Launch L{};
  L.h = h;
  L.w = &w;
  L.sms = sm_count_of(h->device);
  L.spec = spec;
  L.lp = lp;
  L.u_max = u_max;
  L.fixed_dev = fixed_dev;
  L.v_explicit[0] = v0;
  L.v_explicit[1] = v1;
  L.new_explicit[0] = new0;
  L.new_explicit[1] = new1;
  L.stats_explicit = stats;
  L.use_ctl = false;
  count_launches(enqueue_iteration(L, s), 0);
  if (stats) {
    k_decode_stats<<<1, 1, 0, s>>>(stats);
    IMP_CUDA(cudaGetLastError());
    count_launches(1, 0);
  }
  if (policy_dev)
    IMP_CUDA(cudaMemcpyAsync(policy_dev, w.policy.ptr,
                             sizeof(int64_t) * h->k_count,
                             cudaMemcpyDeviceToDevice, s));
  IMP_CUDA(cudaStreamSynchronize(s));
}
}  // namespace
}  // namespace imp

extern "C" int imp_bellman_step(imp_imdp* h, const double* values,
                                int32_t spec, int32_t lp, int32_t u_max,
                                const int64_t* fixed_policy,
                                double* new_values, int64_t* chosen) {
  return guarded([&] {
    IMP_REQUIRE(h && values && new_values, "null argument");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = 0;
    DevBuf<double> v(h->n_s), n0(std::max(h->k_count, 1)),
        n1(std::max(h->k_count, 1));
    DevBuf<int64_t> fx, pol(std::max(h->k_count, 1));
    IMP_CUDA(cudaMemcpy(v.ptr, values, sizeof(double) * h->n_s,
                        cudaMemcpyHostToDevice));
    if (fixed_policy) {
      fx.alloc(h->k_count);
      IMP_CUDA(cudaMemcpy(fx.ptr, fixed_policy, sizeof(int64_t) * h->k_count,
                          cudaMemcpyHostToDevice));
    }
    explicit_step(h, v.ptr, v.ptr, spec, lp, u_max,
                  fixed_policy ? fx.ptr : nullptr, n0.ptr, n1.ptr, pol.ptr,
                  nullptr, s);
    IMP_CUDA(cudaMemcpy(new_values, n0.ptr, sizeof(double) * h->k_count,
                        cudaMemcpyDeviceToHost));
    if (chosen)
      IMP_CUDA(cudaMemcpy(chosen, pol.ptr, sizeof(int64_t) * h->k_count,
                          cudaMemcpyDeviceToHost));
  });
}

extern "C" int imp_shard_sweep(imp_imdp* h, const double* v0,
                               const double* v1, int32_t spec, int32_t lp,
                               int32_t u_max, const int64_t* fixed_dev,
                               double* new0, double* new1, int64_t* policy,
                               double* stats, void* stream) {
  return guarded([&] {
    IMP_REQUIRE(h && v0 && v1 && new0 && new1 && stats, "null argument");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    IMP_CUDA(cudaMemsetAsync(stats, 0, 5 * sizeof(double), s));
    explicit_step(h, v0, v1, spec, lp, u_max, fixed_dev, new0, new1, policy,
                  stats, s);
  });
}

extern "C" int imp_row_values(imp_imdp* h, const double* weights, int32_t lp,
                              double* out, int32_t on_device) {
  return guarded([&] {
    IMP_REQUIRE(h && weights && out, "null argument");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = 0;
    const int n = h->n_s + 2;
    std::vector<double> hw(n);
    if (on_device)
      IMP_CUDA(cudaMemcpy(hw.data(), weights, sizeof(double) * n,
                          cudaMemcpyDeviceToHost));
    else
      std::copy(weights, weights + n, hw.begin());
    // The sweep prices (values, d1, d2); feed the two virtual weights
    // through a spec-agnostic path: run with explicit values and patch the
    // virtual-slot weights via a custom spec encoding.
    Work w;
    w.init(h, h->n_rows);
    DevBuf<double> v(h->n_s);
    IMP_CUDA(cudaMemcpy(v.ptr, hw.data(), sizeof(double) * h->n_s,
                        cudaMemcpyHostToDevice));
    OrderArgs oa{};
    for (int t = 0; t < 2; ++t)
      for (int p = 0; p < 2; ++p) oa.v[t][p] = v.ptr;
    oa.n_s = h->n_s;
    oa.n = n;
    oa.d1 = hw[h->n_s];
    oa.d2 = hw[h->n_s + 1];
    oa.lp_max = lp == IMP_LP_MAX;
    for (int t = 0; t < 2; ++t) {
      oa.keys[t] = w.keys_in[t].ptr;
      oa.idx[t] = w.idx_in[t].ptr;
    }
    oa.colw = w.colw.ptr;
    k_order_keys<<<(n + 255) / 256, 256, 0, s>>>(oa);
    IMP_CUDA(cudaGetLastError());
    {
      uint64_t* const kin[2] = {w.keys_in[0].ptr, w.keys_in[1].ptr};
      uint64_t* const kout[2] = {w.keys_out[0].ptr, w.keys_out[1].ptr};
      int* const iin[2] = {w.idx_in[0].ptr, w.idx_in[1].ptr};
      int* const pout[2] = {w.perm[0].ptr, w.perm[1].ptr};
      launch_sort(nullptr, n, kin, iin, kout, pout, s);
    }
    RankArgs ra{};
    ra.n = n;
    ra.perm[0] = w.perm[0].ptr;
    ra.perm[1] = w.perm[1].ptr;
    ra.colw = w.colw.ptr;
    ra.rank = w.rank.ptr;
    ra.ws[0] = w.ws[0].ptr;
    ra.ws[1] = w.ws[1].ptr;
    k_ranks<<<(n + 1 + 255) / 256, 256, 0, s>>>(ra);
    IMP_CUDA(cudaGetLastError());
    if (!w.wide) {
      k_pack_ranks<<<(n + 255) / 256, 256, 0, s>>>(nullptr, n, w.rank.ptr,
                                                   w.rank16.ptr);
      IMP_CUDA(cudaGetLastError());
    }
    SweepArgs sa{};
    sa.row_ptr = h->row_ptr.ptr;
    sa.col = h->col.ptr;
    sa.lo = h->lo.ptr;
    sa.hi = h->hi.ptr;
    sa.hd = h->hd.ptr;
    sa.r_min = h->r_min.ptr;
    sa.r_max = h->r_max.ptr;
    sa.a_min = h->a_min.ptr;
    sa.a_max = h->a_max.ptr;
    sa.slack = h->slack.ptr;
    sa.colw = w.colw.ptr;
    sa.rank = w.rank.ptr;
    sa.rank16 = w.rank16.ptr;
    sa.ws0 = w.ws[0].ptr;
    sa.ws1 = w.ws[1].ptr;
    sa.n_phase_rows = h->n_rows;
    sa.n_u = h->n_u;
    sa.n_w = h->n_w;
    sa.n_s = h->n_s;
    sa.n = n;
    sa.nbits = w.nbits;
    sa.out0 = w.val[0].ptr;
    sa.out1 = w.val[1].ptr;
    build_classes(h, w, nullptr, h->n_rows, s);
    launch_sweep(sa, w, w.wide, sm_count_of(h->device), s);
    IMP_CUDA(cudaMemcpy(out, w.val[0].ptr, sizeof(double) * h->n_rows,
                        on_device ? cudaMemcpyDeviceToDevice
                                  : cudaMemcpyDeviceToHost));
  });
}

// K5 alone, for the HBM roofline: one iteration sets up the orders for a
// scrambled value vector, then `reps` twin sweeps over every phase-1 row are
// timed with CUDA events on the launching stream.  *ms = mean per sweep.
extern "C" int imp_time_sweep(imp_imdp* h, int32_t spec, int32_t lp,
                              int32_t reps, double* ms) {
  return guarded([&] {
    IMP_REQUIRE(h && ms && reps > 0, "bad argument");
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s;
    IMP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
    std::vector<double> hv(h->n_s);
    for (int c = 0; c < h->n_s; ++c) {
      double f = c * 0.6180339887498949;
      hv[c] = f - std::floor(f);
    }
    DevBuf<double> v0(h->n_s), v1(h->n_s), n0(std::max(h->k_count, 1)),
        n1(std::max(h->k_count, 1)), st(4);
    IMP_CUDA(cudaMemcpy(v0.ptr, hv.data(), sizeof(double) * h->n_s,
                        cudaMemcpyHostToDevice));
    for (auto& x : hv) x = 1.0 - x;
    IMP_CUDA(cudaMemcpy(v1.ptr, hv.data(), sizeof(double) * h->n_s,
                        cudaMemcpyHostToDevice));
    Work w;
    w.init(h, h->n_rows);
    Launch L{};
    L.h = h;
    L.w = &w;
    L.sms = sm_count_of(h->device);
    L.spec = spec;
    L.lp = lp;
    L.u_max = spec == IMP_SPEC_REACH;
    L.v_explicit[0] = v0.ptr;
    L.v_explicit[1] = v1.ptr;
    L.new_explicit[0] = n0.ptr;
    L.new_explicit[1] = n1.ptr;
    L.stats_explicit = st.ptr;
    L.use_ctl = false;
    build_classes(h, w, nullptr, h->n_rows, s);
    enqueue_iteration(L, s);
    const SweepArgs sa = w.last_sweep;
    cudaEvent_t e0, e1;
    IMP_CUDA(cudaEventCreate(&e0));
    IMP_CUDA(cudaEventCreate(&e1));
    IMP_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) launch_sweep(sa, w, w.wide, L.sms, s);
    IMP_CUDA(cudaEventRecord(e1, s));
    IMP_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    count_launches(reps, 0);
    *ms = t / reps;
  });
}

// ---------------------------------------------------------------------------
// Device-resident sharded phase loop (multi-GPU; reference _run_phase,
// synthesis.py:145-205, over state shards).  Per iteration the caller
// enqueues, on one stream and without host synchronisation:
//   imp_shard_loop_sweep    orders, K5 and the Bellman step of this shard,
//                           writing its [V0' | V1'] chunk into the packed
//                           buffer of the iteration and its statistics;
//   all-gather (NCCL, in place) of the chunk and all-reduce(max) of the
//                           5 statistics -- torch.distributed, the caller;
//   imp_shard_loop_control  the termination logic of every rank on the
//                           reduced statistics (k_control).
// Kernels of an iteration after termination exit at once, so a CUDA graph
// of G iterations can be replayed until imp_shard_loop_poll reports done:
// one host round trip per G sweeps.
// ---------------------------------------------------------------------------

struct imp_shard_loop {
  imp_imdp* h = nullptr;
  imp::Work w;
  imp::DevBuf<int64_t> sb;
  std::vector<int64_t> hsb;
  imp::Launch L{};
  double* stats = nullptr;
  int world = 1, rank = 0;
  int64_t pw = 0;
  double* buf[2] = {nullptr, nullptr};
  double eps = 0.0;
};

namespace imp {
namespace {
__global__ void k_pack_init(double* b0, double* b1, int64_t total, int64_t pw) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= total) return;
  const double v = ((q / pw) & 1) ? 1.0 : 0.0;   // track 0: zeros, 1: ones
  b0[q] = v;
  b1[q] = v;
}

// this device's statistics slots -> the 5 doubles the all-reduce combines
__global__ void k_export_stats(Ctl* c, double* st) {
  const unsigned long long u[3] = {c->slot_d0, c->slot_d1, c->slot_gap};
  for (int q = 0; q < 3; ++q) st[q] = u[q] ? key_value(u[q]) : -INFINITY;
  st[3] = (c->slot_flags & 1u) ? 1.0 : 0.0;
  st[4] = (c->slot_flags & 2u) ? 1.0 : 0.0;
  c->slot_d0 = c->slot_d1 = c->slot_gap = 0ull;
  c->slot_flags = 0u;
}
}  // namespace
}  // namespace imp

extern "C" int imp_shard_loop_begin(imp_imdp* h, const imp_phase_desc* d,
                                    const int64_t* shard_begin, int32_t world,
                                    double* vbuf0, double* vbuf1, int64_t pw,
                                    double* stats, void* stream,
                                    imp_shard_loop** out) {
  imp_shard_loop* L = nullptr;
  int st = guarded([&] {
    IMP_REQUIRE(h && d && shard_begin && vbuf0 && vbuf1 && stats && out,
                "null argument");
    IMP_REQUIRE(world >= 1 && world <= 64, "world size %d unsupported", world);
    IMP_REQUIRE(d->eps > 0 || d->horizon > 0, "eps must be positive");
    IMP_REQUIRE(shard_begin[0] == 0 && shard_begin[world] == h->n_s,
                "shard table must cover the %d safe states", h->n_s);
    int rank = -1;
    int64_t widest = 0;
    for (int r = 0; r < world; ++r) {
      IMP_REQUIRE(shard_begin[r + 1] >= shard_begin[r], "shard table not sorted");
      widest = std::max<int64_t>(widest, shard_begin[r + 1] - shard_begin[r]);
      if (shard_begin[r] == h->k_begin &&
          shard_begin[r + 1] == (int64_t)h->k_begin + h->k_count)
        rank = r;
    }
    IMP_REQUIRE(rank >= 0, "this handle's states [%d, %d) are not a shard of "
                "the table", h->k_begin, h->k_begin + h->k_count);
    IMP_REQUIRE(pw >= widest && pw >= 1, "packed width %lld below the widest "
                "shard (%lld)", (long long)pw, (long long)widest);
    IMP_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    L = new imp_shard_loop();
    L->h = h;
    L->world = world;
    L->rank = rank;
    L->pw = pw;
    L->buf[0] = vbuf0;
    L->buf[1] = vbuf1;
    L->stats = stats;
    L->eps = d->eps;
    L->hsb.assign(shard_begin, shard_begin + world + 1);
    L->sb.alloc(world + 1);
    IMP_CUDA(cudaMemcpyAsync(L->sb.ptr, shard_begin,
                             sizeof(int64_t) * (world + 1),
                             cudaMemcpyHostToDevice, s));
    const int64_t phase_rows = d->fixed_policy ? (int64_t)h->k_count * h->n_w
                                               : h->n_rows;
    Work& w = L->w;
    w.init(h, phase_rows);
    if (d->fixed_policy) {
      w.fixed.alloc(std::max(h->k_count, 1));
      IMP_CUDA(cudaMemcpyAsync(w.fixed.ptr, d->fixed_policy,
                               sizeof(int64_t) * h->k_count,
                               cudaMemcpyHostToDevice, s));
    }
    build_classes(h, w, d->fixed_policy ? w.fixed.ptr : nullptr, phase_rows, s);
    const int64_t total = (int64_t)world * 2 * pw;
    k_pack_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(vbuf0, vbuf1,
                                                                total, pw);
    IMP_CUDA(cudaGetLastError());
    Ctl c{};
    c.k0 = c.k1 = -1;
    c.mode = d->mode;
    c.eps = d->eps;
    c.horizon = d->horizon > 0 ? d->horizon : 0;
    c.max_iter = d->max_iterations > 0 ? d->max_iterations : (1ll << 62);
    IMP_CUDA(cudaMemcpyAsync(w.ctl.ptr, &c, sizeof(Ctl),
                             cudaMemcpyHostToDevice, s));
    Launch& la = L->L;
    la.h = h;
    la.w = &w;
    la.sms = sm_count_of(h->device);
    la.spec = d->spec;
    la.lp = d->lp;
    la.u_max = d->u_max;
    la.fixed_dev = d->fixed_policy ? w.fixed.ptr : nullptr;
    la.use_ctl = true;
    la.skip_control = true;
    la.pk = Packed{L->sb.ptr, world, pw};
    la.vbuf[0] = vbuf0;
    la.vbuf[1] = vbuf1;
    la.stats_reduced = stats;
    IMP_CUDA(cudaStreamSynchronize(s));
    *out = L;
  });
  if (st != IMP_OK) delete L;
  return st;
}

extern "C" int imp_shard_loop_sweep(imp_shard_loop* L, void* stream) {
  return guarded([&] {
    IMP_REQUIRE(L, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    count_launches(enqueue_iteration(L->L, s), 0);
    k_export_stats<<<1, 1, 0, s>>>(L->w.ctl.ptr, L->stats);
    IMP_CUDA(cudaGetLastError());
    count_launches(1, 0);
  });
}

extern "C" int imp_shard_loop_control(imp_shard_loop* L, void* stream) {
  return guarded([&] {
    IMP_REQUIRE(L, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    k_control<<<1, 1, 0, s>>>(L->w.ctl.ptr, L->stats);
    IMP_CUDA(cudaGetLastError());
    count_launches(1, 0);
  });
}

extern "C" int imp_shard_loop_poll(imp_shard_loop* L, imp_phase_out* out,
                                   int32_t* done, void* stream) {
  return guarded([&] {
    IMP_REQUIRE(L && out && done, "null argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Ctl hc{};
    IMP_CUDA(cudaMemcpyAsync(&hc, L->w.ctl.ptr, sizeof(Ctl),
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaStreamSynchronize(s));
    *done = hc.done;
    out->iterations = hc.it;
    out->sweeps = hc.it;
    out->k0 = hc.k0;
    out->k1 = hc.k1;
    out->fallback = hc.fallback;
    out->gap = hc.gap;
    if (out->gap_log) {
      const int nlog = std::min<int>(hc.gap_log_n, (int)out->gap_log_cap);
      std::copy(hc.gap_log, hc.gap_log + nlog, out->gap_log);
      out->gap_log_n = nlog;
    }
    if (!hc.done) return;
    const imp_imdp* h = L->h;
    if (out->v0 || out->v1) {   // unpack the current full vectors
      const int64_t total = (int64_t)L->world * 2 * L->pw;
      std::vector<double> hb(total);
      IMP_CUDA(cudaMemcpy(hb.data(), L->buf[hc.cur], sizeof(double) * total,
                          cudaMemcpyDeviceToHost));
      for (int r = 0; r < L->world; ++r)
        for (int64_t c = L->hsb[r]; c < L->hsb[r + 1]; ++c) {
          const int64_t base = (int64_t)r * 2 * L->pw + (c - L->hsb[r]);
          if (out->v0) out->v0[c] = hb[base];
          if (out->v1) out->v1[c] = hb[base + L->pw];
        }
    }
    if (out->policy)
      IMP_CUDA(cudaMemcpy(out->policy, L->w.policy.ptr,
                          sizeof(int64_t) * h->k_count,
                          cudaMemcpyDeviceToHost));
    if (hc.status != IMP_OK) {
      if (hc.status == IMP_E_CONVERGENCE)
        set_error("gap %.17g above eps=%.17g after %lld iterations", hc.gap,
                  L->eps, hc.it);
      else if (hc.status == IMP_E_MONOTONE)
        set_error("value iterates lost monotonicity; abstraction bounds "
                  "inconsistent (iteration %lld)", hc.it);
      else
        set_error("interval iteration bracket violated (v0 > v1); "
                  "abstraction bounds inconsistent (iteration %lld)", hc.it);
      throw Failure{hc.status};
    }
  });
}

extern "C" void imp_shard_loop_free(imp_shard_loop* L) { delete L; }
