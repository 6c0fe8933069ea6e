// IMDP construction kernels, JIT-compiled by NVRTC per dynamics spec.
//
// The module source is  ndtr.h + <generated config> + <generated dynamics>
// + this file.  The generated config defines
//   IMP_N, IMP_NC             state dimension, folded constants per (j, i)
//   kNDeps[IMP_N]             state dependencies of each f_d
//   kDeps[IMP_N][IMP_N]       their indices (ascending, -1 padded)
// and the dynamics provide imp_f<d>(x, k) / imp_fd(d, x, k), x = full state
// vector, k = the row's folded x-free subexpressions.  Compiled with
// --fmad=false so every expression, centroid and Horner step rounds like
// the reference's numpy evaluation.
//
// Stages (reference pkg/src/impact/abstraction.py):
//   1 k_mean_ranges  per (row, d, sign): NM over the dependency sub-cell,
//                    min over starts                       (:256-284)
//   2 k_outer        per row (CTA): exact per-dimension extremes (:287-297),
//                    pruned enumeration of the lattice box whose outer
//                    product can exceed the cutoff, cutoff / live window,
//                    CSR count + write (two launches), separable values,
//                    r / a terms and cover leak           (:442-508, :300-319)
//   3 k_refine       coupled dynamics: one thread per NM instance
//                    (row, live box, min|max) running all `multistart`
//                    starts through a one-evaluation-per-step state machine,
//                    simplex held in shared memory      (:322-375, :465-495;
//                                                        optimize.py:47-155)
//   4 k_assemble     clip, low-cost, row-sum repair, hard errors (:607-659)

#define IMP_INF __longlong_as_double(0x7ff0000000000000ll)

__device__ __forceinline__ double imp_min(double a, double b) {
  return (a < b || a != a) ? a : b;   // numpy.minimum propagates NaN
}
__device__ __forceinline__ double imp_max(double a, double b) {
  return (a > b || a != a) ? a : b;
}
// np.clip on non-NaN values, signed zeros included: numpy's clip loop is
// min(max(x, lo), hi) with max(a, b) = a > b ? a : b, min(a, b) = a < b ? a : b
__device__ __forceinline__ double imp_clip(double x, double lo, double hi) {
  const double t = x > lo ? x : lo;
  return t < hi ? t : hi;
}
__device__ __forceinline__ bool imp_finite(double x) {
  return x - x == 0.0;
}

struct BuildParams {
  int n_u, n_w, k_begin, k_count;
  long long n_rows;
  int n_s, n_t, n_a, total;
  const int* counts;          // (N)
  const int* edge_off;        // (N) offsets into edges
  const int* strides;         // (N) flat-index strides (row-major)
  const double* eta;          // (N)
  const double* sigma;        // (N)
  const double* edges;
  const double* cover_lo;
  const double* cover_hi;
  const double* src_lo;       // (n_s, N) clipped source cells, global k
  const double* src_hi;
  const double* consts;       // (n_u * n_w, NC)
  const int* label;           // (total) >= 0 safe pos, -1-t target,
                              // -1-n_t-a avoid; nullptr: every point safe
  const int* safe_flat;       // (n_s)
  const int* target_flat;     // (n_t)
  const int* avoid_flat;      // (n_a)
  double cutoff, tol;
  int low_cost, separable;
  int max_evals_fixed;        // 0: 200 * dim
  int multistart;             // 0: 1 + 2 * dim
  // stage 1
  double* mlo;                // (n_rows, N)
  double* mhi;
  // stage 2
  int write;                  // 0: count pass, 1: write pass
  long long* t_count;         // (n_rows) count pass output
  long long* x_count;         // (n_rows) aux items (coupled)
  const long long* row_ptr;   // (n_rows + 1)
  const long long* aux_ptr;   // (n_rows + 1)
  int* col;
  double* lo;
  double* hi;
  int* aux_code;              // >= 0 target index, < 0: -1 - avoid index
  double* aux_min;
  double* aux_max;
  double* raw;                // (n_rows, 6): r_min r_max av_min av_max
                              //              leak_min leak_max
  // stage 3
  long long n_items;          // nnz + n_aux + n_rows
  long long* evals;           // counters (atomic): [0] refinement evals,
                              // [1] lane slots, [2] work cursor, [3] shared
                              // simplex values, [4] live entries, [5]
                              // mean-range evals
  // stage 4
  double* r_min;
  double* r_max;
  double* a_min;
  double* a_max;
  // errors
  unsigned long long* err;    // [0]: first non-finite row, [1]: first
                              // min-side excess row, [2]: max-side deficit
  double* err_val;            // [1], [2]: the offending magnitudes
  // noise scales by value (kernel-parameter space: constant-bank operands)
  // and RN(1/sigma) for imp_div_rcp (NaN when sigma is outside 2^+-100)
  double sig[16];
  double sig_rcp[16];
  // separable dynamics: per-key mean ranges and 1-D tables (k_sep_tables)
  int sep;
  const double* dim_lo;       // (sum counts) clipped coordinate cells
  const double* dim_hi;
  double* sep_mr;             // (keys, 2)
  double* sep_tab;            // per key: counts[d] x {min, max}
  // Monte Carlo noise (IMP_MC modules)
  long long row0;             // global index of local row 0 (seeding)
  int mc_samples;
  unsigned long long mc_seed;
  double mc_norm;
  const double* inv_cov;      // (N, N)
  // destination boxes: {edges[b_d], edges[b_d + 1]} of every lattice state,
  // (total, N), so k_refine's item setup needs no integer divisions
  const double2* box;
};

__device__ __forceinline__ int imp_max_evals(const BuildParams& P, int dim) {
  return P.max_evals_fixed ? P.max_evals_fixed : 200 * (dim > 1 ? dim : 1);
}
__device__ __forceinline__ int imp_multistart(const BuildParams& P, int dim) {
  return P.multistart ? P.multistart : 1 + 2 * dim;
}

__device__ __forceinline__ void imp_row_kji(const BuildParams& P, long long r,
                                            int& k, int& j, int& i) {
  i = (int)(r % P.n_w);
  long long rest = r / P.n_w;
  j = (int)(rest % P.n_u);
  k = P.k_begin + (int)(rest / P.n_u);
}

// Deterministic start list (optimize.py:28-44) for a D-dim box.
template <int D>
__device__ __forceinline__ void imp_start_point(const double* lo,
                                                const double* hi, int s,
                                                double* out) {
  double c[D];
#pragma unroll
  for (int d = 0; d < D; ++d) c[d] = (lo[d] + hi[d]) / 2;
  int b = s;
  if (s > 2 * D) b = (s - 2 * D) % (1 + 2 * D);
#pragma unroll
  for (int d = 0; d < D; ++d) out[d] = c[d];
  if (b > 0) {
    int dd = (b - 1) >> 1;
    bool up = (b - 1) & 1;
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d == dd) out[d] = up ? hi[d] : lo[d];
  }
  if (s > 2 * D) {
#pragma unroll
    for (int d = 0; d < D; ++d) out[d] = (out[d] + c[d]) / 2;
  }
}

// ---------------------------------------------------------------------------
// Nelder-Mead (optimize.py:47-155) as a one-evaluation-per-step state
// machine.  point() gives the next point to evaluate, feed() consumes its
// objective value.  Vertices live in shared memory in fixed physical slots
// (conflict-free stride = block size); the sorted order is a packed 4-bit
// permutation `ord` in a register, recomputed by a branch-free stable rank
// (key = value, ties by current position -- numpy's stable argsort).  All
// lanes that finish a step in any phase run the single iterate() site
// together, so the bookkeeping does not serialise a warp per phase.
// ---------------------------------------------------------------------------
enum { NM_INIT = 0, NM_REFLECT = 1, NM_SECOND = 2, NM_SHRINK = 3 };
enum { NM_EXPAND = 0, NM_OUTSIDE = 1, NM_INSIDE = 2 };

// Shared-memory doubles per thread: D + 4 points (the D + 1 vertices, then
// centroid, reflection and candidate -- kept out of registers so the
// objective has room) and D + 1 vertex values.
template <int D>
__host__ __device__ constexpr int imp_nm_doubles() { return (D + 4) * D + D + 1; }

template <int D, int S>   // S: threads per block = shared-memory stride
struct NelderMead {
  static_assert(D + 1 <= 16, "4-bit permutation");
  static constexpr int CEN = D + 1, REF = D + 2, CAND = D + 3;
  double* X;   // X[(point * D + d) * S], points 0..D vertices, CEN, REF, CAND
  double* F;   // F[slot * S]
  unsigned long long ord;
  double lo[D], hi[D];
  double fr, tol, best;
  int phase, v, evals, kind, max_evals;
  int pend;    // iterate() owed: 0 no, 1 insert the new worst, 2 full sort
  bool done;

  __device__ __forceinline__ int slot(int q) const {
    return (int)((ord >> (4 * q)) & 15ull);
  }
  __device__ __forceinline__ double& xs(int s, int d) { return X[(s * D + d) * S]; }
  __device__ __forceinline__ double& fs(int s) { return F[s * S]; }

  __device__ void start(const double* s) {
    ord = 0;
#pragma unroll
    for (int q = 0; q <= D; ++q) ord |= (unsigned long long)q << (4 * q);
#pragma unroll
    for (int d = 0; d < D; ++d) xs(0, d) = s[d];
#pragma unroll
    for (int e = 0; e < D; ++e) {
      const double step = 0.25 * (hi[e] - lo[e]);
#pragma unroll
      for (int d = 0; d < D; ++d) xs(e + 1, d) = s[d];
      const double up = s[e] + step;
      xs(e + 1, e) = up <= hi[e] ? up : s[e] - step;
    }
    phase = NM_INIT;
    v = 0;
    evals = 0;
    pend = 0;
    done = false;
  }

  // The max instance of a box starts from the same simplex as its min
  // instance (optimize.py:60-72: the starts and the cell are shared), so
  // its initial values are the min run's, negated (the objective is
  // prob * -1.0, _BoxProbObjective:349): no evaluations, same bits.
  // Fi[q * S] holds the min run's values in vertex order.
  __device__ void start_shared(const double* s, const double* Fi) {
    start(s);
#pragma unroll
    for (int q = 0; q <= D; ++q) fs(q) = Fi[q * S] * -1.0;
    v = D + 1;
    evals = D + 1;
    pend = 2;
  }

  // A shrink (optimize.py:140-148) moves vertex v towards the best vertex
  // here, when v is about to be evaluated, instead of all D vertices at the
  // shrink decision: the same arithmetic per vertex, but done on the trip
  // every lane runs instead of in a rarely-taken branch that serialises.
  __device__ __forceinline__ void point(double* p) {
#if IMP_NM_UNIFIED
    // Every phase's next point is base + coef * (x - y) (clipped to the
    // cell except for shrinks; the initial simplex: the vertex itself), so
    // all lanes run ONE path here whatever their phase, instead of the
    // reflection point in iterate() and the second candidate in feed()
    // running as separate divergent blocks.  Same operands, same order,
    // same bits (optimize.py:88, 104-117, 140-143).
    const int ph = phase;
    const int sv = slot(v), s0 = slot(0), sw = slot(D);
    const bool init = ph == NM_INIT, shr = ph == NM_SHRINK;
    const bool sec = ph == NM_SECOND;
    const int b = shr ? s0 : (init ? sv : CEN);
    const int x = shr || init ? sv
                  : (sec && kind == NM_OUTSIDE ? REF
                     : (sec && kind == NM_INSIDE ? sw : CEN));
    const int y = shr ? s0 : (init ? sv
                  : (sec && kind != NM_EXPAND ? CEN : sw));
    const double coef = shr ? 0.5 : (init ? 0.0
                        : (!sec ? 1.0 : (kind == NM_EXPAND ? 2.0 : 0.5)));
    const int dst = shr || init ? sv : (sec ? CAND : REF);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double bv = xs(b, d);
      double t = bv + coef * (xs(x, d) - xs(y, d));
      t = shr ? t : imp_clip(t, lo[d], hi[d]);
      t = init ? bv : t;
      xs(dst, d) = t;
      p[d] = t;
    }
#else
    const bool shr = phase == NM_SHRINK;
    const bool vert = phase == NM_INIT || shr;
    const int ps = vert ? slot(v) : (phase == NM_REFLECT ? REF : CAND);
    const int s0 = slot(0);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double q = xs(ps, d);
      if (shr) {
        const double b = xs(s0, d);
        q = b + 0.5 * (q - b);
        xs(ps, d) = q;
      }
      p[d] = q;
    }
#endif
  }

  // stable sort, termination test, centroid and reflection point.
  // full: every vertex may have moved (initial simplex, shrink) -- rank all
  // D + 1 keys.  Otherwise only the worst slot got a new value while the
  // others stay sorted: numpy's stable argsort of [sorted prefix, new] puts
  // the new key after every prefix key <= it, so one pass of D compares
  // finds its rank (optimize.py:75-78).
  __device__ void iterate(bool full) {
    pend = 0;
    if (full) {
      double key[D + 1];
      int sl[D + 1];
#pragma unroll
      for (int q = 0; q <= D; ++q) {
        sl[q] = slot(q);
        key[q] = fs(sl[q]);
      }
      unsigned long long nord = 0;
#pragma unroll
      for (int q = 0; q <= D; ++q) {
        int rk = 0;
#pragma unroll
        for (int u = 0; u <= D; ++u)
          rk += (key[u] < key[q]) || (u < q && key[u] == key[q]);
        nord |= (unsigned long long)sl[q] << (4 * rk);
      }
      ord = nord;
    } else {
      const int sw = slot(D);
      const double fn = fs(sw);
      int r = 0;
#pragma unroll
      for (int q = 0; q < D; ++q) r += fs(slot(q)) <= fn;
      const unsigned long long low = (1ull << (4 * r)) - 1;
      const unsigned long long mid = ord & ~low & ((1ull << (4 * D)) - 1);
      ord = (ord & low) | ((unsigned long long)sw << (4 * r)) | (mid << 4);
    }
    const double f0 = fs(slot(0));
    const double spread = fs(slot(D)) - f0;
    if (!(spread > tol && evals < max_evals)) {
      done = true;
      best = f0;
      return;
    }
    const int sw = slot(D);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double s = xs(slot(0), d);
#pragma unroll
      for (int vv = 1; vv < D; ++vv) s += xs(slot(vv), d);
      const double cd = imp_div_rcp(s, (double)D, 1.0 / D);
      xs(CEN, d) = cd;
#if !IMP_NM_UNIFIED
      xs(REF, d) = imp_clip(cd + 1.0 * (cd - xs(sw, d)), lo[d], hi[d]);
#endif
    }
    phase = NM_REFLECT;
  }

  // consume the value of the last point(); the iterate() it may owe is left
  // in `pend` so that a kernel can run it at one site for all its lanes
  __device__ void feed(double fp) {
    // decisions per phase, then ONE block that moves an accepted point into
    // the worst slot (a warp runs each divergent block once per trip, so the
    // reflect-accept and second-candidate-take moves share it)
    bool iter = false, full = false, replace = false;
    int from = REF;
    double newf = fp;
    const int sw = slot(D);
    if (phase == NM_INIT || phase == NM_SHRINK) {
      fs(slot(v)) = fp;
      if (++v > D) {
        evals += phase == NM_INIT ? D + 1 : D;
        iter = full = true;
      }
    } else if (phase == NM_REFLECT) {
      fr = fp;
      evals += 1;
      const double f0 = fs(slot(0)), fsw = fs(slot(D - 1)), fw = fs(sw);
      if (fr < f0 || fr >= fsw) {
        kind = fr < f0 ? NM_EXPAND : (fr < fw ? NM_OUTSIDE : NM_INSIDE);
#if !IMP_NM_UNIFIED
        const double coef = kind == NM_EXPAND ? 2.0 : 0.5;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double w = xs(sw, d), cd = xs(CEN, d);
          const double dir = kind == NM_EXPAND ? cd - w
                             : (kind == NM_OUTSIDE ? xs(REF, d) - cd : w - cd);
          xs(CAND, d) = imp_clip(cd + coef * dir, lo[d], hi[d]);
        }
#endif
        phase = NM_SECOND;
      } else {
        replace = true;          // from REF, value fr
      }
    } else {  // NM_SECOND
      evals += 1;
      const bool take = kind == NM_EXPAND ||
                        (kind == NM_OUTSIDE ? fp < fr : fp < fs(sw));
      if (take) {
        const bool use_c = kind != NM_EXPAND || fp < fr;
        replace = true;
        from = use_c ? CAND : REF;
        newf = use_c ? fp : fr;
      } else {   // shrink: vertices 1..D move in point()
        v = 1;
        phase = NM_SHRINK;
      }
    }
    if (replace) {
#pragma unroll
      for (int d = 0; d < D; ++d) xs(sw, d) = xs(from, d);
      fs(sw) = newf;
      iter = true;
    }
    if (iter) pend = full ? 2 : 1;
  }

  __device__ void step(double fp) {
    feed(fp);
    if (pend) iterate(pend == 2);
  }
};


// Division of 0 <= n < 2^31 by a run-time divisor d >= 1 fixed per row
// (the pruned box's extents): q = umulhi(n, mul) >> shr with mul =
// ceil(2^p / d), p = 31 + ceil(log2 d) -- exact for every such n, two
// instructions instead of the integer-division sequence.
struct ImpFastDiv {
  unsigned mul;   // 0: d == 1
  int shr;
};
__device__ __forceinline__ ImpFastDiv imp_fastdiv(int d) {
  ImpFastDiv f{0u, 0};
  if (d > 1) {
    const int l = 32 - __clz(d - 1);
    const int p = 31 + l;
    f.mul = (unsigned)(((1ull << p) + (unsigned long long)d - 1) /
                       (unsigned long long)d);
    f.shr = p - 32;
  }
  return f;
}
__device__ __forceinline__ int imp_fdiv(int n, ImpFastDiv f) {
  return f.mul ? (int)(__umulhi((unsigned)n, f.mul) >> f.shr) : n;
}

__device__ __forceinline__ void imp_flag_nonfinite(const BuildParams& P,
                                                   long long row) {
  atomicMin(P.err, (unsigned long long)row);
}

// ---------------------------------------------------------------------------
// Stage 1: per-dimension mean ranges (abstraction.py:256-284)
// ---------------------------------------------------------------------------

// min (sgn 0) or max (sgn 1) of f_DI over the dependency sub-cell
// [lo, hi] (the source cell's coordinates of kDeps[DI]) with folded
// constants K; `flag_row` is reported if f is non-finite.  Returns the
// number of objective evaluations.
template <int DI>
__device__ long long imp_mean_box(const BuildParams& P, const double* K,
                                  const double* lo, const double* hi, int sgn,
                                  long long flag_row, double* smem, int S,
                                  double* out) {
  constexpr int D = kNDeps[DI];
  double xfull[IMP_N];
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) xfull[d] = 0.0;
  if constexpr (D == 0) {
    double v = imp_fd(DI, xfull, K);
    if (!imp_finite(v)) imp_flag_nonfinite(P, flag_row);
    *out = v;
    return 0;
  } else {
    NelderMead<D, IMP_MEAN_BLOCK> nm;
    nm.X = smem;
    nm.F = smem + (D + 4) * D * S;
    nm.tol = P.tol;
    nm.max_evals = imp_max_evals(P, D);
#pragma unroll
    for (int q = 0; q < D; ++q) {
      nm.lo[q] = lo[q];
      nm.hi[q] = hi[q];
    }
    const int ms = imp_multistart(P, D);
    const double sign = sgn ? -1.0 : 1.0;
    double best = IMP_INF;
    long long ev = 0;
    for (int s = 0; s < ms; ++s) {
      double st[D];
      imp_start_point<D>(nm.lo, nm.hi, s, st);
      nm.start(st);
      while (!nm.done) {
        double p[D];
        nm.point(p);
#pragma unroll
        for (int q = 0; q < D; ++q) xfull[kDeps[DI][q]] = p[q];
        double val = imp_fd(DI, xfull, K) * sign;
        if (!imp_finite(val)) {
          imp_flag_nonfinite(P, flag_row);
          val = 0.0;
        }
        nm.step(val);
        ++ev;
      }
      best = fmin(best, nm.best);
    }
    *out = sgn ? -best : best;
    return ev;
  }
}

template <int DI>
__device__ long long imp_mean_task(const BuildParams& P, long long r, int sgn,
                                   double* smem, int S) {
  constexpr int D = kNDeps[DI];
  int k, j, i;
  imp_row_kji(P, r, k, j, i);
  const double* K = P.consts + (long long)(j * P.n_w + i) * IMP_NC;
  double lo[D > 0 ? D : 1], hi[D > 0 ? D : 1];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    lo[q] = P.src_lo[(long long)k * IMP_N + kDeps[DI][q]];
    hi[q] = P.src_hi[(long long)k * IMP_N + kDeps[DI][q]];
  }
  double v;
  const long long ev = imp_mean_box<DI>(P, K, lo, hi, sgn, r, smem, S, &v);
  if (sgn == 0) P.mlo[r * IMP_N + DI] = v;
  else P.mhi[r * IMP_N + DI] = v;
  return ev;
}

// --- separable dynamics: tables per (dimension, coordinate, input, dist.) --
// f_d depends on x_d alone, so a row's mean range and 1-D extremes table
// in dimension d are functions of (d, c_d(k), j, i) only: k_sep_tables
// computes each once (the same NM and interval probabilities, hence the
// same bits) and k_outer gathers them per row instead of recomputing them
// (robot2d_reachavoid: 41 x 441 keys per dimension vs 694 575 rows).
__device__ __forceinline__ long long imp_sep_key(const BuildParams& P, int d,
                                                 int c, int j, int i) {
  long long off = 0;
  for (int e = 0; e < d; ++e) off += (long long)kCounts[e] * P.n_u * P.n_w;
  return off + ((long long)c * P.n_u + j) * P.n_w + i;
}

__device__ __forceinline__ long long imp_sep_tab(const BuildParams& P, int d,
                                                 int c, int j, int i) {
  long long off = 0;
  for (int e = 0; e < d; ++e)
    off += 2ll * kCounts[e] * kCounts[e] * P.n_u * P.n_w;
  return off + (((long long)c * P.n_u + j) * P.n_w + i) * 2 * kCounts[d];
}

template <int DI>
__device__ __forceinline__ long long imp_sep_dispatch(
    int d, const BuildParams& P, const double* K, const double* lo,
    const double* hi, int sgn, double* smem, int S, double* out) {
  if constexpr (DI < IMP_N) {
    if (d == DI) return imp_mean_box<DI>(P, K, lo, hi, sgn, 0, smem, S, out);
    return imp_sep_dispatch<DI + 1>(d, P, K, lo, hi, sgn, smem, S, out);
  }
  return 0;
}

// P.write == 0: one thread per (key, sign) -> mean ranges sep_mr;
// P.write == 1: one thread per (key, bin) -> the 1-D extremes table
extern "C" __global__ void __launch_bounds__(IMP_MEAN_BLOCK)
    k_sep_tables(BuildParams P) {
  extern __shared__ double smem[];
  constexpr int S = IMP_MEAN_BLOCK;
  long long nkeys = 0, nbins = 0;
  for (int e = 0; e < IMP_N; ++e) {
    nkeys += (long long)kCounts[e] * P.n_u * P.n_w;
    nbins += (long long)kCounts[e] * kCounts[e] * P.n_u * P.n_w;
  }
  unsigned long long ev = 0;
  const long long ntask = P.write ? nbins : 2 * nkeys;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       t < ntask; t += (long long)gridDim.x * blockDim.x) {
    // task -> (d, key within d, bin or sign)
    int d = 0, coord0 = 0;
    long long rem = P.write ? t : t >> 1, koff = 0;
    for (;;) {
      const long long kd = (long long)kCounts[d] * P.n_u * P.n_w;
      const long long per = P.write ? kd * kCounts[d] : kd;
      if (rem < per) break;
      rem -= per;
      koff += kd;
      coord0 += kCounts[d];
      ++d;
    }
    int q = 0;
    if (P.write) {
      q = (int)(rem % kCounts[d]);
      rem /= kCounts[d];
    }
    const int i = (int)(rem % P.n_w);
    const long long rest = rem / P.n_w;
    const int j = (int)(rest % P.n_u);
    const int c = (int)(rest / P.n_u);
    const long long kk = koff + rem;
    if (!P.write) {
      const double* K = P.consts + (long long)(j * P.n_w + i) * IMP_NC;
      const double lo = P.dim_lo[coord0 + c], hi = P.dim_hi[coord0 + c];
      const int sgn = (int)(t & 1);
      double v;
      ev += imp_sep_dispatch<0>(d, P, K, &lo, &hi, sgn, smem + threadIdx.x,
                                S, &v);
      P.sep_mr[2 * kk + sgn] = v;
    } else {
      // exact 1-D extremes (abstraction.py:287-297), as k_outer computes
      const double ml = P.sep_mr[2 * kk], mh = P.sep_mr[2 * kk + 1];
      const double* e = P.edges + P.edge_off[d];
      const double sg = P.sigma[d];
      const double plo = imp_interval_prob(sg, ml, e[q], e[q + 1]);
      const double phi = imp_interval_prob(sg, mh, e[q], e[q + 1]);
      const double mid = (e[q] + e[q + 1]) / 2;
      double top;
      if (mid < ml) top = plo;
      else if (mid > mh) top = phi;
      else top = imp_interval_prob(sg, 0.0, -P.eta[d] / 2, P.eta[d] / 2);
      double* tab = P.sep_tab + imp_sep_tab(P, d, c, j, i);
      tab[2 * q] = fmin(plo, phi);
      tab[2 * q + 1] = top;
    }
  }
  if (ev) atomicAdd((unsigned long long*)P.evals + 5, ev);   // mean-range NM
}

template <int DI>
__device__ __forceinline__ long long imp_mean_dispatch(int d,
                                                       const BuildParams& P,
                                                       long long r, int sgn,
                                                       double* smem, int S) {
  if constexpr (DI < IMP_N) {
    if (d == DI) return imp_mean_task<DI>(P, r, sgn, smem, S);
    return imp_mean_dispatch<DI + 1>(d, P, r, sgn, smem, S);
  }
  return 0;
}

extern "C" __global__ void __launch_bounds__(IMP_MEAN_BLOCK)
    k_mean_ranges(BuildParams P) {
  extern __shared__ double smem[];
  constexpr int S = IMP_MEAN_BLOCK;
  const long long ntask = P.n_rows * IMP_N * 2;
  unsigned long long ev = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
       t < ntask; t += (long long)gridDim.x * blockDim.x) {
    const long long r = t % P.n_rows;
    const int ds = (int)(t / P.n_rows);
    ev += imp_mean_dispatch<0>(ds >> 1, P, r, ds & 1, smem + threadIdx.x, S);
  }
  if (ev) atomicAdd((unsigned long long*)P.evals + 5, ev);   // mean-range NM
}

// ---------------------------------------------------------------------------
// Stage 2: per-row extremes tables, pruned lattice enumeration, CSR
// ---------------------------------------------------------------------------

// Deterministic block sum (fixed tree over the block, result in all threads).
__device__ double imp_block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = lane < nw ? red[lane] : 0.0;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// Block exclusive scan of 0/1 flags; returns this thread's offset, *total
// gets the block count.
__device__ int imp_block_scan(int flag, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  const int pre = __popc(b & ((1u << lane) - 1u));
  __syncthreads();
  if (lane == 0) wsum[w] = __popc(b);
  __syncthreads();
  int off = 0, tot = 0;
  const int nw = blockDim.x >> 5;
  for (int q = 0; q < nw; ++q) {
    int c = wsum[q];
    if (q < w) off += c;
    tot += c;
  }
  *total = tot;
  return off + pre;
}

struct RowTables {
  double* gmin;   // per dim d: [edge_off[d] - d, + counts[d])
  double* gmax;
  int blo[IMP_N], bext[IMP_N];
  long long box;
};

extern "C" __global__ void k_outer(BuildParams P) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ int wsum[32];
  __shared__ int s_blo[IMP_N], s_bext[IMP_N];
  __shared__ ImpFastDiv s_fdiv[IMP_N];
  __shared__ int s_lo[IMP_N], s_hi[IMP_N];
  __shared__ unsigned long long s_pm[IMP_N];
  __shared__ double s_ml[IMP_N], s_mh[IMP_N];
  __shared__ double s_cov[3 * IMP_N];
  int nbins = 0;
  for (int d = 0; d < IMP_N; ++d) nbins += kCounts[d];
  double* gmin = smem;
  double* gmax = smem + nbins;

  for (long long r = blockIdx.x; r < P.n_rows; r += gridDim.x) {
    int rk, rj, ri;
    imp_row_kji(P, r, rk, rj, ri);
    const int rflat = P.sep ? P.safe_flat[rk] : 0;
    if (threadIdx.x < IMP_N) {
      if (P.sep) {
        const int d = threadIdx.x;
        const int c = (rflat / kStrides[d]) % kCounts[d];
        const long long kk = imp_sep_key(P, d, c, rj, ri);
        s_ml[d] = P.sep_mr[2 * kk];
        s_mh[d] = P.sep_mr[2 * kk + 1];
      } else {
        s_ml[threadIdx.x] = P.mlo[r * IMP_N + threadIdx.x];
        s_mh[threadIdx.x] = P.mhi[r * IMP_N + threadIdx.x];
      }
    }
    __syncthreads();
    if (P.sep) {   // separable: gather this row's tables (k_sep_tables)
      int d = 0, base = 0;
      for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        while (b >= base + kCounts[d]) { base += kCounts[d]; ++d; }
        const int c = (rflat / kStrides[d]) % kCounts[d];
        const double* tab = P.sep_tab + imp_sep_tab(P, d, c, rj, ri);
        const int q = b - base;
        gmin[b] = tab[2 * q];
        gmax[b] = tab[2 * q + 1];
        d = 0;
        base = 0;
      }
    }
    // exact per-dimension extremes (abstraction.py:287-297); Monte Carlo
    // rows have no closed form: every destination is an NM item
    // (abstraction.py:511-540)
    if (!IMP_MC && !P.sep) {
      int d = 0, base = 0;
      for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        while (b >= base + kCounts[d]) { base += kCounts[d]; ++d; }
        const int q = b - base;
        const double* e = P.edges + P.edge_off[d];
        const double s = P.sigma[d], ml = s_ml[d], mh = s_mh[d];
        const double plo = imp_interval_prob(s, ml, e[q], e[q + 1]);
        const double phi = imp_interval_prob(s, mh, e[q], e[q + 1]);
        const double mid = (e[q] + e[q + 1]) / 2;
        double top;
        if (mid < ml) top = plo;
        else if (mid > mh) top = phi;
        else top = imp_interval_prob(s, 0.0, -P.eta[d] / 2, P.eta[d] / 2);
        gmin[b] = fmin(plo, phi);
        gmax[b] = top;
        d = 0;
        base = 0;
      }
    }
    __syncthreads();
    // pruned box: a lattice point can only pass the cutoff if every factor
    // exceeds cutoff / prod_{e != d} max gmax_e (factors are <= 1); the
    // superlevel sets of the unimodal gmax_d are index intervals.
    // Block-parallel: per-dimension maxima, then the index intervals, with
    // shared-memory integer atomics (exact: order-free max / min).
    if (IMP_MC) {
      if (threadIdx.x < IMP_N) {
        s_blo[threadIdx.x] = 0;
        s_bext[threadIdx.x] = kCounts[threadIdx.x];
      }
      __syncthreads();
    } else {
      if (threadIdx.x < IMP_N) {
        s_pm[threadIdx.x] = 0ull;
        s_lo[threadIdx.x] = kCounts[threadIdx.x];
        s_hi[threadIdx.x] = -1;
      }
      __syncthreads();
      {   // pm_d = max_q gmax_d[q] (gmax >= 0: bit order = value order)
        int d = 0, base = 0;
        for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
          while (b >= base + kCounts[d]) { base += kCounts[d]; ++d; }
          const double gm = gmax[b] > 0.0 ? gmax[b] : 0.0;
          atomicMax(&s_pm[d], (unsigned long long)__double_as_longlong(gm));
          d = 0;
          base = 0;
        }
      }
      __syncthreads();
      {   // superlevel interval of gmax_d above cutoff / prod_{e != d} pm_e
        int d = 0, base = 0;
        for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
          while (b >= base + kCounts[d]) { base += kCounts[d]; ++d; }
          double rest = 1.0;
          for (int e = 0; e < IMP_N; ++e)
            if (e != d) rest *= __longlong_as_double((long long)s_pm[e]);
          const double thr = P.cutoff * (1.0 - 1e-9) / rest;
          if (gmax[b] > thr) {
            atomicMin(&s_lo[d], b - base);
            atomicMax(&s_hi[d], b - base);
          }
          d = 0;
          base = 0;
        }
      }
      __syncthreads();
      if (threadIdx.x < IMP_N) {
        const int d = threadIdx.x;
        s_blo[d] = s_lo[d];
        s_bext[d] = s_hi[d] >= s_lo[d] ? s_hi[d] - s_lo[d] + 1 : 0;
      }
      __syncthreads();
    }
    if (threadIdx.x < IMP_N) s_fdiv[threadIdx.x] = imp_fastdiv(s_bext[threadIdx.x]);
    __syncthreads();
    int box = 1;   // < 2^31: a sub-box of the state lattice
    for (int d = 0; d < IMP_N; ++d) box *= s_bext[d];

    // --- safe destinations: t entries ------------------------------------
    long long out = P.write ? P.row_ptr[r] : 0;
    long long cnt = 0;
    for (int q0 = 0; q0 < box; q0 += blockDim.x) {
      const int q = q0 + threadIdx.x;
      int live = 0, pos = -1;
      double tmin = 0.0, tmax = 0.0;
      if (q < box) {
        int rem = q;
        int flat = 0;
        int bidx[IMP_N];
#pragma unroll
        for (int d = IMP_N - 1; d >= 0; --d) {
          const int qd = imp_fdiv(rem, s_fdiv[d]);
          const int b = s_blo[d] + (rem - qd * s_bext[d]);
          rem = qd;
          bidx[d] = b;
          flat += b * kStrides[d];
        }
        pos = P.label ? P.label[flat] : flat;
        if (pos >= 0) {
          int base = 0;
#pragma unroll
          for (int d = 0; d < IMP_N; ++d) {
            const double a = gmax[base + bidx[d]], c = gmin[base + bidx[d]];
            tmax = d == 0 ? a : tmax * a;
            tmin = d == 0 ? c : tmin * c;
            base += kCounts[d];
          }
          live = IMP_MC ? 1 : tmax > P.cutoff;
        }
      }
      int tot;
      const int off = imp_block_scan(live, wsum, &tot);
      if (P.write && live) {
        const long long at = out + cnt + off;
        P.col[at] = pos;
        if (P.separable) {
          P.lo[at] = fmin(tmin, tmax);
          P.hi[at] = tmax;
        }
      }
      cnt += tot;
    }
    if (!P.write && threadIdx.x == 0) P.t_count[r] = cnt;

    // --- target / avoid masses: full lists ------------------------------
    double rs[2] = {0.0, 0.0}, as[2] = {0.0, 0.0};
    long long xo = P.write && !P.separable ? P.aux_ptr[r] : 0;
    long long xc = 0;
    for (int kind = 0; kind < 2; ++kind) {
      const int n_list = kind == 0 ? P.n_t : P.n_a;
      const int* flats = kind == 0 ? P.target_flat : P.avoid_flat;
      for (int q0 = 0; q0 < n_list; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        double tmin = 0.0, tmax = 0.0;
        int live = 0;
        if (q < n_list) {
          int flat = flats[q];
          int base = 0;
#pragma unroll
          for (int d = 0; d < IMP_N; ++d) {
            const int b = (flat / kStrides[d]) % kCounts[d];
            const double a = gmax[base + b], c = gmin[base + b];
            tmax = d == 0 ? a : tmax * a;
            tmin = d == 0 ? c : tmin * c;
            base += kCounts[d];
          }
          live = IMP_MC ? 1 : tmax > P.cutoff;
          if (kind == 0) { rs[0] += tmin; rs[1] += tmax; }
          else { as[0] += tmin; as[1] += tmax; }
        }
        if (!P.separable) {
          int tot;
          const int off = imp_block_scan(live, wsum, &tot);
          if (P.write && live)
            P.aux_code[xo + xc + off] = kind == 0 ? q : -1 - q;
          xc += tot;
        }
      }
    }
    if (!P.write && !P.separable && threadIdx.x == 0) P.x_count[r] = xc;

    if (P.write && P.separable) {
      const double r0 = imp_block_sum(rs[0], red);
      const double r1 = imp_block_sum(rs[1], red);
      const double a0 = imp_block_sum(as[0], red);
      const double a1 = imp_block_sum(as[1], red);
      // cover leak (abstraction.py:300-309): per-dimension factors in
      // parallel, products in dimension order on thread 0
      if (threadIdx.x < IMP_N) {
        const int d = threadIdx.x;
        const double lo = P.cover_lo[d], hi = P.cover_hi[d];
        const double mu = imp_clip((lo + hi) / 2, s_ml[d], s_mh[d]);
        const double s = P.sigma[d];
        s_cov[3 * d] = imp_interval_prob(s, mu, lo, hi);
        s_cov[3 * d + 1] = imp_interval_prob(s, s_ml[d], lo, hi);
        s_cov[3 * d + 2] = imp_interval_prob(s, s_mh[d], lo, hi);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double pmax = 1.0, pmin = 1.0;
        for (int d = 0; d < IMP_N; ++d) {
          const double pa = s_cov[3 * d], pl = s_cov[3 * d + 1],
                       ph = s_cov[3 * d + 2];
          pmax = d == 0 ? pa : pmax * pa;
          pmin = d == 0 ? fmin(pl, ph) : pmin * fmin(pl, ph);
        }
        double* raw = P.raw + r * 6;
        raw[0] = r0;
        raw[1] = r1;
        raw[2] = a0;
        raw[3] = a1;
        raw[4] = fmax(0.0, 1.0 - pmax);
        raw[5] = fmax(0.0, 1.0 - pmin);
      }
    }
    __syncthreads();
  }
}

// Separable rows, one warp per row (k_outer's work without block barriers):
// the row's 1-D tables are gathered from k_sep_tables' output (L1/L2 hot),
// the pruned box is found with warp max / ballots, lattice points are
// compacted with ballot + popc, and the target / avoid sums use the warp's
// fixed xor tree.  P.write = 0: counts; 1: CSR values, r / a sums, leak.
extern "C" __global__ void __launch_bounds__(256) k_outer_sep(BuildParams P) {
  const int lane = threadIdx.x & 31;
  __shared__ ImpFastDiv s_fd[8][IMP_N];   // per warp: the box extents'
  ImpFastDiv* fd = s_fd[threadIdx.x >> 5];
  // per warp: the row's 1-D tables (small lattices; else read in place)
  constexpr bool STAGE = IMP_TAB_DOUBLES <= 256;
  __shared__ double s_tab[8][STAGE ? IMP_TAB_DOUBLES : 1];
  double* stab = s_tab[threadIdx.x >> 5];
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < P.n_rows; r += nw) {
    int rk, rj, ri;
    imp_row_kji(P, r, rk, rj, ri);
    const int rflat = P.safe_flat[rk];
    const double* tab[IMP_N];
    double ml[IMP_N], mh[IMP_N];
    int cnt_d[IMP_N];
    if (STAGE) __syncwarp();   // the previous row's reads are done
#pragma unroll
    for (int d = 0; d < IMP_N; ++d) {
      const int c = (rflat / kStrides[d]) % kCounts[d];
      tab[d] = P.sep_tab + imp_sep_tab(P, d, c, rj, ri);
      const long long kk = imp_sep_key(P, d, c, rj, ri);
      ml[d] = P.sep_mr[2 * kk];
      mh[d] = P.sep_mr[2 * kk + 1];
      cnt_d[d] = kCounts[d];
      if (STAGE) {
        for (int q = lane; q < 2 * kCounts[d]; q += 32)
          stab[kTabOff[d] + q] = tab[d][q];
      }
    }
    if (STAGE) __syncwarp();
    // table value idx of dimension d (shared-memory copy when staged)
    auto tv = [&](int d, int idx) -> double {
      return STAGE ? stab[kTabOff[d] + idx] : tab[d][idx];
    };
    // pm_d = max gmax_d (exact), then the superlevel index interval
    double pm[IMP_N];
#pragma unroll
    for (int d = 0; d < IMP_N; ++d) {
      double m = 0.0;
      for (int q = lane; q < cnt_d[d]; q += 32) m = fmax(m, tv(d, 2 * q + 1));
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      pm[d] = m;
    }
    int blo[IMP_N], bext[IMP_N];
    int box = 1;
#pragma unroll
    for (int d = 0; d < IMP_N; ++d) {
      double rest = 1.0;
#pragma unroll
      for (int e = 0; e < IMP_N; ++e)
        if (e != d) rest *= pm[e];
      const double thr = P.cutoff * (1.0 - 1e-9) / rest;
      int lo = cnt_d[d], hi = -1;
      for (int q0 = 0; q0 < cnt_d[d]; q0 += 32) {
        const int q = q0 + lane;
        const unsigned b = __ballot_sync(0xffffffffu,
                                         q < cnt_d[d] && tv(d, 2 * q + 1) > thr);
        if (b) {
          lo = min(lo, q0 + __ffs(b) - 1);
          hi = q0 + 31 - __clz(b);
        }
      }
      blo[d] = lo;
      bext[d] = hi >= lo ? hi - lo + 1 : 0;
      box *= bext[d];
    }
    // safe destinations
    __syncwarp();
#pragma unroll
    for (int d = 0; d < IMP_N; ++d)
      if (lane == d) fd[d] = imp_fastdiv(bext[d]);
    __syncwarp();
    long long out = P.write ? P.row_ptr[r] : 0;
    long long cnt = 0;
    for (int q0 = 0; q0 < box; q0 += 32) {
      const int q = q0 + lane;
      int live = 0, pos = -1;
      double tmin = 0.0, tmax = 0.0;
      if (q < box) {
        int rem = q, flat = 0;
        int bidx[IMP_N];
#pragma unroll
        for (int d = IMP_N - 1; d >= 0; --d) {
          const int qd = imp_fdiv(rem, fd[d]);
          const int b = blo[d] + (rem - qd * bext[d]);
          rem = qd;
          bidx[d] = b;
          flat += b * kStrides[d];
        }
        pos = P.label ? P.label[flat] : flat;
        if (pos >= 0) {
#pragma unroll
          for (int d = 0; d < IMP_N; ++d) {
            const double a = tv(d, 2 * bidx[d] + 1), c = tv(d, 2 * bidx[d]);
            tmax = d == 0 ? a : tmax * a;
            tmin = d == 0 ? c : tmin * c;
          }
          live = tmax > P.cutoff;
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, live);
      if (P.write && live) {
        const long long at = out + cnt + __popc(b & ((1u << lane) - 1u));
        P.col[at] = pos;
        P.lo[at] = fmin(tmin, tmax);
        P.hi[at] = tmax;
      }
      cnt += __popc(b);
    }
    if (!P.write) {
      if (lane == 0) P.t_count[r] = cnt;
      continue;
    }
    // target / avoid masses (full lists) and the cover leak
    double rs0 = 0.0, rs1 = 0.0, as0 = 0.0, as1 = 0.0;
    for (int kind = 0; kind < 2; ++kind) {
      const int n_list = kind == 0 ? P.n_t : P.n_a;
      const int* flats = kind == 0 ? P.target_flat : P.avoid_flat;
      for (int q = lane; q < n_list; q += 32) {
        const int flat = flats[q];
        double tmin = 0.0, tmax = 0.0;
#pragma unroll
        for (int d = 0; d < IMP_N; ++d) {
          const int bb = (flat / kStrides[d]) % kCounts[d];
          const double a = tv(d, 2 * bb + 1), c = tv(d, 2 * bb);
          tmax = d == 0 ? a : tmax * a;
          tmin = d == 0 ? c : tmin * c;
        }
        if (kind == 0) { rs0 += tmin; rs1 += tmax; }
        else { as0 += tmin; as1 += tmax; }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, o);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, o);
      as0 += __shfl_xor_sync(0xffffffffu, as0, o);
      as1 += __shfl_xor_sync(0xffffffffu, as1, o);
    }
    // cover leak (abstraction.py:300-309): lane d computes dimension d
    double pa = 1.0, pl = 1.0, ph = 1.0;
    if (lane < IMP_N) {
      const int d = lane;
      double mld = ml[0], mhd = mh[0];
#pragma unroll
      for (int e = 1; e < IMP_N; ++e)
        if (e == d) { mld = ml[e]; mhd = mh[e]; }
      const double lo = P.cover_lo[d], hi = P.cover_hi[d];
      const double mu = imp_clip((lo + hi) / 2, mld, mhd);
      const double sg = P.sigma[d];
      pa = imp_interval_prob(sg, mu, lo, hi);
      pl = imp_interval_prob(sg, mld, lo, hi);
      ph = imp_interval_prob(sg, mhd, lo, hi);
    }
    double pmax = 1.0, pmin = 1.0;
#pragma unroll
    for (int d = 0; d < IMP_N; ++d) {
      const double a = __shfl_sync(0xffffffffu, pa, d);
      const double l = __shfl_sync(0xffffffffu, pl, d);
      const double h = __shfl_sync(0xffffffffu, ph, d);
      pmax = d == 0 ? a : pmax * a;
      pmin = d == 0 ? fmin(l, h) : pmin * fmin(l, h);
    }
    if (lane == 0) {
      double* raw = P.raw + r * 6;
      raw[0] = rs0;
      raw[1] = rs1;
      raw[2] = as0;
      raw[3] = as1;
      raw[4] = fmax(0.0, 1.0 - pmax);
      raw[5] = fmax(0.0, 1.0 - pmin);
    }
  }
}


// ---------------------------------------------------------------------------
// Stage 3: coupled refinement, one thread per NM instance
// ---------------------------------------------------------------------------

// One per thread, in shared memory (AoS: the 8-byte fields of a warp fall on
// distinct banks for the sizes that occur); registers stay for the objective.
struct Instance {
  long long row;               // row
  long long t0, x0;            // CSR / aux offsets of the row
  long long slot;              // CSR / aux index
  const double* K;             // folded dynamics constants of the row
  int rel;                     // item index within the row
  int nt, nx;                  // live t entries / aux items of the row
  int sgn;
  int kind;                    // 0: t entry, 1: aux (target/avoid), 2: cover
  double blo[IMP_N], bhi[IMP_N];
#if IMP_MC
  unsigned long long seed;     // derive_seed(mc_seed, row, destination)
#endif
};
static_assert(sizeof(Instance) == 64 + 16 * IMP_N + 8 * IMP_MC,
              "build.cu inst_bytes");

__device__ void imp_load_row(const BuildParams& P, Instance& I) {
  const long long r = I.row;
  I.t0 = P.row_ptr[r];
  I.nt = (int)(P.row_ptr[r + 1] - I.t0);
  I.x0 = P.aux_ptr[r];
  I.nx = (int)(P.aux_ptr[r + 1] - I.x0);
  int k, j, i;
  imp_row_kji(P, r, k, j, i);
  I.K = P.consts + (long long)(j * P.n_w + i) * IMP_NC;
}

__device__ void imp_load_item(const BuildParams& P, Instance& I) {
  int flat = -1;
  if (I.rel < I.nt) {
    I.kind = 0;
    I.slot = I.t0 + I.rel;
    flat = P.safe_flat[P.col[I.slot]];
  } else if (I.rel < I.nt + I.nx) {
    I.kind = 1;
    I.slot = I.x0 + (I.rel - I.nt);
    const int code = P.aux_code[I.slot];
    flat = code >= 0 ? P.target_flat[code] : P.avoid_flat[-1 - code];
  } else {
    I.kind = 2;
    I.slot = I.row;
  }
#if IMP_MC
  {   // noise.py:121-125 derive_seed(mc_seed, row, dest), dest = flat state
      // index (cover: the lattice size, abstraction.py:538-539)
    const unsigned long long key[2] = {
        (unsigned long long)(P.row0 + I.row),
        (unsigned long long)(flat >= 0 ? flat : P.total)};
    imp_seedseq(P.mc_seed, key, 2, &I.seed, 1);
  }
#endif
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) {
    double lo = P.cover_lo[d], hi = P.cover_hi[d];
    if (flat >= 0) {
      const double2 e = P.box[(long long)flat * IMP_N + d];
      lo = e.x;
      hi = e.y;
    }
    I.blo[d] = lo;
    I.bhi[d] = hi;
  }
}

// Source cell of a row: the NM box (clipped cell of the row's state k).
__device__ __forceinline__ void imp_source_cell(const BuildParams& P,
                                                long long r, double* lo,
                                                double* hi) {
  int k, j, i;
  imp_row_kji(P, r, k, j, i);
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) {
    lo[d] = P.src_lo[(long long)k * IMP_N + d];
    hi[d] = P.src_hi[(long long)k * IMP_N + d];
  }
}

// Instance g = 2 * item + sign; items of row r are its live t entries, then
// its live target / avoid boxes, then the cover box.
__device__ void imp_seek_instance(const BuildParams& P, long long g,
                                  Instance& I) {
  const long long item = g >> 1;
  I.sgn = (int)(g & 1);
  long long lo = 0, hi = P.n_rows - 1;
  while (lo < hi) {   // last row with item_ptr[row] <= item
    const long long mid = (lo + hi + 1) >> 1;
    if (P.row_ptr[mid] + P.aux_ptr[mid] + mid <= item) lo = mid;
    else hi = mid - 1;
  }
  I.row = lo;
  imp_load_row(P, I);
  I.rel = (int)(item - (I.t0 + I.x0 + I.row));
  imp_load_item(P, I);
}

// Next item (box): its min and max instances run together, start by start
// (k_refine), so the item index advances by one and the sign restarts at 0.
__device__ void imp_next_instance(const BuildParams& P, Instance& I) {
  I.sgn = 0;
  if (++I.rel == I.nt + I.nx + 1) {
    ++I.row;
    I.rel = 0;
    imp_load_row(P, I);
  }
  imp_load_item(P, I);
}

// P(f(x) + noise in box) * sign  (abstraction.py:333-349)
__device__ __forceinline__ double imp_box_objective(const BuildParams& P,
                                                    const Instance& I,
                                                    const double* x,
                                                    const double* ndtr_tab,
                                                    const double2* exp_tab) {
  // all 2N normal CDFs of one evaluation in one branch-free batch
  double arg[2 * IMP_N], cdf[2 * IMP_N], mean[IMP_N];
  imp_f_all(x, I.K, mean);
#ifndef IMP_NDTR_CHUNK
#define IMP_NDTR_CHUNK 1
#endif
#if IMP_EXACT
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) {
    const double m = mean[d];
    const double s = P.sig[d];
    arg[2 * d] = imp_div_rcp(I.bhi[d] - m, s, P.sig_rcp[d]);
    arg[2 * d + 1] = imp_div_rcp(I.blo[d] - m, s, P.sig_rcp[d]);
  }
#if IMP_NDTR_LEGACY
  (void)exp_tab;
  imp_ndtr_chunks<2 * IMP_N, IMP_NDTR_CHUNK>(arg, cdf, ndtr_tab);
#elif IMP_NDTR_UNROLL   // measured slower (profiles/r02/k_refine_exact_knobs)
#pragma unroll
  for (int j = 0; j < 2 * IMP_N; j += IMP_NDTR_CHUNK)
    imp_ndtr_batch_x<IMP_NDTR_CHUNK>(arg + j, cdf + j, ndtr_tab, exp_tab);
#elif IMP_OBJ_FUSED
  // each dimension's factor as soon as its two CDFs are known: no cdf
  // array in local memory, the same products in the same order
  double pr = 1.0, c_hi = 0.0;
#pragma unroll 1
  for (int j = 0; j < 2 * IMP_N; ++j) {
    double c;
#if IMP_OBJ_FUSED == 2   // the argument by a select chain, not local memory
    double aj = arg[0];
#pragma unroll
    for (int q = 1; q < 2 * IMP_N; ++q) aj = j == q ? arg[q] : aj;
    imp_ndtr_batch_x<1>(&aj, &c, ndtr_tab, exp_tab);
#else
    imp_ndtr_batch_x<1>(arg + j, &c, ndtr_tab, exp_tab);
#endif
    if (j & 1) pr *= c_hi - c;
    else c_hi = c;
  }
  (void)cdf;
  return I.sgn ? pr * -1.0 : pr;
#else
#pragma unroll 1
  for (int j = 0; j < 2 * IMP_N; j += IMP_NDTR_CHUNK)
    imp_ndtr_batch_x<IMP_NDTR_CHUNK>(arg + j, cdf + j, ndtr_tab, exp_tab);
#endif
#else
  // (b - m) / sigma correctly rounded by an unchecked Markstein step
  // (sigma in [2^-100, 2^100], build.cu exact_mode): the reference's args
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) {
    const double m = mean[d];
    const double s = P.sig[d], y = P.sig_rcp[d];
    const double nh = I.bhi[d] - m, nl = I.blo[d] - m;
    const double qh = nh * y, ql = nl * y;
    arg[2 * d] = fma(fma(-qh, s, nh), y, qh);
    arg[2 * d + 1] = fma(fma(-ql, s, nl), y, ql);
  }
#pragma unroll 1
  for (int j = 0; j < 2 * IMP_N; j += IMP_NDTR_CHUNK)
    imp_ndtr_batch_fast<IMP_NDTR_CHUNK>(arg + j, cdf + j, ndtr_tab, exp_tab);
#endif
  double prob = 1.0;
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) prob *= cdf[2 * d] - cdf[2 * d + 1];
  return I.sgn ? prob * -1.0 : prob;
}

#if IMP_MC
// Monte Carlo cell probability (noise.py:133-153 mc_box_probability with
// FullNormal.density, :63-73): volume * mean(density(lo + (hi - lo) * U))
// over mc_samples rows of U from the instance's Philox stream, the mean in
// numpy's pairwise summation order (np.mean = add.reduce / n), generated
// on the fly in stream order.  exp is glibc's (numpy's SIMD exp differs by
// an ulp on ~5% of arguments), so values agree to ulps, not bits.
struct ImpMc {
  ImpPhilox g;
  const BuildParams* P;
  double lo[IMP_N], w[IMP_N], mean[IMP_N];
  bool bad;
};

__device__ __forceinline__ double imp_mc_density(ImpMc& c) {
  double y[IMP_N];
#pragma unroll
  for (int d = 0; d < IMP_N; ++d)
    y[d] = c.lo[d] + c.w[d] * imp_philox_double(&c.g);
#if IMP_MC_CUSTOM
  // CustomNoise.density (noise.py:84-95): the lowered expression over the
  // point and the mean; non-finite or negative -> NoiseError
  const double v = imp_density(y, c.mean);
  if (!imp_finite(v) || v < 0.0) c.bad = true;
  return v;
#else
  double diff[IMP_N];
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) diff[d] = y[d] - c.mean[d];
  double q = 0.0;   // einsum("ki,ij,kj->k", diff, inv_cov, diff)
#pragma unroll
  for (int i = 0; i < IMP_N; ++i)
#pragma unroll
    for (int j = 0; j < IMP_N; ++j)
      q += diff[i] * c.P->inv_cov[i * IMP_N + j] * diff[j];
  const double v = c.P->mc_norm * imp_exp(-0.5 * q);
  if (!imp_finite(v)) c.bad = true;
  return v;
#endif
}

// numpy pairwise_sum of the next n densities (PW_BLOCKSIZE 128, 8 lanes):
// leaves of <= 128 values summed as numpy does, split n -> (n2, n - n2) with
// n2 = n/2 rounded down to a multiple of 8, combined left + right.  The
// recursion runs on an explicit stack in stream order (no device
// recursion, so the stack frame is static).
__device__ double imp_mc_leaf(ImpMc& c, long long n) {
  if (n < 8) {
    double r = 0.0;
    for (long long i = 0; i < n; ++i) r += imp_mc_density(c);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = imp_mc_density(c);
  long long i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += imp_mc_density(c);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += imp_mc_density(c);
  return res;
}

__device__ double imp_mc_pairwise(ImpMc& c, long long n) {
  long long right[24];   // pending right halves (-1: right in progress)
  double left[24];
  int sp = 0;
  long long cur = n;
  for (;;) {
    while (cur > 128) {
      long long n2 = cur / 2;
      n2 -= n2 % 8;
      right[sp] = cur - n2;
      ++sp;
      cur = n2;
    }
    double val = imp_mc_leaf(c, cur);
    for (;;) {
      if (sp == 0) return val;
      if (right[sp - 1] >= 0) {       // left subtree done: descend right
        left[sp - 1] = val;
        cur = right[sp - 1];
        right[sp - 1] = -1;
        break;
      }
      val = left[sp - 1] + val;       // right subtree done: combine
      --sp;
    }
  }
}

__device__ double imp_mc_objective(const BuildParams& P, const Instance& I,
                                   const double* x) {
  double vol = 1.0;
#pragma unroll
  for (int d = 0; d < IMP_N; ++d) vol = d == 0 ? I.bhi[0] - I.blo[0]
                                               : vol * (I.bhi[d] - I.blo[d]);
  double est = 0.0;
  if (vol != 0.0) {
    ImpMc c;
    c.P = &P;
    c.bad = false;
    imp_f_all(x, I.K, c.mean);
#pragma unroll
    for (int d = 0; d < IMP_N; ++d) {
      c.lo[d] = I.blo[d];
      c.w[d] = I.bhi[d] - I.blo[d];
    }
    imp_philox_seed(&c.g, I.seed);
    est = vol * (imp_mc_pairwise(c, P.mc_samples) / (double)P.mc_samples);
    if (c.bad) est = IMP_INF - IMP_INF;   // NaN: flagged by the caller
    else est = est > 0.0 ? (est < 1.0 ? est : 1.0) : 0.0;  // min(max(e,0),1)
  }
  return I.sgn ? est * -1.0 : est;
}
#endif

__device__ void imp_store_instance(const BuildParams& P, const Instance& I,
                                   double best) {
  const double v = I.sgn ? -best : best;
  if (I.kind == 0) {
    if (I.sgn) P.hi[I.slot] = v;
    else P.lo[I.slot] = v;
  } else if (I.kind == 1) {
    if (I.sgn) P.aux_max[I.slot] = v;
    else P.aux_min[I.slot] = v;
  } else {
    // cover: leak bounds from the box probability extremes
    double* raw = P.raw + I.row * 6;
    if (I.sgn) raw[4] = fmax(0.0, 1.0 - v);   // leak_min = 1 - p_max
    else raw[5] = fmax(0.0, 1.0 - v);         // leak_max = 1 - p_min
  }
}

// Work is handed out in batches of consecutive items from a global counter
// (a lane that finishes grabs the next batch, so warps stay full until the
// pool drains; NM costs vary 8..max_evals evaluations per run).  A lane
// runs an item's 2 x multistart Nelder-Mead runs in the order
// (start 0, min), (start 0, max), (start 1, min), ...: the max run of a
// start reuses the min run's initial simplex values (start_shared), and the
// per-sign results are the minimum over starts (order-free).
extern "C" __global__ void __launch_bounds__(IMP_REFINE_BLOCK, IMP_REFINE_MINB)
    k_refine(BuildParams P) {
  extern __shared__ double smem[];
  __shared__ double2 s_ndtr[IMP_NDTR_TAB / 2];
  for (int q = threadIdx.x; q < IMP_NDTR_TAB; q += blockDim.x)
    imp_ndtr_fill_one(reinterpret_cast<double*>(s_ndtr), q);
#if IMP_EXACT && IMP_NDTR_LEGACY
  const double2* exp_tab = nullptr;
#else
  __shared__ double2 s_exp[128];
  for (int q = threadIdx.x; q < 128; q += blockDim.x)
    s_exp[q] = make_double2(imp_asd(imp_exp_tab[2 * q]),
                            imp_asd(imp_exp_tab[2 * q + 1]));
  const double2* exp_tab = s_exp;
#endif
  __syncthreads();
  const double* ndtr_tab = reinterpret_cast<const double*>(s_ndtr);
  constexpr int S = IMP_REFINE_BLOCK;
  NelderMead<IMP_N, S> nm;
  nm.X = smem + threadIdx.x;
  nm.F = smem + (IMP_N + 4) * IMP_N * S + threadIdx.x;
  // the min run's initial simplex values of the current start
  double* Fi = smem + imp_nm_doubles<IMP_N>() * S + threadIdx.x;
#if IMP_INST_SMEM
  Instance& I = reinterpret_cast<Instance*>(
      smem + (imp_nm_doubles<IMP_N>() + IMP_N + 1) * S)[threadIdx.x];
#else
  Instance I;
#endif
  nm.tol = P.tol;
  nm.max_evals = imp_max_evals(P, IMP_N);
  const int ms = imp_multistart(P, IMP_N);
  const long long total = P.n_items;
  constexpr long long B = IMP_REFINE_BATCH / 2 > 0 ? IMP_REFINE_BATCH / 2 : 1;
  unsigned long long* counter = (unsigned long long*)P.evals + 2;
  long long g = (long long)atomicAdd(counter, (unsigned long long)B);
  long long g_end = min(total, g + B);
  if (g >= total) return;
  imp_seek_instance(P, 2 * g, I);
  imp_source_cell(P, I.row, nm.lo, nm.hi);
  int s = 0;
  double best0 = IMP_INF, best1 = IMP_INF;
  unsigned int ev = 0, shared = 0, slots = 0;   // per thread: far below 2^32
  {
    double st[IMP_N];
    imp_start_point<IMP_N>(nm.lo, nm.hi, 0, st);
    nm.start(st);
  }
  // One objective evaluation per trip for every live lane; run changes are
  // a nested loop that reconverges before the next evaluation, so a warp
  // never splits into groups evaluating the objective separately.
  bool live = true;
  while (__any_sync(__activemask(), live)) {
    ++slots;
    if (live) {
      double p[IMP_N];
      nm.point(p);
#if IMP_MC
      double val = imp_mc_objective(P, I, p);
#else
      double val = imp_box_objective(P, I, p, ndtr_tab, exp_tab);
#endif
      if (!imp_finite(val)) {
        imp_flag_nonfinite(P, I.row);
        val = 0.0;
      }
      ++ev;
      nm.feed(val);
      if (nm.pend == 2 && nm.phase == NM_INIT && I.sgn == 0) {
#pragma unroll
        for (int q = 0; q <= IMP_N; ++q) Fi[q * S] = nm.fs(q);
      }
      for (;;) {
        if (nm.pend) nm.iterate(nm.pend == 2);   // the one iterate() site
        if (!nm.done) break;
        double st[IMP_N];
        if (I.sgn == 0) {
          best0 = fmin(best0, nm.best);
          I.sgn = 1;
          imp_start_point<IMP_N>(nm.lo, nm.hi, s, st);
          nm.start_shared(st, Fi);
          shared += IMP_N + 1;
          continue;
        }
        best1 = fmin(best1, nm.best);
        I.sgn = 0;
        if (++s == ms) {
          I.sgn = 0;
          imp_store_instance(P, I, best0);
          I.sgn = 1;
          imp_store_instance(P, I, best1);
          I.sgn = 0;
          bool more = ++g < g_end;
          if (more) {
            imp_next_instance(P, I);
          } else {
            g = (long long)atomicAdd(counter, (unsigned long long)B);
            g_end = min(total, g + B);
            more = g < total;
            if (more) imp_seek_instance(P, 2 * g, I);
          }
          if (!more) {
            live = false;
            break;
          }
          imp_source_cell(P, I.row, nm.lo, nm.hi);
          s = 0;
          best0 = best1 = IMP_INF;
        }
        imp_start_point<IMP_N>(nm.lo, nm.hi, s, st);
        nm.start(st);
      }
    }
    __syncwarp(__activemask());
  }
  // [0] the reference's objective evaluations (performed + shared initial
  // simplices), [1] lane slots, [3] evaluations saved by sharing
  atomicAdd((unsigned long long*)P.evals, (unsigned long long)(ev + shared));
  atomicAdd((unsigned long long*)P.evals + 1, (unsigned long long)slots);
  atomicAdd((unsigned long long*)P.evals + 3, (unsigned long long)shared);
}


// ---------------------------------------------------------------------------
// Stage 4: assemble (abstraction.py:607-659), one warp per row
// ---------------------------------------------------------------------------

__device__ __forceinline__ double imp_warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

extern "C" __global__ void k_assemble(BuildParams P) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < P.n_rows; r += nw) {
    const long long b = P.row_ptr[r], e = P.row_ptr[r + 1];
    double* raw = P.raw + r * 6;
    double rmin, rmax, avmin, avmax;
    if (P.separable) {
      rmin = raw[0]; rmax = raw[1]; avmin = raw[2]; avmax = raw[3];
    } else {
      // sums of the refined target / avoid terms (non-live terms are 0)
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      const long long xb = P.aux_ptr[r], xe = P.aux_ptr[r + 1];
      for (long long q = xb + lane; q < xe; q += 32) {
        const int code = P.aux_code[q];
        const int off = code >= 0 ? 0 : 2;
        double mn = P.aux_min[q], mx = P.aux_max[q];
        if (IMP_MC) {   // abstraction.py:518-522: cutoff, then min(pmin, pmax)
          if (mx <= P.cutoff) mn = mx = 0.0;
          mn = fmin(mn, mx);
        }
        s[off] += mn;
        s[off + 1] += mx;
      }
      rmin = imp_warp_sum(s[0]);
      rmax = imp_warp_sum(s[1]);
      avmin = imp_warp_sum(s[2]);
      avmax = imp_warp_sum(s[3]);
    }
    // clip t entries, t_min = min(t_min, t_max), low-cost zeroing
    double smin = 0.0, smax = 0.0;
    unsigned live = 0;   // t_max > cutoff (the reference's sparsity log)
    for (long long q = b + lane; q < e; q += 32) {
      const double hv0 = P.hi[q], lv0 = P.lo[q];
      double hv = hv0, lv = lv0;
      if (IMP_MC) {     // abstraction.py:518-522
        if (hv <= P.cutoff) lv = hv = 0.0;
        lv = fmin(lv, hv);
      }
      double hi = imp_clip(hv, 0.0, 1.0);
      double lo = imp_clip(lv, 0.0, 1.0);
      if (P.low_cost && hi <= P.cutoff) lo = 0.0;
      lo = fmin(lo, hi);
      // store only what changed (bitwise): the writers already clip and
      // order most entries, so this halves the kernel's HBM traffic
      if (__double_as_longlong(lo) != __double_as_longlong(lv0)) P.lo[q] = lo;
      if (__double_as_longlong(hi) != __double_as_longlong(hv0)) P.hi[q] = hi;
      smin += lo;
      smax += hi;
      live += hi > P.cutoff;
    }
    smin = imp_warp_sum(smin);
    smax = imp_warp_sum(smax);
    for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if (lane == 0 && live)
      atomicAdd((unsigned long long*)P.evals + 4, (unsigned long long)live);
    rmin = imp_clip(rmin, 0.0, 1.0);
    rmax = imp_clip(rmax, 0.0, 1.0);
    rmin = fmin(rmin, rmax);
    avmin = imp_clip(avmin, 0.0, 1.0);
    avmax = imp_clip(avmax, 0.0, 1.0);
    avmin = fmin(avmin, avmax);
    double lkmin = imp_clip(raw[4], 0.0, 1.0), lkmax = imp_clip(raw[5], 0.0, 1.0);
    lkmin = fmin(lkmin, lkmax);
    double amin = imp_clip(lkmin + avmin, 0.0, 1.0);
    double amax = imp_clip(lkmax + avmax, 0.0, 1.0);
    // row-sum repair: shave min-side excess off a_min, then scale
    // closed-form rows must balance to 1e-6; Monte Carlo rows carry
    // independent sampling error per destination and are only repaired
    // (abstraction.py:620-632, `if not monte_carlo`)
    const double excess = fmax(smin + rmin + amin - 1.0, 0.0);
    if (!IMP_MC && excess > 1e-6 && lane == 0) {
      if (atomicMin(P.err + 1, (unsigned long long)r) > (unsigned long long)r)
        P.err_val[1] = excess;
    }
    const double shaved = fmin(excess, amin);
    amin = amin - shaved;
    const double rest = excess - shaved;
    if (rest > 0) {
      const double s = smin + rmin;
      const double scale = s > 0 ? 1.0 - rest / fmax(s, 1e-300) : 1.0;
      for (long long q = b + lane; q < e; q += 32) P.lo[q] *= scale;
      rmin *= scale;
    }
    const double deficit = fmax(1.0 - (smax + rmax + amax), 0.0);
    if (!IMP_MC && deficit > 1e-6 && lane == 0) {
      if (atomicMin(P.err + 2, (unsigned long long)r) > (unsigned long long)r)
        P.err_val[2] = deficit;
    }
    amax = fmin(amax + deficit, 1.0);
    amin = fmin(amin, amax);
    if (lane == 0) {
      P.r_min[r] = rmin;
      P.r_max[r] = rmax;
      P.a_min[r] = amin;
      P.a_max[r] = amax;
    }
  }
}


// ---------------------------------------------------------------------------
// Test entry (imp_ndtr_eval): the module's device normal CDFs on n
// arguments.  which = 0: imp_ndtr_batch (round-1 exact form), 1:
// imp_ndtr_batch_x (the IMP_EXACT objective's), 2: imp_ndtr_batch_fast.
// ---------------------------------------------------------------------------
extern "C" __global__ void k_ndtr_eval(const double* x, double* y,
                                       long long n, int which) {
  __shared__ double2 s_ndtr[IMP_NDTR_TAB / 2];
  __shared__ double2 s_exp[128];
  for (int q = threadIdx.x; q < IMP_NDTR_TAB; q += blockDim.x)
    imp_ndtr_fill_one(reinterpret_cast<double*>(s_ndtr), q);
  for (int q = threadIdx.x; q < 128; q += blockDim.x)
    s_exp[q] = make_double2(imp_asd(imp_exp_tab[2 * q]),
                            imp_asd(imp_exp_tab[2 * q + 1]));
  __syncthreads();
  const double* tab = reinterpret_cast<const double*>(s_ndtr);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = x[i];
    double r;
    if (which == 0) imp_ndtr_batch<1>(&a, &r, tab);
    else if (which == 1) imp_ndtr_batch_x<1>(&a, &r, tab, s_exp);
    else imp_ndtr_batch_fast<1>(&a, &r, tab, s_exp);
    y[i] = r;
  }
}
