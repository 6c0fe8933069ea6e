/*
 * impact_b200.h -- C-ABI of the B200 IMDP construction + interval-iteration
 * library (libimpact_b200.so).
 *
 * The reference (arxiv 2401.03555's Python package `impact`) has no FFI; its
 * boundary for this path is the module-level Python API
 * (pkg/src/impact/__init__.py:4-17).  Each entry point below is what that
 * API's hot calls bind to; INTEGRATION.md shows the ctypes stubs a maintainer
 * would add to the reference.  Plain pointers and sizes only, no torch types.
 *
 * Conventions
 *   - every function returns an imp_status; imp_last_error() gives the
 *     message of the calling thread's last failure (plus row / iteration
 *     counts where meaningful);
 *   - row r = (k * n_u + j) * n_w + i  (reference abstraction.py:79-85);
 *   - columns 0..n_s-1 are safe states, virtual slot n_s is the target
 *     (r_min/r_max) and n_s+1 the avoid mass (a_min/a_max)
 *     (reference synthesis.py:79-83);
 *   - all probabilities / values are IEEE float64;
 *   - an imp_imdp owns its device memory (one GPU, one shard of rows);
 *   - one in-flight call per handle; handles are not shared across threads.
 */
#ifndef IMPACT_B200_H
#define IMPACT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum imp_status {
  IMP_OK = 0,
  IMP_E_ARG = 1,          /* -> ValueError                                  */
  IMP_E_CUDA = 2,         /* -> RuntimeError                                */
  IMP_E_ABSTRACTION = 3,  /* -> AbstractionError (row sums, validate)       */
  IMP_E_NONFINITE = 4,    /* -> AbstractionError("non-finite objective ...") */
  IMP_E_CONVERGENCE = 5,  /* -> ConvergenceError(k0, k1)                    */
  IMP_E_MONOTONE = 6,     /* -> ImpactError (iterates lost monotonicity)    */
  IMP_E_BRACKET = 7,      /* -> ImpactError (v0 > v1 + 1e-9)                */
  IMP_E_JIT = 8,          /* -> RuntimeError (NVRTC / module load)          */
  IMP_E_NOMEM = 9         /* -> MemoryError                                 */
} imp_status;

typedef struct imp_imdp imp_imdp;

/* Message of the calling thread's last failure; returns its full length. */
size_t imp_last_error(char* buf, size_t len);

/* Library / device facts: SM count, compute capability, library version. */
int imp_device_query(int device, int* sm_count, int* cc_major, int* cc_minor);
const char* imp_version(void);

/* ---------------------------------------------------------------------- */
/* Abstraction handles                                                     */
/* ---------------------------------------------------------------------- */

typedef struct imp_imdp_info {
  int64_t n_rows;      /* rows held by this handle (its shard)             */
  int64_t row_begin;   /* global index of the first row                    */
  int64_t nnz;         /* stored t entries (cutoff-sparse)                 */
  int32_t n_s, n_u, n_w;
  int32_t k_begin;     /* first safe state of the shard                     */
  int32_t k_count;     /* safe states in the shard                          */
  int32_t max_row;     /* longest stored row                                */
  int32_t device;
} imp_imdp_info;

/*
 * Import a cutoff-sparse abstraction shard (CSR over the t columns plus the
 * r/a vectors) from HOST memory.  Replaces constructing
 * impact.abstraction.Imdp(...) (reference abstraction.py:88-137) from
 * arrays, e.g. after impact.fileio.load_abstraction (fileio.py:303-328).
 * row_ptr has n_rows+1 entries (row_ptr[0] == 0); columns must be
 * ascending within a row.  The shard covers safe states
 * [k_begin, k_begin + n_rows / (n_u*n_w)).
 */
int imp_imdp_import(int device, int32_t n_s, int32_t n_u, int32_t n_w,
                    int32_t k_begin, int64_t n_rows, const int64_t* row_ptr,
                    const int32_t* col, const double* t_lo,
                    const double* t_hi, const double* r_min,
                    const double* r_max, const double* a_min,
                    const double* a_max, imp_imdp** out);

int imp_imdp_info_get(const imp_imdp* h, imp_imdp_info* out);

/* Copy the shard back to HOST memory (row_ptr: n_rows+1, col/t_lo/t_hi:
 * nnz, vectors: n_rows).  Any pointer may be NULL to skip that array.
 * Lazy materialisation for fileio / tests (reference Imdp fields). */
int imp_imdp_export(const imp_imdp* h, int64_t* row_ptr, int32_t* col,
                    double* t_lo, double* t_hi, double* r_min, double* r_max,
                    double* a_min, double* a_max);

/* Row-sum / interval invariants of Imdp.validate (abstraction.py:121-137),
 * evaluated on the device.  Returns IMP_E_ABSTRACTION with the first bad
 * row in the message. */
int imp_imdp_validate(const imp_imdp* h, double tol);

void imp_imdp_free(imp_imdp* h);

/* ---------------------------------------------------------------------- */
/* Construction (reference build_abstraction, abstraction.py:551-599)      */
/* ---------------------------------------------------------------------- */

typedef struct imp_build_desc {
  int32_t device;
  int32_t n, m, p;           /* state / input / disturbance dimensions     */
  int32_t n_u, n_w;          /* input / disturbance lattice sizes           */
  int32_t separable;         /* DynamicsSpec.is_separable()                 */
  /* host geometry, computed with the reference's float64 formulas */
  const int32_t* counts;     /* (n) lattice points per dimension            */
  const double* eta;         /* (n)                                         */
  const double* sigma;       /* (n) diagonal noise                          */
  const double* edges;       /* (sum(counts)+n) cell edges, dim-major       */
  const double* cover_lo;    /* (n) [lb - eta/2]                            */
  const double* cover_hi;    /* (n) [ub + eta/2]                            */
  int32_t n_s, n_t, n_a;     /* safe / target / avoid counts                */
  const int32_t* safe_multi;   /* (n_s, n) lattice indices                  */
  const int32_t* target_multi; /* (n_t, n)                                  */
  const int32_t* avoid_multi;  /* (n_a, n)                                  */
  const double* src_lo;      /* (n_s, n) clipped source cells               */
  const double* src_hi;      /* (n_s, n)                                    */
  /* dynamics: CUDA source of imp_f<d>(x, k) (expr.lower_dynamics) and the
   * per-(j,i) folded constants */
  const char* dyn_source;
  int32_t n_consts;
  const double* consts;      /* (n_u*n_w, n_consts)                         */
  const int32_t* deps;       /* (n, n) dependency lists, -1 padded          */
  const int32_t* n_deps;     /* (n)                                         */
  /* AbstractionOptions */
  double zero_cutoff;
  double tol;
  int32_t low_cost;
  int32_t max_evals_per_dim; /* 0: 200*dim (default); < 0: fixed -v evals   */
  int32_t multistart;        /* 0 -> 1 + 2*dim                              */
  /* shard: safe states [k_begin, k_begin + k_count) */
  int32_t k_begin, k_count;
  /* Monte Carlo noise (FullNormal, noise.py:41-73, 133-153): mc = 1 runs
   * the reference's _row_monte_carlo (abstraction.py:511-540) -- every
   * destination, NM over the MC cell probability of mc_samples samples
   * from Generator(Philox(SeedSequence(derive_seed(mc_seed, row, dest)))) */
  int32_t mc;
  int32_t mc_samples;
  uint64_t mc_seed;
  double mc_norm;            /* sqrt(det(inv_cov)) * (2 pi)^(-n/2), numpy  */
  const double* inv_cov;     /* (n, n)                                      */
  /* clipped cell bounds of every lattice coordinate, dimension-major
   * (sum(counts)): lets separable dynamics compute one mean range / table
   * per (dimension, coordinate, input, disturbance); NULL: per row */
  const double* dim_lo;
  const double* dim_hi;
  /* 1 (the Python default): the k_refine objective's normal CDFs are
   * scipy's bit for bit (cephes with unfused Horner steps, IEEE quotient);
   * 0: the fast objective -- the same cephes formula with fused Horner
   * steps and a reciprocal-seeded quotient, within a few ulps per CDF
   * (tests/test_construct_gpu.py).  The outer-bound tables, and with them
   * the live sets, are bit-exact in both modes. */
  int32_t exact;
  /* non-NULL: count only -- run the mean ranges and the outer count pass,
   * write each shard state's construction work (coupled: live entries +
   * aux boxes + 1 per row, the Nelder-Mead items; separable: live entries
   * + 1 per row) to state_cost[k_count], and return without building
   * (*out = NULL).  The multi-GPU driver balances shards with it. */
  int64_t* state_cost;
} imp_build_desc;

/* Per-build timings (device milliseconds, CUDA events) and counters. */
typedef struct imp_build_stats {
  double ms_total, ms_mean_ranges, ms_outer, ms_refine, ms_assemble;
  int64_t nnz;
  int64_t nm_instances;
  int64_t nm_evals;          /* refinement objective evaluations (k_refine,
                                shared initial simplices included)        */
  int64_t nm_lane_slots;     /* refine-loop lane slots (warp trips x 32):
                                nm_evals / nm_lane_slots = SIMT efficiency */
  int64_t nm_evals_shared;   /* of nm_evals: initial-simplex values a max
                                run took from its min run (not evaluated) */
  int64_t nnz_live;          /* stored entries with t_max > zero_cutoff   */
  int64_t nm_evals_mean;     /* mean-range NM evaluations (k_mean_ranges /
                                k_sep_tables: one dynamics component each) */
} imp_build_stats;

int imp_build(const imp_build_desc* desc, imp_imdp** out,
              imp_build_stats* stats);

/* NVRTC-compile (only) the construction module imp_build would use for
 * desc's dynamics; no device needed.  Writes the sm_100a cubin to
 * cubin_path when non-NULL (for cuobjdump).  IMP_E_JIT carries the NVRTC
 * log in imp_last_error(). */
int imp_jit_compile(const imp_build_desc* desc, const char* cubin_path);

/* Test entry: the construction module's device normal CDFs (reference
 * scipy.special.ndtr, noise.py:14, 116-118) on n host values.  which = 0:
 * the round-1 branch-free cephes form, 1: the form the default (exact)
 * k_refine objective uses -- both bit-identical to scipy -- 2: the fast
 * objective's fused form (a few ulps). */
int imp_ndtr_eval(const imp_build_desc* desc, const double* x, double* y,
                  int64_t n, int32_t which);

/* ---------------------------------------------------------------------- */
/* Interval iteration (reference synthesis.py:97-361)                      */
/* ---------------------------------------------------------------------- */

enum { IMP_SPEC_REACH = 0, IMP_SPEC_SAFETY = 1 };
enum { IMP_LP_MIN = 0, IMP_LP_MAX = 1 };
enum { IMP_MODE_PHASE = 0, IMP_MODE_DIAGNOSE = 1 };

typedef struct imp_phase_desc {
  int32_t spec;          /* IMP_SPEC_*: terminal weights [V, 1, 0] / [V, 0, 1] */
  int32_t lp;            /* IMP_LP_*: feasible-distribution direction        */
  int32_t u_max;         /* 1: inputs maximise (reach), 0: minimise (safety) */
  int32_t mode;          /* IMP_MODE_PHASE (_run_phase) or DIAGNOSE          */
  double eps;
  int64_t horizon;       /* <= 0: infinite                                   */
  int64_t max_iterations;
  const int64_t* fixed_policy; /* host (k_count) or NULL (phase 1)           */
} imp_phase_desc;

typedef struct imp_phase_out {
  double* v0;            /* host (n_s) final lower-track values              */
  double* v1;            /* host (n_s) final upper-track values              */
  int64_t* policy;       /* host (n_s) or NULL                               */
  int64_t iterations;
  int64_t k0, k1;        /* first self-converged iteration, -1 if never      */
  int32_t fallback;      /* stalled-gap fallback fired                       */
  double gap;            /* final max(v1 - v0)                               */
  double ms_device;      /* device time of the loop (CUDA events)            */
  int64_t sweeps;        /* twin sweeps executed                             */
  double ms_sweep;       /* device time of the K5 launches alone, summed over
                          * the executed iterations (events captured into
                          * the loop's CUDA graph around each K5 group)      */
  double* gap_log;       /* host (gap_log_cap) or NULL: max(v1 - v0) at every
                          * 1000th iteration that continued -- the values the
                          * reference logs (synthesis.py:204-205)           */
  int64_t gap_log_cap;
  int64_t gap_log_n;     /* entries written                                 */
} imp_phase_out;

/* Run one synthesis phase to termination (reference _run_phase,
 * synthesis.py:145-205; diagnose_convergence :321-361 with
 * IMP_MODE_DIAGNOSE).  Single-shard handles only; the loop, the stable
 * sorts, the sweeps and the termination logic all run on the device in
 * CUDA graphs.  IMP_E_CONVERGENCE / _MONOTONE / _BRACKET carry the
 * reference's error semantics (k0/k1 are filled in either way). */
int imp_run_phase(imp_imdp* h, const imp_phase_desc* desc,
                  imp_phase_out* out);

/* One robust Bellman update (reference bellman_step, synthesis.py:97-135)
 * from host values (n_s) -> new values (k_count) and chosen inputs. */
int imp_bellman_step(imp_imdp* h, const double* values, int32_t spec,
                     int32_t lp, int32_t u_max, const int64_t* fixed_policy,
                     double* new_values, int64_t* chosen);

/* Row-level greedy LP values (reference RowsSolver.values,
 * feasible.py:96-111) for every stored row: out[r] for weights w (n_s+2).
 * Device pointers are accepted when on_device != 0. */
int imp_row_values(imp_imdp* h, const double* weights, int32_t lp,
                   double* out, int32_t on_device);

/* ---------------------------------------------------------------------- */
/* Sharded iteration (multi-GPU): the host exchanges V between sweeps.     */
/* ---------------------------------------------------------------------- */

/* One twin sweep of this shard against the full value vectors v0/v1
 * (device pointers, n_s each): writes this shard's new values to
 * new0/new1 (device, k_count each), chosen inputs to policy (device,
 * k_count) and the shard's max |dV0|, max |dV1|, max(v1'-v0') and the
 * monotone/bracket flags (0/1) to stats[0..4] (5 device doubles; an empty
 * shard reports -inf maxima).  stream is a cudaStream_t (NULL = legacy
 * default); the call returns after the stream work completed. */
int imp_shard_sweep(imp_imdp* h, const double* v0, const double* v1,
                    int32_t spec, int32_t lp, int32_t u_max,
                    const int64_t* fixed_policy_dev, double* new0,
                    double* new1, int64_t* policy, double* stats,
                    void* stream);

/* Device-resident sharded phase loop (reference _run_phase over state
 * shards; the multi-GPU hot loop).  shard_begin (host, world + 1) is the
 * partition of the n_s safe states; this handle must be one of its shards.
 * vbuf0 / vbuf1 (device, world * 2 * pw doubles; pw >= the widest shard)
 * are the ping-pong value buffers in the packed layout [rank][V0|V1][pw]:
 * iteration i (1-based) writes this rank's chunk of vbuf[i % 2] at offset
 * rank * 2 * pw, and the caller's in-place all-gather of that chunk
 * (2 * pw doubles per rank) completes the full vectors.  stats (device, 5
 * doubles) receives this shard's [max|dV0|, max|dV1|, max(V1'-V0'),
 * monotone, bracket]; the caller all-reduces it (max) before
 * imp_shard_loop_control.  No call but begin / poll synchronises, so G
 * iterations can be captured in one CUDA graph (with the collectives) and
 * replayed; kernels of iterations after termination exit at once.
 * desc->fixed_policy: this shard's phase-2 policy (host, k_count).
 * poll reads the control block (a stream sync): *done, iterations, k0, k1,
 * fallback, gap; once done it fills out->v0 / v1 (host, n_s, may be NULL)
 * and out->policy (host, k_count: this shard's choices) and returns the
 * reference's termination errors as imp_run_phase does. */
typedef struct imp_shard_loop imp_shard_loop;
int imp_shard_loop_begin(imp_imdp* h, const imp_phase_desc* desc,
                         const int64_t* shard_begin, int32_t world,
                         double* vbuf0, double* vbuf1, int64_t pw,
                         double* stats, void* stream, imp_shard_loop** out);
int imp_shard_loop_sweep(imp_shard_loop* loop, void* stream);
int imp_shard_loop_control(imp_shard_loop* loop, void* stream);
int imp_shard_loop_poll(imp_shard_loop* loop, imp_phase_out* out,
                        int32_t* done, void* stream);
void imp_shard_loop_free(imp_shard_loop* loop);

/* Microbenchmark used for the FP64 roofline denominator: DFMA throughput
 * (GFLOP/s, 2 flops per DFMA) measured with CUDA events. */
int imp_fp64_peak(int device, double* gflops);

/* K5 sweep kernel alone: mean device milliseconds of one twin sweep over
 * all of h's rows (reps back-to-back launches, CUDA events) -- the HBM
 * roofline measurement. */
int imp_time_sweep(imp_imdp* h, int32_t spec, int32_t lp, int32_t reps,
                   double* ms);

/* ---------------------------------------------------------------------- */
/* Closed-loop simulation (cli.py:163-251, cmd_simulate)                   */
/* ---------------------------------------------------------------------- */

typedef struct imp_sim_desc {
  int32_t rollouts, steps;
  uint64_t seed;             /* [synthesis] seed (derive_seed(seed, r, 0))  */
  int32_t reach_like;        /* spec reach / reach-avoid                     */
  int32_t n_starts;
  const int32_t* starts;     /* (n_starts) controller slots                  */
  int32_t n_ctrl;
  const double* coords;      /* (n_ctrl, n) controller state coordinates     */
  const int32_t* slot_input; /* (n_ctrl) input index of each slot's policy   */
  int64_t total;             /* state lattice size                           */
  const int32_t* slot_of;    /* (total) controller slot of a flat state, -1  */
  const uint8_t* kind;       /* (total) 1 avoid, 2 target, 0 other           */
  const double* lb;          /* (n) state space                              */
  const double* ub;
  /* desc->consts here: (n_u, n_consts) folded at (u_j, disturbance centre) */
} imp_sim_desc;

/* All rollouts at once, one GPU thread each, bit-identical to the
 * reference's loop for dynamics without x-dependent library calls.
 * trace: (rollouts, steps + 1, n) visited points (the first length[r] rows
 * of each rollout are valid); satisfied: (rollouts) 0/1.  A non-finite
 * dynamics value -> IMP_E_NONFINITE (EvalError). */
int imp_simulate(const imp_build_desc* d, const imp_sim_desc* s,
                 double* trace, int32_t* length, int32_t* satisfied);

/* ---------------------------------------------------------------------- */
/* Text export in the reference's file formats (fileio.py)                 */
/* ---------------------------------------------------------------------- */

/* Dense text lines of rows [row_begin, row_end) of t_min (which = 0) or
 * t_max (which = 1), exactly as the reference's save_matrix writes them
 * (fileio.py:94-101: format(x, ".17g") per field, one space between fields,
 * '\n' per row; the header line is the caller's).  Rendered on the device
 * from the sparse rows, zeros included.  buf == NULL: size query only
 * (*out_len = bytes needed).  Replaces the per-row Python formatting loop
 * of fileio.save_matrix / save_abstraction (:285-299). */
int imp_export_text_rows(const imp_imdp* h, int32_t which, int64_t row_begin,
                         int64_t row_end, char* buf, int64_t cap,
                         int64_t* out_len);

/* Text body of n host doubles as lines of `cols` fields (row-major; n a
 * multiple of cols): format(x, ".17g"), ' ' between fields, '\n' after each
 * line -- the body of save_matrix (cols = C) and save_vector (cols = 1),
 * fileio.py:94-101, :118-123, formatted on the device.  buf == NULL: size
 * query. */
int imp_format_values(const double* x, int64_t n, int64_t cols,
                      int32_t device, char* buf, int64_t cap,
                      int64_t* out_len);

/* Cumulative kernel launches issued by the library: our own kernels and
 * CUB primitive calls (radix sort / scan), graph replays included. */
void imp_launch_count(unsigned long long* mine, unsigned long long* cub);

#ifdef __cplusplus
}
#endif
#endif /* IMPACT_B200_H */
