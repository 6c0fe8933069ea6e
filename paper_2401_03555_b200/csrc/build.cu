// IMDP construction host driver (reference build_abstraction,
// pkg/src/impact/abstraction.py:551-599).
//
// The construction kernels (jit/construct.cuh) are specialised per dynamics
// spec with NVRTC: the generated source fixes the state dimension, the
// dependency structure and the x-dependent residual of every f_d, so the
// Nelder-Mead objective is straight-line FP64 code with the simplex
// dimension known at compile time.  Compiled for sm_100a with --fmad=false
// (numpy's rounding of a*b + c); modules are cached per source in-process.
//
// Pipeline on one stream: stage 1 mean ranges -> stage 2 count -> CUB scan
// -> stage 2 write -> [stage 3 NM refinement, coupled only] -> stage 4
// assemble -> slack / row stats.  Device time per stage via CUDA events.
#include <nvrtc.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "common.h"
#include "_jit_source.inc"

namespace imp {
namespace {

// Host mirror of BuildParams in jit/construct.cuh (identical layout).
struct BuildParams {
  int n_u, n_w, k_begin, k_count;
  long long n_rows;
  int n_s, n_t, n_a, total;
  const int* counts;
  const int* edge_off;
  const int* strides;
  const double* eta;
  const double* sigma;
  const double* edges;
  const double* cover_lo;
  const double* cover_hi;
  const double* src_lo;
  const double* src_hi;
  const double* consts;
  const int* label;
  const int* safe_flat;
  const int* target_flat;
  const int* avoid_flat;
  double cutoff, tol;
  int low_cost, separable;
  int max_evals_fixed;
  int multistart;
  double* mlo;
  double* mhi;
  int write;
  long long* t_count;
  long long* x_count;
  const long long* row_ptr;
  const long long* aux_ptr;
  int* col;
  double* lo;
  double* hi;
  int* aux_code;
  double* aux_min;
  double* aux_max;
  double* raw;
  long long n_items;
  long long* evals;
  double* r_min;
  double* r_max;
  double* a_min;
  double* a_max;
  unsigned long long* err;
  double* err_val;
  double sig[16];
  double sig_rcp[16];
  int sep;
  const double* dim_lo;
  const double* dim_hi;
  double* sep_mr;
  double* sep_tab;
  long long row0;
  int mc_samples;
  unsigned long long mc_seed;
  double mc_norm;
  const double* inv_cov;
  const double2* box;
};

// JIT modules go through the runtime's library API (cudaLibrary_t /
// cudaKernel_t), so libimpact_b200.so never links libcuda directly and
// loads on hosts without a driver (the CPU build check).
struct JitModule {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t mean = nullptr, outer = nullptr, refine = nullptr,
               assemble = nullptr, simulate = nullptr, sep_tables = nullptr,
               outer_sep = nullptr, ndtr_eval = nullptr;
};

std::mutex g_jit_mu;
std::map<std::string, JitModule> g_jit_cache;

// Threads per block of the NM kernels: the shared-memory simplex of every
// thread ((N+1)*N + N+1 doubles) must fit in ~200 KB.
int nm_block(int n) {
  const size_t per = ((size_t)(n + 4) * n + 2 * (n + 1)) * sizeof(double) +
                     (64 + 16 * (size_t)n);
  int b = 128;
  while (b > 32 && b * per > 200 * 1024) b /= 2;
  return b;
}

// k_refine keeps its per-thread Instance record in shared memory (1) or in
// registers (0)
int inst_smem() {
  const char* e = getenv("IMPACT_INST_SMEM");
  return e ? atoi(e) : 0;
}

// The fast k_refine objective needs RN(1/sigma) for an unchecked Markstein
// quotient; noise scales outside 2^+-100 (never in practice) take the exact
// module.
bool exact_mode(const imp_build_desc* d) {
  if (d->exact) return true;
  for (int q = 0; q < d->n; ++q) {
    const double sg = d->sigma[q];
    if (!(sg >= 0x1p-100 && sg <= 0x1p100)) return true;
  }
  return false;
}

std::string config_header(const imp_build_desc* d) {
  std::ostringstream o;
  o << "#define IMP_EXACT " << (exact_mode(d) ? 1 : 0) << "\n";
  o << "#define IMP_N " << d->n << "\n#define IMP_NC "
    << std::max(d->n_consts, 1) << "\n";
  o << "#define IMP_MC " << (d->mc ? 1 : 0) << "\n";
  o << "#define IMP_MC_CUSTOM " << (d->mc == 2 ? 1 : 0) << "\n";
  o << "#define IMP_MEAN_BLOCK " << nm_block(d->n) << "\n";
  o << "#define IMP_REFINE_BLOCK " << nm_block(d->n) << "\n";
  // tuning knobs (environment overrides for experiments)
  const char* minb = getenv("IMPACT_REFINE_MINB");
  // defaults measured on the full vehicle3d / room5d builds (subsets mislead)
  // (n = 5: shared memory admits 3 blocks of 128 per SM, so a register
  // cap for 4 only adds spills -- room5d refine 17.86 -> 17.27 s with 3;
  // n >= 6: 2 blocks fit.  profiles/r02/k_refine_minb_ab.txt)
  o << "#define IMP_REFINE_MINB "
    << (minb ? atoi(minb) : (d->n <= 4 ? 5 : d->n == 5 ? 3 : 2))
    << "\n";
  const char* ch = getenv("IMPACT_NDTR_CHUNK");
  // CDF chains interleaved per step: fast objective 2 (full vehicle3d
  // build: 1.56e10 vs 1.53e10 evaluations/s for one), exact 1 (12.72 vs
  // 12.87 s; profiles/r02/k_refine_exact_knobs_vehicle3d.txt)
  o << "#define IMP_NDTR_CHUNK " << (ch ? atoi(ch) : exact_mode(d) ? 1 : 2)
    << "\n";
  const char* unr = getenv("IMPACT_NDTR_UNROLL");
  o << "#define IMP_NDTR_UNROLL " << (unr ? atoi(unr) : 0) << "\n";
  o << "#define IMP_INST_SMEM " << inst_smem() << "\n";
  const char* leg = getenv("IMPACT_NDTR_LEGACY");   // round-1 exact ndtr
  o << "#define IMP_NDTR_LEGACY " << (leg ? atoi(leg) : 0) << "\n";
  const char* ftab = getenv("IMPACT_NDTR_FAST_TABLE");
  o << "#define IMP_NDTR_FAST_TABLE " << (ftab ? atoi(ftab) : 0) << "\n";
  // Nelder-Mead next point on one shared path for every phase (same bits;
  // vehicle3d refine 12.73 -> 12.48 s, room5d 19.39 -> 18.49 s:
  // profiles/r02/k_refine_nm_unified_ab.txt)
  const char* nmu = getenv("IMPACT_NM_UNIFIED");
  o << "#define IMP_NM_UNIFIED " << (nmu ? atoi(nmu) : 1) << "\n";
  // exact objective: each dimension's factor formed as soon as its two
  // CDFs are known, no cdf array in local memory (same bits; vehicle3d
  // refine 12.48 -> 12.25 s, room5d 18.49 -> 17.82 s:
  // profiles/r02/k_refine_obj_fused_ab.txt)
  const char* ofu = getenv("IMPACT_OBJ_FUSED");
  o << "#define IMP_OBJ_FUSED " << (ofu ? atoi(ofu) : 1) << "\n";
  // (IMPACT_REFINE_CARVEOUT: the k_refine shared-memory carve-out hint, an
  // experiment knob; the driver's default is the fastest measured)
  const char* batch = getenv("IMPACT_REFINE_BATCH");
  // k_refine work grab: 8 boxes per atomic (fewer binary-search seeks;
  // vehicle3d 12.25 -> 12.11 s, profiles/r02/k_refine_batch_ab.txt)
  o << "#define IMP_REFINE_BATCH " << (batch ? atoi(batch) : 16) << "\n";
  // the lattice shape as compile-time constants: index arithmetic by
  // multiply-shift instead of the integer-division sequence
  o << "__device__ constexpr int kCounts[IMP_N] = {";
  for (int q = 0; q < d->n; ++q) o << (q ? ", " : "") << d->counts[q];
  o << "};\n";
  // a separable row's 1-D tables ({min, max} per coordinate of every
  // dimension): offsets and size, for staging them per warp in k_outer_sep
  {
    int tot = 0;
    o << "__device__ constexpr int kTabOff[IMP_N] = {";
    for (int q = 0; q < d->n; ++q) {
      o << (q ? ", " : "") << tot;
      tot += 2 * d->counts[q];
    }
    o << "};\n#define IMP_TAB_DOUBLES " << tot << "\n";
  }
  o << "__device__ constexpr int kStrides[IMP_N] = {";   // row-major
  {
    std::vector<long long> st(d->n);
    long long t = 1;
    for (int q = d->n - 1; q >= 0; --q) {
      st[q] = t;
      t *= d->counts[q];
    }
    for (int q = 0; q < d->n; ++q) o << (q ? ", " : "") << st[q];
  }
  o << "};\n";
  o << "__device__ constexpr int kNDeps[IMP_N] = {";
  for (int q = 0; q < d->n; ++q) o << (q ? ", " : "") << d->n_deps[q];
  o << "};\n__device__ constexpr int kDeps[IMP_N][IMP_N] = {";
  for (int q = 0; q < d->n; ++q) {
    o << (q ? ", {" : "{");
    for (int e = 0; e < d->n; ++e) o << (e ? ", " : "") << d->deps[q * d->n + e];
    o << "}";
  }
  o << "};\n";
  return o.str();
}

// config header (macros, dependency tables) + ndtr prelude + generated
// dynamics + kernels
std::string jit_source(const std::string& config, const std::string& dyn) {
  return config + std::string(kJitPrelude) + "\n" +
         "__device__ __forceinline__ double imp_min(double, double);\n"
         "__device__ __forceinline__ double imp_max(double, double);\n" +
         dyn + "\n" + kJitKernels;
}

// NVRTC: source -> sm_100a cubin (no device needed).
std::vector<char> compile_cubin(const std::string& src) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "impact_construct.cu", 0,
                         nullptr, nullptr) != NVRTC_SUCCESS)
    fail(IMP_E_JIT, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false",
                        "-std=c++17", "-lineinfo"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    set_error("NVRTC compile of the construction module failed:\n%s",
              log.c_str());
    throw Failure{IMP_E_JIT};
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  return cubin;
}

JitModule& jit(int device, const std::string& config, const std::string& dyn) {
  const std::string src = jit_source(config, dyn);
  const std::string key = std::to_string(device) + "\n" + src;
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto it = g_jit_cache.find(key);
  if (it != g_jit_cache.end()) return it->second;
  if (getenv("IMPACT_DUMP_JIT")) {  // for ncu --import-source
    if (FILE* f = fopen("impact_construct.cu", "w")) {
      fwrite(src.data(), 1, src.size(), f);
      fclose(f);
    }
  }
  std::vector<char> cubin = compile_cubin(src);
  IMP_CUDA(cudaSetDevice(device));
  IMP_CUDA(cudaFree(nullptr));  // bind the primary context
  JitModule m;
  IMP_CUDA(cudaLibraryLoadData(&m.lib, cubin.data(), nullptr, nullptr, 0,
                               nullptr, nullptr, 0));
  IMP_CUDA(cudaLibraryGetKernel(&m.mean, m.lib, "k_mean_ranges"));
  IMP_CUDA(cudaLibraryGetKernel(&m.outer, m.lib, "k_outer"));
  IMP_CUDA(cudaLibraryGetKernel(&m.refine, m.lib, "k_refine"));
  IMP_CUDA(cudaLibraryGetKernel(&m.assemble, m.lib, "k_assemble"));
  IMP_CUDA(cudaLibraryGetKernel(&m.simulate, m.lib, "k_simulate"));
  IMP_CUDA(cudaLibraryGetKernel(&m.sep_tables, m.lib, "k_sep_tables"));
  IMP_CUDA(cudaLibraryGetKernel(&m.outer_sep, m.lib, "k_outer_sep"));
  IMP_CUDA(cudaLibraryGetKernel(&m.ndtr_eval, m.lib, "k_ndtr_eval"));
  return g_jit_cache.emplace(key, m).first->second;
}

void launch(cudaKernel_t f, unsigned grid, unsigned block, size_t smem,
            cudaStream_t s, BuildParams& P) {
  const void* fn = reinterpret_cast<const void*>(f);
  if (smem > 48 * 1024)
    IMP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  void* args[] = {&P};
  IMP_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, s));
}

template <class T>
DevBuf<T> upload(const T* src, size_t n, cudaStream_t s) {
  DevBuf<T> b(std::max<size_t>(n, 1));
  if (n) IMP_CUDA(cudaMemcpyAsync(b.ptr, src, n * sizeof(T),
                                  cudaMemcpyHostToDevice, s));
  return b;
}

void exclusive_scan(long long* counts, long long* out, int64_t n,
                    cudaStream_t s) {
  device_exclusive_scan(reinterpret_cast<const int64_t*>(counts),
                        reinterpret_cast<int64_t*>(out), n, s);
}

struct Events {
  cudaEvent_t e[6];
  Events() { for (auto& x : e) cudaEventCreate(&x); }
  ~Events() { for (auto& x : e) cudaEventDestroy(x); }
  float ms(int a, int b) {
    float v = 0.f;
    cudaEventElapsedTime(&v, e[a], e[b]);
    return v;
  }
};

}  // namespace
}  // namespace imp

using namespace imp;

extern "C" int imp_build(const imp_build_desc* d, imp_imdp** out,
                         imp_build_stats* stats) {
  imp_imdp* h = nullptr;
  int st = guarded([&] {
    IMP_REQUIRE(d && out, "null argument");
    const int N = d->n;
    IMP_REQUIRE(N >= 1 && N <= 16, "state dimension %d unsupported", N);
    IMP_REQUIRE(d->n_s >= 1, "no safe states to abstract");
    IMP_REQUIRE(d->k_begin >= 0 && d->k_count >= 0 &&
                    d->k_begin + d->k_count <= d->n_s,
                "bad shard range");
    IMP_REQUIRE(d->dyn_source, "missing dynamics source");
    IMP_CUDA(cudaSetDevice(d->device));
    int sms = 0;   // queried below
    IMP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount,
                                    d->device));
    JitModule& M = jit(d->device, config_header(d), d->dyn_source);

    cudaStream_t s;
    IMP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
    Events ev;

    // --- host geometry -> device ------------------------------------------
    std::vector<int> edge_off(N), strides(N);
    int total = 1, off = 0;
    for (int q = 0; q < N; ++q) {
      edge_off[q] = off;
      off += d->counts[q] + 1;
    }
    for (int q = N - 1; q >= 0; --q) {
      strides[q] = total;
      total *= d->counts[q];
    }
    auto flat_of = [&](const int32_t* multi, int cnt) {
      std::vector<int> f(cnt);
      for (int i = 0; i < cnt; ++i) {
        int v = 0;
        for (int q = 0; q < N; ++q) v += multi[(int64_t)i * N + q] * strides[q];
        f[i] = v;
      }
      return f;
    };
    std::vector<int> sflat = flat_of(d->safe_multi, d->n_s);
    std::vector<int> tflat = flat_of(d->target_multi, d->n_t);
    std::vector<int> aflat = flat_of(d->avoid_multi, d->n_a);
    std::vector<int> label;
    const bool identity = d->n_t == 0 && d->n_a == 0 && d->n_s == total;
    if (!identity) {
      label.assign(total, INT32_MIN);
      for (int i = 0; i < d->n_s; ++i) label[sflat[i]] = i;
      for (int i = 0; i < d->n_t; ++i) label[tflat[i]] = -1 - i;
      for (int i = 0; i < d->n_a; ++i) label[aflat[i]] = -1 - d->n_t - i;
    }
    auto g_counts = upload(d->counts, N, s);
    auto g_eoff = upload(edge_off.data(), N, s);
    auto g_strides = upload(strides.data(), N, s);
    auto g_eta = upload(d->eta, N, s);
    auto g_sigma = upload(d->sigma, N, s);
    auto g_edges = upload(d->edges, (size_t)off, s);
    // destination boxes per lattice state (k_refine item setup)
    const bool refines = !d->separable || d->mc;
    std::vector<double2> hbox(refines ? (size_t)total * N : 1);
    for (int f = 0; refines && f < total; ++f)
      for (int q = 0; q < N; ++q) {
        const int b = (f / strides[q]) % d->counts[q];
        hbox[(size_t)f * N + q] = make_double2(d->edges[edge_off[q] + b],
                                               d->edges[edge_off[q] + b + 1]);
      }
    auto g_box = upload(hbox.data(), hbox.size(), s);
    auto g_clo = upload(d->cover_lo, N, s);
    auto g_chi = upload(d->cover_hi, N, s);
    auto g_slo = upload(d->src_lo, (size_t)d->n_s * N, s);
    auto g_shi = upload(d->src_hi, (size_t)d->n_s * N, s);
    const int nc = std::max(d->n_consts, 1);
    auto g_consts = upload(d->consts, (size_t)d->n_u * d->n_w * nc, s);
    auto g_label = upload(label.data(), label.size(), s);
    auto g_sflat = upload(sflat.data(), sflat.size(), s);
    auto g_tflat = upload(tflat.data(), tflat.size(), s);
    auto g_aflat = upload(aflat.data(), aflat.size(), s);

    const long long n_rows = (long long)d->k_count * d->n_u * d->n_w;
    h = new imp_imdp();
    h->device = d->device;
    h->n_s = d->n_s;
    h->n_u = d->n_u;
    h->n_w = d->n_w;
    h->k_begin = d->k_begin;
    h->k_count = d->k_count;
    h->n_rows = n_rows;

    DevBuf<double> mlo(n_rows * N + 1), mhi(n_rows * N + 1), raw(n_rows * 6 + 1);
    DevBuf<long long> tcnt(n_rows + 1), xcnt(n_rows + 1);
    DevBuf<int64_t> row_ptr(n_rows + 1);
    DevBuf<long long> aux_ptr(n_rows + 1);
    DevBuf<unsigned long long> err(3);
    DevBuf<double> err_val(3);
    // [0] objective evals (the reference's count), [1] refine lane slots,
    // [2] refine work counter, [3] evals saved by shared initial simplices,
    // [4] stored entries with t_max > zero_cutoff (k_assemble)
    DevBuf<long long> evals(6);
    IMP_CUDA(cudaMemsetAsync(err.ptr, 0xff, 3 * sizeof(unsigned long long), s));
    IMP_CUDA(cudaMemsetAsync(err_val.ptr, 0, 3 * sizeof(double), s));
    IMP_CUDA(cudaMemsetAsync(evals.ptr, 0, 6 * sizeof(long long), s));
    IMP_CUDA(cudaMemsetAsync(tcnt.ptr, 0, (n_rows + 1) * sizeof(long long), s));
    IMP_CUDA(cudaMemsetAsync(xcnt.ptr, 0, (n_rows + 1) * sizeof(long long), s));
    IMP_CUDA(cudaMemsetAsync(raw.ptr, 0, (n_rows * 6 + 1) * sizeof(double), s));

    BuildParams P{};
    P.n_u = d->n_u;
    P.n_w = d->n_w;
    P.k_begin = d->k_begin;
    P.k_count = d->k_count;
    P.n_rows = n_rows;
    P.n_s = d->n_s;
    P.n_t = d->n_t;
    P.n_a = d->n_a;
    P.total = total;
    P.counts = g_counts.ptr;
    P.edge_off = g_eoff.ptr;
    P.strides = g_strides.ptr;
    P.eta = g_eta.ptr;
    P.sigma = g_sigma.ptr;
    for (int q = 0; q < 16; ++q) {
      const double sg = q < N ? d->sigma[q] : 1.0;
      P.sig[q] = sg;
      P.sig_rcp[q] = (sg >= 0x1p-100 && sg <= 0x1p100) ? 1.0 / sg : NAN;
    }
    P.edges = g_edges.ptr;
    P.box = g_box.ptr;
    P.cover_lo = g_clo.ptr;
    P.cover_hi = g_chi.ptr;
    P.src_lo = g_slo.ptr;
    P.src_hi = g_shi.ptr;
    P.consts = g_consts.ptr;
    P.label = identity ? nullptr : g_label.ptr;
    P.safe_flat = g_sflat.ptr;
    P.target_flat = g_tflat.ptr;
    P.avoid_flat = g_aflat.ptr;
    P.cutoff = d->zero_cutoff;
    P.tol = d->tol;
    P.low_cost = d->low_cost;
    P.separable = d->separable;
    P.max_evals_fixed = d->max_evals_per_dim < 0 ? -d->max_evals_per_dim : 0;
    P.multistart = d->multistart;
    P.mlo = mlo.ptr;
    P.mhi = mhi.ptr;
    P.t_count = tcnt.ptr;
    P.x_count = xcnt.ptr;
    P.row_ptr = reinterpret_cast<const long long*>(row_ptr.ptr);
    P.aux_ptr = aux_ptr.ptr;
    P.raw = raw.ptr;
    P.evals = evals.ptr;
    P.err = err.ptr;
    P.err_val = err_val.ptr;

    // Monte Carlo noise: every destination of every row is an NM item
    P.row0 = (long long)d->k_begin * d->n_u * d->n_w;
    P.mc_samples = d->mc_samples;
    P.mc_seed = d->mc_seed;
    P.mc_norm = d->mc_norm;
    DevBuf<double> g_inv;
    if (d->mc) {
      IMP_REQUIRE(d->inv_cov && d->mc_samples >= 2, "bad Monte Carlo noise");
      IMP_REQUIRE(d->mc == 1 || d->mc == 2, "bad Monte Carlo noise kind");
      g_inv = upload(d->inv_cov, (size_t)N * N, s);
      P.inv_cov = g_inv.ptr;
    }

    // IMPACT_SYNC_STAGES=1: synchronize after every stage (fault isolation)
    const bool sync_stages = getenv("IMPACT_SYNC_STAGES") != nullptr;
    auto stage_done = [&](const char* name) {
      if (!sync_stages) return;
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        set_error("stage %s: %s", name, cudaGetErrorString(e));
        throw Failure{IMP_E_CUDA};
      }
    };

    // --- stage 1: mean ranges -------------------------------------------------
    // per-thread shared memory of the NM kernels (jit/construct.cuh:
    // imp_nm_doubles; k_refine adds its Instance record)
    const size_t nm_doubles = (size_t)(N + 4) * N + (N + 1);
    // k_refine also keeps the min run's initial simplex values (N + 1)
    const size_t refine_doubles = nm_doubles + (N + 1);
    const size_t inst_bytes = 5 * 8 + 5 * 4 + 4 + 2 * N * 8 + (d->mc ? 8 : 0);
    const int block1 = nm_block(N);
    // separable dynamics: one table per (dimension, coordinate, input,
    // disturbance) instead of per row.  The choice depends on the system
    // only (never on the shard), because it selects k_outer_sep, whose r / a
    // sums use a warp tree: every shard of a system must take the same path
    // for the bits to be shard-independent.  (IMPACT_SEP_TABLES set: per-row
    // path, for A/B timing only.)
    long long nkeys = 0, tab_doubles = 0;
    for (int q = 0; q < N; ++q) {
      nkeys += (long long)d->counts[q] * d->n_u * d->n_w;
      tab_doubles += 2ll * d->counts[q] * d->counts[q] * d->n_u * d->n_w;
    }
    const bool sep = d->separable && !d->mc && d->dim_lo && d->dim_hi &&
                     getenv("IMPACT_SEP_TABLES") == nullptr &&
                     tab_doubles < (1ll << 29);
    DevBuf<double> g_dlo, g_dhi, sep_mr, sep_tab;
    P.sep = sep ? 1 : 0;
    if (sep && n_rows > 0) {
      int csum = 0;
      for (int q = 0; q < N; ++q) csum += d->counts[q];
      g_dlo = upload(d->dim_lo, csum, s);
      g_dhi = upload(d->dim_hi, csum, s);
      sep_mr.alloc(2 * nkeys);
      sep_tab.alloc(std::max<long long>(tab_doubles, 1));
      P.dim_lo = g_dlo.ptr;
      P.dim_hi = g_dhi.ptr;
      P.sep_mr = sep_mr.ptr;
      P.sep_tab = sep_tab.ptr;
    }
    // device timing starts here: host geometry, uploads and allocations
    // above are part of the end-to-end time, not of the kernels'
    IMP_CUDA(cudaEventRecord(ev.e[0], s));
    if (sep && n_rows > 0) {
      P.write = 0;   // mean ranges, one thread per (key, sign)
      unsigned grid = (unsigned)std::min<long long>(
          (2 * nkeys + block1 - 1) / block1, (long long)sms * 64);
      launch(M.sep_tables, grid, block1, block1 * nm_doubles * 8, s, P);
      P.write = 1;   // tables, one thread per (key, bin)
      grid = (unsigned)std::min<long long>(
          (tab_doubles / 2 + block1 - 1) / block1, (long long)sms * 64);
      launch(M.sep_tables, grid, block1, block1 * nm_doubles * 8, s, P);
    }
    if (n_rows > 0 && !d->mc && !sep) {
      const long long ntask = n_rows * N * 2;
      unsigned grid = (unsigned)std::min<long long>((ntask + block1 - 1) / block1,
                                                    (long long)sms * 64);
      launch(M.mean, grid, block1, block1 * nm_doubles * 8, s, P);
    }
    stage_done("mean_ranges");
    IMP_CUDA(cudaEventRecord(ev.e[1], s));

    // --- stage 2: count, scan, write ---------------------------------------
    int nbins = 0;
    for (int q = 0; q < N; ++q) nbins += d->counts[q];
    const size_t smem2 = 2 * (size_t)nbins * sizeof(double);
    const unsigned grid2 = (unsigned)std::max<long long>(
        1, std::min<long long>(n_rows, (long long)sms * 32));
    // separable rows with per-key tables: one warp per row
    const unsigned grid_sep = (unsigned)std::max<long long>(
        1, std::min<long long>((n_rows * 32 + 255) / 256, (long long)sms * 64));
    auto outer = [&]() {
      if (n_rows <= 0) return;
      if (sep) launch(M.outer_sep, grid_sep, 256, 0, s, P);
      else launch(M.outer, grid2, 128, smem2, s, P);
    };
    P.write = 0;
    outer();
    stage_done("outer count");
    if (d->state_cost) {   // count only: per-state construction work
      std::vector<long long> tc(std::max<long long>(n_rows, 1)),
          xc(std::max<long long>(n_rows, 1));
      if (n_rows > 0) {
        IMP_CUDA(cudaMemcpyAsync(tc.data(), tcnt.ptr, sizeof(long long) * n_rows,
                                 cudaMemcpyDeviceToHost, s));
        IMP_CUDA(cudaMemcpyAsync(xc.data(), xcnt.ptr, sizeof(long long) * n_rows,
                                 cudaMemcpyDeviceToHost, s));
      }
      IMP_CUDA(cudaStreamSynchronize(s));
      const long long per = (long long)d->n_u * d->n_w;
      const bool refine = !d->separable || d->mc;
      for (int k = 0; k < d->k_count; ++k) {
        long long c = 0;
        for (long long r = k * per; r < (k + 1) * per; ++r)
          c += tc[r] + (refine ? xc[r] : 0) + 1;
        d->state_cost[k] = c;
      }
      delete h;
      h = nullptr;
      *out = nullptr;
      return;
    }
    exclusive_scan(tcnt.ptr, reinterpret_cast<long long*>(row_ptr.ptr), n_rows + 1, s);
    exclusive_scan(xcnt.ptr, aux_ptr.ptr, n_rows + 1, s);
    long long nnz = 0, naux = 0;
    IMP_CUDA(cudaMemcpyAsync(&nnz, row_ptr.ptr + n_rows, sizeof(long long),
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaMemcpyAsync(&naux, aux_ptr.ptr + n_rows, sizeof(long long),
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaStreamSynchronize(s));
    h->nnz = nnz;
    h->col.alloc(std::max<long long>(nnz, 1));
    h->lo.alloc(std::max<long long>(nnz, 1));
    h->hi.alloc(std::max<long long>(nnz, 1));
    DevBuf<int> aux_code(std::max<long long>(naux, 1));
    DevBuf<double> aux_min(std::max<long long>(naux, 1)),
        aux_max(std::max<long long>(naux, 1));
    P.col = h->col.ptr;
    P.lo = h->lo.ptr;
    P.hi = h->hi.ptr;
    P.aux_code = aux_code.ptr;
    P.aux_min = aux_min.ptr;
    P.aux_max = aux_max.ptr;
    P.write = 1;
    outer();
    stage_done("outer write");
    IMP_CUDA(cudaEventRecord(ev.e[2], s));

    // --- stage 3: NM refinement of the live window (coupled) ---------------
    long long instances = 0;
    if ((!d->separable || d->mc) && n_rows > 0) {
      P.n_items = nnz + naux + n_rows;
      instances = 2 * P.n_items;
      const int block3 = nm_block(N);
      const size_t smem3 =
          block3 * (refine_doubles * sizeof(double) + (inst_smem() ? inst_bytes : 0));
      const void* rfn = reinterpret_cast<const void*>(M.refine);
      if (smem3 > 48 * 1024)
        IMP_CUDA(cudaFuncSetAttribute(
            rfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
      if (const char* co = getenv("IMPACT_REFINE_CARVEOUT"))   // experiment
        IMP_CUDA(cudaFuncSetAttribute(
            rfn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(co)));
      int per_sm = 0;
      IMP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rfn,
                                                             block3, smem3));
      per_sm = std::max(per_sm, 1);
      const long long need = (instances + block3 - 1) / block3;
      const unsigned grid3 = (unsigned)std::max<long long>(
          1, std::min<long long>(need, (long long)sms * per_sm));
      launch(M.refine, grid3, block3, smem3, s, P);
      stage_done("refine");
    }
    IMP_CUDA(cudaEventRecord(ev.e[3], s));

    // --- stage 4: assemble ---------------------------------------------------
    for (auto* b : {&h->r_min, &h->r_max, &h->a_min, &h->a_max})
      b->alloc(std::max<long long>(n_rows, 1));
    P.r_min = h->r_min.ptr;
    P.r_max = h->r_max.ptr;
    P.a_min = h->a_min.ptr;
    P.a_max = h->a_max.ptr;
    if (n_rows > 0) {
      const unsigned grid4 = (unsigned)std::max<long long>(
          1, std::min<long long>((n_rows * 32 + 255) / 256, (long long)sms * 64));
      launch(M.assemble, grid4, 256, 0, s, P);
    }
    IMP_CUDA(cudaEventRecord(ev.e[4], s));
    IMP_CUDA(cudaStreamSynchronize(s));

    unsigned long long herr[3];
    double hval[3];
    long long hev = 0, hslots = 0, hshared = 0, hlive = 0, hmean = 0;
    IMP_CUDA(cudaMemcpy(herr, err.ptr, sizeof(herr), cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(hval, err_val.ptr, sizeof(hval), cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(&hev, evals.ptr, sizeof(hev), cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(&hslots, evals.ptr + 1, sizeof(hslots),
                        cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(&hshared, evals.ptr + 3, sizeof(hshared),
                        cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(&hlive, evals.ptr + 4, sizeof(hlive),
                        cudaMemcpyDeviceToHost));
    IMP_CUDA(cudaMemcpy(&hmean, evals.ptr + 5, sizeof(hmean),
                        cudaMemcpyDeviceToHost));
    const long long row0 = (long long)d->k_begin * d->n_u * d->n_w;
    if (herr[0] != ~0ull) {
      set_error("row %lld", row0 + (long long)herr[0]);
      throw Failure{IMP_E_NONFINITE};
    }
    if (herr[1] != ~0ull) {
      set_error("row %lld: min-side sum exceeds 1 by %.17g",
                row0 + (long long)herr[1], hval[1]);
      throw Failure{IMP_E_ABSTRACTION};
    }
    if (herr[2] != ~0ull) {
      set_error("row %lld: max-side sum falls short of 1 by %.17g",
                row0 + (long long)herr[2], hval[2]);
      throw Failure{IMP_E_ABSTRACTION};
    }
    h->row_ptr = std::move(row_ptr);
    finalize_imdp(h, s);
    if (n_rows > 0)
      count_launches(5 + (d->separable ? 0 : 1), 0);  // + slack kernel (scans count themselves)
    IMP_CUDA(cudaEventRecord(ev.e[5], s));
    IMP_CUDA(cudaEventSynchronize(ev.e[5]));
    if (stats) {
      stats->ms_total = ev.ms(0, 5);
      stats->ms_mean_ranges = ev.ms(0, 1);
      stats->ms_outer = ev.ms(1, 2);
      stats->ms_refine = ev.ms(2, 3);
      stats->ms_assemble = ev.ms(3, 5);
      stats->nnz = nnz;
      stats->nm_instances = instances;
      stats->nm_evals = hev;
      stats->nm_lane_slots = hslots;
      stats->nm_evals_shared = hshared;
      stats->nnz_live = hlive;
      stats->nm_evals_mean = hmean;
    }
    *out = h;
  });
  if (st != IMP_OK) delete h;
  return st;
}

// Compile (only) the construction module for a dynamics spec and optionally
// write the cubin to `cubin_path`: used by the CPU build check and to
// inspect SASS (cuobjdump) without a GPU.
extern "C" int imp_jit_compile(const imp_build_desc* d, const char* cubin_path) {
  return guarded([&] {
    IMP_REQUIRE(d && d->dyn_source, "null argument");
    std::vector<char> cubin =
        compile_cubin(jit_source(config_header(d), d->dyn_source));
    if (cubin_path) {
      FILE* f = fopen(cubin_path, "wb");
      IMP_REQUIRE(f, "cannot open %s", cubin_path);
      fwrite(cubin.data(), 1, cubin.size(), f);
      fclose(f);
    }
  });
}

// The device normal CDFs of desc's construction module on n host values
// (test entry: parity of the k_refine objective's CDF forms with scipy).
extern "C" int imp_ndtr_eval(const imp_build_desc* d, const double* x,
                             double* y, int64_t n, int32_t which) {
  return guarded([&] {
    IMP_REQUIRE(d && d->dyn_source && x && y && n >= 0, "null argument");
    IMP_REQUIRE(which >= 0 && which <= 2, "which must be 0, 1 or 2");
    IMP_CUDA(cudaSetDevice(d->device));
    JitModule& M = jit(d->device, config_header(d), d->dyn_source);
    if (n == 0) return;
    DevBuf<double> gx(n), gy(n);
    IMP_CUDA(cudaMemcpy(gx.ptr, x, n * sizeof(double), cudaMemcpyHostToDevice));
    const void* fn = reinterpret_cast<const void*>(M.ndtr_eval);
    long long nn = n;
    int w = which;
    void* args[] = {&gx.ptr, &gy.ptr, &nn, &w};
    const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 4096);
    IMP_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(256), args, 0, 0));
    IMP_CUDA(cudaMemcpy(y, gy.ptr, n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

// ---------------------------------------------------------------------------
// Closed-loop simulation (cli.py:177-251): k_simulate of the JIT module
// ---------------------------------------------------------------------------

namespace imp {
namespace {
// Mirror of the JIT module's SimParams (jit/simulate.cuh); same layout.
struct SimParamsHost {
  int rollouts, steps, n_starts, reach_like;
  unsigned long long seed;
  const int* starts;
  const double* coords;
  const int* slot_of;
  const unsigned char* kind;
  const int* slot_input;
  const double* consts;
  const double* lb;
  const double* ub;
  const double* eta;
  const int* counts;
  const double* sigma;
  double* trace;
  int* length;
  int* satisfied;
  unsigned long long* err;
};
}  // namespace
}  // namespace imp

extern "C" int imp_simulate(const imp_build_desc* d, const imp_sim_desc* sd,
                            double* trace, int32_t* length,
                            int32_t* satisfied) {
  return guarded([&] {
    IMP_REQUIRE(d && sd && trace && length && satisfied, "null argument");
    IMP_REQUIRE(d->n >= 1 && d->n <= 16, "state dimension unsupported");
    IMP_REQUIRE(sd->rollouts >= 1 && sd->steps >= 1,
                "rollouts and steps must be >= 1");
    IMP_REQUIRE(sd->n_starts >= 1 && sd->n_ctrl >= 1, "empty controller");
    IMP_REQUIRE(d->dyn_source, "missing dynamics source");
    const int N = d->n;
    IMP_CUDA(cudaSetDevice(d->device));
    JitModule& M = jit(d->device, config_header(d), d->dyn_source);
    cudaStream_t s;
    IMP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
    const int64_t npts = (int64_t)sd->rollouts * (sd->steps + 1) * N;
    auto starts = upload(sd->starts, sd->n_starts, s);
    auto coords = upload(sd->coords, (size_t)sd->n_ctrl * N, s);
    auto slot_of = upload(sd->slot_of, sd->total, s);
    auto kind = upload(sd->kind, sd->total, s);
    auto slot_input = upload(sd->slot_input, sd->n_ctrl, s);
    auto consts = upload(d->consts, (size_t)d->n_u * std::max(d->n_consts, 1), s);
    auto lb = upload(sd->lb, N, s);
    auto ub = upload(sd->ub, N, s);
    auto eta = upload(d->eta, N, s);
    auto counts = upload(d->counts, N, s);
    auto sigma = upload(d->sigma, N, s);
    DevBuf<double> tr(npts);
    DevBuf<int> len(sd->rollouts), sat(sd->rollouts);
    DevBuf<unsigned long long> err(1);
    IMP_CUDA(cudaMemsetAsync(err.ptr, 0xff, sizeof(unsigned long long), s));
    SimParamsHost P{};
    P.rollouts = sd->rollouts;
    P.steps = sd->steps;
    P.n_starts = sd->n_starts;
    P.reach_like = sd->reach_like;
    P.seed = sd->seed;
    P.starts = starts.ptr;
    P.coords = coords.ptr;
    P.slot_of = slot_of.ptr;
    P.kind = kind.ptr;
    P.slot_input = slot_input.ptr;
    P.consts = consts.ptr;
    P.lb = lb.ptr;
    P.ub = ub.ptr;
    P.eta = eta.ptr;
    P.counts = counts.ptr;
    P.sigma = sigma.ptr;
    P.trace = tr.ptr;
    P.length = len.ptr;
    P.satisfied = sat.ptr;
    P.err = err.ptr;
    void* args[] = {&P};
    const unsigned block = 128;
    IMP_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(M.simulate),
                              dim3((sd->rollouts + block - 1) / block),
                              dim3(block), args, 0, s));
    count_launches(1, 0);
    unsigned long long e = 0;
    IMP_CUDA(cudaMemcpyAsync(&e, err.ptr, sizeof(e), cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaMemcpyAsync(trace, tr.ptr, sizeof(double) * npts,
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaMemcpyAsync(length, len.ptr, sizeof(int) * sd->rollouts,
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaMemcpyAsync(satisfied, sat.ptr, sizeof(int) * sd->rollouts,
                             cudaMemcpyDeviceToHost, s));
    IMP_CUDA(cudaStreamSynchronize(s));
    if (e != ~0ull) {
      set_error("domain error evaluating the dynamics (rollout %llu)", e);
      throw Failure{IMP_E_NONFINITE};
    }
  });
}
