// Closed-loop rollouts of a synthesized controller,
// appended to the JIT construction module (same generated dynamics).
//
// Reference: pkg/src/impact/cli.py:163-251 (cmd_simulate, _noise_sampler),
// grid.py:118-132 (quantize), noise.py:121-131 (derive_seed, mc_generator).
// One thread per rollout r:
//   rng     Generator(Philox(SeedSequence(derive_seed(seed, r, 0)))) (rng.h)
//   start   controller slot starts[r % n_starts], x = its coordinates
//   step    state = quantize(x) (outside the covered domain: fail); avoid:
//           fail; reach-like and target: success; no controller entry:
//           fail; else x = f(x, u_slot, w_center) + normal(0, sigma)
//   end     after `steps` steps without an event: success iff safety
// Every operation is the reference's IEEE sequence (--fmad=false), so for
// dynamics without x-dependent library calls the trace is bit-identical.

struct SimParams {
  int rollouts, steps, n_starts, reach_like;
  unsigned long long seed;
  const int* starts;           // (n_starts) controller slots
  const double* coords;        // (n_ctrl, N) controller state coordinates
  const int* slot_of;          // (total) controller slot of a flat state, -1
  const unsigned char* kind;   // (total) 1 avoid, 2 target, 0 other
  const int* slot_input;       // (n_ctrl) row of `consts` (policy input)
  const double* consts;        // (n_u, NC) folded constants at (u_j, w_c)
  const double* lb;            // (N) state space
  const double* ub;
  const double* eta;
  const int* counts;
  const double* sigma;         // (N) noise scales
  double* trace;               // (rollouts, steps + 1, N)
  int* length;                 // (rollouts) trace points written
  int* satisfied;              // (rollouts)
  unsigned long long* err;     // first rollout with a non-finite state
};

// grid.py:118-132: nearest representative point, ties to the lower index;
// -1 outside the covered domain (lb - eta/2 - tol, ub + eta/2 + tol)
__device__ long long imp_sim_quantize(const SimParams& P, const double* x) {
  long long flat = 0;
  for (int d = 0; d < IMP_N; ++d) {
    const double half = P.eta[d] / 2;
    const double tol = 1e-9 * (P.eta[d] > 1.0 ? P.eta[d] : 1.0);
    if (x[d] < P.lb[d] - half - tol || x[d] > P.ub[d] + half + tol) return -1;
  }
  for (int d = 0; d < IMP_N; ++d) {
    const double r = (x[d] - P.lb[d]) / P.eta[d];
    double c = ceil(r - 0.5);
    long long idx = (long long)c;
    if (idx < 0) idx = 0;
    if (idx > P.counts[d] - 1) idx = P.counts[d] - 1;
    flat = flat * P.counts[d] + idx;
  }
  return flat;
}

extern "C" __global__ void k_simulate(SimParams P) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.rollouts) return;
  ImpPhilox g;
  {
    const unsigned long long key[2] = {(unsigned long long)r, 0ull};
    unsigned long long s;
    imp_seedseq(P.seed, key, 2, &s, 1);
    imp_philox_seed(&g, s);
  }
  const int k = P.starts[r % P.n_starts];
  double x[IMP_N];
  double* tr = P.trace + (long long)r * (P.steps + 1) * IMP_N;
  for (int d = 0; d < IMP_N; ++d) tr[d] = x[d] = P.coords[(long long)k * IMP_N + d];
  int sat = !P.reach_like, len = 1;
  for (int step = 1; step <= P.steps; ++step) {
    const long long state = imp_sim_quantize(P, x);
    if (state < 0) { sat = 0; break; }
    const int kd = P.kind[state];
    if (kd == 1) { sat = 0; break; }
    if (P.reach_like && kd == 2) { sat = 1; break; }
    const int slot = P.slot_of[state];
    if (slot < 0) { sat = 0; break; }
    const double* K = P.consts + (long long)P.slot_input[slot] * IMP_NC;
    double mean[IMP_N];
    imp_f_all(x, K, mean);
    bool finite = true;
    for (int d = 0; d < IMP_N; ++d) finite &= imp_finite(mean[d]);
    if (!finite) {   // DynamicsSpec.eval raises EvalError
      atomicMin(P.err, (unsigned long long)r);
      break;
    }
    for (int d = 0; d < IMP_N; ++d) {
      const double z = imp_std_normal(&g);
      x[d] = mean[d] + (0.0 + P.sigma[d] * z);   // f(...) + normal(0, sigma)
    }
    for (int d = 0; d < IMP_N; ++d) tr[(long long)len * IMP_N + d] = x[d];
    ++len;
  }
  P.length[r] = len;
  P.satisfied[r] = sat;
}
