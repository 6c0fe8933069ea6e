"""Benchmark: IMDP construction + infinite-horizon interval iteration.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME]
    python bench.py --impl reference ...      (CPU oracle port, host cores)

One step = the hot path of BASELINE.json's north star on one synthetic
batch: build_abstraction of the whole config on the GPU (cutoff-sparse CSR
in HBM) followed by the two-phase synthesis (synthesize_reach /
synthesize_safe / verify) to termination.  Default workload: configs[1],
the 3D autonomous-vehicle reach-avoid IMDP (pkg/benchmarks/vehicle3d.cfg:
166 860 rows x 5 562 columns), which fits one B200.

Reported (one JSON line on rank 0):
  value       IMDP bound entries/s built (rows * n_s / device construction
              time, the reference's `d`, abstraction.py:140-157), all ranks
  sweeps      interval-iteration twin sweeps/s of phase 1 (device time)
  e2e         the same entries/s through the public API (build_abstraction
              + synthesis from host inputs to a host Controller), wall time
  roofline    dominant kernel (k_refine, FP64 Nelder-Mead) vs the measured
              FP64 DFMA peak; roofline_sweep: K5 vs measured HBM copy peak
  cpu_baseline  the oracle port (numpy restatement of the reference) on a
              bounded row sample, 1 host core
Inputs are generated from the config (no dataset); outputs (9.8 GB CSR per
step for vehicle3d) are far larger than L2, so no flush is needed.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = ("IMDP bound entries/sec built; interval-iteration "
                   "sweeps/sec; 1/2/4/8 B200")
DEFAULT_CONFIG = "vehicle3d"


_JSON_FD = None   # original stdout of a sharded run (see run_b200)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def _ncu_traffic(config):
    """DRAM bytes per algorithmic unit from the committed ncu --set full
    captures (profiles/*/ncu_traffic.json, dram__bytes_read.sum +
    dram__bytes_write.sum of one launch / its units), newest round first."""
    base = os.path.join(ROOT, "profiles")
    try:
        rounds = sorted(os.listdir(base), reverse=True)
    except OSError:
        return None
    for r in rounds:
        path = os.path.join(base, r, "ncu_traffic.json")
        if os.path.exists(path):
            with open(path) as fh:
                return json.load(fh).get(config)
    return None


from paper_2401_03555_b200.benchutil import ClockSampler, h2d_bytes as _h2d_bytes  # noqa: E402,F401


# --- algorithmic flop model of one Nelder-Mead objective evaluation ---------

def _dyn_flops(dyn):
    """Arithmetic nodes of the x-dependent residual of every f_d, library
    calls counted as 20 (F_dyn)."""
    from paper_2401_03555_b200.expr import _vars

    def walk(node):
        if not any(v.startswith("x") for v in _vars(node, set())):
            return 0
        tag = node[0]
        if tag == "var":
            return 0
        if tag == "neg":
            return 1 + walk(node[1])
        if tag == "bin":
            return 1 + walk(node[2]) + walk(node[3])
        if tag == "call":
            return 20 + sum(walk(a) for a in node[2])
        return 0
    return sum(walk(e.node) for e in dyn.exprs)


def objective_flops(dyn):
    """F_obj = n * (2 * F_ndtr + 6) + F_dyn, F_ndtr = 50."""
    n = dyn.dims[0]
    return n * (2 * 50 + 6) + _dyn_flops(dyn)


# --- CPU baseline (oracle port) ------------------------------------------------

_ORACLE_CTX = None


def _oracle_init(name):
    """Pool initializer: the oracle's context once per worker process (the
    reference builds its context once per run too, abstraction.py:198-228),
    so steps time row computation only."""
    global _ORACLE_CTX
    from oracle import construct as OC
    from paper_2401_03555_b200.config import benchmark
    cfg = benchmark(name)
    _ORACLE_CTX = OC.make_context(cfg.dynamics, cfg.noise, cfg.spaces,
                                  cfg.labels(), cfg.abstraction_options())


def _oracle_rows(rows):
    from oracle import construct as OC
    t0 = time.perf_counter()
    for r in rows:
        OC.row_bounds(_ORACLE_CTX, int(r))
    return time.perf_counter() - t0


class OraclePool:
    """The oracle port of the reference construction on `procs` host
    processes (fork pool, one row per task like the reference's workers)."""

    def __init__(self, name, procs):
        import multiprocessing
        self.procs = procs
        self.pool = multiprocessing.get_context("fork").Pool(
            procs, initializer=_oracle_init, initargs=(name,))

    def run(self, rows):
        """Wall seconds to build `rows` (split over the processes)."""
        chunks = [rows[p::self.procs] for p in range(self.procs)]
        t0 = time.perf_counter()
        self.pool.map(_oracle_rows, chunks)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(name, n_rows, n_s, rows_sample, procs=1, seed=7):
    """Oracle construction of a seeded row sample; entries/s on `procs`
    host processes (context built once per process, outside the timing)."""
    rng = np.random.default_rng(seed)
    rows = rng.choice(n_rows, size=min(rows_sample * procs, n_rows),
                      replace=False)
    pool = OraclePool(name, procs)
    try:
        pool.run(rows[:procs])          # warm-up (imports, first row)
        dt = pool.run(rows)
    finally:
        pool.close()
    return len(rows) * n_s / dt, dt, len(rows)


def cpu_sweep_baseline(name, n_rows, n_s, rows_sample=4, tile=2000,
                       seed=11):
    """The reference's sweep (RowsSolver.values, feasible.py:80-111, the
    oracle restatement) on REAL rows of the config: `rows_sample` seeded
    rows built by the oracle construction, tiled to `tile` rows, one twin
    sweep (V0 and V1) timed; sweeps/s extrapolated linearly in rows.  One
    process, like the reference's synthesis."""
    from oracle import construct as OC
    from oracle.lp import Rows
    from paper_2401_03555_b200.config import benchmark
    cfg = benchmark(name)
    ctx = OC.make_context(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                          cfg.abstraction_options())
    rng = np.random.default_rng(seed)
    rows = rng.choice(n_rows, size=min(rows_sample, n_rows), replace=False)
    lo, hi = [], []
    for r in rows:
        b = OC.row_bounds(ctx, int(r))
        t_min, t_max, r0, r1, av0, av1, lk0, lk1 = b
        a0 = min(max(lk0 + av0, 0.0), 1.0)
        a1 = min(max(lk1 + av1, 0.0), 1.0)
        lo.append(np.concatenate([np.clip(t_min, 0, 1), [r0, a0]]))
        hi.append(np.concatenate([np.clip(t_max, 0, 1), [r1, a1]]))
    reps = max(1, tile // len(rows))
    solver = Rows(np.tile(np.array(lo), (reps, 1)),
                  np.tile(np.array(hi), (reps, 1)))
    w0 = np.concatenate([rng.uniform(0, 1, n_s), [1.0, 0.0]])
    w1 = np.concatenate([rng.uniform(0, 1, n_s), [1.0, 0.0]])
    t0 = time.perf_counter()
    solver.values(w0, "min")
    solver.values(w1, "min")
    dt = time.perf_counter() - t0
    nrows = reps * len(rows)
    return {"sweeps_per_s": nrows / (n_rows * dt),
            "sample": f"oracle RowsSolver.values twin sweep on {len(rows)} "
                      f"real rows of {name} (oracle construction) tiled to "
                      f"{nrows} rows, {dt * 1e3:.0f} ms, extrapolated "
                      f"linearly to {n_rows} rows; 1 process, as the "
                      f"reference iterates (its process pool serves only "
                      f"the construction, abstraction.py:571-592)"}


# --- the GPU step ---------------------------------------------------------------

def _overrides(args):
    # --horizon: a finite horizon for configs whose infinite-horizon run
    # ends, in the reference too, at the 10^6-iteration cap with a
    # ConvergenceError (room5d); the reference suggests max(k0, k1) or any
    # finite horizon for plain value iteration
    return {"horizon": args.horizon} if args.horizon else {}


def _config(args, cfg, rows_total, n_s):
    """The workload description both arms print (identical keys and
    values, so the driver can match the arms)."""
    return {"workload": args.config, "rows": rows_total, "n_s": n_s,
            "entries": rows_total * n_s, "spec": cfg.spec_type,
            "mode": cfg.mode, "eps": cfg.eps, "horizon": cfg.horizon,
            "step": "build_abstraction + two-phase synthesis"}


def _spec_call(cfg, imdp):
    from paper_2401_03555_b200 import synthesize_reach, synthesize_safe, verify
    kw = dict(mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon,
              max_iterations=cfg.max_iterations)
    if imdp.input_space is None:
        return verify(imdp, spec="safety" if cfg.spec_type == "safety"
                      else "reach", **kw)
    if cfg.spec_type == "safety":
        return synthesize_safe(imdp, **kw)
    return synthesize_reach(imdp, **kw)


def run_b200(args):
    import torch
    from paper_2401_03555_b200 import _lib
    from paper_2401_03555_b200.abstraction import build_abstraction
    from paper_2401_03555_b200.config import benchmark

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # IMP_BENCH_FORCE_SHARDED=1 runs the sharded (multi-GPU) step even at
    # world size 1 (to exercise that path on a single-GPU box)
    sharded_path = world > 1 or os.environ.get("IMP_BENCH_FORCE_SHARDED") == "1"
    if sharded_path:
        import torch.distributed as dist
        # NCCL writes its version banner to fd 1 when the communicator is
        # created: route fd 1 to stderr for the whole run and keep the
        # original stdout for the one JSON line of rank 0
        global _JSON_FD
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local
    cfg = benchmark(args.config, **_overrides(args))
    labels = cfg.labels()
    n_s = len(labels.safe)
    n_u = cfg.input_space.total if cfg.input_space is not None else 1
    n_w = cfg.disturb_space.total if cfg.disturb_space is not None else 1
    rows_total = n_s * n_u * n_w
    if sharded_path:
        return run_sharded(args, cfg, labels, world, rank, device)

    _lib.load()
    from paper_2401_03555_b200.abstraction import exact_default
    imdp_exact = exact_default()
    t_build, t_ph1, t_step_dev, wall, sweeps1, launches = [], [], [], [], [], []
    k5_ph1 = []
    report = None
    ctrl_bytes = 0
    sampler = ClockSampler(device)
    for step in range(args.warmup + args.steps):
        timed = step >= args.warmup
        if step == max(args.warmup - 1, 0):
            sampler.start()     # nvidia-smi start-up stays out of the timing
        if timed and step == args.warmup:
            sampler.mark()
            l0 = _lib.launch_count()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                                 cfg.abstraction_options(), device=device)
        ctrl = _spec_call(cfg, imdp)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        rep = imdp.build_report
        if timed:
            t_build.append(rep.ms_total)
            ms = ctrl.meta["device_ms"]
            t_ph1.append(ms[0])
            k5_ph1.append(ctrl.meta["sweep_ms"][0])
            t_step_dev.append(rep.ms_total + sum(ms))
            wall.append((w1 - w0) * 1e3)
            sweeps1.append(ctrl.meta["iterations"][0])
            report = rep
            ctrl_bytes = sum(a.nbytes for a in (ctrl.p_min, ctrl.p_max)
                             if a is not None)
            if ctrl.policy is not None:
                ctrl_bytes += ctrl.policy.nbytes
        if step < args.warmup + args.steps - 1:
            del imdp
    clocks = sampler.stop()
    l1 = _lib.launch_count()
    launches = l1[0] - l0[0]

    entries = rows_total * n_s
    ms_build = float(np.mean(t_build))
    ms_step = float(np.mean(t_step_dev))
    value = entries / (ms_build * 1e-3)
    sweeps_per_s = float(np.mean([s / (t * 1e-3) for s, t in
                                  zip(sweeps1, t_ph1)]))
    e2e = entries / (float(np.mean(wall)) * 1e-3)

    # K5 alone for the HBM roofline; FP64 peak microbenchmark
    spec = _lib.SPEC_SAFETY if cfg.spec_type == "safety" else _lib.SPEC_REACH
    lp = (_lib.LP_MAX if cfg.spec_type == "safety" else _lib.LP_MIN)
    ms_sweep = _lib.c_dbl(0)
    _lib.check(_lib.load().imp_time_sweep(imdp.device_handle().raw, spec, lp,
                                          10, ms_sweep))
    nnz = report.nnz
    sweep_bytes = nnz * 20 + rows_total * (5 * 8) + (n_s + 1) * 8
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs")
    hbm_note = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm:
        hbm, hbm_note = 6650.0, "fallback (B200_PROFILING.md)"
    sweep_gbs = sweep_bytes / (ms_sweep.value * 1e-3) / 1e9
    fp64_peak = _lib.fp64_peak_gflops(device) / 1e3  # TFLOP/s
    f_obj = objective_flops(cfg.dynamics)
    # roofline of the construction stage that dominates this config:
    # coupled dynamics -> k_refine (FP64 Nelder-Mead); separable -> the
    # CSR writer (k_outer_sep, HBM writes of 20 B per stored entry)
    stage_ms = {"refine": report.ms_refine, "outer": report.ms_outer,
                "mean_ranges": report.ms_mean_ranges,
                "assemble": report.ms_assemble}
    top = max(stage_ms, key=stage_ms.get)
    if top == "refine" and report.nm_evals:
        refine_tflops = report.nm_evals * f_obj / (report.ms_refine * 1e-3) / 1e12
        roofline = {
            "kernel": "k_refine", "bound": "fp64",
            "achieved": refine_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": refine_tflops / fp64_peak, "traffic": None,
            "flops_per_eval": f_obj, "evals_per_step": report.nm_evals,
            "kernel_ms": report.ms_refine,
            "peak_source": "measured DFMA microbenchmark (imp_fp64_peak: "
                           "dependent DFMA chains on every SM, CUDA events; "
                           "2 flops/DFMA; MEASURED_PEAKS.json has no FP64 "
                           "entry and B200_PROFILING.md no FP64 fallback)",
        }
    elif top == "mean_ranges" and report.nm_evals_mean:
        # mean ranges dominate (bas7d: the lattice probabilities vanish
        # under the cutoff, so there is almost nothing to refine or write):
        # Nelder-Mead over each dynamics component, FP64 flops = evals x
        # (the component's share of F_dyn)
        f_comp = max(_dyn_flops(cfg.dynamics), 1) / cfg.dynamics.dims[0]
        mean_tflops = report.nm_evals_mean * f_comp / \
            (report.ms_mean_ranges * 1e-3) / 1e12
        roofline = {
            "kernel": "k_mean_ranges", "bound": "fp64",
            "achieved": mean_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": mean_tflops / fp64_peak, "traffic": None,
            "flops_per_eval": f_comp,
            "evals_per_step": report.nm_evals_mean,
            "kernel_ms": report.ms_mean_ranges,
            "peak_source": "measured DFMA microbenchmark (imp_fp64_peak)",
            "note": "one dynamics component per evaluation: the kernel is "
                    "Nelder-Mead bookkeeping (sort, centroid, accept) bound, "
                    "not FP64-throughput bound",
        }
    else:
        out_bytes = nnz * 20 + rows_total * (8 + 48)
        gbs = out_bytes / (report.ms_outer * 1e-3) / 1e9
        roofline = {
            "kernel": "k_outer_sep" if cfg.dynamics.is_separable() else
                      "k_outer",
            "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
            "frac": gbs / hbm, "traffic": None,
            "bytes_per_build": out_bytes, "kernel_ms": report.ms_outer,
            "peak_source": hbm_note,
            "note": "CSR written by the count + write passes (20 B per "
                    "stored entry, 56 B per row) over both passes' time",
        }
    # K5 measured live in the timed steps: CUDA-graph event nodes around
    # every phase-1 iteration's K5 launches (moved-crossing passes and
    # searches included), averaged per sweep
    k5_ms = float(np.sum(k5_ph1)) / max(float(np.sum(sweeps1)), 1.0)
    live_gbs = sweep_bytes / (k5_ms * 1e-3) / 1e9 if k5_ms > 0 else None
    # the same bytes over the whole in-loop iteration (order keys, sorts,
    # ranks, K5, Bellman, control)
    loop_gbs = sweep_bytes * sweeps_per_s / 1e9
    traffic = _ncu_traffic(args.config)
    roofline_sweep = {
        "kernel": "k_sweep", "bound": "hbm", "achieved": live_gbs,
        "peak": hbm, "unit": "GB/s",
        "frac": live_gbs / hbm if live_gbs else None,
        "traffic": (traffic["k_sweep_bytes_per_entry"] * nnz
                    if traffic and "k_sweep_bytes_per_entry" in traffic
                    else None),
        "bytes_per_sweep": sweep_bytes, "kernel_ms": k5_ms,
        "peak_source": hbm_note,
        "note": "K5 timed live over the timed steps' phase-1 iterations",
        "settled": {"gbs": sweep_gbs, "frac": sweep_gbs / hbm,
                    "kernel_ms": ms_sweep.value,
                    "note": "K5 alone with every row's crossing settled "
                            "(imp_time_sweep, repeated sweeps of one order)"},
        "in_loop": {"gbs": loop_gbs, "frac": loop_gbs / hbm,
                    "note": "phase-1 iterations of the timed steps: same "
                            "algorithmic bytes over the full iteration time"},
    }
    if traffic and "k_refine_fp64_pipe_pct" in traffic:
        roofline["ncu_fp64_pipe_active_pct"] = traffic["k_refine_fp64_pipe_pct"]
        roofline["note"] = ("algorithmic flops (SURVEY.md 8d) over the DFMA "
                            "peak; bit parity keeps cephes' Horner steps as "
                            "unfused DMUL + DADD, so the FP64 pipe (ncu) is "
                            "busier than the algorithmic fraction shows")
    if traffic and "k_refine_dram_bytes_per_eval" in traffic:
        roofline["traffic"] = traffic["k_refine_dram_bytes_per_eval"] * \
            report.nm_evals

    cpu = None
    if not args.no_cpu_baseline:
        cpu_v, cpu_dt, cpu_rows = cpu_baseline(args.config, rows_total, n_s,
                                               args.cpu_rows, procs=1)
        cpu_sw = cpu_sweep_baseline(args.config, rows_total, n_s)
        cpu = {"value": cpu_v, "unit": "entries/s", "cores": 1,
               "kind": "port",
               "sample": f"{cpu_rows} seeded rows of {args.config} through "
                         f"oracle/construct.py (numpy restatement of the "
                         f"reference, scipy ndtr) in {cpu_dt:.1f} s",
               "sweeps_per_s": cpu_sw["sweeps_per_s"],
               "sweeps_sample": cpu_sw["sample"]}

    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "entries/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": _config(args, cfg, rows_total, n_s),
        "nnz": nnz,
        "l2": "outputs/inputs >> L2 (CSR %.1f GB)" % (nnz * 20 / 1e9),
        "parallelism": "rows of every state on 1 GPU",
        "construction": "exact (bit-identical objective)" if
                        imdp_exact else "fast objective (exact=False)",
        "sweeps_per_s": sweeps_per_s,
        "phase1_sweeps": int(sweeps1[-1]),
        "ms_build": ms_build, "ms_phase1": float(np.mean(t_ph1)),
        "build_stages_ms": {"mean_ranges": report.ms_mean_ranges,
                            "outer": report.ms_outer,
                            "refine": report.ms_refine,
                            "assemble": report.ms_assemble},
        "e2e": {"value": e2e, "unit": "entries/s",
                "h2d_bytes_per_step": _h2d_bytes(cfg, labels),
                "d2h_bytes_per_step": int(ctrl_bytes),
                "ms_per_step_wall": float(np.mean(wall))},
        "roofline": roofline, "roofline_sweep": roofline_sweep,
        "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": int(launches),
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, cfg, labels, world, rank, device):
    import torch.distributed as dist
    from paper_2401_03555_b200 import sharded
    line = sharded.bench_step(args, cfg, labels, world, rank, device)
    if rank == 0 and line is not None:
        sys.stdout.flush()
        os.write(_JSON_FD if _JSON_FD is not None else 1,
                 (json.dumps(line) + "\n").encode())
    dist.destroy_process_group()


# --- reference arm ---------------------------------------------------------------

def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2401_03555_b200.config import benchmark
    cfg = benchmark(args.config, **_overrides(args))
    labels = cfg.labels()
    n_s = len(labels.safe)
    n_u = cfg.input_space.total if cfg.input_space is not None else 1
    n_w = cfg.disturb_space.total if cfg.disturb_space is not None else 1
    rows_total = n_s * n_u * n_w
    procs = len(os.sched_getaffinity(0))
    pool = OraclePool(args.config, procs)
    rng = np.random.default_rng(100)
    try:
        # rows per process per step: enough for ~2 s of work (>= 1)
        probe = rng.choice(rows_total, size=procs, replace=False)
        pool.run(probe)                        # imports, first rows
        per_row = pool.run(probe)              # one row per process
        per_proc = int(max(1, min(256, 2.0 / max(per_row, 1e-6))))
        vals, dts = [], []
        for step in range(args.warmup + args.steps):
            rows = rng.choice(rows_total, size=min(per_proc * procs,
                                                   rows_total),
                              replace=False)
            dt = pool.run(rows)
            if step >= args.warmup:
                vals.append(len(rows) * n_s / dt)
                dts.append(dt)
    finally:
        pool.close()
    nrows = per_proc * procs
    value = float(np.mean(vals))
    sw = cpu_sweep_baseline(args.config, rows_total, n_s)
    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "entries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(dts)) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": _config(args, cfg, rows_total, n_s),
        "sweeps_per_s": sw["sweeps_per_s"],
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": procs,
                         "kind": "port",
                         "sample": f"{nrows} seeded rows per step "
                                   f"({per_proc} per host core, fork pool, "
                                   "contexts built once) through the oracle "
                                   "port of the reference construction",
                         "sweeps_per_s": sw["sweeps_per_s"],
                         "sweeps_sample": sw["sample"]},
        "e2e": {"value": value, "unit": "entries/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--cpu-rows", type=int, default=3)
    ap.add_argument("--horizon", type=int, default=0,
                    help="finite horizon (0: the config's, infinite)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
