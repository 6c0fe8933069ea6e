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

def _oracle_rows_worker(args):
    name, rows = args
    from oracle import construct as OC
    from paper_2401_03555_b200.config import benchmark
    cfg = benchmark(name)
    ctx = OC.make_context(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                          cfg.abstraction_options())
    t0 = time.perf_counter()
    for r in rows:
        OC.row_bounds(ctx, int(r))
    return time.perf_counter() - t0


def cpu_baseline(name, n_rows, n_s, rows_sample, procs=1, seed=7):
    """Oracle construction of a seeded row sample; entries/s on `procs`
    host processes (each process one row at a time, like the reference's
    fork pool)."""
    import multiprocessing
    rng = np.random.default_rng(seed)
    rows = rng.choice(n_rows, size=rows_sample * procs, replace=False)
    chunks = [(name, rows[p::procs]) for p in range(procs)]
    t0 = time.perf_counter()
    if procs == 1:
        _oracle_rows_worker(chunks[0])
    else:
        with multiprocessing.get_context("fork").Pool(procs) as pool:
            pool.map(_oracle_rows_worker, chunks)
    dt = time.perf_counter() - t0
    return len(rows) * n_s / dt, dt, len(rows)


def cpu_sweep_baseline(n_rows, n_s, live, sample=2000, seed=7):
    """Oracle RowsSolver (feasible.py:80-111 restated) twin sweep on a
    sample of synthetic Dirichlet rows of the config's width and sparsity;
    sweeps/s extrapolated linearly in rows."""
    from oracle.lp import Rows
    rng = np.random.default_rng(seed)
    width = n_s + 2
    lo = np.zeros((sample, width))
    hi = np.zeros((sample, width))
    k = max(1, min(width, int(live)))
    for r in range(sample):
        cols = rng.choice(width, size=k, replace=False)
        q = rng.dirichlet(np.ones(k))
        lo[r, cols] = 0.8 * q
        hi[r, cols] = np.minimum(1.0, 1.3 * q + 1e-4)
    rows = Rows(lo, hi)
    w0 = rng.uniform(0, 1, width)
    w1 = rng.uniform(0, 1, width)
    t0 = time.perf_counter()
    rows.values(w0, "min")
    rows.values(w1, "min")
    dt = time.perf_counter() - t0
    return sample / (n_rows * dt)


# --- the GPU step ---------------------------------------------------------------

def _overrides(args):
    # --horizon: a finite horizon for configs whose infinite-horizon run
    # ends, in the reference too, at the 10^6-iteration cap with a
    # ConvergenceError (room5d); the reference suggests max(k0, k1) or any
    # finite horizon for plain value iteration
    return {"horizon": args.horizon} if args.horizon else {}


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
            "peak_source": "measured DFMA microbenchmark (imp_fp64_peak), "
                           "2 flops/DFMA",
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
        cpu_sw = cpu_sweep_baseline(rows_total, n_s, nnz / rows_total)
        cpu = {"value": cpu_v, "unit": "entries/s", "cores": 1,
               "kind": "port",
               "sample": f"{cpu_rows} seeded rows of {args.config} through "
                         f"oracle/construct.py (numpy restatement of the "
                         f"reference, scipy ndtr) in {cpu_dt:.1f} s",
               "sweeps_per_s": cpu_sw,
               "sweeps_sample": "oracle Rows.values twin sweep on 2000 "
                                "synthetic rows of the same width/sparsity, "
                                "extrapolated linearly in rows"}

    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "entries/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "rows": rows_total, "n_s": n_s,
                   "entries": entries, "nnz": nnz,
                   "spec": cfg.spec_type, "mode": cfg.mode, "eps": cfg.eps,
                   "horizon": cfg.horizon,
                   "step": "build_abstraction + two-phase synthesis",
                   "l2": "outputs/inputs >> L2 (CSR %.1f GB)" % (
                       nnz * 20 / 1e9),
                   "parallelism": "rows sharded by state (1 GPU)"},
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
    vals, dts = [], []
    for step in range(args.warmup + args.steps):
        v, dt, nrows = cpu_baseline(args.config, rows_total, n_s, 1,
                                    procs=procs, seed=100 + step)
        if step >= args.warmup:
            vals.append(v)
            dts.append(dt)
    value = float(np.mean(vals))
    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": "entries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(dts)) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.config, "rows": rows_total, "n_s": n_s,
                   "entries": rows_total * n_s},
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": procs,
                         "kind": "port",
                         "sample": f"{procs} seeded rows per step (one per "
                                   "host core, fork pool) through the oracle "
                                   "port of the reference construction"},
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
