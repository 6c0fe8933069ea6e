"""Multi-GPU interval iteration: safe states sharded across ranks.

SURVEY.md 8(e): rows are sharded by contiguous blocks of source states, so
construction needs no communication (each rank builds its shard into its
own HBM, `build_abstraction(..., k_range=...)`) and the min over
disturbances / max over inputs stays local.  Every sweep each rank prices
its rows against the full value vectors, then
  1. all-gather of the new V0' / V1' shards (one NCCL all_gather_into_tensor
     over NVLink per track), and
  2. all-reduce(max) of [max|dV0|, max|dV1|, gap, monotone, bracket].
Every rank then runs the same termination logic (the reference's
_run_phase, synthesis.py:145-205) on identical numbers, so all ranks stop at
the same iteration.  Max is the only cross-rank floating-point reduction and
it is exact, so results are bitwise independent of the rank count.

The per-shard sweep is an engine object: CudaShard calls the C-ABI
(imp_shard_sweep) on the rank's GPU; tests substitute a CPU engine to cover
the exchange and control logic with gloo on world_size 2.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConvergenceError, ImpactError

__all__ = ["shard_range", "CudaShard", "run_phase", "synthesize",
           "bench_step"]


def shard_range(n_s, world, rank):
    """Contiguous block of safe states for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_s, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


class CudaShard:
    """One rank's shard on its GPU; device tensors are torch (plumbing)."""

    def __init__(self, imdp, device):
        import torch
        self.torch = torch
        self.imdp = imdp
        info = imdp.device_handle().info()
        self.k_begin, self.k_count = info.k_begin, info.k_count
        self.n_s, self.n_u, self.n_w = info.n_s, info.n_u, info.n_w
        self.device = torch.device("cuda", device)
        kc = max(self.k_count, 1)
        self.new0 = torch.empty(kc, dtype=torch.float64, device=self.device)
        self.new1 = torch.empty_like(self.new0)
        self.pol = torch.empty(kc, dtype=torch.int64, device=self.device)
        self.stats = torch.empty(5, dtype=torch.float64, device=self.device)
        self.fixed = None

    def set_policy(self, local_policy):
        t = self.torch
        self.fixed = None if local_policy is None else t.as_tensor(
            np.ascontiguousarray(local_policy, dtype=np.int64),
            device=self.device)

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64,
                                device=self.device)

    def ones(self, n):
        return self.torch.ones(n, dtype=self.torch.float64,
                               device=self.device)

    def sweep(self, v0, v1, spec, lp, u_max):
        stream = self.torch.cuda.current_stream(self.device).cuda_stream
        fixed = self.fixed.data_ptr() if self.fixed is not None else None
        _lib.check(_lib.load().imp_shard_sweep(
            self.imdp.device_handle().raw, v0.data_ptr(), v1.data_ptr(),
            spec, lp, u_max, fixed, self.new0.data_ptr(),
            self.new1.data_ptr(), self.pol.data_ptr(),
            self.stats.data_ptr(), ctypes.c_void_p(stream)))
        k = self.k_count
        return self.new0[:k], self.new1[:k], self.pol[:k], self.stats


@dataclass
class ShardedPhase:
    v0: object
    v1: object
    policy: np.ndarray
    iterations: int
    k0: int | None
    k1: int | None
    fallback: bool
    gap: float


def _gather(dist, local, n_total, world, counts, like_fn):
    """All-gather variable-size contiguous shards into one vector."""
    import torch
    width = max(counts)
    buf = like_fn(width)
    buf[:local.shape[0]] = local
    out = torch.empty(world * width, dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(out, buf)
    parts = [out[r * width:r * width + counts[r]] for r in range(world)]
    return torch.cat(parts)[:n_total]


def run_phase(engine, dist, spec, lp, u_obj, eps, horizon, max_iterations,
              fixed_policy=None):
    """One reference phase (synthesis.py:145-205) over all ranks."""
    import torch
    world = dist.get_world_size()
    rank = dist.get_rank()
    n_s = engine.n_s
    counts = [shard_range(n_s, world, r)[1] for r in range(world)]
    b0, kc = shard_range(n_s, world, rank)
    assert (b0, kc) == (engine.k_begin, engine.k_count), "shard mismatch"
    engine.set_policy(None if fixed_policy is None
                      else np.asarray(fixed_policy)[b0:b0 + kc])
    spec_c = _lib.SPEC_REACH if spec == "reach" else _lib.SPEC_SAFETY
    lp_c = _lib.LP_MAX if lp == "max" else _lib.LP_MIN
    u_max = 1 if u_obj == "max" else 0
    v0, v1 = engine.zeros(n_s), engine.ones(n_s)
    k0 = k1 = None
    prev = None
    it = 0
    while True:
        it += 1
        n0, n1, pol, st = engine.sweep(v0, v1, spec_c, lp_c, u_max)
        st = st.clone()
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        # the gathers are queued before the host reads the statistics, so
        # their launches overlap the sweep instead of following the sync
        v0 = _gather(dist, n0, n_s, world, counts, engine.zeros)
        v1 = _gather(dist, n1, n_s, world, counts, engine.zeros)
        d0, d1, gap, mono, brk = (float(x) for x in st.cpu().tolist())
        if mono > 0:
            raise ImpactError("value iterates lost monotonicity; "
                              "abstraction bounds inconsistent")
        if k0 is None and d0 <= eps:
            k0 = it
        if k1 is None and d1 <= eps:
            k1 = it
        if brk > 0:
            raise ImpactError("interval iteration bracket violated (v0 > v1);"
                              " abstraction bounds inconsistent")
        done = fallback = False
        if horizon is not None:
            done = it >= horizon
        elif gap <= eps:
            done = True
        else:
            stalled = prev is not None and prev - gap <= 1e-15 * max(1.0, gap)
            if k0 is not None and k1 is not None and stalled:
                done = fallback = True
            else:
                prev = gap
                if it >= max_iterations:
                    rk = (lambda k: None if k is None else max(k - 1, 1))
                    raise ConvergenceError(
                        f"gap {gap!r} above eps={eps!r} after {it} "
                        "iterations", k0=rk(k0), k1=rk(k1))
        if done:
            polf = _gather(dist, pol.to(torch.float64), n_s, world, counts,
                           engine.zeros)
            return ShardedPhase(v0, v1, polf.cpu().numpy().astype(np.int64),
                                it, k0, k1, fallback, gap)


def synthesize(engine, dist, spec, mode="pessimistic", eps=1e-6, horizon=None,
               max_iterations=10**6):
    """Two-phase synthesis over shards (synthesis.py:238-303): returns
    (p_min, p_max, policy, iterations, fallback) on every rank."""
    if spec == "reach":
        lp1 = "min" if mode == "pessimistic" else "max"
        u_obj = "max"
    else:
        lp1 = "max" if mode == "pessimistic" else "min"
        u_obj = "min"
    lp2 = "max" if lp1 == "min" else "min"
    ph1 = run_phase(engine, dist, spec, lp1, u_obj, eps, horizon,
                    max_iterations)
    ph2 = run_phase(engine, dist, spec, lp2, u_obj, eps, horizon,
                    max_iterations, fixed_policy=ph1.policy)

    def track(ph, lp):
        if horizon is not None or ph.fallback:
            return ph.v0
        if spec == "reach":
            return ph.v0 if lp == "min" else ph.v1
        return ph.v0 if lp == "max" else ph.v1

    a = track(ph1, lp1).cpu().numpy()
    b = track(ph2, lp2).cpu().numpy()
    if spec == "reach":
        p_min, p_max = (a, b) if lp1 == "min" else (b, a)
    else:
        p_min, p_max = (1.0 - a, 1.0 - b) if lp1 == "max" else \
            (1.0 - b, 1.0 - a)
    return (p_min, np.maximum(p_min, p_max), ph1.policy,
            (ph1.iterations, ph2.iterations), (ph1.fallback, ph2.fallback))


def _h2d(cfg, labels):
    from .benchutil import h2d_bytes
    return h2d_bytes(cfg, labels)


def bench_step(args, cfg, labels, world, rank, device):
    """bench.py at N > 1: each rank builds its shard, then the sharded
    two-phase synthesis.  Device time (CUDA events on the launching stream,
    max over ranks) with a barrier + synchronize around every timed step;
    e2e is the same step through the public API from host inputs to the
    host controller (wall time, max over ranks)."""
    import time
    import torch
    import torch.distributed as dist
    from .abstraction import build_abstraction
    n_s = len(labels.safe)
    n_u = cfg.input_space.total if cfg.input_space is not None else 1
    n_w = cfg.disturb_space.total if cfg.disturb_space is not None else 1
    k_range = shard_range(n_s, world, rank)
    spec = "safety" if cfg.spec_type == "safety" else "reach"
    builds, synths, sweeps, walls = [], [], [], []
    sampler = None
    if rank == 0:
        from .benchutil import ClockSampler
        sampler = ClockSampler(device)
    l0 = None
    ctrl_bytes = 0
    for step in range(args.warmup + args.steps):
        timed = step >= args.warmup
        if sampler and step == max(args.warmup - 1, 0):
            sampler.start()     # nvidia-smi start-up stays out of the timing
        if timed and l0 is None:
            if sampler:
                sampler.mark()
            l0 = _lib.launch_count()
        dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                                 cfg.abstraction_options(), device=device,
                                 k_range=k_range)
        eng = CudaShard(imdp, device)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e1.record()
        res = synthesize(eng, dist, spec, cfg.mode, cfg.eps, cfg.horizon,
                         cfg.max_iterations)
        e2.record()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        if timed:
            builds.append(imdp.build_report.ms_total)
            synths.append(e1.elapsed_time(e2))
            sweeps.append(res[3][0])
            walls.append((w1 - w0) * 1e3)
            ctrl_bytes = sum(np.asarray(a).nbytes for a in res[:3]
                             if a is not None)
        if step < args.warmup + args.steps - 1:
            del eng, imdp   # the next build reuses the pooled CSR blocks
    l1 = _lib.launch_count()
    clocks = sampler.stop() if sampler else None
    mx = torch.tensor([np.mean(builds), np.mean(synths), np.mean(walls)],
                      dtype=torch.float64, device=torch.device("cuda", device))
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms_build, ms_synth, ms_wall = (float(x) for x in mx.cpu().tolist())
    entries = n_s * n_u * n_w * n_s
    if rank != 0:
        return None
    return {
        "metric": "IMDP bound entries/sec built; interval-iteration "
                  "sweeps/sec; 1/2/4/8 B200",
        "value": entries / (ms_build * 1e-3), "unit": "entries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_build + ms_synth, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.config, "rows": n_s * n_u * n_w,
                   "n_s": n_s, "entries": entries, "horizon": cfg.horizon,
                   "step": "build_abstraction (shard) + two-phase synthesis",
                   "parallelism": f"states sharded over {world} ranks; V "
                                  "all-gathered per sweep (NCCL)"},
        "sweeps_per_s": float(np.mean(sweeps)) / (ms_synth * 1e-3),
        "ms_build": ms_build, "ms_synthesis": ms_synth,
        "e2e": {"value": entries / (ms_wall * 1e-3), "unit": "entries/s",
                "h2d_bytes_per_step": _h2d(cfg, labels),
                "d2h_bytes_per_step": int(ctrl_bytes),
                "ms_per_step_wall": ms_wall},
        "clocks": clocks,
        "gpu_launches": int(l1[0] - l0[0]),
    }
