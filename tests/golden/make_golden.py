"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

TEST INFRASTRUCTURE ONLY.  This script imports the reference package
(`impact`, /root/reference/pkg/src) read-only, runs its own public API and
row-level internals on the benchmark configs and on reduced "mini" grids,
and writes small compressed .npz fixtures.  Nothing at run time (tests on the
GPU box, smoke(), bench.py) reads /root/reference; they read these files.

Usage:  python tests/golden/make_golden.py [--only NAME ...] [--workers 8]

Fixture kinds
  ndtr.npz            scipy.special.ndtr on a spread of points (noise.py:116-118)
  pairwise.npz        np.sum (numpy pairwise) on odd lengths (abstraction.py:506)
  rows_<cfg>.npz      seeded row samples of a full benchmark config:
                      raw _compute_one_row outputs (abstraction.py:430-508) and
                      the same rows after _assemble (abstraction.py:607-659)
  full_<cfg>.npz      full reference abstraction (sparse) + synthesis/verify
                      controller, iteration counts, phase-1 top-2 margins
"""

import argparse
import multiprocessing
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))

import impact  # noqa: E402
from impact import abstraction as A  # noqa: E402
from impact import synthesis as S  # noqa: E402
from impact.config import load_config  # noqa: E402
from impact.errors import ConvergenceError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# Reduced grids of the BASELINE.json config families (same dynamics, noise
# and predicates as pkg/benchmarks/*.cfg, coarser lattices) so the reference
# can build and synthesize them in full within minutes.
MINI = {
    "robot2d_ra_mini": """
[state]
lb = -10 -10
ub = 10 10
eta = 2 2
[input]
lb = -1 -1
ub = 1 1
eta = 0.5 0.5
[dynamics]
f1 = x1 + 10*u1*cos(u2)
f2 = x2 + 10*u2*sin(u2)
[noise]
type = diagonal
sigma = 0.8660254037844386 0.8660254037844386
[spec]
type = reach-avoid
target = (x1 >= 5) & (x1 <= 7) & (x2 >= 5) & (x2 <= 7)
avoid = (x1 >= -2) & (x1 <= 2) & (x2 >= -2) & (x2 <= 2)
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = infinite
""",
    "vehicle3d_mini": """
[state]
lb = -5 -5 -3.4
ub = 5 5 3.4
eta = 2 2 1.7
[input]
lb = -1 -0.4
ub = 4 0.4
eta = 2.5 0.4
[dynamics]
f1 = x1 + (u1*cos(atan(tan(u2)/2) + x3)/cos(atan(tan(u2)/2)))*0.1
f2 = x2 + (u1*sin(atan(tan(u2)/2) + x3)/cos(atan(tan(u2)/2)))*0.1
f3 = x3 + (u1*tan(u2))*0.1
[noise]
type = diagonal
sigma = 0.81649658092772603 0.81649658092772603 0.81649658092772603
[spec]
type = reach-avoid
target = (x1 >= -5.75) & (x1 <= 0.25) & (x2 >= -0.25) & (x2 <= 5.75) & (x3 >= -3.45) & (x3 <= 3.45)
avoid = (x1 >= -5.75) & (x1 <= 0.25) & (x2 >= -3.5) & (x2 <= -0.25) & (x3 >= -3.45) & (x3 <= 3.45)
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = infinite
""",
    "room5d_mini": """
[state]
lb = 19 19 19 19 19
ub = 21 21 21 21 21
eta = 1 1 1 1 1
[input]
lb = 0 0
ub = 1 1
eta = 0.5 0.5
[dynamics]
f1 = (0.378 - 0.05*u1)*x1 + 0.3*(x2 + x5) + 2.5*u1 - 0.022
f2 = 0.378*x2 + 0.3*(x1 + x3) - 0.022
f3 = (0.378 - 0.05*u2)*x3 + 0.3*(x4 + x2) + 2.5*u2 - 0.022
f4 = 0.378*x4 + 0.3*(x3 + x5) - 0.022
f5 = 0.378*x5 + 0.3*(x4 + x1) - 0.022
[noise]
type = diagonal
sigma = 0.1 0.1 0.1 0.1 0.1
[spec]
type = safety
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = infinite
""",
    "bas4d_mini": """
[state]
lb = 19 19 30 30
ub = 21 21 36 36
eta = 1 1 2 2
[input]
lb = 17
ub = 20
eta = 1.0
[dynamics]
f1 = 0.6682*x1 + 0.02632*x3 + 0.1320*u1 + 3.4378
f2 = 0.683*x2 + 0.02096*x4 + 0.1402*u1 + 2.9272
f3 = 1.0005*x1 - 0.000499*x3 + 13.0207
f4 = 0.8004*x2 + 0.1996*x4 + 10.4166
[noise]
type = diagonal
sigma = 3.5944262407232674 3.5944262407232674 1.6070469812671937 1.796635744941083
[spec]
type = safety
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = infinite
""",
    "dim6_mini": """
[state]
lb = -0.5 -0.5 -0.5 -0.5 -0.5 -0.5
ub = 0.5 0.5 0.5 0.5 0.5 0.5
eta = 1 1 1 1 1 1
[dynamics]
f1 = 0.8*x1
f2 = 0.8*x2
f3 = 0.8*x3
f4 = 0.8*x4
f5 = 0.8*x5
f6 = 0.8*x6
[noise]
type = diagonal
sigma = 0.2 0.2 0.2 0.2 0.2 0.2
[spec]
type = safety
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = 40
""",
    "bas7d_mini": """
[state]
lb = -0.5 -0.5 -0.5 -0.5 -0.5 -0.5 -0.5
ub = 0.5 0.5 0.5 0.5 0.5 0.5 0.5
eta = 0.5 0.5 1 1 1 1 1
[dynamics]
f1 = 0.968*x1 + 0.004*x3 + 0.004*x5 + 0.004*x7
f2 = 0.968*x2 + 0.003*x4 + 0.003*x6 + 0.003*x7
f3 = 0.011*x1 + 0.949*x3
f4 = 0.010*x2 + 0.952*x4
f5 = 0.011*x1 + 0.949*x5
f6 = 0.010*x2 + 0.952*x6
f7 = 0.011*x1 + 0.010*x2 + 0.979*x7
[noise]
type = diagonal
sigma = 0.7162401831787993 0.7071067811865476 0.4669047011971501 0.4847679857416329 0.5019960159204453 0.5147815070493500 0.9576011695899289
[spec]
type = safety
[synthesis]
policy = pessimistic
epsilon = 1e-6
horizon = infinite
""",
    "robot2d_reach": None,     # the full benchmark config, built in full
}

# Full-size benchmark configs sampled row-wise (BASELINE.json configs 1-5).
# The first count is the seeded uniform draw (kept from round 1 so earlier
# rows stay in the fixtures); STRATA adds stratified rows on top.
SAMPLES = {
    "robot2d_reachavoid": 96,
    "vehicle3d": 12,
    "room5d": 12,
    "bas7d_verify": 24,
    "dim14_verify": 8,
    "robot2d_reach": 64,
}
# Stratified extra rows per config: boundary states (a coordinate on the
# grid's edge), states next to a target / avoid state, and random interior
# states, with the input index cycling so every input appears.
STRATA = {
    "vehicle3d": 72,
    "room5d": 64,
    "bas7d_verify": 48,
}


def cfg_text(name):
    if MINI.get(name):
        return MINI[name].strip() + "\n"
    with open(os.path.join(REF, "benchmarks", name + ".cfg")) as fh:
        return fh.read()


def load(name):
    path = os.path.join("/tmp", f"golden_{name}.cfg")
    with open(path, "w") as fh:
        fh.write(cfg_text(name))
    return load_config(path)


def sparse_rows(t_min, t_max):
    """CSR of the entries where either bound is nonzero."""
    ptr = [0]
    cols, lo, hi = [], [], []
    for r in range(t_min.shape[0]):
        nz = np.nonzero((t_min[r] != 0) | (t_max[r] != 0))[0]
        cols.append(nz)
        lo.append(t_min[r, nz])
        hi.append(t_max[r, nz])
        ptr.append(ptr[-1] + len(nz))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs
           else np.zeros(0, dt))
    return (np.asarray(ptr, np.int64), cat(cols, np.int32),
            cat(lo, np.float64), cat(hi, np.float64))


# --- row samples -----------------------------------------------------------

_CTX = None


def _one_row(row):
    k, j, i = A.RowIndex(_CTX.n_u, _CTX.n_w).kji(row)
    return A._compute_one_row(_CTX, row, k, j, i)


def stratified_rows(space, labels, n_u, n_w, n, seed):
    """n rows: a third boundary states, a third states with a target / avoid
    neighbour (one lattice step in one dimension), the rest random; input
    index cycling over all inputs, disturbance index random."""
    rng = np.random.default_rng(seed)
    counts = np.asarray(space.counts, dtype=np.int64)
    safe = np.asarray(labels.safe, dtype=np.int64)
    multi = np.stack(np.unravel_index(safe, tuple(counts)), axis=1)
    edge = np.any((multi == 0) | (multi == counts - 1), axis=1)
    special = np.zeros(space.total, dtype=bool)
    special[np.asarray(labels.target, dtype=np.int64)] = True
    special[np.asarray(labels.avoid, dtype=np.int64)] = True
    near = np.zeros(len(safe), dtype=bool)
    for d in range(len(counts)):
        for step in (-1, 1):
            m = multi.copy()
            m[:, d] += step
            ok = (m[:, d] >= 0) & (m[:, d] < counts[d])
            flat = np.ravel_multi_index(tuple(np.clip(m, 0, counts - 1).T),
                                        tuple(counts))
            near |= ok & special[flat]
    pools = [np.flatnonzero(edge), np.flatnonzero(near),
             np.arange(len(safe))]
    per = [n // 3, n // 3, n - 2 * (n // 3)]
    ks = []
    for pool, c in zip(pools, per):
        if len(pool) == 0:
            pool = pools[2]
        ks.append(rng.choice(pool, size=min(c, len(pool)), replace=False))
    ks = np.concatenate(ks)
    js = (rng.integers(n_u) + np.arange(len(ks))) % n_u
    iw = rng.integers(n_w, size=len(ks))
    return (ks * n_u + js) * n_w + iw


def make_rows(name, nsamp, workers):
    global _CTX
    cfg = load(name)
    labels = cfg.labels()
    spaces = (cfg.state_space, cfg.input_space, cfg.disturb_space)
    opts = cfg.abstraction_options()
    ctx = A._make_context(cfg.dynamics, cfg.noise, spaces, labels, opts)
    n_rows = len(labels.safe) * ctx.n_u * ctx.n_w
    rng = np.random.default_rng(1)
    rows = np.sort(rng.choice(n_rows, size=min(nsamp, n_rows), replace=False))
    extra = np.zeros(0, np.int64)
    if STRATA.get(name):
        extra = stratified_rows(cfg.state_space, labels, ctx.n_u, ctx.n_w,
                                STRATA[name], seed=2)
    # always include the first and last row (boundary cells)
    rows = np.unique(np.concatenate([[0, n_rows - 1], rows, extra]))
    _CTX = ctx
    t0 = time.time()
    with multiprocessing.get_context("fork").Pool(workers) as pool:
        res = pool.map(_one_row, [int(r) for r in rows], chunksize=1)
    dt = time.time() - t0
    _CTX = None
    t_min = np.stack([r[0] for r in res])
    t_max = np.stack([r[1] for r in res])
    vec = {key: np.array([r[2 + q] for r in res]) for q, key in enumerate(
        ("r_min", "r_max", "av_min", "av_max", "leak_min", "leak_max"))}
    raw = sparse_rows(t_min, t_max)
    im = A._assemble(ctx, t_min.copy(), t_max.copy(), vec["r_min"].copy(),
                     vec["r_max"].copy(), vec["av_min"].copy(),
                     vec["av_max"].copy(), vec["leak_min"].copy(),
                     vec["leak_max"].copy())
    asm = sparse_rows(im.t_min, im.t_max)
    out = dict(config=cfg_text(name), rows=rows, n_rows=n_rows,
               n_s=len(labels.safe), n_u=ctx.n_u, n_w=ctx.n_w,
               raw_ptr=raw[0], raw_col=raw[1], raw_lo=raw[2], raw_hi=raw[3],
               ptr=asm[0], col=asm[1], lo=asm[2], hi=asm[3],
               r_min=im.r_min, r_max=im.r_max, a_min=im.a_min, a_max=im.a_max,
               sec_per_row_core=dt * workers / len(rows),
               **{"raw_" + k: v for k, v in vec.items()})
    np.savez_compressed(os.path.join(OUT, f"rows_{name}.npz"), **out)
    print(f"rows_{name}: {len(rows)} rows in {dt:.1f}s "
          f"({dt * workers / len(rows):.3f} s/row/core)", flush=True)


# --- full build + synthesis -------------------------------------------------

def _traced_phase_margins(imdp, spec_kind, mode):
    """Re-run phase 1 through the reference's own bellman_step, recording the
    V0 that produced the final policy; return top-2 margins per state."""
    calls = []
    orig = S.bellman_step

    def spy(imdp_, values, lp_direction, u_objective, spec, fixed_policy=None,
            bounds=None, solver=None):
        if fixed_policy is None:
            calls.append((np.array(values, copy=True), lp_direction,
                          u_objective, spec, solver))
        return orig(imdp_, values, lp_direction, u_objective, spec,
                    fixed_policy, bounds, solver)

    S.bellman_step = spy
    try:
        if spec_kind == "safety":
            S.synthesize_safe(imdp, mode=mode)
        else:
            S.synthesize_reach(imdp, mode=mode)
    finally:
        S.bellman_step = orig
    v0, lp, u_obj, spec, solver = calls[-2]
    d1, d2 = (1.0, 0.0) if spec == "reach" else (0.0, 1.0)
    vals = solver.values(np.concatenate([v0, [d1, d2]]), lp)
    per_uw = vals.reshape(imdp.n_s, imdp.n_u, imdp.n_w)
    per_u = per_uw.min(axis=2) if u_obj == "max" else per_uw.max(axis=2)
    srt = np.sort(per_u, axis=1)
    if imdp.n_u == 1:
        margin = np.full(imdp.n_s, np.inf)
    elif u_obj == "max":
        margin = srt[:, -1] - srt[:, -2]
    else:
        margin = srt[:, 1] - srt[:, 0]
    return margin, per_u, v0


def make_full(name, workers, max_iter=None):
    cfg = load(name)
    labels = cfg.labels()
    spaces = (cfg.state_space, cfg.input_space, cfg.disturb_space)
    cfg.workers = workers
    t0 = time.time()
    imdp = A.build_abstraction(cfg.dynamics, cfg.noise, spaces, labels,
                               cfg.abstraction_options())
    t_build = time.time() - t0
    ptr, col, lo, hi = sparse_rows(imdp.t_min, imdp.t_max)
    out = dict(config=cfg_text(name), n_s=imdp.n_s, n_u=imdp.n_u,
               n_w=imdp.n_w, ptr=ptr, col=col, lo=lo, hi=hi,
               r_min=imdp.r_min, r_max=imdp.r_max, a_min=imdp.a_min,
               a_max=imdp.a_max, t_build=t_build,
               row_sum_min=imdp.t_min.sum(axis=1),
               row_sum_max=imdp.t_max.sum(axis=1))
    kind = cfg.spec_type
    kw = dict(mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon)
    if max_iter is not None:
        kw["max_iterations"] = max_iter
    t0 = time.time()
    try:
        if imdp.input_space is None:
            ctrl = S.verify(imdp, spec="safety" if kind == "safety"
                            else "reach", **kw)
        elif kind == "safety":
            ctrl = S.synthesize_safe(imdp, **kw)
        else:
            ctrl = S.synthesize_reach(imdp, **kw)
        out.update(p_min=ctrl.p_min, p_max=ctrl.p_max,
                   iterations=np.array(ctrl.meta["iterations"]),
                   fallback=np.array(ctrl.meta["fallback"]),
                   policy=(ctrl.policy if ctrl.policy is not None
                           else np.zeros(0, np.int64)),
                   error=np.array(""))
        if ctrl.policy is not None and cfg.horizon is None:
            margin, per_u, v0 = _traced_phase_margins(
                imdp, "safety" if kind == "safety" else "reach", cfg.mode)
            out.update(margin=margin, per_u=per_u, v0_last=v0)
    except ConvergenceError as exc:
        out.update(error=np.array("ConvergenceError"),
                   k0=np.array(-1 if exc.k0 is None else exc.k0),
                   k1=np.array(-1 if exc.k1 is None else exc.k1))
    t_syn = time.time() - t0
    out["t_synth"] = t_syn
    # twin-sweep trace of the first iterations (phase 1) for trace parity
    lp = ("min" if cfg.mode == "pessimistic" else "max") if kind != "safety" \
        else ("max" if cfg.mode == "pessimistic" else "min")
    u_obj = "max" if kind != "safety" else "min"
    prog = "reach" if kind != "safety" else "safety"
    bounds = S._stack_bounds(imdp)
    solver = S._phase_solver(imdp, bounds)
    v0 = np.zeros(imdp.n_s)
    v1 = np.ones(imdp.n_s)
    tr0, tr1, pol = [], [], []
    for _ in range(6):
        v0, p = S.bellman_step(imdp, v0, lp, u_obj, prog, solver=solver)
        v1, _ = S.bellman_step(imdp, v1, lp, u_obj, prog, solver=solver)
        tr0.append(v0)
        tr1.append(v1)
        pol.append(p)
    out.update(trace_v0=np.array(tr0), trace_v1=np.array(tr1),
               trace_pol=np.array(pol))
    np.savez_compressed(os.path.join(OUT, f"full_{name}.npz"), **out)
    print(f"full_{name}: {imdp.n_rows}x{imdp.n_s} built in {t_build:.1f}s, "
          f"synth {t_syn:.1f}s, err={out['error']}", flush=True)


# --- full-size reference runs (controller + traces, no matrices) -----------

def _lean_stack_bounds(imdp):
    """S._stack_bounds, then t_min / t_max re-pointed at views of the stacked
    copies: same values, one dense copy fewer (robot2d_reachavoid: 17.5 GB),
    so the reference's own synthesis fits a 62 GB host."""
    lower, upper = _ORIG_STACK(imdp)
    imdp.t_min = lower[:, :imdp.n_s]
    imdp.t_max = upper[:, :imdp.n_s]
    return lower, upper


_ORIG_STACK = S._stack_bounds


def make_fullsize(name, workers, trace_iters=6, max_iter=None):
    """The reference end to end at full size: build_abstraction (fork pool),
    then synthesize_* / verify through its own _run_phase.  A spy on
    bellman_step records the phase-1 V0 / V1 of the first `trace_iters`
    iterations, every phase-1 policy's change count and gap, and the last
    V0 (for top-2 margins).  Only vectors are stored: the abstraction itself
    is rebuilt by the GPU in the test."""
    cfg = load(name)
    labels = cfg.labels()
    spaces = (cfg.state_space, cfg.input_space, cfg.disturb_space)
    cfg.workers = workers
    t0 = time.time()
    imdp = A.build_abstraction(cfg.dynamics, cfg.noise, spaces, labels,
                               cfg.abstraction_options())
    t_build = time.time() - t0
    print(f"{name}: built {imdp.n_rows}x{imdp.n_s} in {t_build:.0f}s",
          flush=True)
    nnz = int(np.count_nonzero((imdp.t_min != 0) | (imdp.t_max != 0)))
    row_nnz = np.count_nonzero((imdp.t_min != 0) | (imdp.t_max != 0), axis=1)
    out = dict(config=cfg_text(name), n_s=imdp.n_s, n_u=imdp.n_u,
               n_w=imdp.n_w, nnz=nnz, row_nnz=row_nnz.astype(np.int32),
               r_min=imdp.r_min, r_max=imdp.r_max, a_min=imdp.a_min,
               a_max=imdp.a_max, t_build=t_build,
               row_sum_min=imdp.t_min.sum(axis=1),
               row_sum_max=imdp.t_max.sum(axis=1),
               t_max_colsum=imdp.t_max.sum(axis=0),
               t_min_colsum=imdp.t_min.sum(axis=0))
    tr0, tr1, trp, gaps = [], [], [], []
    state = {"pair": None, "phase1": True, "last": None, "calls": 0}
    orig = S.bellman_step

    def spy(imdp_, values, lp_direction, u_objective, spec, fixed_policy=None,
            bounds=None, solver=None):
        res = orig(imdp_, values, lp_direction, u_objective, spec,
                   fixed_policy, bounds, solver)
        if fixed_policy is None:
            state["calls"] += 1
            if state["calls"] % 2 == 1:      # V0 step of an iteration
                state["last"] = (np.array(values, copy=True), lp_direction,
                                 u_objective, spec, solver)
                state["v0"] = res
            else:                             # V1 step
                v0n, pol = state["v0"]
                gaps.append(float(np.max(res[0] - v0n)))
                if len(tr0) < trace_iters:
                    tr0.append(v0n)
                    tr1.append(res[0])
                    trp.append(pol)
        return res

    S.bellman_step = spy
    S._stack_bounds = _lean_stack_bounds
    kind = cfg.spec_type
    kw = dict(mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon)
    if max_iter is not None:
        kw["max_iterations"] = max_iter
    t0 = time.time()
    try:
        if imdp.input_space is None:
            ctrl = S.verify(imdp, spec="safety" if kind == "safety"
                            else "reach", **kw)
        elif kind == "safety":
            ctrl = S.synthesize_safe(imdp, **kw)
        else:
            ctrl = S.synthesize_reach(imdp, **kw)
        out.update(p_min=ctrl.p_min, p_max=ctrl.p_max,
                   iterations=np.array(ctrl.meta["iterations"]),
                   fallback=np.array(ctrl.meta["fallback"]),
                   policy=(ctrl.policy if ctrl.policy is not None
                           else np.zeros(0, np.int64)),
                   error=np.array(""))
        if ctrl.policy is not None and state["last"] is not None:
            v0, lp, u_obj, spec, solver = state["last"]
            d1, d2 = (1.0, 0.0) if spec == "reach" else (0.0, 1.0)
            vals = solver.values(np.concatenate([v0, [d1, d2]]), lp)
            per_u = vals.reshape(imdp.n_s, imdp.n_u, imdp.n_w)
            per_u = per_u.min(axis=2) if u_obj == "max" else per_u.max(axis=2)
            srt = np.sort(per_u, axis=1)
            margin = (srt[:, -1] - srt[:, -2]) if u_obj == "max" \
                else (srt[:, 1] - srt[:, 0])
            out.update(margin=margin, per_u=per_u, v0_last=v0)
    except ConvergenceError as exc:
        out.update(error=np.array("ConvergenceError"),
                   k0=np.array(-1 if exc.k0 is None else exc.k0),
                   k1=np.array(-1 if exc.k1 is None else exc.k1))
    finally:
        S.bellman_step = orig
        S._stack_bounds = _ORIG_STACK
    out.update(t_synth=time.time() - t0, trace_v0=np.array(tr0),
               trace_v1=np.array(tr1), trace_pol=np.array(trp),
               gap_trace=np.array(gaps))
    np.savez_compressed(os.path.join(OUT, f"fullsize_{name}.npz"), **out)
    print(f"fullsize_{name}: synth {out['t_synth']:.0f}s, "
          f"{len(gaps)} phase-1 iterations traced, err={out['error']}",
          flush=True)


# --- the reference's optimistic mode and diagnose_convergence on minis ------

def make_modes(name, workers):
    """full_<name>'s abstraction (rebuilt by the reference), synthesized in
    optimistic mode, and diagnose_convergence in both modes -- pins the
    oracle's restatement of those paths (synthesis.py:238-361)."""
    cfg = load(name)
    labels = cfg.labels()
    spaces = (cfg.state_space, cfg.input_space, cfg.disturb_space)
    cfg.workers = workers
    imdp = A.build_abstraction(cfg.dynamics, cfg.noise, spaces, labels,
                               cfg.abstraction_options())
    kind = cfg.spec_type
    spec = "safety" if kind == "safety" else "reach"
    out = dict(config=cfg_text(name))
    kw = dict(mode="optimistic", eps=cfg.eps, horizon=cfg.horizon)
    if imdp.input_space is None:
        ctrl = S.verify(imdp, spec=spec, **kw)
    elif kind == "safety":
        ctrl = S.synthesize_safe(imdp, **kw)
    else:
        ctrl = S.synthesize_reach(imdp, **kw)
    out.update(opt_p_min=ctrl.p_min, opt_p_max=ctrl.p_max,
               opt_iterations=np.array(ctrl.meta["iterations"]),
               opt_fallback=np.array(ctrl.meta["fallback"]),
               opt_policy=(ctrl.policy if ctrl.policy is not None
                           else np.zeros(0, np.int64)))
    for mode in ("pessimistic", "optimistic"):
        try:
            k0, k1 = S.diagnose_convergence(imdp, spec=spec, mode=mode,
                                            eps=cfg.eps, max_iterations=2000)
            err = ""
        except ConvergenceError as exc:
            k0, k1, err = exc.k0, exc.k1, "ConvergenceError"
        out[f"diag_{mode}"] = np.array([-1 if k0 is None else k0,
                                        -1 if k1 is None else k1])
        out[f"diag_{mode}_error"] = np.array(err)
    np.savez_compressed(os.path.join(OUT, f"modes_{name}.npz"), **out)
    print(f"modes_{name}: optimistic {out['opt_iterations']}, diagnose "
          f"{out['diag_pessimistic']} / {out['diag_optimistic']}", flush=True)


def make_ndtr():
    from scipy.special import ndtr
    rng = np.random.default_rng(2024)
    xs = np.concatenate([
        rng.uniform(-3, 3, 60000), rng.uniform(-40, 40, 20000),
        rng.normal(0, 1, 20000), np.linspace(-0.75, 0.75, 4001),
        np.array([0.0, -0.0, 1e-300, -1e-300, 37.5, -37.5, 38.5, -38.5,
                  8.0, -8.0, 1.0, -1.0, np.sqrt(0.5), -np.sqrt(0.5),
                  np.inf, -np.inf]),
    ])
    np.savez_compressed(os.path.join(OUT, "ndtr.npz"), x=xs, y=ndtr(xs))
    print("ndtr: done", flush=True)


def make_pairwise():
    rng = np.random.default_rng(5)
    lens = [1, 2, 7, 8, 9, 15, 16, 17, 100, 127, 128, 129, 255, 256, 257,
            1000, 1577, 4097, 9261]
    arrs, sums = [], []
    for n in lens:
        a = rng.uniform(0, 1, n) * rng.choice([1.0, 1e-8, 1e-13], n)
        arrs.append(a)
        sums.append(float(np.sum(a)))
    np.savez_compressed(os.path.join(OUT, "pairwise.npz"),
                        lens=np.array(lens), data=np.concatenate(arrs),
                        sums=np.array(sums))
    print("pairwise: done", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    want = set(args.only or [])

    def on(key):
        return not want or key in want

    if on("ndtr"):
        make_ndtr()
    if on("pairwise"):
        make_pairwise()
    for name in ("robot2d_ra_mini", "dim6_mini", "room5d_mini",
                 "vehicle3d_mini", "bas4d_mini", "bas7d_mini"):
        if on("full_" + name):
            make_full(name, args.workers,
                      max_iter=300 if name.startswith("dim") else None)
    for name in ("robot2d_ra_mini", "room5d_mini", "dim6_mini",
                 "bas4d_mini"):
        if on("modes_" + name):
            make_modes(name, args.workers)
    for name, n in SAMPLES.items():
        if on("rows_" + name):
            make_rows(name, n, args.workers)
    if on("full_robot2d_reach"):
        make_full("robot2d_reach", args.workers)
    # explicit only (hours of CPU): the reference end to end at full size
    if "fullsize_dim14_verify" in want:
        # phase 1 needs ~731 sweeps and phase 2 ~1.7 M (SURVEY.md finding 7):
        # stop phase 1 at 30 iterations through the reference's own cap
        make_fullsize("dim14_verify", args.workers, trace_iters=30,
                      max_iter=30)
    if "fullsize_robot2d_reachavoid" in want:
        make_fullsize("robot2d_reachavoid", args.workers)


if __name__ == "__main__":
    main()
