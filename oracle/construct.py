"""IMDP row bounds under diagonal Gaussian noise -- oracle restatement.

TEST INFRASTRUCTURE.  Restates pkg/src/impact/abstraction.py for
DiagonalNormal noise: build context (:198-228), clipped source cell
(:231-235), mean ranges by NM (:238-284), exact per-dimension extremes
(:287-297), cover-box leak (:300-309), product gather (:312-319), coupled
NM refinement of the live window (:322-375, :465-495), separable cutoff
(:496-503), row sums (:505-508) and _assemble (:607-659).
"""

from dataclasses import dataclass

import numpy as np
from scipy.special import ndtr

from paper_2401_03555_b200.errors import AbstractionError
from paper_2401_03555_b200.grid import domain_box, multi_indices

from .nm import minimize_batch, start_points

ROW_SUM_HARD = 1e-6


def interval_probability(sigma, mean, lo, hi):
    """noise.py:116-118 (scipy's cephes ndtr)."""
    return ndtr((hi - mean) / sigma) - ndtr((lo - mean) / sigma)


@dataclass
class Context:
    dyn: object
    sigma: np.ndarray
    state: object
    n_u: int
    n_w: int
    u_reps: np.ndarray
    w_reps: np.ndarray
    safe: np.ndarray
    safe_multi: np.ndarray
    target_multi: np.ndarray
    avoid_multi: np.ndarray
    edges: list
    cover_lo: np.ndarray
    cover_hi: np.ndarray
    separable: bool
    cutoff: float
    low_cost: bool
    max_evals: callable
    multistart: callable
    tol: float


def make_context(dyn, noise, spaces, labels, opts):
    """abstraction.py:198-228."""
    state, inp, dist = spaces
    n = state.dim
    cover = domain_box(state)
    return Context(
        dyn=dyn, sigma=np.asarray(noise.sigma, float), state=state,
        n_u=inp.total if inp is not None else 1,
        n_w=dist.total if dist is not None else 1,
        u_reps=inp.rep_points() if inp is not None else np.zeros((1, 0)),
        w_reps=dist.rep_points() if dist is not None else np.zeros((1, 0)),
        safe=np.asarray(labels.safe),
        safe_multi=multi_indices(state, labels.safe),
        target_multi=multi_indices(state, labels.target),
        avoid_multi=multi_indices(state, labels.avoid),
        edges=[state.edges(d) for d in range(n)],
        cover_lo=cover.lo, cover_hi=cover.hi,
        separable=dyn.is_separable(), cutoff=opts.zero_cutoff,
        low_cost=opts.low_cost,
        max_evals=lambda dim: opts.optimizer_max_evals or 200 * max(dim, 1),
        multistart=lambda dim: opts.multistart or 1 + 2 * dim,
        tol=opts.optimizer_tol)


def source_cell(ctx, flat):
    """Cell of the state clipped to [lb, ub] (abstraction.py:231-235)."""
    sp = ctx.state
    rep = sp.lb + multi_indices(sp, [flat])[0] * sp.eta
    return (np.maximum(rep - sp.eta / 2, sp.lb),
            np.minimum(rep + sp.eta / 2, sp.ub))


def _env(ctx, j, i):
    u, w = ctx.u_reps[j], ctx.w_reps[i]
    env = {f"u{q + 1}": u[q] for q in range(len(u))}
    env.update({f"w{q + 1}": w[q] for q in range(len(w))})
    return env


def mean_ranges(ctx, lo, hi, base):
    """Per-dimension [min, max] of f_d over the cell by NM with signed
    objectives (abstraction.py:256-284)."""
    n = ctx.state.dim
    m_lo, m_hi = np.empty(n), np.empty(n)
    for d in range(n):
        deps = sorted(ctx.dyn.state_dependencies(d))
        expr = ctx.dyn.exprs[d]
        if not deps:
            v = float(expr.evaluate(dict(base)))
            m_lo[d] = m_hi[d] = v
            continue
        slo, shi = lo[deps], hi[deps]
        ms = ctx.multistart(len(deps))
        st = start_points(slo, shi, ms)
        sign = np.repeat([1.0, -1.0], ms)

        def fn(pts, ids, deps=deps, expr=expr, sign=sign):
            env = dict(base)
            for q, e in enumerate(deps):
                env[f"x{e + 1}"] = pts[:, q]
            v = np.broadcast_to(np.asarray(expr.evaluate_env(env), float),
                                (len(pts),))
            return v * sign[ids]

        best = minimize_batch(fn, slo, shi, np.vstack([st, st]),
                              ctx.max_evals(len(deps)), ctx.tol)
        m_lo[d] = float(np.min(best[:ms]))
        m_hi[d] = float(-np.min(best[ms:]))
    return m_lo, m_hi


def dim_extremes(sigma, eta, edges, ml, mh):
    """Exact min/max over the mean interval of each bin's 1-D probability;
    the peak sits at the bin center (abstraction.py:287-297)."""
    a, b = edges[:-1], edges[1:]
    p_lo = interval_probability(sigma, ml, a, b)
    p_hi = interval_probability(sigma, mh, a, b)
    mid = (a + b) / 2
    top = interval_probability(sigma, 0.0, -eta / 2, eta / 2)
    return np.minimum(p_lo, p_hi), np.where(
        mid < ml, p_lo, np.where(mid > mh, p_hi, top))


def products(tables, multi):
    """Left-to-right product of per-dimension table entries (:312-319)."""
    if len(multi) == 0:
        return np.zeros(0)
    out = tables[0][multi[:, 0]].copy()
    for d in range(1, multi.shape[1]):
        out *= tables[d][multi[:, d]]
    return out


def cover_extremes(ctx, ml, mh):
    """abstraction.py:300-309."""
    lo, hi = ctx.cover_lo, ctx.cover_hi
    mu = np.clip((lo + hi) / 2, ml, mh)
    pmax = float(np.prod(interval_probability(ctx.sigma, mu, lo, hi)))
    pmin = float(np.prod(np.minimum(
        interval_probability(ctx.sigma, ml, lo, hi),
        interval_probability(ctx.sigma, mh, lo, hi))))
    return pmin, pmax


def box_extremes(ctx, lo, hi, base, blo, bhi):
    """NM min and max of the box probability over the source cell for each
    box (abstraction.py:322-375): per box a min block then a max block of
    `ms` starts, value = min over starts."""
    nbox = len(blo)
    if nbox == 0:
        return np.zeros(0), np.zeros(0)
    n = ctx.state.dim
    ms = ctx.multistart(n)
    st = start_points(lo, hi, ms)
    sign = np.tile([1.0, -1.0], nbox)
    blo2 = np.repeat(blo, 2, axis=0)
    bhi2 = np.repeat(bhi, 2, axis=0)

    def fn(pts, ids):
        env = dict(base)
        for d in range(n):
            env[f"x{d + 1}"] = pts[:, d]
        means = ctx.dyn.eval_env(env)
        item = ids // ms
        prob = np.ones(len(pts))
        for d in range(n):
            md = np.broadcast_to(np.asarray(means[d], float), (len(pts),))
            prob *= interval_probability(ctx.sigma[d], md, blo2[item, d],
                                         bhi2[item, d])
        return prob * sign[item]

    best = minimize_batch(fn, lo, hi, np.tile(st, (2 * nbox, 1)),
                          ctx.max_evals(n), ctx.tol)
    best = best.reshape(2 * nbox, ms).min(axis=1)
    return best[0::2], -best[1::2]


def _boxes(ctx, multi):
    blo = np.empty((len(multi), ctx.state.dim))
    bhi = np.empty_like(blo)
    for d in range(ctx.state.dim):
        blo[:, d] = ctx.edges[d][multi[:, d]]
        bhi[:, d] = ctx.edges[d][multi[:, d] + 1]
    return blo, bhi


def row_bounds(ctx, row):
    """Raw bounds of one row (abstraction.py:430-508).  Returns
    (t_min, t_max, r_min, r_max, av_min, av_max, leak_min, leak_max)."""
    i = row % ctx.n_w
    k, j = divmod(row // ctx.n_w, ctx.n_u)
    lo, hi = source_cell(ctx, int(ctx.safe[k]))
    base = _env(ctx, j, i)
    ml, mh = mean_ranges(ctx, lo, hi, base)
    n = ctx.state.dim
    gmin, gmax = [], []
    for d in range(n):
        a, b = dim_extremes(ctx.sigma[d], ctx.state.eta[d], ctx.edges[d],
                            ml[d], mh[d])
        gmin.append(a)
        gmax.append(b)
    t_max = products(gmax, ctx.safe_multi)
    t_min = products(gmin, ctx.safe_multi)
    r_hi = products(gmax, ctx.target_multi)
    r_lo = products(gmin, ctx.target_multi)
    a_hi = products(gmax, ctx.avoid_multi)
    a_lo = products(gmin, ctx.avoid_multi)
    p_lo, p_hi = cover_extremes(ctx, ml, mh)
    if not ctx.separable:
        groups = [(ctx.safe_multi, t_max), (ctx.target_multi, r_hi),
                  (ctx.avoid_multi, a_hi)]
        lives = [np.flatnonzero(ub > ctx.cutoff) for _, ub in groups]
        blos, bhis = [], []
        for (multi, _), live in zip(groups, lives):
            if len(live):
                bl, bh = _boxes(ctx, multi[live])
                blos.append(bl)
                bhis.append(bh)
        blos.append(ctx.cover_lo[None, :])
        bhis.append(ctx.cover_hi[None, :])
        mins, maxs = box_extremes(ctx, lo, hi, base, np.vstack(blos),
                                  np.vstack(bhis))
        outs = [(np.zeros_like(t_min), np.zeros_like(t_max)),
                (np.zeros_like(r_lo), np.zeros_like(r_hi)),
                (np.zeros_like(a_lo), np.zeros_like(a_hi))]
        at = 0
        for (omin, omax), live in zip(outs, lives):
            omin[live] = mins[at:at + len(live)]
            omax[live] = maxs[at:at + len(live)]
            at += len(live)
        (t_min, t_max), (r_lo, r_hi), (a_lo, a_hi) = outs
        p_lo, p_hi = mins[at], maxs[at]
    else:
        dead = t_max <= ctx.cutoff
        t_max[dead] = 0.0
        t_min[dead] = 0.0
        t_min = np.minimum(t_min, t_max)
    if ctx.low_cost:
        t_min[t_max <= ctx.cutoff] = 0.0
    return (t_min, t_max, float(np.sum(r_lo)), float(np.sum(r_hi)),
            float(np.sum(a_lo)), float(np.sum(a_hi)),
            max(0.0, 1.0 - p_hi), max(0.0, 1.0 - p_lo))


def assemble(t_min, t_max, r_min, r_max, av_min, av_max, leak_min, leak_max,
             monte_carlo=False):
    """Clip, repair row sums, validate (abstraction.py:607-659, :121-137).
    Works in place on the (rows, n_s) arrays; returns the six bound arrays.
    Monte Carlo rows skip the hard row-sum errors and are only repaired
    (abstraction.py:620-632, 645-650: `if not monte_carlo`)."""
    np.clip(t_min, 0.0, 1.0, out=t_min)
    np.clip(t_max, 0.0, 1.0, out=t_max)
    np.minimum(t_min, t_max, out=t_min)
    for a, b in ((r_min, r_max), (av_min, av_max), (leak_min, leak_max)):
        np.clip(a, 0.0, 1.0, out=a)
        np.clip(b, 0.0, 1.0, out=b)
        np.minimum(a, b, out=a)
    a_min = np.clip(leak_min + av_min, 0.0, 1.0)
    a_max = np.clip(leak_max + av_max, 0.0, 1.0)
    over = np.maximum(t_min.sum(axis=1) + r_min + a_min - 1.0, 0.0)
    if not monte_carlo and (over > ROW_SUM_HARD).any():
        r = int(np.argmax(over > ROW_SUM_HARD))
        raise AbstractionError(f"row {r}: min-side sum exceeds 1 by "
                               f"{float(over[r])!r}")
    cut = np.minimum(over, a_min)
    a_min = a_min - cut
    rest = over - cut
    hot = np.flatnonzero(rest > 0)
    if hot.size:
        s = t_min[hot].sum(axis=1) + r_min[hot]
        f = np.where(s > 0, 1.0 - rest[hot] / np.maximum(s, 1e-300), 1.0)
        t_min[hot] *= f[:, None]
        r_min[hot] *= f
    short = np.maximum(1.0 - (t_max.sum(axis=1) + r_max + a_max), 0.0)
    if not monte_carlo and (short > ROW_SUM_HARD).any():
        r = int(np.argmax(short > ROW_SUM_HARD))
        raise AbstractionError(f"row {r}: max-side sum falls short of 1 by "
                               f"{float(short[r])!r}")
    a_max = np.minimum(a_max + short, 1.0)
    a_min = np.minimum(a_min, a_max)
    validate(t_min, t_max, r_min, r_max, a_min, a_max)
    return t_min, t_max, r_min, r_max, a_min, a_max


def validate(t_min, t_max, r_min, r_max, a_min, a_max, tol=1e-9):
    """Imdp.validate (abstraction.py:121-137)."""
    for name, lo, hi in (("t", t_min, t_max), ("r", r_min, r_max),
                         ("a", a_min, a_max)):
        if (lo < 0).any() or (hi > 1).any() or (lo > hi).any():
            raise AbstractionError(f"{name} bounds violate 0<=min<=max<=1")
    s_lo = t_min.sum(axis=1) + r_min + a_min
    s_hi = t_max.sum(axis=1) + r_max + a_max
    bad = np.flatnonzero((s_lo > 1 + tol) | (s_hi < 1 - tol))
    if bad.size:
        raise AbstractionError(f"row {int(bad[0])} sum invariant violated")


def build(dyn, noise, spaces, labels, opts, rows=None):
    """Dense oracle abstraction (or a subset of rows).  Returns dict of
    t_min, t_max (rows, n_s) and r_min, r_max, a_min, a_max."""
    ctx = make_context(dyn, noise, spaces, labels, opts)
    n_rows = len(ctx.safe) * ctx.n_u * ctx.n_w
    rows = np.arange(n_rows) if rows is None else np.asarray(rows)
    res = [row_bounds(ctx, int(r)) for r in rows]
    t_min = np.stack([x[0] for x in res]) if res else np.zeros((0, len(ctx.safe)))
    t_max = np.stack([x[1] for x in res]) if res else np.zeros((0, len(ctx.safe)))
    vec = [np.array([x[q] for x in res]) for q in range(2, 8)]
    out = assemble(t_min, t_max, *vec)
    return dict(zip(("t_min", "t_max", "r_min", "r_max", "a_min", "a_max"),
                    out))
