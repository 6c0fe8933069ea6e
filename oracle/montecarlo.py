"""Monte Carlo-noise row bounds -- oracle restatement (TEST INFRASTRUCTURE).

Restates pkg/src/impact/abstraction.py's Monte Carlo path for FullNormal
noise: _row_monte_carlo (:511-540) over every destination, _mc_prob_extremes
(:378-397) through optimize_over_cell (optimize.py:165-189), and
mc_box_probability / FullNormal.density / CustomNoise.density /
derive_seed / mc_generator (noise.py:63-95, 121-153) with numpy itself (the reference's dependency), so
its bits equal the reference's; pinned to tests/golden/mc_*.npz.
"""

import math

import numpy as np

from .construct import _env, assemble, make_context, source_cell, _boxes
from .nm import minimize_batch, start_points


def derive_seed(base, row, dest):
    ss = np.random.SeedSequence(entropy=int(base) & (2**64 - 1),
                                spawn_key=(int(row), int(dest)))
    return int(ss.generate_state(1, np.uint64)[0])


def density(noise, y, mean):
    """FullNormal.density (noise.py:63-73) / CustomNoise.density (:84-95)."""
    if hasattr(noise, "inv_cov"):
        diff = y - mean
        quad = np.einsum("ki,ij,kj->k", diff, noise.inv_cov, diff)
        n = noise.inv_cov.shape[0]
        norm = math.sqrt(np.linalg.det(noise.inv_cov)) * \
            (2 * math.pi) ** (-n / 2)
        return norm * np.exp(-0.5 * quad)
    env = {f"y{d + 1}": y[:, d] for d in range(noise.dim)}
    env.update({f"m{d + 1}": mean[d] for d in range(noise.dim)})
    return np.broadcast_to(np.asarray(
        noise.density_expr.evaluate_env(env), dtype=float), (len(y),))


def box_probability(noise, mean, lo, hi, seed):
    """mc_box_probability(...)[0] (noise.py:133-153)."""
    volume = float(np.prod(hi - lo))
    if volume == 0.0:
        return 0.0
    rng = np.random.Generator(np.random.Philox(
        np.random.SeedSequence(entropy=int(seed) & (2**64 - 1))))
    y = lo + (hi - lo) * rng.random((noise.samples, len(lo)))
    dens = density(noise, y, mean)
    est = volume * float(np.mean(dens))
    return min(max(est, 0.0), 1.0)


def extremes(ctx, noise, mc_seed, lo, hi, base, blo, bhi, row, dest):
    """_mc_prob_extremes: (min, max) over the source cell."""
    seed = derive_seed(mc_seed, row, dest)
    n = ctx.state.dim
    ms = ctx.multistart(n)
    out = []
    for sign in (1.0, -1.0):
        def fn(pts, ids, sign=sign):
            vals = []
            for p in pts:
                env = dict(base)
                env.update({f"x{d + 1}": p[d] for d in range(n)})
                mean = np.array([float(e.evaluate(env))
                                 for e in ctx.dyn.exprs])
                vals.append(sign * box_probability(noise, mean, blo, bhi,
                                                   seed))
            return np.array(vals)
        best = minimize_batch(fn, lo, hi, start_points(lo, hi, ms),
                              ctx.max_evals(n), ctx.tol)
        out.append(float(sign * np.min(best)))
    return out[0], out[1]


def row_bounds(ctx, noise, mc_seed, row):
    i = row % ctx.n_w
    k, j = divmod(row // ctx.n_w, ctx.n_u)
    lo, hi = source_cell(ctx, int(ctx.safe[k]))
    base = _env(ctx, j, i)
    sp = ctx.state

    def group(multi):
        mins = np.zeros(len(multi))
        maxs = np.zeros(len(multi))
        if not len(multi):
            return mins, maxs
        blo, bhi = _boxes(ctx, multi)
        for q in range(len(multi)):
            flat = 0
            for d in range(sp.dim):
                flat = flat * int(sp.counts[d]) + int(multi[q, d])
            pmin, pmax = extremes(ctx, noise, mc_seed, lo, hi, base,
                                  blo[q], bhi[q], row, flat)
            if pmax <= ctx.cutoff:
                pmin = pmax = 0.0
            mins[q] = min(pmin, pmax)
            maxs[q] = pmax
        return mins, maxs

    t_min, t_max = group(ctx.safe_multi)
    r_min, r_max = group(ctx.target_multi)
    a_min, a_max = group(ctx.avoid_multi)
    p_lo, p_hi = extremes(ctx, noise, mc_seed, lo, hi, base, ctx.cover_lo,
                          ctx.cover_hi, row, sp.total)
    return (t_min, t_max, float(np.sum(r_min)), float(np.sum(r_max)),
            float(np.sum(a_min)), float(np.sum(a_max)),
            max(0.0, 1.0 - p_hi), max(0.0, 1.0 - p_lo))


def build(dyn, noise, spaces, labels, opts, rows=None):
    ctx = make_context(dyn, _Sigma(spaces[0].dim), spaces, labels, opts)
    n_rows = len(ctx.safe) * ctx.n_u * ctx.n_w
    rows = np.arange(n_rows) if rows is None else np.asarray(rows)
    res = [row_bounds(ctx, noise, opts.mc_seed, int(r)) for r in rows]
    t_min = np.stack([x[0] for x in res])
    t_max = np.stack([x[1] for x in res])
    vec = [np.array([x[q] for x in res]) for q in range(2, 8)]
    out = assemble(t_min, t_max, *vec, monte_carlo=True)
    return dict(zip(("t_min", "t_max", "r_min", "r_max", "a_min", "a_max"),
                    out))


class _Sigma:
    """make_context reads noise.sigma; unused on the Monte Carlo path."""
    def __init__(self, n):
        self.sigma = np.ones(n)
