"""Batched projected Nelder-Mead -- oracle restatement (TEST INFRASTRUCTURE).

Restates pkg/src/impact/optimize.py: deterministic starts (:28-44) and the
lockstep simplex search (:47-155) with coefficients alpha=1, gamma=2,
rho=1/2, sigma=1/2 (:22-25).  Per instance the sequence of objective
evaluations is exactly the reference's; instances never interact, so the
batching here does not change any bits.
"""

import numpy as np

from paper_2401_03555_b200.errors import AbstractionError


def start_points(lo, hi, count):
    """Center, then lo/hi faces per dimension, then midpoints toward the
    center of earlier starts (optimize.py:28-44)."""
    lo = np.asarray(lo, dtype=float)
    hi = np.asarray(hi, dtype=float)
    mid = (lo + hi) / 2
    pts = [mid]
    for d in range(lo.size):
        for face in (lo[d], hi[d]):
            p = mid.copy()
            p[d] = face
            pts.append(p)
    base = 1 + 2 * lo.size
    q = 1
    while len(pts) < count:
        pts.append((pts[q % base] + mid) / 2)
        q += 1
    return np.asarray(pts[:count])


def _call(fn, pts, ids):
    v = np.asarray(fn(pts, ids), dtype=float)
    if not np.isfinite(v).all():
        raise AbstractionError("non-finite objective value encountered")
    return v


def minimize_batch(fn, lo, hi, starts, max_evals, tol):
    """Minimize B independent instances over the box [lo, hi].

    fn(points (A, dim), ids (A,)) -> (A,).  Returns the best value per
    instance (optimize.py:47-155; best = first argmin, :152-155).
    """
    starts = np.asarray(starts, dtype=float)
    nb, dim = starts.shape
    lo = np.asarray(lo, dtype=float)
    hi = np.asarray(hi, dtype=float)
    width = hi - lo
    # initial simplex: quarter-width step away from the nearer face (:61-68)
    xs = np.repeat(starts[:, None, :], dim + 1, axis=1)
    for d in range(dim):
        step = 0.25 * width[d]
        fwd = starts[:, d] + step
        xs[:, d + 1, d] = np.where(fwd <= hi[d], fwd, starts[:, d] - step)
    every = np.arange(nb)
    fs = np.stack([_call(fn, xs[:, v, :], every) for v in range(dim + 1)],
                  axis=1)
    used = np.full(nb, dim + 1)
    while True:
        perm = np.argsort(fs, axis=1, kind="stable")
        fs = np.take_along_axis(fs, perm, axis=1)
        xs = np.take_along_axis(xs, perm[:, :, None], axis=1)
        live = ((fs[:, -1] - fs[:, 0]) > tol) & (used < max_evals)
        if not live.any():
            break
        ids = np.flatnonzero(live)
        f = fs[ids]
        cen = xs[ids, :-1, :].mean(axis=1)
        bad = xs[ids, -1, :]
        xr = np.clip(cen + 1.0 * (cen - bad), lo, hi)
        fr = _call(fn, xr, ids)
        used[ids] += 1
        put_x, put_f = xr.copy(), fr.copy()
        shrink = np.zeros(ids.size, dtype=bool)
        grow = fr < f[:, 0]
        pull = fr >= f[:, -2]
        two = grow | pull
        if two.any():
            out = pull & (fr < f[:, -1])
            inn = pull & ~out
            cand = np.empty((ids.size, dim))
            cand[grow] = np.clip(cen[grow] + 2.0 * (cen[grow] - bad[grow]),
                                 lo, hi)
            cand[out] = np.clip(cen[out] + 0.5 * (xr[out] - cen[out]), lo, hi)
            cand[inn] = np.clip(cen[inn] + 0.5 * (bad[inn] - cen[inn]), lo, hi)
            fc = np.full(ids.size, np.inf)
            fc[two] = _call(fn, cand[two], ids[two])
            used[ids[two]] += 1
            acc = (grow & (fc < fr)) | (out & (fc < fr)) | (inn & (fc < f[:, -1]))
            put_x[acc] = cand[acc]
            put_f[acc] = fc[acc]
            shrink = (out | inn) & ~acc
        keep = ids[~shrink]
        xs[keep, -1, :] = put_x[~shrink]
        fs[keep, -1] = put_f[~shrink]
        if shrink.any():
            sid = ids[shrink]
            best = xs[sid, :1, :]
            moved = best + 0.5 * (xs[sid, 1:, :] - best)
            fv = _call(fn, moved.reshape(-1, dim), np.repeat(sid, dim))
            xs[sid, 1:, :] = moved
            fs[sid, 1:] = fv.reshape(sid.size, dim)
            used[sid] += dim
    return fs[every, np.argmin(fs, axis=1)]
