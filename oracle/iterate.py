"""Twin interval iteration and the synthesis API -- oracle restatement.

TEST INFRASTRUCTURE.  Restates pkg/src/impact/synthesis.py: virtual r/a
slots (:79-83), phase row subsets (:86-94), the robust Bellman step
(:97-135), the two-phase loop with monotone / bracket / gap / stall / cap
logic (:145-205), value-track selection and the safety complement
(:238-318) and diagnose_convergence (:321-361).

`Model` is any object with n_s, n_u, n_w, t_min, t_max, r_min, r_max, a_min,
a_max (dense numpy) -- e.g. a dict-backed namespace built from oracle
construction or from golden fixtures.
"""

from dataclasses import dataclass

import numpy as np

from paper_2401_03555_b200.errors import ConvergenceError, ImpactError

from .lp import Rows

BRACKET_TOL = 1e-9
MONOTONE_TOL = 1e-12


@dataclass
class Model:
    n_s: int
    n_u: int
    n_w: int
    t_min: np.ndarray
    t_max: np.ndarray
    r_min: np.ndarray
    r_max: np.ndarray
    a_min: np.ndarray
    a_max: np.ndarray


def stacked(m):
    lo = np.hstack([m.t_min, m.r_min[:, None], m.a_min[:, None]])
    hi = np.hstack([m.t_max, m.r_max[:, None], m.a_max[:, None]])
    return lo, hi


def phase_rows(m, bounds, policy=None):
    lo, hi = bounds
    if policy is None:
        return Rows(lo, hi)
    base = (np.arange(m.n_s) * m.n_u + np.asarray(policy)) * m.n_w
    idx = (base[:, None] + np.arange(m.n_w)).ravel()
    return Rows(lo[idx], hi[idx])


def bellman(m, v, lp, u_obj, spec, policy=None, rows=None):
    """One robust Bellman update (synthesis.py:97-135) -> (V', choice)."""
    if rows is None:
        rows = phase_rows(m, stacked(m), policy)
    if spec not in ("reach", "safety"):
        raise ValueError(f"bad spec {spec!r}")
    tail = [1.0, 0.0] if spec == "reach" else [0.0, 1.0]
    vals = rows.values(np.concatenate([np.asarray(v, float), tail]), lp)
    per = vals.reshape(m.n_s, 1 if policy is not None else m.n_u, m.n_w)
    if u_obj == "max":
        per_u = per.min(axis=2)
        pick = np.argmax(per_u, axis=1)
    elif u_obj == "min":
        per_u = per.max(axis=2)
        pick = np.argmin(per_u, axis=1)
    else:
        raise ValueError(f"bad u_objective {u_obj!r}")
    new = per_u[np.arange(m.n_s), pick]
    if policy is not None:
        pick = np.asarray(policy).copy()
    return new, pick


def report_k(k):
    return None if k is None else max(k - 1, 1)


@dataclass
class PhaseResult:
    v0: np.ndarray
    v1: np.ndarray
    policy: np.ndarray
    iterations: int
    k0: int | None
    k1: int | None
    fallback: bool
    gaps: list


def run_phase(m, bounds, spec, lp, u_obj, eps, horizon, max_iterations,
              policy=None):
    """synthesis.py:145-205."""
    rows = phase_rows(m, bounds, policy)
    v0 = np.zeros(m.n_s)
    v1 = np.ones(m.n_s)
    pol = np.zeros(m.n_s, dtype=np.int64)
    k0 = k1 = None
    prev = None
    it = 0
    gaps = []
    while True:
        it += 1
        n0, pol = bellman(m, v0, lp, u_obj, spec, policy, rows)
        n1, _ = bellman(m, v1, lp, u_obj, spec, policy, rows)
        if (n0 < v0 - MONOTONE_TOL).any() or (n1 > v1 + MONOTONE_TOL).any():
            raise ImpactError("value iterates lost monotonicity; "
                              "abstraction bounds inconsistent")
        if k0 is None and np.max(np.abs(n0 - v0)) <= eps:
            k0 = it
        if k1 is None and np.max(np.abs(n1 - v1)) <= eps:
            k1 = it
        v0, v1 = n0, n1
        if (v0 > v1 + BRACKET_TOL).any():
            raise ImpactError("interval iteration bracket violated")
        if horizon is not None:
            if it >= horizon:
                return PhaseResult(v0, v1, pol, it, k0, k1, False, gaps)
            continue
        gap = float(np.max(v1 - v0))
        gaps.append(gap)
        if gap <= eps:
            return PhaseResult(v0, v1, pol, it, k0, k1, False, gaps)
        stalled = prev is not None and prev - gap <= 1e-15 * max(1.0, gap)
        if k0 is not None and k1 is not None and stalled:
            return PhaseResult(v0, v1, pol, it, k0, k1, True, gaps)
        prev = gap
        if it >= max_iterations:
            raise ConvergenceError(f"gap {gap!r} above eps={eps!r} after {it} "
                                   "iterations", k0=report_k(k0),
                                   k1=report_k(k1))


def synthesize(m, spec, mode="pessimistic", eps=1e-6, horizon=None,
               max_iterations=10**6):
    """synthesize_reach (spec 'reach') / synthesize_safe (spec 'safety'),
    synthesis.py:238-303.  Returns dict(p_min, p_max, policy, iterations,
    fallback)."""
    b = stacked(m)
    if spec == "reach":
        lp1 = "min" if mode == "pessimistic" else "max"
        u_obj = "max"
    else:
        lp1 = "max" if mode == "pessimistic" else "min"
        u_obj = "min"
    lp2 = "max" if lp1 == "min" else "min"
    ph1 = run_phase(m, b, spec, lp1, u_obj, eps, horizon, max_iterations)
    ph2 = run_phase(m, b, spec, lp2, u_obj, eps, horizon, max_iterations,
                    policy=ph1.policy)

    def pick(ph, lp, from_max_lp):
        if horizon is not None or ph.fallback:
            return ph.v0
        if spec == "reach":
            return ph.v0 if lp == "min" else ph.v1
        return ph.v0 if lp == "max" else ph.v1

    val1 = pick(ph1, lp1, None)
    val2 = pick(ph2, lp2, None)
    if spec == "reach":
        p_min, p_max = (val1, val2) if lp1 == "min" else (val2, val1)
    else:
        p_min, p_max = ((1.0 - val1, 1.0 - val2) if lp1 == "max"
                        else (1.0 - val2, 1.0 - val1))
    p_max = np.maximum(p_min, p_max)
    return dict(p_min=p_min, p_max=p_max, policy=ph1.policy,
                iterations=(ph1.iterations, ph2.iterations),
                fallback=(ph1.fallback, ph2.fallback), phase1=ph1, phase2=ph2)


def diagnose(m, spec="reach", mode="pessimistic", eps=1e-6,
             max_iterations=10**6):
    """diagnose_convergence (synthesis.py:321-361): each phase-1 bound
    iterated on its own until its own step drops to eps -> (k0, k1)."""
    if spec == "safety":
        lp = "max" if mode == "pessimistic" else "min"
        u_obj = "min"
    else:
        lp = "min" if mode == "pessimistic" else "max"
        u_obj = "max"
    rows = phase_rows(m, stacked(m))
    v0 = np.zeros(m.n_s)
    v1 = np.ones(m.n_s)
    k0 = k1 = None
    for it in range(1, max_iterations + 1):
        if k0 is None:
            n0, _ = bellman(m, v0, lp, u_obj, spec, rows=rows)
            if np.max(np.abs(n0 - v0)) <= eps:
                k0 = it
            v0 = n0
        if k1 is None:
            n1, _ = bellman(m, v1, lp, u_obj, spec, rows=rows)
            if np.max(np.abs(n1 - v1)) <= eps:
                k1 = it
            v1 = n1
        if k0 is not None and k1 is not None:
            return report_k(k0), report_k(k1)
    raise ConvergenceError(f"no self-convergence within {max_iterations} "
                           "iterations", k0=report_k(k0), k1=report_k(k1))
