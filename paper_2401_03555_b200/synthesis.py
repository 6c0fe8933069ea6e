"""Controller synthesis / verification by interval iteration on the B200.

Drop-in for pkg/src/impact/synthesis.py: ValuePair (:45-57), Controller
(:60-76), bellman_step (:97-135), synthesize_reach (:238-266),
synthesize_safe (:269-303), verify (:306-318), diagnose_convergence
(:321-361).  Each phase of the reference's _run_phase (:145-205) is one
imp_run_phase call: the stable orders, the twin greedy-LP sweeps, the robust
Bellman reduction and every termination test (monotone, k0/k1, bracket,
gap, stalled-gap fallback, horizon, iteration cap) run on the GPU inside
replayed CUDA graphs; the host only picks value tracks and complements.
"""

import ctypes
import logging
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConvergenceError, ImpactError

__all__ = ["ValuePair", "Controller", "bellman_step", "synthesize_reach",
           "synthesize_safe", "verify", "diagnose_convergence",
           "PhaseReport"]

log = logging.getLogger(__name__)

GAP_LOG = 256   # gaps kept by the device loop: iterations 1000, 2000, ...


def log_phase(gaps, iterations, fallback, gap, k0, k1):
    """The reference's log lines for one phase (synthesis.py:190-194,
    204-205), emitted after the device loop: the gap at every 1000th
    iteration that continued, and the stalled-gap fallback warning."""
    if log.isEnabledFor(logging.INFO):
        for j, g in enumerate(gaps):
            log.info("iteration %d: gap %.3e", 1000 * (j + 1), g)
        if iterations // 1000 > len(gaps):
            log.info("(gap log kept for the first %d thousand iterations)",
                     len(gaps))
    if fallback:
        log.warning(
            "gap stuck at %.3e with both bounds self-converged "
            "(k0=%s, k1=%s); falling back to the value-iteration "
            "result on the lower track", gap, _report_k(k0), _report_k(k1))


DEFAULT_EPS = 1e-6
DEFAULT_MAX_ITERATIONS = 10**6
_BRACKET_TOL = 1e-9


@dataclass
class ValuePair:
    """Twin interval-iteration iterates (v0 from zeros, v1 from ones)."""
    v0: np.ndarray
    v1: np.ndarray

    def gap(self):
        return float(np.max(self.v1 - self.v0))

    def check_bracket(self):
        if np.any(self.v0 > self.v1 + _BRACKET_TOL):
            raise ImpactError("interval iteration bracket violated "
                              "(v0 > v1); abstraction bounds inconsistent")


@dataclass
class Controller:
    """Synthesis output: lookup table over the safe states."""
    states: np.ndarray
    coords: np.ndarray
    policy: np.ndarray | None
    inputs: np.ndarray | None
    p_min: np.ndarray
    p_max: np.ndarray
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if np.any(self.p_min > self.p_max):
            raise ImpactError("controller has p_min > p_max")


@dataclass
class PhaseReport:
    """One phase as run on the device."""
    pair: ValuePair
    policy: np.ndarray
    iterations: int
    k0: int | None
    k1: int | None
    fallback: bool
    gap: float
    ms_device: float
    ms_sweep: float = 0.0   # K5 launches alone (live, CUDA graph events)


def _report_k(k):
    return None if k is None else max(k - 1, 1)


def _spec_code(spec):
    if spec not in ("reach", "safety"):
        raise ValueError(f"bad spec {spec!r}")
    return _lib.SPEC_REACH if spec == "reach" else _lib.SPEC_SAFETY


def _lp_code(lp):
    if lp not in ("min", "max"):
        raise ValueError(f"bad direction {lp!r}")
    return _lib.LP_MAX if lp == "max" else _lib.LP_MIN


def _u_code(u_objective):
    if u_objective not in ("min", "max"):
        raise ValueError(f"bad u_objective {u_objective!r}")
    return 1 if u_objective == "max" else 0


def run_phase(imdp, spec, lp_direction, u_objective, eps, horizon,
              max_iterations, fixed_policy=None, mode=_lib.MODE_PHASE):
    """One reference _run_phase (synthesis.py:145-205) on the GPU."""
    h = imdp.device_handle()
    n_s = imdp.n_s
    desc = _lib.PhaseDesc()
    desc.spec = _spec_code(spec)
    desc.lp = _lp_code(lp_direction)
    desc.u_max = _u_code(u_objective)
    desc.mode = mode
    desc.eps = float(eps) if eps is not None else 0.0
    desc.horizon = int(horizon) if horizon is not None else 0
    desc.max_iterations = int(max_iterations)
    fixed = None
    if fixed_policy is not None:
        fixed = _lib.as_i64(fixed_policy)
        desc.fixed_policy = _lib.ptr(fixed, _lib.c_i64)
    v0 = np.empty(n_s)
    v1 = np.empty(n_s)
    pol = np.empty(n_s, dtype=np.int64)
    gaps = np.empty(GAP_LOG)
    out = _lib.PhaseOut()
    out.v0 = _lib.ptr(v0, _lib.c_dbl)
    out.v1 = _lib.ptr(v1, _lib.c_dbl)
    out.policy = _lib.ptr(pol, _lib.c_i64)
    out.gap_log = _lib.ptr(gaps, _lib.c_dbl)
    out.gap_log_cap = GAP_LOG
    st = _lib.load().imp_run_phase(h.raw, ctypes.byref(desc),
                                   ctypes.byref(out))
    k0 = None if out.k0 < 0 else int(out.k0)
    k1 = None if out.k1 < 0 else int(out.k1)
    log_phase(gaps[:out.gap_log_n], out.iterations, bool(out.fallback),
              float(out.gap), k0, k1)
    if st == _lib.IMP_E_CONVERGENCE:
        if mode == _lib.MODE_DIAGNOSE:
            raise ConvergenceError(
                f"no self-convergence within {max_iterations} iterations",
                k0=_report_k(k0), k1=_report_k(k1))
        raise ConvergenceError(
            f"gap {out.gap!r} above eps={eps!r} after {out.iterations} "
            f"iterations; per-bound self-convergence k0={_report_k(k0)}, "
            f"k1={_report_k(k1)} (use the larger as a finite horizon for "
            "plain value iteration)", k0=_report_k(k0), k1=_report_k(k1))
    _lib.check(st)
    return PhaseReport(ValuePair(v0, v1), pol, int(out.iterations), k0, k1,
                       bool(out.fallback), float(out.gap),
                       float(out.ms_device), float(out.ms_sweep))


def bellman_step(imdp, values, lp_direction, u_objective, spec,
                 fixed_policy=None, bounds=None, solver=None):
    """One robust Bellman update over all safe states -> (V', choice)."""
    spec_c = _spec_code(spec)
    lp_c = _lp_code(lp_direction)
    u_c = _u_code(u_objective)
    h = imdp.device_handle()
    v = _lib.as_f64(values)
    out = np.empty(imdp.n_s)
    pick = np.empty(imdp.n_s, dtype=np.int64)
    fixed = None if fixed_policy is None else _lib.as_i64(fixed_policy)
    _lib.check(_lib.load().imp_bellman_step(
        h.raw, _lib.ptr(v, _lib.c_dbl), spec_c, lp_c, u_c,
        _lib.ptr(fixed, _lib.c_i64), _lib.ptr(out, _lib.c_dbl),
        _lib.ptr(pick, _lib.c_i64)))
    if fixed is not None:
        pick = fixed.copy()
    return out, pick


def _check_args(eps, horizon, mode):
    if mode not in ("pessimistic", "optimistic"):
        raise ValueError(f"bad mode {mode!r}")
    if horizon is None:
        if not eps > 0:
            raise ValueError("eps must be positive for infinite horizon")
    elif not (isinstance(horizon, (int, np.integer)) and horizon >= 1):
        raise ValueError("horizon must be a positive integer or None")


def _make_controller(imdp, policy, p_min, p_max, kind, mode, eps, horizon,
                     phases, with_policy=True):
    p_max = np.maximum(p_min, p_max)
    coords = imdp.state_space.rep_points()[imdp.labels.safe]
    if with_policy and imdp.input_space is not None:
        inputs = imdp.input_space.rep_points()[policy]
    else:
        policy = None
        inputs = None
    meta = {"spec": kind, "mode": mode, "eps": eps,
            "horizon": "infinite" if horizon is None else int(horizon),
            "iterations": tuple(p.iterations for p in phases),
            "fallback": tuple(p.fallback for p in phases),
            "device_ms": tuple(p.ms_device for p in phases),
            "sweep_ms": tuple(p.ms_sweep for p in phases)}
    return Controller(states=np.asarray(imdp.labels.safe).copy(),
                      coords=coords, policy=policy, inputs=inputs,
                      p_min=p_min, p_max=p_max, meta=meta)


def _two_phases(imdp, spec, lp1, u_obj, eps, horizon, max_iterations):
    lp2 = "max" if lp1 == "min" else "min"
    ph1 = run_phase(imdp, spec, lp1, u_obj, eps, horizon, max_iterations)
    ph2 = run_phase(imdp, spec, lp2, u_obj, eps, horizon, max_iterations,
                    fixed_policy=ph1.policy)
    return ph1, ph2, lp2


def synthesize_reach(imdp, mode="pessimistic", eps=DEFAULT_EPS, horizon=None,
                     max_iterations=DEFAULT_MAX_ITERATIONS,
                     _with_policy=True, _kind="reach"):
    """Reachability / reach-avoid synthesis (synthesis.py:238-266)."""
    _check_args(eps, horizon, mode)
    lp1 = "min" if mode == "pessimistic" else "max"
    ph1, ph2, lp2 = _two_phases(imdp, "reach", lp1, "max", eps, horizon,
                                max_iterations)
    if horizon is not None or ph1.fallback:
        val1 = ph1.pair.v0
    else:
        val1 = ph1.pair.v0 if lp1 == "min" else ph1.pair.v1
    if horizon is not None or ph2.fallback:
        val2 = ph2.pair.v0
    else:
        val2 = ph2.pair.v1 if lp2 == "max" else ph2.pair.v0
    p_min, p_max = (val1, val2) if lp1 == "min" else (val2, val1)
    return _make_controller(imdp, ph1.policy, p_min, p_max, _kind, mode, eps,
                            horizon, (ph1, ph2), with_policy=_with_policy)


def synthesize_safe(imdp, mode="pessimistic", eps=DEFAULT_EPS, horizon=None,
                    max_iterations=DEFAULT_MAX_ITERATIONS,
                    _with_policy=True):
    """Safety via the complement of avoid-reach (synthesis.py:269-303)."""
    _check_args(eps, horizon, mode)
    if len(imdp.labels.target) != 0:
        raise ValueError("safety requires an empty target set")
    lp1 = "max" if mode == "pessimistic" else "min"
    ph1, ph2, lp2 = _two_phases(imdp, "safety", lp1, "min", eps, horizon,
                                max_iterations)
    if horizon is not None or ph1.fallback:
        avoid1 = ph1.pair.v0
    else:
        avoid1 = ph1.pair.v0 if lp1 == "max" else ph1.pair.v1
    if horizon is not None or ph2.fallback:
        avoid2 = ph2.pair.v0
    else:
        avoid2 = ph2.pair.v1 if lp2 == "min" else ph2.pair.v0
    if lp1 == "max":
        p_min, p_max = 1.0 - avoid1, 1.0 - avoid2
    else:
        p_min, p_max = 1.0 - avoid2, 1.0 - avoid1
    return _make_controller(imdp, ph1.policy, p_min, p_max, "safety", mode,
                            eps, horizon, (ph1, ph2),
                            with_policy=_with_policy)


def verify(imdp, mode="pessimistic", eps=DEFAULT_EPS, horizon=None,
           spec="safety", max_iterations=DEFAULT_MAX_ITERATIONS):
    """Verification of an input-free abstraction (synthesis.py:306-318)."""
    if imdp.input_space is not None:
        raise ValueError("verify requires an abstraction without inputs")
    if spec == "safety":
        return synthesize_safe(imdp, mode, eps, horizon, max_iterations,
                               _with_policy=False)
    if spec in ("reach", "reach-avoid"):
        return synthesize_reach(imdp, mode, eps, horizon, max_iterations,
                                _with_policy=False, _kind=spec)
    raise ValueError(f"bad spec {spec!r}")


def diagnose_convergence(imdp, spec="reach", mode="pessimistic",
                         eps=DEFAULT_EPS, max_iterations=DEFAULT_MAX_ITERATIONS):
    """Per-bound self-convergence iterations (synthesis.py:321-361)."""
    if spec == "safety":
        lp = "max" if mode == "pessimistic" else "min"
        u_obj, prog = "min", "safety"
    else:
        lp = "min" if mode == "pessimistic" else "max"
        u_obj, prog = "max", "reach"
    ph = run_phase(imdp, prog, lp, u_obj, eps, None, max_iterations,
                   mode=_lib.MODE_DIAGNOSE)
    return _report_k(ph.k0), _report_k(ph.k1)


def row_values(t_min, t_max, r_min, r_max, a_min, a_max, weights, lp,
               device=0):
    """Greedy-LP values of dense rows (the reference's RowsSolver.values,
    feasible.py:80-111) through K5: one value per row for the (n_s + 2)
    weights [V, w_target, w_avoid].  Rows of any stored length (< 2^20)."""
    from .abstraction import csr_from_dense, import_csr
    t_min = np.asarray(t_min, dtype=float)
    n_s = t_min.shape[1]
    ptr, col, lo, hi = csr_from_dense(t_min, t_max)
    h = import_csr(n_s, 1, 1, ptr, col, lo, hi, r_min, r_max, a_min, a_max,
                   device=device)
    w = _lib.as_f64(weights)
    if len(w) != n_s + 2:
        raise ValueError("weights must have n_s + 2 entries")
    out = np.empty(t_min.shape[0])
    _lib.check(_lib.load().imp_row_values(
        h.raw, _lib.ptr(w, _lib.c_dbl), 1 if lp == "max" else 0,
        _lib.ptr(out, _lib.c_dbl), 0))
    return out
