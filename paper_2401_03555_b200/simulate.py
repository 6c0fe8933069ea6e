"""Closed-loop rollouts of a controller on the GPU.

Drop-in for the reference's `impact simulate` (pkg/src/impact/cli.py:
163-251, cmd_simulate): the same rollout semantics, random streams, CSV
format and summary, with every rollout a GPU thread of the JIT module
(csrc/jit/simulate.cuh; numpy's SeedSequence / Philox / ziggurat normal
restated in csrc/rng.h).  For dynamics without x-dependent library calls
the CSV is byte-identical to the reference's.

    res = simulate(cfg, controller, rollouts=1000, steps=50)
    res.write_csv("rollouts.csv"); print(res.summary())
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .abstraction import describe
from .errors import ConfigError, EvalError, FileFormatError
from .expr import lower_dynamics
from .fileio import format_reals
from .noise import CustomNoise, DiagonalNormal, FullNormal

__all__ = ["simulate", "Rollouts"]


@dataclass
class Rollouts:
    trace: np.ndarray        # (rollouts, steps + 1, n); rows < length valid
    length: np.ndarray       # (rollouts,) trace points per rollout
    satisfied: np.ndarray    # (rollouts,) bool
    visited: np.ndarray      # controller slots the rollouts started from
    p_min: np.ndarray        # controller bounds (for the summary)
    p_max: np.ndarray

    @property
    def rollouts(self):
        return len(self.length)

    def csv_bytes(self, device=0) -> bytes:
        """cli.py:231-240: header, then per rollout and step
        `r,step,x1,...,xn,satisfied` with format(v, ".17g")."""
        n = self.trace.shape[2]
        pts = np.concatenate([self.trace[r, :self.length[r]]
                              for r in range(self.rollouts)])
        text = format_reals(pts, n, device).decode().split("\n")
        head = "rollout,step," + ",".join(f"x{d + 1}" for d in range(n)) + \
            ",satisfied\n"
        out = [head]
        q = 0
        for r in range(self.rollouts):
            sat = int(self.satisfied[r])
            for step in range(int(self.length[r])):
                out.append(f"{r},{step},{text[q].replace(' ', ',')},{sat}\n")
                q += 1
        return "".join(out).encode()

    def write_csv(self, path, device=0):
        try:
            with open(path, "wb") as fh:
                fh.write(self.csv_bytes(device))
        except OSError as exc:
            raise FileFormatError(f"cannot write {path}: {exc}")

    def summary(self, steps=None):
        frac = float(np.mean(self.satisfied)) if self.rollouts else 0.0
        v = self.visited
        lines = [f"rollouts: {self.rollouts}, steps: "
                 f"{steps if steps is not None else self.trace.shape[1] - 1}",
                 f"empirical satisfaction: {frac:.4f}",
                 f"controller bounds over start states: "
                 f"[{float(np.mean(self.p_min[v])):.4f}, "
                 f"{float(np.mean(self.p_max[v])):.4f}]"]
        return "\n".join(lines)


def simulate(cfg, ctrl, rollouts, steps, start_pmin=None, device=0):
    """Rollouts of `ctrl` under cfg's dynamics and noise (cli.py:177-251).

    cfg: a RunConfig (config.load_config / parse_config_text); ctrl: a
    Controller (synthesis result or fileio.load_controller)."""
    if ctrl.coords.shape[1] != cfg.state_space.dim:
        raise ConfigError("controller dimension does not match [state]")
    if rollouts < 1 or steps < 1:
        raise ConfigError("--rollouts and --steps must be >= 1")
    noise = cfg.noise
    if isinstance(noise, CustomNoise):
        raise ConfigError("simulate supports normal noise only; custom "
                          "densities have no built-in sampler")
    if isinstance(noise, FullNormal):
        raise ConfigError("full-covariance noise: simulate on the B200 path "
                          "samples diagonal normal noise only")
    if not isinstance(noise, DiagonalNormal):
        raise ConfigError("no noise model configured")
    labels = cfg.labels()
    state = cfg.state_space
    starts = np.arange(len(ctrl.states))
    if start_pmin is not None:
        starts = starts[ctrl.p_min >= start_pmin]
        if len(starts) == 0:
            raise ConfigError(f"no states with p_min >= {start_pmin}")
    reach_like = cfg.spec_type in ("reach", "reach-avoid")
    inp, dist = cfg.input_space, cfg.disturb_space
    w_center = ((dist.lb + dist.ub) / 2 if dist is not None
                else np.zeros(0))
    u_reps = inp.rep_points() if inp is not None else np.zeros((1, 0))

    # geometry + generated dynamics of the construction module, constants
    # folded at (u_j, disturbance centre)
    desc, keep = describe(cfg.dynamics, noise, cfg.spaces, labels,
                          cfg.abstraction_options(), device=device)
    lowered = lower_dynamics(cfg.dynamics, u_reps, w_center[None, :])
    consts = _lib.as_f64(lowered.consts)
    desc.consts = _lib.ptr(consts, _lib.c_dbl)
    desc.n_consts = lowered.consts.shape[1]

    total = int(state.total)
    slot_of = np.full(total, -1, dtype=np.int32)
    slot_of[np.asarray(ctrl.states, dtype=np.int64)] = \
        np.arange(len(ctrl.states), dtype=np.int32)
    kind = np.zeros(total, dtype=np.uint8)
    kind[np.asarray(labels.target, dtype=np.int64)] = 2
    kind[np.asarray(labels.avoid, dtype=np.int64)] = 1
    if ctrl.policy is not None:
        slot_input = np.asarray(ctrl.policy, dtype=np.int32)
    else:
        slot_input = np.zeros(len(ctrl.states), dtype=np.int32)
    if slot_input.size and (slot_input.min() < 0 or
                            slot_input.max() >= len(u_reps)):
        raise ConfigError("controller inputs do not match [input]")
    arrays = dict(starts=_lib.as_i32(starts), slot_input=_lib.as_i32(slot_input),
                  slot_of=slot_of, coords=_lib.as_f64(ctrl.coords),
                  lb=_lib.as_f64(state.lb), ub=_lib.as_f64(state.ub),
                  kind=np.ascontiguousarray(kind))
    sd = _lib.SimDesc()
    sd.rollouts, sd.steps = int(rollouts), int(steps)
    sd.seed = int(cfg.seed) & (2**64 - 1)
    sd.reach_like = int(reach_like)
    sd.n_starts = len(starts)
    sd.starts = _lib.ptr(arrays["starts"], _lib.c_i32)
    sd.n_ctrl = len(ctrl.states)
    sd.coords = _lib.ptr(arrays["coords"], _lib.c_dbl)
    sd.slot_input = _lib.ptr(arrays["slot_input"], _lib.c_i32)
    sd.total = total
    sd.slot_of = _lib.ptr(arrays["slot_of"], _lib.c_i32)
    sd.kind = arrays["kind"].ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    sd.lb = _lib.ptr(arrays["lb"], _lib.c_dbl)
    sd.ub = _lib.ptr(arrays["ub"], _lib.c_dbl)
    n = state.dim
    trace = np.zeros((rollouts, steps + 1, n))
    length = np.zeros(rollouts, dtype=np.int32)
    sat = np.zeros(rollouts, dtype=np.int32)
    st = _lib.load().imp_simulate(ctypes.byref(desc), ctypes.byref(sd),
                                  _lib.ptr(trace, _lib.c_dbl),
                                  _lib.ptr(length, _lib.c_i32),
                                  _lib.ptr(sat, _lib.c_i32))
    if st == _lib.IMP_E_NONFINITE:
        raise EvalError(_lib.last_error())
    _lib.check(st)
    del keep
    visited = np.array(sorted(set(int(starts[r % len(starts)])
                                  for r in range(rollouts))))
    return Rollouts(trace=trace, length=length, satisfied=sat.astype(bool),
                    visited=visited, p_min=np.asarray(ctrl.p_min),
                    p_max=np.asarray(ctrl.p_max))
