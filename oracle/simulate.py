"""Closed-loop rollouts -- oracle restatement (TEST INFRASTRUCTURE).

Restates pkg/src/impact/cli.py:163-251 (`impact simulate`): per rollout r
the generator Generator(Philox(SeedSequence(derive_seed(seed, r, 0))))
(noise.py:121-131), start state ctrl slot starts[r % len(starts)], steps of
quantize (grid.py:118-132) -> avoid / target / controller lookup ->
x = f(x, u, w_centre) + rng.normal(0, sigma), and the CSV / summary text.
numpy is the reference's own dependency for the random streams.  Pinned to
the reference CLI's output (tests/golden/simulate_digests.json).
"""

import numpy as np


def derive_seed(base, row, dest):
    ss = np.random.SeedSequence(entropy=int(base) & (2**64 - 1),
                                spawn_key=(int(row), int(dest)))
    return int(ss.generate_state(1, np.uint64)[0])


def generator(seed):
    return np.random.Generator(np.random.Philox(
        np.random.SeedSequence(entropy=int(seed) & (2**64 - 1))))


def quantize(lb, ub, eta, counts, x):
    """grid.py:118-132; None outside the covered domain."""
    half = eta / 2
    tol = 1e-9 * np.maximum(eta, 1.0)
    if np.any(x < lb - half - tol) or np.any(x > ub + half + tol):
        return None
    idx = np.ceil((x - lb) / eta - 0.5).astype(int)
    idx = np.clip(idx, 0, counts - 1)
    flat = 0
    for d in range(len(counts)):
        flat = flat * int(counts[d]) + int(idx[d])
    return flat


def simulate(cfg, ctrl, rollouts, steps, start_pmin=None):
    """-> (csv bytes, summary text) exactly as the reference CLI."""
    labels = cfg.labels()
    sp = cfg.state_space
    target = set(int(i) for i in labels.target)
    avoid = set(int(i) for i in labels.avoid)
    by_state = {int(s): k for k, s in enumerate(ctrl.states)}
    starts = np.arange(len(ctrl.states))
    if start_pmin is not None:
        starts = starts[ctrl.p_min >= start_pmin]
    w_c = ((cfg.disturb_space.lb + cfg.disturb_space.ub) / 2
           if cfg.disturb_space is not None else np.zeros(0))
    reach_like = cfg.spec_type in ("reach", "reach-avoid")
    sigma = cfg.noise.sigma
    n = sp.dim
    rows, ok, visited = [], 0, []
    for r in range(rollouts):
        rng = generator(derive_seed(cfg.seed, r, 0))
        k = int(starts[r % len(starts)])
        visited.append(k)
        x = ctrl.coords[k].copy()
        sat = not reach_like
        trace = [(0, x.copy())]
        for step in range(1, steps + 1):
            s = quantize(sp.lb, sp.ub, sp.eta, sp.counts, x)
            if s is None or s in avoid:
                sat = False
                break
            if reach_like and s in target:
                sat = True
                break
            slot = by_state.get(s)
            if slot is None:
                sat = False
                break
            u = ctrl.inputs[slot] if ctrl.inputs is not None else np.zeros(0)
            x = cfg.dynamics.eval(x, u, w_c) + rng.normal(0.0, sigma)
            trace.append((step, x.copy()))
        ok += bool(sat)
        rows += [(r, st, pt, int(sat)) for st, pt in trace]
    head = "rollout,step," + ",".join(f"x{d + 1}" for d in range(n)) + \
        ",satisfied\n"
    body = "".join(f"{r},{st}," + ",".join(format(v, ".17g") for v in pt)
                   + f",{sat}\n" for r, st, pt, sat in rows)
    v = np.array(sorted(set(visited)))
    summary = (f"rollouts: {rollouts}, steps: {steps}\n"
               f"empirical satisfaction: {ok / rollouts:.4f}\n"
               f"controller bounds over start states: "
               f"[{float(np.mean(ctrl.p_min[v])):.4f}, "
               f"{float(np.mean(ctrl.p_max[v])):.4f}]\n")
    return (head + body).encode(), summary
