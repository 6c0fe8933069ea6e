"""Full BASELINE-size checks through size-independent properties.

The CPU reference cannot build or solve these configs in test time (room5d
alone is ~450 core-hours), so parity at full size rests on
properties that must hold for the reference's exact semantics:

* construction: the validate() invariants of every row (abstraction.py:
  121-137) and, for sampled rows, bitwise agreement with one-state shard
  builds (position independence);
* synthesis: the bracket p_min <= p_max in [0, 1]; the returned bounds are
  (eps-)fixed points of the reference's Bellman operator (synthesis.py:
  97-135) evaluated through the same API; sharded sweeps equal the single
  handle bit for bit;
* dim14: the scalar recursion V' = a + (1 - a) V of its symmetric rows
  (SURVEY.md finding 7) for the first sweeps.
"""

import numpy as np
import pytest

from paper_2401_03555_b200 import (bellman_step, build_abstraction,
                                   synthesize_reach, verify)
from paper_2401_03555_b200.config import benchmark

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ra():
    cfg = benchmark("robot2d_reachavoid")
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                           cfg.abstraction_options())
    return cfg, im


def test_robot2d_reachavoid_rows_valid_and_position_independent(ra):
    cfg, im = ra
    im.validate()
    ptr, col, lo, hi, r0, r1, a0, a1 = im.csr()
    rng = np.random.default_rng(4)
    n_u = im.n_u
    for k in rng.choice(im.n_s, 3, replace=False):
        sh = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                               cfg.labels(), cfg.abstraction_options(),
                               k_range=(int(k), 1))
        sp, sc, sl, shh, s0, s1, t0, t1 = sh.csr()
        b, e = ptr[k * n_u], ptr[(k + 1) * n_u]
        assert np.array_equal(sc, col[b:e])
        assert np.array_equal(sl, lo[b:e])
        assert np.array_equal(shh, hi[b:e])
        rows = slice(k * n_u, (k + 1) * n_u)
        for got, want in ((s0, r0), (s1, r1), (t0, a0), (t1, a1)):
            assert np.array_equal(got, want[rows])


def test_robot2d_reachavoid_controller_is_a_bellman_fixed_point(ra):
    cfg, im = ra
    eps = cfg.eps
    c = synthesize_reach(im, mode=cfg.mode, eps=eps)
    assert np.all((0 <= c.p_min) & (c.p_min <= c.p_max) & (c.p_max <= 1))
    # pessimistic reach: p_min is phase 1's lower iterate under the min-LP
    nxt, pol = bellman_step(im, c.p_min, "min", "max", "reach")
    assert np.all(nxt >= c.p_min - 1e-12)         # monotone from below
    assert np.max(nxt - c.p_min) <= eps           # converged to eps
    # the returned policy (extracted one sweep earlier) is eps-optimal at
    # the fixed point
    fixed, _ = bellman_step(im, c.p_min, "min", "max", "reach",
                            fixed_policy=c.policy)
    assert np.all(fixed <= nxt + 1e-12)
    assert np.max(nxt - fixed) <= eps


def test_robot2d_reachavoid_shards_bitwise(ra):
    import torch
    from paper_2401_03555_b200.sharded import shard_range, shard_sweep
    cfg, im = ra
    rng = np.random.default_rng(9)
    v = rng.uniform(0, 1, im.n_s)
    want, wpick = bellman_step(im, v, "min", "max", "reach")
    vt = torch.tensor(v, dtype=torch.float64, device="cuda")
    got, gpick = [], []
    for r in range(4):
        sh = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                               cfg.labels(), cfg.abstraction_options(),
                               k_range=shard_range(im.n_s, 4, r))
        n0, _, pol, _ = shard_sweep(sh, vt, vt, 0, 0, 1)
        got.append(n0.cpu().numpy())
        gpick.append(pol.cpu().numpy())
    assert np.array_equal(np.concatenate(got), want)
    assert np.array_equal(np.concatenate(gpick), wpick)


def test_dim14_scalar_recursion():
    """dim14 (16 384 states, every row identical up to symmetry): after k
    phase-1 sweeps V0_k = 1 - (1 - a)^k: the scalar
    recursion V' = a + (1 - a) V of the max-LP (SURVEY.md finding 7)."""
    cfg = benchmark("dim14_verify")
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                           cfg.abstraction_options())
    a = im.a_max
    assert np.max(a) - np.min(a) <= 1e-12
    c = verify(im, spec="safety", horizon=10)
    want = (1.0 - a) ** 10          # p_min = 1 - V0_10, V0_k = 1 - (1-a)^k
    assert np.max(np.abs(c.p_min - want)) <= 1e-12
