"""GPU construction vs the reference's golden abstractions (tests/golden).

Parity rules: bounds within 1e-9 absolute -- bit-for-bit for
dynamics without x-dependent library calls; live index sets
(t_max > zero_cutoff) exact except entries whose reference t_max lies within
1e-12 relative of the cutoff.
"""

import numpy as np
import pytest

from paper_2401_03555_b200 import (AbstractionError, AbstractionOptions,
                                   DiagonalNormal, DynamicsSpec,
                                   LabeledStates, build_abstraction,
                                   build_space, label_states,
                                   parse_expression, parse_predicate,
                                   synthesize_reach)
from paper_2401_03555_b200.expr import has_x_transcendental

from . import golden_io as G

pytestmark = pytest.mark.gpu
TOL = 1e-9
SINGLE_CELL_PROB = 0.3829249225480262


def make_dyn(texts, dims):
    return DynamicsSpec(tuple(parse_expression(t, dims) for t in texts), dims)


def all_safe(space):
    return LabeledStates(safe=np.arange(space.total),
                         target=np.array([], dtype=np.int64),
                         avoid=np.array([], dtype=np.int64),
                         total=space.total)


def compare_dense(got_min, got_max, ref_min, ref_max, cutoff=1e-12,
                  trig=False):
    """Bounds within TOL; for dynamics with x-dependent library calls
    (CUDA vs numpy sin/cos bits steer a few Nelder-Mead paths apart) at
    least 99% of entries within 1e-12 and all within the NM's own
    resolution (1e-6).  Live index sets exact (near-cutoff excepted)."""
    assert got_min.shape == ref_min.shape
    for got, ref in ((got_min, ref_min), (got_max, ref_max)):
        d = np.abs(got - ref)
        if trig:
            assert np.mean(d <= 1e-12) >= 0.99
            assert d.max() <= 1e-6
        else:
            assert d.max() <= TOL
    live_g = got_max > cutoff
    live_r = ref_max > cutoff
    near = np.abs(ref_max - cutoff) <= 1e-12 * cutoff
    assert not np.any((live_g != live_r) & ~near)


class TestKnownAnswers:
    def test_single_cell(self):
        sp = build_space([0.0], [0.0], [1.0])
        imdp = build_abstraction(make_dyn(["x1"], (1, 0, 0)),
                                 DiagonalNormal(np.array([1.0])),
                                 (sp, None, None), all_safe(sp))
        assert imdp.t_min[0, 0] == pytest.approx(SINGLE_CELL_PROB, abs=1e-12)
        assert imdp.t_max[0, 0] == pytest.approx(SINGLE_CELL_PROB, abs=1e-12)
        assert imdp.a_min[0] == pytest.approx(1 - SINGLE_CELL_PROB, abs=1e-12)
        assert imdp.a_max[0] == pytest.approx(1 - SINGLE_CELL_PROB, abs=1e-12)
        imdp.validate()

    def test_coupled_form_matches_separable(self):
        sp = build_space([-1, -1], [1, 1], [1, 1])
        noise = DiagonalNormal(np.array([0.8, 0.8]))
        dims = (2, 0, 0)
        sep = make_dyn(["0.6*x1", "0.9*x2"], dims)
        cpl = make_dyn(["0.6*x1 + 0*x2", "0.9*x2"], dims)
        assert sep.is_separable() and not cpl.is_separable()
        a = build_abstraction(sep, noise, (sp, None, None), all_safe(sp))
        b = build_abstraction(cpl, noise, (sp, None, None), all_safe(sp))
        for key in ("t_min", "t_max", "a_min", "a_max"):
            assert np.allclose(getattr(a, key), getattr(b, key), atol=1e-9)

    def test_row_invariants_and_low_cost(self):
        sp = build_space([-1, -1], [1, 1], [1, 1])
        noise = DiagonalNormal(np.array([0.8, 0.8]))
        dyn = make_dyn(["0.5*x1 + 0.3*x2", "x2"], (2, 0, 0))
        a = build_abstraction(dyn, noise, (sp, None, None), all_safe(sp),
                              AbstractionOptions(low_cost=False))
        b = build_abstraction(dyn, noise, (sp, None, None), all_safe(sp),
                              AbstractionOptions(low_cost=True))
        a.validate()
        assert np.array_equal(a.t_max, b.t_max)
        live = a.t_max > 1e-12
        assert np.array_equal(a.t_min[live], b.t_min[live])
        assert np.all(b.t_min[~live] == 0.0)

    def test_target_avoid_columns(self):
        sp = build_space([0], [4], [1])
        labels = label_states(sp, parse_predicate("x1 >= 4", 1),
                              parse_predicate("x1 <= 0", 1))
        imdp = build_abstraction(make_dyn(["x1"], (1, 0, 0)),
                                 DiagonalNormal(np.array([1.5])),
                                 (sp, None, None), labels)
        assert imdp.n_s == 3
        imdp.validate()
        assert imdp.r_max[1] > 0 and imdp.a_max[1] > 0
        assert imdp.t_min.shape == (3, 3)

    def test_inputs_and_disturbances_layout(self):
        sp = build_space([0], [4], [1])
        inp = build_space([0], [1], [1])
        imdp = build_abstraction(make_dyn(["x1 + 2*u1"], (1, 1, 0)),
                                 DiagonalNormal(np.array([0.8])),
                                 (sp, inp, None), all_safe(sp))
        assert imdp.n_rows == 10
        assert imdp.t_max[imdp.rows.row(0, 1), 2] > \
            imdp.t_max[imdp.rows.row(0, 0), 2]
        dist = build_space([-0.5], [0.5], [0.5])
        with_w = build_abstraction(make_dyn(["x1 + w1"], (1, 0, 1)),
                                   DiagonalNormal(np.array([0.8])),
                                   (sp, None, dist), all_safe(sp))
        without = build_abstraction(make_dyn(["x1"], (1, 0, 0)),
                                    DiagonalNormal(np.array([0.8])),
                                    (sp, None, None), all_safe(sp))
        assert with_w.n_rows == 15
        assert with_w.t_max[with_w.rows.row(0, 0, 1), 0] == pytest.approx(
            without.t_max[0, 0], abs=1e-12)

    def test_nonfinite_objective_raises(self):
        sp = build_space([0], [1], [1])
        dyn = make_dyn(["log(x1 - 5)"], (1, 0, 0))
        with pytest.raises(AbstractionError):
            build_abstraction(dyn, DiagonalNormal(np.array([1.0])),
                              (sp, None, None), all_safe(sp))


@pytest.mark.parametrize("name", G.MINIS)
def test_golden_abstraction(name):
    if not G.have("full_" + name):
        pytest.skip("fixture not generated")
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                             cfg.labels(), cfg.abstraction_options())
    ref_min, ref_max = G.dense(g)
    trig = has_x_transcendental(cfg.dynamics)
    compare_dense(imdp.t_min, imdp.t_max, ref_min, ref_max, trig=trig)
    for key in ("r_min", "r_max", "a_min", "a_max"):
        d = np.abs(getattr(imdp, key) - g[key])
        assert d.max() <= (1e-6 if trig else TOL), key
    if not trig:
        # affine dynamics: the whole construction is bit-for-bit the
        # reference's (cephes ndtr + glibc exp restated, --fmad=false)
        assert np.array_equal(imdp.t_min, ref_min)
        assert np.array_equal(imdp.t_max, ref_max)
    imdp.validate()


ROW_SAMPLES = ("robot2d_reachavoid", "vehicle3d", "room5d", "bas7d_verify",
               "dim14_verify", "robot2d_reach")


@pytest.mark.parametrize("name", ROW_SAMPLES)
def test_golden_rows_full_size(name):
    """Seeded rows of the full BASELINE configs, built as one-state shards
    (k_range) so the test does not need the whole abstraction."""
    if not G.have("rows_" + name):
        pytest.skip("fixture not generated")
    g = G.load("rows_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    per_k = int(g["n_u"]) * int(g["n_w"])
    trig = has_x_transcendental(cfg.dynamics)
    ptr, col, lo, hi = g["ptr"], g["col"], g["lo"], g["hi"]
    for q, row in enumerate(g["rows"]):
        k, rel = divmod(int(row), per_k)
        im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                               cfg.abstraction_options(), k_range=(k, 1))
        sp, scol, slo, shi, r0, r1, a0, a1 = im.csr()
        got_min = np.zeros(int(g["n_s"]))
        got_max = np.zeros_like(got_min)
        b, e = sp[rel], sp[rel + 1]
        got_min[scol[b:e]] = slo[b:e]
        got_max[scol[b:e]] = shi[b:e]
        ref_min = np.zeros_like(got_min)
        ref_max = np.zeros_like(got_min)
        rb, re_ = ptr[q], ptr[q + 1]
        ref_min[col[rb:re_]] = lo[rb:re_]
        ref_max[col[rb:re_]] = hi[rb:re_]
        compare_dense(got_min[None], got_max[None], ref_min[None],
                      ref_max[None], trig=trig)
        for key, got in (("r_min", r0), ("r_max", r1), ("a_min", a0),
                         ("a_max", a1)):
            assert abs(got[rel] - g[key][q]) <= (1e-6 if trig else TOL), key


def test_golden_robot2d_reach_end_to_end():
    """Full robot2d_reach (52 272 x 432): abstraction and controller against
    the reference run in full (BASELINE config 1's small sibling)."""
    if not G.have("full_robot2d_reach"):
        pytest.skip("fixture not generated")
    g = G.load("full_robot2d_reach")
    cfg = G.config_of(g)
    imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                             cfg.labels(), cfg.abstraction_options())
    ref_min, ref_max = G.dense(g)
    assert np.array_equal(imdp.t_min, ref_min)
    assert np.array_equal(imdp.t_max, ref_max)
    for key in ("r_min", "r_max", "a_min", "a_max"):
        assert np.max(np.abs(getattr(imdp, key) - g[key])) <= TOL
    c = synthesize_reach(imdp, mode=cfg.mode, eps=cfg.eps)
    assert tuple(c.meta["iterations"]) == tuple(g["iterations"])
    assert np.max(np.abs(c.p_min - g["p_min"])) <= TOL
    assert np.max(np.abs(c.p_max - g["p_max"])) <= TOL
    diff = c.policy != g["policy"]
    tight = g["margin"] <= 1e-12
    assert not np.any(diff & ~tight)
    k = np.flatnonzero(diff)
    per_u = g["per_u"]
    assert np.all(np.abs(per_u[k, c.policy[k]] - per_u[k, g["policy"][k]])
                  <= 1e-12)
