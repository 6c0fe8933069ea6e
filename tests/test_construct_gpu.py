"""GPU construction vs the reference's golden abstractions (tests/golden).

Parity rules:
  * live index sets (t_max > zero_cutoff) exact in both construction modes,
    except entries whose reference t_max lies within 1e-12 relative of the
    cutoff;
  * default (exact=True) and dynamics without x-dependent library calls:
    bit for bit;
  * default and x-dependent trig (vehicle3d: CUDA vs numpy sin / cos): a
    Nelder-Mead run whose comparisons flip on an ulp-level near-tie follows
    a different path and stops elsewhere inside its own stopping tolerance
    (optimize.py:80-83, tol = 1e-8 on the simplex spread): >= 99.9 % of
    entries within FAST_TOL = 1e-12 and all within NM_TOL = 1e-8.
    Observed on the 237 896 golden vehicle3d entries: 11 above 1e-12, max
    1.0e-9; the REFERENCE against itself with its sin / cos results moved
    one ulp: 60 above 1e-12, max 3.2e-9 (profiles/r02/row_parity_*.json,
    ref_floor_*.json);
  * opt-in fast objective (exact=False, CDFs within a few ulps of scipy's):
    >= 99.9 % of entries within 1e-12 -- a flipped near-tie can also send a
    run to another local optimum (once, 1.0e-3, on room5d_mini).
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
FAST_TOL = 1e-12
NM_TOL = 1e-8
SINGLE_CELL_PROB = 0.3829249225480262
MODES = (True, False)    # exact, fast


def make_dyn(texts, dims):
    return DynamicsSpec(tuple(parse_expression(t, dims) for t in texts), dims)


def all_safe(space):
    return LabeledStates(safe=np.arange(space.total),
                         target=np.array([], dtype=np.int64),
                         avoid=np.array([], dtype=np.int64),
                         total=space.total)


def compare_dense(got_min, got_max, ref_min, ref_max, cutoff=1e-12,
                  trig=False, exact=True):
    """The module docstring's rules; returns the largest deviation."""
    assert got_min.shape == ref_min.shape
    worst = 0.0
    for got, ref in ((got_min, ref_min), (got_max, ref_max)):
        d = np.abs(got - ref)
        worst = max(worst, float(d.max(initial=0.0)))
        if not exact:
            # opt-in fast objective: NM paths that flip on an ulp-level
            # near-tie may stop at another local optimum (observed once on
            # room5d_mini: 1.0e-3), so only the bulk is bounded
            assert np.mean(d <= FAST_TOL) >= 0.999
        elif trig:
            assert np.mean(d <= FAST_TOL) >= 0.999
            assert d.max() <= NM_TOL
        else:
            assert np.array_equal(got, ref)
    live_g = got_max > cutoff
    live_r = ref_max > cutoff
    near = np.abs(ref_max - cutoff) <= 1e-12 * cutoff
    assert not np.any((live_g != live_r) & ~near)
    return worst


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


def vec_tol(trig, exact):
    """r / a vectors: sums of entries, in block-tree order (not numpy's
    pairwise order), so never compared bitwise."""
    if not exact:
        return 1e-2
    return TOL if not trig else NM_TOL


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("name", G.MINIS)
def test_golden_abstraction(name, exact):
    if not G.have("full_" + name):
        pytest.skip("fixture not generated")
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                             cfg.labels(), cfg.abstraction_options(),
                             exact=exact)
    ref_min, ref_max = G.dense(g)
    trig = has_x_transcendental(cfg.dynamics)
    # affine dynamics, exact: the whole construction is bit-for-bit the
    # reference's (cephes ndtr + glibc exp restated, --fmad=false)
    compare_dense(imdp.t_min, imdp.t_max, ref_min, ref_max, trig=trig,
                  exact=exact)
    for key in ("r_min", "r_max", "a_min", "a_max"):
        d = np.abs(getattr(imdp, key) - g[key])
        assert d.max() <= vec_tol(trig, exact), key
    imdp.validate()


ROW_SAMPLES = ("robot2d_reachavoid", "vehicle3d", "room5d", "bas7d_verify",
               "dim14_verify", "robot2d_reach")


@pytest.mark.parametrize("exact", MODES)
@pytest.mark.parametrize("name", ROW_SAMPLES)
def test_golden_rows_full_size(name, exact):
    """Seeded + stratified rows of the full BASELINE configs (boundary
    states, states next to target / avoid, every input), built as
    one-state shards (k_range) so the test does not need the whole
    abstraction.  Trig dynamics: the >= 99.9 % rule over all sampled
    entries together."""
    if not G.have("rows_" + name):
        pytest.skip("fixture not generated")
    g = G.load("rows_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    per_k = int(g["n_u"]) * int(g["n_w"])
    trig = has_x_transcendental(cfg.dynamics)
    ptr, col, lo, hi = g["ptr"], g["col"], g["lo"], g["hi"]
    got_all, ref_all = [], []
    built = {}
    for q, row in enumerate(g["rows"]):
        k, rel = divmod(int(row), per_k)
        if k not in built:
            built = {k: build_abstraction(
                cfg.dynamics, cfg.noise, cfg.spaces, labels,
                cfg.abstraction_options(), k_range=(k, 1),
                exact=exact).csr()}
        sp, scol, slo, shi, r0, r1, a0, a1 = built[k]
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
        got_all.append(np.stack([got_min, got_max]))
        ref_all.append(np.stack([ref_min, ref_max]))
        for key, got in (("r_min", r0), ("r_max", r1), ("a_min", a0),
                         ("a_max", a1)):
            assert abs(got[rel] - g[key][q]) <= vec_tol(trig, exact), key
    got_all, ref_all = np.stack(got_all), np.stack(ref_all)
    compare_dense(got_all[:, 0], got_all[:, 1], ref_all[:, 0], ref_all[:, 1],
                  trig=trig, exact=exact)


def test_golden_robot2d_reach_end_to_end():
    """Full robot2d_reach (52 272 x 432): abstraction and controller against
    the reference run in full (BASELINE config 1's small sibling)."""
    if not G.have("full_robot2d_reach"):
        pytest.skip("fixture not generated")
    g = G.load("full_robot2d_reach")
    cfg = G.config_of(g)
    imdp = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                             cfg.labels(), cfg.abstraction_options(),
                             exact=True)
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


@pytest.mark.parametrize("which", (0, 1, 2))
def test_device_ndtr_forms_vs_scipy(which):
    """The k_refine objective's device CDFs on the 104 k scipy golden
    samples (noise.py:116-118): the exact forms (0: round 1, 1: the default
    objective's integer-classified / inline-quotient form) bit for bit;
    the fast fused form (2) within 16 ulps relative and 4.5e-16 absolute
    (measured: <= 12 ulps, worst next to cephes' erf / erfc switch where
    1 - erf cancels; profiles/r02/ndtr_fast_err.txt)."""
    from paper_2401_03555_b200.abstraction import device_ndtr
    g = G.load("ndtr")
    got = device_ndtr(g["x"], which)
    want = g["y"]
    if which < 2:
        assert np.array_equal(got, want, equal_nan=True)
    else:
        # the fused form stands in P / Q for cephes' R / S at |x| >= 8 sqrt2
        # (CDF 1 exactly, or below 1e-29): absolute agreement there
        x = g["x"]
        fin = np.isfinite(x)
        err = np.abs(got[fin] - want[fin])
        core = np.abs(x[fin]) < 8 * np.sqrt(2)
        assert np.all(err[core] <= 16 * np.spacing(np.abs(want[fin][core])))
        assert np.all(err[core] <= 4.5e-16)
        assert np.all(err[~core] <= 1e-28)
        assert np.array_equal(got[~fin], want[~fin], equal_nan=True)
