"""GPU interval iteration vs the oracle and the reference's golden outputs.

Parity rules: values within 1e-9 (expected ~1e-15);
policies equal wherever the reference's top-2 margin exceeds 1e-12, else
the GPU's input must be epsilon-optimal; iteration counts equal.
"""

import numpy as np
import pytest

from paper_2401_03555_b200 import (ConvergenceError, Imdp, LabeledStates,
                                   bellman_step, build_space,
                                   diagnose_convergence, synthesize_reach,
                                   synthesize_safe, verify)
from paper_2401_03555_b200.synthesis import run_phase

from oracle import iterate as ORI

from . import golden_io as G

pytestmark = pytest.mark.gpu
TOL = 1e-9


def make_imdp(t_min, t_max, r_min, r_max, a_min, a_max, n_u=1, n_w=1):
    t_min = np.asarray(t_min, dtype=float)
    n_s = t_min.shape[1]
    state = build_space([0.0], [float(n_s - 1)], [1.0])
    labels = LabeledStates(safe=np.arange(n_s),
                           target=np.array([], dtype=np.int64),
                           avoid=np.array([], dtype=np.int64), total=n_s)
    inp = build_space([0.0], [float(n_u - 1)], [1.0]) if n_u > 1 else None
    dist = build_space([0.0], [float(n_w - 1)], [1.0]) if n_w > 1 else None
    return Imdp(state, inp, dist, labels, t_min, np.asarray(t_max, float),
                np.asarray(r_min, float), np.asarray(r_max, float),
                np.asarray(a_min, float), np.asarray(a_max, float))


def chain(r, a, t):
    return make_imdp([[t]], [[t]], [r], [r], [a], [a])


def oracle_model(m):
    return ORI.Model(m.n_s, m.n_u, m.n_w, m.t_min, m.t_max, m.r_min,
                     m.r_max, m.a_min, m.a_max)


def random_imdp(rng, n_s, n_u=1, n_w=1, width=0.3, density=1.0):
    rows = n_s * n_u * n_w
    full = rng.dirichlet(np.ones(n_s + 2), size=rows)
    if density < 1.0:
        keep = rng.random((rows, n_s + 2)) < density
        keep[:, -1] = True
        full = full * keep
        full /= full.sum(axis=1, keepdims=True)
    lo = full * (1 - width)
    hi = np.minimum(1.0, full * (1 + width) + 1e-4 * (full > 0))
    return make_imdp(lo[:, :n_s], hi[:, :n_s], lo[:, n_s], hi[:, n_s],
                     lo[:, n_s + 1], hi[:, n_s + 1], n_u=n_u, n_w=n_w)


def per_input(om, v, lp, u_obj, spec):
    """Oracle per-(state, input) values after the min / max over
    disturbances (synthesis.py:118-131)."""
    rows = ORI.phase_rows(om, ORI.stacked(om))
    tail = [1.0, 0.0] if spec == "reach" else [0.0, 1.0]
    vals = rows.values(np.concatenate([np.asarray(v, float), tail]), lp)
    per = vals.reshape(om.n_s, om.n_u, om.n_w)
    return per.min(axis=2) if u_obj == "max" else per.max(axis=2)


def assert_policy_margin_aware(om, v, lp, u_obj, spec, pick, wpick,
                               tie=1e-12):
    """equal choices wherever the oracle's top-2 margin
    exceeds `tie`; elsewhere the GPU's choice must be tie-optimal."""
    per_u = per_input(om, v, lp, u_obj, spec)
    srt = np.sort(per_u, axis=1)
    if om.n_u == 1:
        assert np.array_equal(pick, wpick)
        return
    margin = srt[:, -1] - srt[:, -2] if u_obj == "max" else srt[:, 1] - srt[:, 0]
    diff = np.asarray(pick) != np.asarray(wpick)
    assert not np.any(diff & (margin > tie))
    k = np.flatnonzero(diff)
    assert np.all(np.abs(per_u[k, np.asarray(pick)[k]] -
                         per_u[k, np.asarray(wpick)[k]]) <= tie)


class TestBellmanStep:
    def test_scalar_affine_map(self):
        m = chain(0.2, 0.0, 0.8)
        for v in (0.0, 0.3, 1.0):
            out, _ = bellman_step(m, np.array([v]), "min", "max", "reach")
            assert out[0] == pytest.approx(0.2 + 0.8 * v, abs=1e-15)

    def test_two_inputs_safety_picks_smaller_avoid(self):
        t = np.array([[0.8], [0.5]])
        m = make_imdp(t, t, [0, 0], [0, 0], [0.2, 0.5], [0.2, 0.5], n_u=2)
        vals, chosen = bellman_step(m, np.ones(1), "max", "min", "safety")
        assert chosen[0] == 0
        assert vals[0] == pytest.approx(1.0, abs=1e-15)

    def test_fixed_policy_only_prices_chosen_input(self):
        t = np.array([[0.5], [0.9]])
        m = make_imdp(t, t, [0.5, 0.1], [0.5, 0.1], [0, 0], [0, 0], n_u=2)
        _, chosen = bellman_step(m, np.zeros(1), "min", "max", "reach")
        assert chosen[0] == 0
        forced, _ = bellman_step(m, np.zeros(1), "min", "max", "reach",
                                 fixed_policy=np.array([1]))
        assert forced[0] == pytest.approx(0.1, abs=1e-15)

    @pytest.mark.parametrize("seed", range(6))
    @pytest.mark.parametrize("lp", ["min", "max"])
    def test_random_rows_match_oracle(self, seed, lp):
        rng = np.random.default_rng(seed)
        n_s = int(rng.integers(3, 300))
        n_u = int(rng.integers(1, 5))
        n_w = int(rng.integers(1, 3))
        m = random_imdp(rng, n_s, n_u, n_w, density=rng.uniform(0.05, 1.0))
        om = oracle_model(m)
        v = rng.uniform(0, 1, n_s)
        v[rng.random(n_s) < 0.2] = 0.5        # exact ties in the order
        for spec, u_obj in (("reach", "max"), ("safety", "min")):
            got, pick = bellman_step(m, v, lp, u_obj, spec)
            want, wpick = ORI.bellman(om, v, lp, u_obj, spec)
            assert np.max(np.abs(got - want)) <= 1e-13
            assert_policy_margin_aware(om, v, lp, u_obj, spec, pick, wpick)


    @pytest.mark.parametrize("n_s", [20000, 70000])
    def test_rows_wider_than_16384_entries(self, n_s):
        """Rows of 20 k / 70 k stored entries (beyond round 1's 16 384-entry
        cap; 70 k also needs 32-bit ranks) against the oracle's Rows.values
        (feasible.py:80-111), both LP directions.  A one-state-per-row shard
        swept repeatedly through imp_shard_sweep keeps its crossing hints,
        so small value moves take the window walk and large ones the
        bucketed search; imp_row_values (no hints) searches every row."""
        import ctypes
        import torch
        from paper_2401_03555_b200 import _lib
        from paper_2401_03555_b200.abstraction import (csr_from_dense,
                                                       import_csr)
        from paper_2401_03555_b200.synthesis import row_values
        from oracle.lp import Rows
        rng = np.random.default_rng(11)
        rows = 6
        full = rng.dirichlet(np.ones(n_s + 2), size=rows)
        lo = full * 0.7
        hi = np.minimum(1.0, full * 1.3 + 1e-7)
        t_min, t_max = lo[:, :n_s], hi[:, :n_s]
        orows = Rows(lo, hi)
        ptr, col, clo, chi = csr_from_dense(t_min, t_max)
        vec = (lo[:, n_s], hi[:, n_s], lo[:, n_s + 1], hi[:, n_s + 1])
        h = import_csr(n_s, 1, 1, ptr, col, clo, chi, *vec)
        dev = torch.device("cuda", 0)
        new0 = torch.empty(rows, dtype=torch.float64, device=dev)
        new1 = torch.empty_like(new0)
        pol = torch.empty(rows, dtype=torch.int64, device=dev)
        stats = torch.empty(5, dtype=torch.float64, device=dev)
        v = rng.uniform(0, 1, n_s)
        for sweep in range(6):
            if sweep == 3:
                v = rng.uniform(0, 1, n_s)            # far move: search
            else:
                v = np.clip(v + rng.normal(0, 1e-4, n_s), 0, 1)  # walk
            v[rng.random(n_s) < 0.05] = 0.25       # exact ties
            w = np.concatenate([v, [1.0, 0.0]])
            vt = torch.tensor(v, dtype=torch.float64, device=dev)
            for lp in ("min", "max"):
                want = orows.values(w, lp)
                got = row_values(t_min, t_max, *vec, w, lp)
                assert np.max(np.abs(got - want)) <= 1e-12
                stream = torch.cuda.current_stream(dev).cuda_stream
                _lib.check(_lib.load().imp_shard_sweep(
                    h.raw, vt.data_ptr(), vt.data_ptr(), 0,
                    1 if lp == "max" else 0, 1, None, new0.data_ptr(),
                    new1.data_ptr(), pol.data_ptr(), stats.data_ptr(),
                    ctypes.c_void_p(stream)))
                got = new0.cpu().numpy()
                assert np.max(np.abs(got - want)) <= 1e-12
                assert np.array_equal(got, new1.cpu().numpy())


class TestHandChains:
    def test_reach_infinite_geometric(self):
        c = synthesize_reach(chain(0.2, 0.0, 0.8), eps=1e-10)
        assert c.p_min[0] == pytest.approx(1.0, abs=1e-9)
        assert c.p_max[0] == pytest.approx(1.0, abs=1e-9)

    def test_reach_two_steps(self):
        c = synthesize_reach(chain(0.2, 0.0, 0.8), horizon=2)
        assert c.p_min[0] == pytest.approx(0.36, abs=1e-9)

    def test_certain_target_one_iteration(self):
        c = synthesize_reach(chain(1.0, 0.0, 0.0), eps=1e-9)
        assert c.p_min[0] == 1.0 and c.p_max[0] == 1.0
        assert c.meta["iterations"][0] == 1

    def test_safety_infinite_zero(self):
        c = synthesize_safe(chain(0.0, 0.2, 0.8), eps=1e-10)
        assert c.p_min[0] == pytest.approx(0.0, abs=1e-9)

    def test_safety_two_steps(self):
        c = synthesize_safe(chain(0.0, 0.2, 0.8), horizon=2)
        assert c.p_min[0] == pytest.approx(0.64, abs=1e-9)

    def test_safety_no_leakage(self):
        ident = np.eye(3)
        z = np.zeros(3)
        c = synthesize_safe(make_imdp(ident, ident, z, z, z, z), eps=1e-9)
        assert np.allclose(c.p_min, 1.0) and np.allclose(c.p_max, 1.0)


class TestOracleAgreement:
    def test_degenerate_chains_match_value_iteration(self):
        rng = np.random.default_rng(99)
        for trial in range(40):
            n_s = int(rng.integers(2, 21))
            full = rng.dirichlet(np.ones(n_s + 2), size=n_s)
            t, r = 0.95 * full[:, :n_s], full[:, n_s]
            r = r + (1 - t.sum(axis=1) - r - full[:, n_s + 1]) / 2
            a = 1 - t.sum(axis=1) - r
            m = make_imdp(t, t, r, r, a, a)
            v = np.zeros(n_s)
            while True:
                nv = t @ v + r
                if np.max(np.abs(nv - v)) <= 1e-12:
                    break
                v = nv
            for mode in ("pessimistic", "optimistic"):
                c = synthesize_reach(m, mode=mode, eps=1e-11)
                assert np.allclose(c.p_min, nv, atol=1e-9), trial
                assert np.allclose(c.p_max, nv, atol=1e-9), trial

    @pytest.mark.parametrize("seed", range(4))
    def test_random_interval_synthesis_matches_oracle(self, seed):
        rng = np.random.default_rng(100 + seed)
        m = random_imdp(rng, int(rng.integers(20, 200)), int(rng.integers(1, 4)),
                        1, density=0.3)
        om = oracle_model(m)
        for spec, fn in (("reach", synthesize_reach),
                         ("safety", synthesize_safe)):
            c = fn(m, eps=1e-8)
            o = ORI.synthesize(om, spec, eps=1e-8)
            assert c.meta["iterations"] == o["iterations"]
            assert np.max(np.abs(c.p_min - o["p_min"])) <= TOL
            assert np.max(np.abs(c.p_max - o["p_max"])) <= TOL

    def test_complement_identity_bitwise(self):
        rng = np.random.default_rng(8)
        full = rng.dirichlet(np.ones(7), size=5)
        t = 0.9 * full[:, :5]
        a = 1 - t.sum(axis=1)
        z = np.zeros(5)
        m = make_imdp(t, t, z, z, a, a)
        safe = synthesize_safe(m, eps=1e-10)
        v = np.zeros(5)
        for _ in range(safe.meta["iterations"][0]):
            v, _ = bellman_step(m, v, "max", "min", "safety")
        assert np.array_equal(safe.p_min, 1.0 - v)


class TestDiagnostics:
    def test_geometric_rate(self):
        k0, k1 = diagnose_convergence(chain(0.2, 0.0, 0.8), spec="reach",
                                      eps=1e-6)
        assert 50 <= k0 <= 60
        assert k1 >= 1

    def test_immediate_absorption(self):
        assert diagnose_convergence(chain(1.0, 0.0, 0.0)) == (1, 1)

    def test_absorbing_safe_state_fallback(self):
        m = chain(0.0, 0.0, 1.0)
        assert diagnose_convergence(m, spec="reach", eps=1e-6) == (1, 1)
        c = synthesize_reach(m, eps=1e-6, max_iterations=50)
        assert c.meta["fallback"] == (True, True)
        assert c.p_min[0] == 0.0 and c.p_max[0] == 0.0

    def test_slow_chain_hits_iteration_cap(self):
        with pytest.raises(ConvergenceError) as info:
            synthesize_reach(chain(0.2, 0.0, 0.8), eps=1e-10,
                             max_iterations=20)
        assert info.value.k0 is None
        assert info.value.k1 == 1

    def test_verify_rejects_inputs(self):
        t = np.array([[0.5], [0.9]])
        m = make_imdp(t, t, [0.5, 0.1], [0.5, 0.1], [0, 0], [0, 0], n_u=2)
        with pytest.raises(ValueError):
            verify(m)


def _golden_controller_check(name):
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    m = G.imdp(g)
    spec = G.spec_of(cfg)
    kw = dict(mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon)
    if m.input_space is None:
        if str(g["error"]) == "ConvergenceError":
            with pytest.raises(ConvergenceError) as info:
                verify(m, spec=spec, max_iterations=300, **kw)
            assert info.value.k0 == (None if g["k0"] < 0 else int(g["k0"]))
            assert info.value.k1 == (None if g["k1"] < 0 else int(g["k1"]))
            return
        c = verify(m, spec=spec, **kw)
    elif spec == "safety":
        c = synthesize_safe(m, **kw)
    else:
        c = synthesize_reach(m, **kw)
    assert tuple(c.meta["iterations"]) == tuple(g["iterations"])
    assert tuple(c.meta["fallback"]) == tuple(bool(x) for x in g["fallback"])
    assert np.max(np.abs(c.p_min - g["p_min"])) <= TOL
    assert np.max(np.abs(c.p_max - g["p_max"])) <= TOL
    if c.policy is not None and "margin" in g:
        diff = c.policy != g["policy"]
        tight = g["margin"] <= 1e-12
        assert not np.any(diff & ~tight), np.flatnonzero(diff & ~tight)
        per_u = g["per_u"]
        k = np.flatnonzero(diff)
        assert np.all(np.abs(per_u[k, c.policy[k]] -
                             per_u[k, g["policy"][k]]) <= 1e-12)


@pytest.mark.parametrize("name", G.MINIS)
def test_golden_controller(name):
    if not G.have("full_" + name):
        pytest.skip("fixture not generated")
    _golden_controller_check(name)


@pytest.mark.parametrize("name", G.MINIS)
def test_golden_sweep_trace(name):
    """First six twin sweeps of phase 1 against the reference's trace."""
    if not G.have("full_" + name):
        pytest.skip("fixture not generated")
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    m = G.imdp(g)
    spec = G.spec_of(cfg)
    if spec == "reach":
        lp = "min" if cfg.mode == "pessimistic" else "max"
        u_obj = "max"
    else:
        lp = "max" if cfg.mode == "pessimistic" else "min"
        u_obj = "min"
    v0 = np.zeros(m.n_s)
    v1 = np.ones(m.n_s)
    for it in range(6):
        v0, pol = bellman_step(m, v0, lp, u_obj, spec)
        v1, _ = bellman_step(m, v1, lp, u_obj, spec)
        assert np.max(np.abs(v0 - g["trace_v0"][it])) <= 1e-12
        assert np.max(np.abs(v1 - g["trace_v1"][it])) <= 1e-12
        ph = run_phase(m, spec, lp, u_obj, 1e-6, it + 1, 10**6)
        assert np.array_equal(ph.pair.v0, v0)
        assert np.array_equal(ph.pair.v1, v1)


@pytest.mark.parametrize("name", ["robot2d_ra_mini", "room5d_mini"])
def test_shard_sweeps_bitwise_equal_single_handle(name):
    """Sweeping the abstraction as 3 state shards (the multi-GPU layout,
    here on one device) gives bit-identical values and choices to the
    single handle: no reduction depends on a row's position or shard."""
    import torch
    from paper_2401_03555_b200 import build_abstraction
    from paper_2401_03555_b200.sharded import shard_range, shard_sweep
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    full = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels)
    n_s = full.n_s
    rng = np.random.default_rng(3)
    v = rng.uniform(0, 1, n_s)
    spec = G.spec_of(cfg)
    u_obj = "max" if spec == "reach" else "min"
    for lp in ("min", "max"):
        want, wpick = bellman_step(full, v, lp, u_obj, spec)
        got, gpick = [], []
        vt = torch.tensor(v, dtype=torch.float64, device="cuda")
        for r in range(3):
            shard = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                                      labels, k_range=shard_range(n_s, 3, r))
            n0, _, pol, _ = shard_sweep(shard, vt, vt,
                                        0 if spec == "reach" else 1,
                                        1 if lp == "max" else 0,
                                        1 if u_obj == "max" else 0)
            got.append(n0.cpu().numpy())
            gpick.append(pol.cpu().numpy())
        assert np.array_equal(np.concatenate(got), want)
        assert np.array_equal(np.concatenate(gpick), wpick)


# --- optimistic mode, finite horizon, diagnose_convergence
# as first-class flags of the same device loop, against the oracle ----------

def _mini_case(name):
    if not G.have("full_" + name):
        pytest.skip("fixture not generated")
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    return cfg, G.imdp(g), G.model(g), G.spec_of(cfg)


def _gpu_synth(m, spec, **kw):
    if m.input_space is None:
        return verify(m, spec=spec, **kw)
    if spec == "safety":
        return synthesize_safe(m, **kw)
    return synthesize_reach(m, **kw)


def _check_against_oracle(c, want, m, spec):
    assert tuple(c.meta["iterations"]) == tuple(want["iterations"])
    assert tuple(c.meta["fallback"]) == tuple(want["fallback"])
    assert np.max(np.abs(c.p_min - want["p_min"])) <= TOL
    assert np.max(np.abs(c.p_max - want["p_max"])) <= TOL
    if c.policy is not None:
        # margin-aware policy rule: where the inputs differ,
        # the GPU's must be eps-optimal under the oracle's phase-1 values
        diff = np.flatnonzero(c.policy != want["policy"])
        if len(diff):
            lp = "min" if spec == "reach" else "max"
            if c.meta["mode"] == "optimistic":
                lp = "max" if lp == "min" else "min"
            u_obj = "max" if spec == "reach" else "min"
            om = oracle_model(m)
            v0 = want["phase1"].v0
            ref, _ = ORI.bellman(om, v0, lp, u_obj, spec, want["policy"])
            alt, _ = ORI.bellman(om, v0, lp, u_obj, spec, c.policy)
            assert np.max(np.abs(ref - alt)) <= 1e-12


@pytest.mark.parametrize("name", ["robot2d_ra_mini", "room5d_mini",
                                  "vehicle3d_mini", "bas4d_mini"])
def test_optimistic_mode_matches_oracle(name):
    cfg, m, om, spec = _mini_case(name)
    c = _gpu_synth(m, spec, mode="optimistic", eps=1e-6)
    want = ORI.synthesize(om, spec, mode="optimistic", eps=1e-6)
    _check_against_oracle(c, want, m, spec)


@pytest.mark.parametrize("name", ["robot2d_ra_mini", "room5d_mini",
                                  "bas4d_mini"])
@pytest.mark.parametrize("horizon", [1, 3, 10])
def test_finite_horizon_matches_oracle(name, horizon):
    cfg, m, om, spec = _mini_case(name)
    c = _gpu_synth(m, spec, horizon=horizon)
    want = ORI.synthesize(om, spec, horizon=horizon)
    assert c.meta["horizon"] == horizon
    _check_against_oracle(c, want, m, spec)


@pytest.mark.parametrize("name", ["robot2d_ra_mini", "room5d_mini",
                                  "vehicle3d_mini", "bas4d_mini",
                                  "bas7d_mini"])
@pytest.mark.parametrize("mode", ["pessimistic", "optimistic"])
def test_diagnose_convergence_matches_oracle(name, mode):
    cfg, m, om, spec = _mini_case(name)
    got = diagnose_convergence(m, spec=spec, mode=mode, eps=1e-6)
    assert got == ORI.diagnose(om, spec=spec, mode=mode, eps=1e-6)


def test_diagnose_convergence_cap_reports_partial_horizons():
    """dim6 (0.8 x contraction, like dim14) does not self-converge within a
    short cap: ConvergenceError carries the same k0 / k1 as the oracle."""
    cfg, m, om, spec = _mini_case("dim6_mini")
    with pytest.raises(ConvergenceError) as got:
        diagnose_convergence(m, spec=spec, eps=1e-6, max_iterations=60)
    with pytest.raises(ConvergenceError) as want:
        ORI.diagnose(om, spec=spec, eps=1e-6, max_iterations=60)
    assert (got.value.k0, got.value.k1) == (want.value.k0, want.value.k1)


def test_reference_log_lines(caplog):
    """The reference's log contract (abstraction.py:596-598, synthesis.py:
    190-194, 204-205): the sparsity INFO line after a build, the gap INFO
    line every 1000 iterations, and the stalled-gap fallback WARNING."""
    import logging
    from paper_2401_03555_b200 import build_abstraction
    g = G.load("full_robot2d_ra_mini")
    cfg = G.config_of(g)
    with caplog.at_level(logging.INFO):
        im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                               cfg.labels(), cfg.abstraction_options())
    dense = G.dense(g)[1]
    want = 100 * float(np.mean(dense <= 1e-12))
    assert f"abstraction built: {im.n_rows} rows x {im.n_s} cols, " \
           f"{want:.1f}% of t_max at zero" in caplog.text
    caplog.clear()
    # 2500 iterations of a slowly contracting chain: two gap lines
    m = chain(0.0, 0.001, 0.999)
    with caplog.at_level(logging.INFO):
        synthesize_safe(m, eps=1e-300, horizon=2500)
    assert "iteration 1000: gap" in caplog.text
    assert "iteration 2000: gap" in caplog.text
    assert "iteration 3000" not in caplog.text
    caplog.clear()
    # absorbing safe state: gap pinned at 1, both bounds self-converge ->
    # fallback warning
    ident = np.eye(2)
    z = np.zeros(2)
    with caplog.at_level(logging.WARNING):
        c = synthesize_safe(make_imdp(ident, ident, z, z, z, z), eps=1e-6)
    assert any(c.meta["fallback"])
    assert "falling back to the value-iteration result" in caplog.text
