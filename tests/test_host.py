"""Host-side surface (CPU only): grids, expressions, configs, lowering.

Mirrors the reference's unit tests for the model layer (pkg/tests/
test_grid.py, test_expr.py, test_acceptance.py criterion 1) on this
package's own implementation, plus the CUDA lowering of the dynamics.
"""

import math
import re

import numpy as np
import pytest

from paper_2401_03555_b200 import (ConfigError, GridError, ParseError,
                                   build_space, cell_of, label_states,
                                   parse_expression, parse_predicate,
                                   quantize, rep_point)
from paper_2401_03555_b200.abstraction import RowIndex, estimate_cost
from paper_2401_03555_b200.config import (BENCHMARKS, benchmark,
                                          parse_config_text)
from paper_2401_03555_b200.expr import has_x_transcendental, lower_dynamics

from . import golden_io as G


class TestGrid:
    def test_cardinalities_of_benchmarks(self):
        expect = {"robot2d_reach_disturb": (441, 121, 11),
                  "robot2d_reachavoid": (1681, 441, None),
                  "vehicle3d": (7938, 30, None), "room3d": (9261, 36, None),
                  "room5d": (7776, 36, None), "bas4d": (1225, 4, None),
                  "bas7d_verify": (107163, None, None),
                  "dim14_verify": (16384, None, None)}
        for name, (nx, nu, nw) in expect.items():
            cfg = benchmark(name)
            got = (cfg.state_space.total,
                   cfg.input_space.total if cfg.input_space else None,
                   cfg.disturb_space.total if cfg.disturb_space else None)
            assert got == (nx, nu, nw), name

    def test_rep_points_and_cells(self):
        sp = build_space([-10, -10], [10, 10], [1, 1])
        assert sp.total == 441
        assert np.array_equal(rep_point(sp, 0), [-10, -10])
        assert np.array_equal(rep_point(sp, 440), [10, 10])
        c = cell_of(sp, quantize(sp, [0.0, 0.0]))
        assert np.array_equal(c.lo, [-0.5, -0.5])
        assert np.array_equal(sp.rep_points()[17], rep_point(sp, 17))

    def test_quantize_ties_and_domain(self):
        sp = build_space([-10, -10], [10, 10], [1, 1])
        assert quantize(sp, [0.5, 0.0]) == quantize(sp, [0.0, 0.0])
        assert quantize(sp, [0.2, -0.3]) == quantize(sp, [0.0, 0.0])
        with pytest.raises(GridError):
            quantize(sp, [11.0, 0.0])

    def test_bad_lattice(self):
        with pytest.raises(GridError):
            build_space([0], [1], [0.3])
        with pytest.raises(GridError):
            build_space([0], [1], [0.0])

    def test_labels_avoid_wins(self):
        sp = build_space([-10, -10], [10, 10], [1, 1])
        t = parse_predicate("(x1 >= 5) & (x1 <= 7) & (x2 >= 5) & (x2 <= 7)",
                            2)
        a = parse_predicate("(x1 >= -2) & (x1 <= 2) & (x2 >= -2) & (x2 <= 2)",
                            2)
        lab = label_states(sp, t, a)
        assert len(lab.target) == 9 and len(lab.avoid) == 25
        assert len(lab.safe) == 441 - 34
        both = label_states(sp, parse_predicate("x1 >= 0", 2),
                            parse_predicate("x1 >= 5", 2))
        assert not set(both.target) & set(both.avoid)

    def test_row_index_and_cost(self):
        idx = RowIndex(n_u=3, n_w=2)
        seen = {idx.row(k, j, i) for k in range(4) for j in range(3)
                for i in range(2)}
        assert seen == set(range(24))
        assert all(idx.kji(idx.row(k, j, i)) == (k, j, i)
                   for k in range(4) for j in range(3) for i in range(2))
        d, nbytes, over = estimate_cost(10, 2, 1)
        assert d == 200 and nbytes == 2 * 200 * 8 + 6 * 20 * 8 and not over
        assert estimate_cost(10**12, 10**6, 1)[2]


class TestExpr:
    def test_precedence(self):
        env = {"x1": 2.0}
        assert parse_expression("-x1^2", (1, 0, 0)).evaluate(env) == -4.0
        assert parse_expression("2^3^2", (1, 0, 0)).evaluate(env) == 512.0
        assert parse_expression("1 - 2 - 3", (1, 0, 0)).evaluate(env) == -4.0
        assert parse_expression("8 / 2 / 2", (1, 0, 0)).evaluate(env) == 2.0
        assert parse_expression("2*x1^-1", (1, 0, 0)).evaluate(env) == 1.0

    def test_errors(self):
        for bad in ("x1 +", "x3", "sin(x1, x1)", "x1 $ 2", "(x1", "min(x1)"):
            with pytest.raises(ParseError):
                parse_expression(bad, (2, 0, 0))
        with pytest.raises(ParseError):
            parse_predicate("x1 + 2", 1)

    def test_random_expressions_match_python(self):
        rng = np.random.default_rng(0)
        ops = ["+", "-", "*"]
        for _ in range(300):
            terms = [f"{rng.uniform(-3, 3):.4f}" if rng.random() < 0.5
                     else f"x{rng.integers(1, 3)}" for _ in range(5)]
            text = terms[0]
            for t in terms[1:]:
                text = f"({text} {ops[rng.integers(0, 3)]} {t})"
            env = {"x1": 0.7, "x2": -1.3}
            got = parse_expression(text, (2, 0, 0)).evaluate(env)
            assert got == pytest.approx(eval(text, {}, env), rel=1e-12)

    def test_predicates(self):
        p = parse_predicate("!(x1 > 1) | (x1 + 1) * 2 >= 9", 1)
        assert p.evaluate([0.5]) and not p.evaluate([2.0])
        assert p.evaluate([4.0])


def _eval_cuda_expr(text, x, k):
    """Evaluate the generated CUDA C expression with Python floats (IEEE
    doubles, same association) to check the lowering."""
    py = text.replace("sincos", "_sincos")
    py = re.sub(r"x\[(\d+)\]", r"x[\1]", py)
    env = {"x": x, "k": k, "sin": math.sin, "cos": math.cos,
           "tan": math.tan, "atan": math.atan, "sqrt": math.sqrt,
           "exp": math.exp, "log": math.log, "fabs": abs, "pow": math.pow,
           "imp_min": min, "imp_max": max, "imp_div": lambda a, b: a / b,
           "imp_div_rcp": lambda a, b, r: a / b}
    return eval(py, env)


@pytest.mark.parametrize("name", sorted(BENCHMARKS))
def test_lowering_matches_numpy_evaluation(name):
    """Folded constants + emitted residual == the reference-order numpy
    evaluation, bitwise for affine dynamics."""
    cfg = benchmark(name)
    dyn = cfg.dynamics
    u = cfg.input_space.rep_points() if cfg.input_space else np.zeros((1, 0))
    w = cfg.disturb_space.rep_points() if cfg.disturb_space else \
        np.zeros((1, 0))
    low = lower_dynamics(dyn, u, w)
    bodies = dict(re.findall(r"double imp_f(\d+)\(const double\* x, const "
                             r"double\* k\) \{ return (.*); \}", low.source))
    assert len(bodies) == dyn.dims[0]
    rng = np.random.default_rng(1)
    n, m, p = dyn.dims
    trig = has_x_transcendental(dyn)
    for trial in range(5):
        j = int(rng.integers(0, len(u)))
        i = int(rng.integers(0, len(w)))
        x = cfg.state_space.lb + rng.uniform(0, 1, n) * (
            cfg.state_space.ub - cfg.state_space.lb)
        env = {f"x{q + 1}": float(x[q]) for q in range(n)}
        env.update({f"u{q + 1}": u[j][q] for q in range(m)})
        env.update({f"w{q + 1}": w[i][q] for q in range(p)})
        k = list(low.consts[j * len(w) + i])
        for d in range(n):
            want = float(dyn.exprs[d].evaluate_env(env))
            got = _eval_cuda_expr(bodies[str(d)], list(map(float, x)), k)
            if trig:
                assert got == pytest.approx(want, rel=1e-14, abs=1e-14)
            else:
                assert got == want


class TestConfig:
    def test_text_config_matches_benchmark(self):
        g = G.load("full_robot2d_ra_mini")
        cfg = G.config_of(g)
        assert cfg.spec_type == "reach-avoid" and cfg.state_space.total == 121
        assert cfg.input_space.total == 25

    def test_config_errors(self):
        with pytest.raises(ConfigError):
            parse_config_text("[state]\nlb = 0\nub = 1\neta = 0.3\n")
        with pytest.raises(ConfigError):
            parse_config_text("[state]\nlb = 0\nub = 1\neta = 1\n"
                              "[spec]\ntype = reach\n")
        with pytest.raises(ConfigError):
            parse_config_text("[state]\nlb = 0\nub = 1\neta = 1\n"
                              "[synthesis]\nepsilon = 0\n")

    def test_bench_horizon_override(self):
        # bench.py --horizon: finite horizon for configs whose infinite-horizon
        # run ends at the reference's iteration cap (room5d, dim14)
        import argparse
        import bench
        cfg = benchmark("room5d", **bench._overrides(
            argparse.Namespace(horizon=200)))
        assert cfg.horizon == 200
        assert benchmark("room5d", **bench._overrides(
            argparse.Namespace(horizon=0))).horizon is None
