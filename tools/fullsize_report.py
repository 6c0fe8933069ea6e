"""Observed deviations of the GPU against the reference's full-size runs
(tests/golden/fullsize_*.npz) as JSON -- the numbers behind
tests/test_fullsize_parity_gpu.py.  Usage (GPU): python tools/fullsize_report.py"""
import json
import sys
import numpy as np
sys.path.insert(0, ".")
import tests.golden_io as G  # noqa: E402
from paper_2401_03555_b200 import build_abstraction, synthesize_reach  # noqa: E402
from paper_2401_03555_b200.synthesis import run_phase  # noqa: E402

out = {}
g = G.load("fullsize_robot2d_reachavoid")
cfg = G.config_of(g)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
ptr, col, lo, hi, r0, r1, a0, a1 = im.csr()
c = synthesize_reach(im, mode=cfg.mode, eps=cfg.eps)
tr = max(float(np.max(np.abs(run_phase(im, "reach", "min", "max", cfg.eps, k,
                                       10**6).pair.v0 - g["trace_v0"][k - 1])))
         for k in range(1, 7))
diff = c.policy != g["policy"]
out["robot2d_reachavoid"] = dict(
    rows=int(len(ptr) - 1), nnz=int(ptr[-1]), nnz_ref=int(g["nnz"]),
    row_nnz_equal=bool(np.array_equal(np.diff(ptr), g["row_nnz"])),
    vec_max_abs=float(max(np.max(np.abs(r0 - g["r_min"])),
                          np.max(np.abs(r1 - g["r_max"])),
                          np.max(np.abs(a0 - g["a_min"])),
                          np.max(np.abs(a1 - g["a_max"])))),
    iterations=list(map(int, c.meta["iterations"])),
    iterations_ref=list(map(int, g["iterations"])),
    p_min_max_abs=float(np.max(np.abs(c.p_min - g["p_min"]))),
    p_max_max_abs=float(np.max(np.abs(c.p_max - g["p_max"]))),
    trace_v0_max_abs=tr,
    policy_diffs=int(diff.sum()),
    policy_diffs_with_margin_above_1e12=int(np.sum(diff & (g["margin"] > 1e-12))),
    ref_ties_margin_le_1e12=int(np.sum(g["margin"] <= 1e-12)))
g = G.load("fullsize_dim14_verify")
cfg = G.config_of(g)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
worst = 0.0
for k in range(1, len(g["trace_v0"]) + 1):
    rep = run_phase(im, "safety", "max", "min", cfg.eps, k, 10**6)
    worst = max(worst, float(np.max(np.abs(rep.pair.v0 - g["trace_v0"][k - 1]))),
                float(np.max(np.abs(rep.pair.v1 - g["trace_v1"][k - 1]))))
out["dim14_verify"] = dict(trace_iterations=len(g["trace_v0"]),
                           trace_max_abs=worst)
print(json.dumps(out, indent=1))
