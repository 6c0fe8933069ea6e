"""Reference Monte Carlo abstractions for the MC-noise parity tests.

TEST INFRASTRUCTURE ONLY.  Runs the REFERENCE build_abstraction
(/root/reference/pkg/src/impact/abstraction.py:511-540 _row_monte_carlo,
noise.py:41-153 FullNormal / mc_box_probability) on a small full-covariance
system and stores the abstraction (dense t bounds, r/a vectors) in
tests/golden/mc_<name>.npz together with its config text.

Usage:  python tests/golden/make_mc_golden.py
"""

import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from impact import abstraction as A  # noqa: E402
from impact.config import load_config  # noqa: E402

SYSTEMS = {
    "mc2d_full": """
[state]
lb = 0 0
ub = 3 3
eta = 1 1
[input]
lb = -0.5
ub = 0.5
eta = 1
[dynamics]
f1 = 0.8*x1 + 0.1*x2 + u1 + 0.3
f2 = 0.1*x1 + 0.7*x2 + 0.5
[noise]
type = full
inv_cov = 4 1 1 3
det = 11
samples = 128
[spec]
type = reach-avoid
target = (x1 >= 2.5) & (x2 >= 2.5)
avoid = (x1 <= 0.5) & (x2 >= 2.5)
[synthesis]
seed = 3
""",
    "mc2d_custom": """
[state]
lb = 0 0
ub = 3 3
eta = 1 1
[input]
lb = -0.5
ub = 0.5
eta = 1
[dynamics]
f1 = 0.8*x1 + 0.1*x2 + u1 + 0.3
f2 = 0.1*x1 + 0.7*x2 + 0.5
[noise]
type = custom
density = exp(-((y1-m1)^2 + (y2-m2)^2) / 0.5) / (0.5*3.141592653589793) * (1 + 0.2*(y1-m1)*(y2-m2)/(1 + (y1-m1)^2 + (y2-m2)^2))
samples = 128
[spec]
type = reach-avoid
target = (x1 >= 2.5) & (x2 >= 2.5)
avoid = (x1 <= 0.5) & (x2 >= 2.5)
[synthesis]
seed = 5
""",
    # small cells (eta << sigma) and few samples: every destination's
    # estimate carries its own sampling error, so min-side row sums overshoot
    # 1 by far more than 1e-6 and max-side sums fall short -- the branch the
    # reference repairs instead of raising (abstraction.py:620-650)
    "mc2d_fine": """
[state]
lb = 0 0
ub = 1.5 1.5
eta = 0.25 0.25
[input]
lb = -0.1
ub = 0.1
eta = 0.2
[dynamics]
f1 = 0.8*x1 + 0.1*x2 + u1 + 0.15
f2 = 0.1*x1 + 0.7*x2 + 0.25
[noise]
type = full
inv_cov = 16 2 2 12
det = 188
samples = 16
[spec]
type = reach-avoid
target = (x1 >= 1.25) & (x2 >= 1.25)
avoid = (x1 <= 0.25) & (x2 >= 1.25)
[synthesis]
seed = 11
""",
}


def main():
    only = sys.argv[1:]
    for name, text in SYSTEMS.items():
        if only and name not in only:
            continue
        with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as fh:
            fh.write(text)
        cfg = load_config(fh.name)
        os.unlink(fh.name)
        t0 = time.time()
        im = A.build_abstraction(cfg.dynamics, cfg.noise,
                                 (cfg.state_space, cfg.input_space,
                                  cfg.disturb_space), cfg.labels(),
                                 cfg.abstraction_options())
        np.savez_compressed(os.path.join(HERE, f"mc_{name}.npz"),
                            config=text, t_min=im.t_min, t_max=im.t_max,
                            r_min=im.r_min, r_max=im.r_max, a_min=im.a_min,
                            a_max=im.a_max, seconds=time.time() - t0)
        print(name, im.t_min.shape, f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
