"""GPU Monte Carlo abstraction vs the reference fixture: error profile."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from paper_2401_03555_b200 import build_abstraction, parse_config_text

g = np.load("tests/golden/mc_mc2d_full.npz")
cfg = parse_config_text(str(g["config"]))
t0 = time.time()
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
dt = time.time() - t0
print("build", dt, "s", im.build_report)
for k in ("t_min", "t_max", "r_min", "r_max", "a_min", "a_max"):
    d = np.abs(getattr(im, k) - g[k])
    print(k, "max", d.max(), "frac>1e-12", np.mean(d > 1e-12),
          "frac>1e-9", np.mean(d > 1e-9), "bitwise", np.mean(d == 0))
