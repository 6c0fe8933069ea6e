"""Build a config and run its synthesis; dump the controller for A/B checks.

    python tools/ab_stream.py NAME OUT.npz      (env IMP_SWEEP_STREAM=0|1)
"""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
from bench import _spec_call
from paper_2401_03555_b200.config import benchmark
from paper_2401_03555_b200.abstraction import build_abstraction
import tests.golden_io as G

name, out = sys.argv[1], sys.argv[2]
cfg = G.config_of(G.load("full_" + name)) if G.have("full_" + name) \
    else benchmark(name)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
_spec_call(cfg, im)                       # warm
t0 = time.perf_counter()
c = _spec_call(cfg, im)
dt = time.perf_counter() - t0
np.savez(out, p_min=c.p_min, p_max=c.p_max,
         policy=c.policy if c.policy is not None else np.zeros(0))
print(f"{name}: iterations {c.meta['iterations']} device_ms "
      f"{tuple(round(x, 2) for x in c.meta['device_ms'])} wall {dt:.2f}s")
