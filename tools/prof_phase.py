"""Build a benchmark config and run its synthesis once (optionally with a
finite horizon): a target for ncu captures of the in-loop K5 launches.

    python tools/prof_phase.py NAME [horizon]
"""
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2401_03555_b200.abstraction import build_abstraction  # noqa: E402
from paper_2401_03555_b200.config import benchmark  # noqa: E402

name = sys.argv[1]
over = {"horizon": int(sys.argv[2])} if len(sys.argv) > 2 else {}
cfg = benchmark(name, **over)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
ctrl = bench._spec_call(cfg, im)
print(name, ctrl.meta.get("iterations"), ctrl.meta.get("device_ms"))
