"""Build one config (benchmark name or golden mini fixture) once; for ncu.

    python tools/prof_build.py NAME [k_begin k_count]
"""
import sys
sys.path.insert(0, ".")
from paper_2401_03555_b200.config import benchmark
from paper_2401_03555_b200.abstraction import build_abstraction
import tests.golden_io as G

name = sys.argv[1]
k_range = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else None
if G.have("full_" + name):
    cfg = G.config_of(G.load("full_" + name))
else:
    cfg = benchmark(name)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options(), k_range=k_range)
print(im.build_report)
