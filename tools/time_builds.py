"""Build a config R times; print the device build times (ms_total)."""
import sys
sys.path.insert(0, ".")
from paper_2401_03555_b200.abstraction import build_abstraction
from paper_2401_03555_b200.config import benchmark

name, reps = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = benchmark(name)
args = (cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
        cfg.abstraction_options())
ms = []
for _ in range(reps):
    im = build_abstraction(*args)
    r = im.build_report
    ms.append((round(r.ms_total, 1), round(r.ms_mean_ranges, 1),
               round(r.ms_outer, 1), round(r.ms_assemble, 1)))
    del im
print(name, ms)
