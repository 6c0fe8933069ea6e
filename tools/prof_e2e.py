"""Host-side profile of one warm bench step (build_abstraction + synthesis).

    python tools/prof_e2e.py CONFIG

Prints wall time per stage and the top cProfile entries of the timed step,
to find host overhead between the device-timed step and the e2e wall time.
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2401_03555_b200.abstraction import build_abstraction  # noqa: E402
from paper_2401_03555_b200.config import benchmark  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "robot2d_reachavoid"
cfg = benchmark(name)
labels = cfg.labels()


def step():
    t0 = time.perf_counter()
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                           cfg.abstraction_options(), device=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctrl = bench._spec_call(cfg, im)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del im
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return ctrl, (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3


for _ in range(2):
    step()
pr = cProfile.Profile()
pr.enable()
ctrl, b, s, f = step()
pr.disable()
print(f"{name}: build wall {b:.1f} ms (device {ctrl.meta.get('device_ms')}), "
      f"synthesis wall {s:.1f} ms, free {f:.1f} ms")
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
