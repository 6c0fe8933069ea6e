"""Does the nvidia-smi clock sampler perturb the timed step?  Steps of one
config without, then with, the sampler running; per step: wall ms, device
build ms, device phase ms.

    python tools/sampler_ab.py CONFIG [interval_ms]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2401_03555_b200.abstraction import build_abstraction  # noqa: E402
from paper_2401_03555_b200.benchutil import ClockSampler  # noqa: E402
from paper_2401_03555_b200.config import benchmark  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "robot2d_reachavoid"
if len(sys.argv) > 2:
    ClockSampler.INTERVAL_MS = int(sys.argv[2])
cfg = benchmark(name)
labels = cfg.labels()


def step(tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                           cfg.abstraction_options(), device=0)
    ctrl = bench._spec_call(cfg, im)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{tag}: wall {(t1 - t0) * 1e3:8.1f} ms  build "
          f"{im.build_report.ms_total:7.1f} ms  phases "
          f"{ctrl.meta['device_ms']}", flush=True)
    del im


for _ in range(3):
    step("warm   ")
for _ in range(3):
    step("plain  ")
s = ClockSampler(0)
s.start()
time.sleep(2.0)
s.mark()
for _ in range(3):
    step("sampler")
print(s.stop())
for _ in range(2):
    step("after  ")
