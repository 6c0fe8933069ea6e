"""Phase-1 sweeps/s of a benchmark config's synthesis (build once, run the
synthesis 3 times, report the best).  Usage: python tools/time_synth.py NAME [horizon]"""
import hashlib
import sys
import time
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2401_03555_b200.abstraction import build_abstraction  # noqa: E402
from paper_2401_03555_b200.config import benchmark  # noqa: E402

name = sys.argv[1]
over = {"horizon": int(sys.argv[2])} if len(sys.argv) > 2 else {}
cfg = benchmark(name, **over)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
best = None
for _ in range(3):
    t0 = time.perf_counter()
    ctrl = bench._spec_call(cfg, im)
    wall = time.perf_counter() - t0
    it = ctrl.meta["iterations"]
    ms = ctrl.meta.get("device_ms")
    rate = it[0] / (ms[0] * 1e-3) if ms else it[0] / wall
    best = max(best or 0, rate)
dig = hashlib.sha1(ctrl.p_min.tobytes() + ctrl.p_max.tobytes() + (
    ctrl.policy.tobytes() if ctrl.policy is not None else b"")).hexdigest()[:12]
print(f"{name}: iterations {it} device_ms {ms} phase-1 sweeps/s {best:.1f} "
      f"result {dig}")
