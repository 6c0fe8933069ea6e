"""Time one GPU build (+ optional synthesis) of a benchmark config."""
import sys, time
sys.path.insert(0, ".")
from paper_2401_03555_b200.config import benchmark
from paper_2401_03555_b200.abstraction import build_abstraction
import bench

name = sys.argv[1]
synth = len(sys.argv) > 2 and sys.argv[2] == "synth"
reps = 1 if len(sys.argv) > 2 and sys.argv[2] == "once" else 2
cfg = benchmark(name)
labels = cfg.labels()
for rep in range(reps):
    t0 = time.perf_counter()
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels, cfg.abstraction_options())
    t1 = time.perf_counter()
    r = im.build_report
    print(name, f"wall {t1-t0:.2f}s", r, f"evals/s {r.nm_evals/max(r.ms_refine,1e-9)*1e3:.3e}", flush=True)
if synth:
    t0 = time.perf_counter()
    c = bench._spec_call(cfg, im)
    print("synth", time.perf_counter() - t0, c.meta)
