"""Time build_abstraction of a benchmark config (second build: JIT cached).

    python tools/time_build.py NAME [once]
JIT knobs via env: IMPACT_NDTR_CHUNK, IMPACT_REFINE_MINB, IMPACT_REFINE_BATCH,
IMPACT_INST_SMEM.
"""
import hashlib
import sys
sys.path.insert(0, ".")
from paper_2401_03555_b200.abstraction import build_abstraction
from paper_2401_03555_b200.config import benchmark

name = sys.argv[1]
cfg = benchmark(name)
args = (cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
        cfg.abstraction_options())
im = build_abstraction(*args)
if len(sys.argv) < 3:
    del im
    im = build_abstraction(*args)
r = im.build_report
dig = hashlib.sha1(b"".join(a.tobytes() for a in im.csr())).hexdigest()[:12]
print(f"{name}: ms_total={r.ms_total:.1f} ms_refine={r.ms_refine:.1f} "
      f"evals/s {r.nm_evals / (r.ms_refine * 1e-3):.4g} "
      f"simt={r.nm_evals / max(r.nm_lane_slots, 1) / 32:.3f} csr {dig}")
