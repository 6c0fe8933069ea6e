"""Build (a shard of) a config and time the K5 sweep kernel alone.

    python tools/prof_sweep.py NAME [k_begin k_count] [reps]
"""
import sys
sys.path.insert(0, ".")
from paper_2401_03555_b200 import _lib
from paper_2401_03555_b200.config import benchmark
from paper_2401_03555_b200.abstraction import build_abstraction
import tests.golden_io as G

name = sys.argv[1]
k_range = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
cfg = G.config_of(G.load("full_" + name)) if G.have("full_" + name) \
    else benchmark(name)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options(), k_range=k_range)
info = im.device_handle().info()
spec = _lib.SPEC_SAFETY if cfg.spec_type == "safety" else _lib.SPEC_REACH
lp = _lib.LP_MAX if cfg.spec_type == "safety" else _lib.LP_MIN
ms = _lib.c_dbl(0)
_lib.check(_lib.load().imp_time_sweep(im.device_handle().raw, spec, lp, reps,
                                      ms))
nbytes = info.nnz * 20 + info.n_rows * 40
print(f"{name}: rows {info.n_rows} nnz {info.nnz} max_row {info.max_row} "
      f"n_s {info.n_s}: {ms.value:.3f} ms/sweep, "
      f"{nbytes / ms.value / 1e6:.1f} GB/s")
