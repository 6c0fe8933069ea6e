"""Per-row construction diffs vs the reference's row samples (GPU)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import tests.golden_io as G
from paper_2401_03555_b200 import build_abstraction

for name in sys.argv[1:]:
    g = G.load("rows_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    per_k = int(g["n_u"]) * int(g["n_w"])
    for q, row in enumerate(g["rows"]):
        k, rel = divmod(int(row), per_k)
        im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                               cfg.abstraction_options(), k_range=(k, 1))
        sp, scol, slo, shi, *_ = im.csr()
        n = int(g["n_s"])
        gm, gx, rm, rx = (np.zeros(n) for _ in range(4))
        b, e = sp[rel], sp[rel + 1]
        gm[scol[b:e]] = slo[b:e]; gx[scol[b:e]] = shi[b:e]
        rb, re_ = g["ptr"][q], g["ptr"][q + 1]
        rm[g["col"][rb:re_]] = g["lo"][rb:re_]; rx[g["col"][rb:re_]] = g["hi"][rb:re_]
        dm, dx = np.abs(gm - rm), np.abs(gx - rx)
        print(f"{name} row {row}: live {np.sum(rx > 1e-12)} min: max {dm.max():.2e} n>1e-12 {np.sum(dm > 1e-12)} "
              f"| max: max {dx.max():.2e} n>1e-12 {np.sum(dx > 1e-12)} n>1e-9 {np.sum(dx > 1e-9)} "
              f"rel {np.max(dx / np.maximum(rx, 1e-300)):.2e} bitwise {np.array_equal(gm, rm) and np.array_equal(gx, rx)}")
