"""The reference against itself under one-ulp perturbations: how far do the
reference's own vehicle3d bounds move when

  mode libm:  its dynamics' sin / cos / tan / atan come from Python's
              `math` (glibc scalar) instead of numpy's loops,
  mode trig:  every sin / cos / tan / atan result is moved up one ulp
              (np.nextafter) -- a different faithful libm,
  mode ndtr:  every scipy ndtr result is moved up one ulp -- a different
              faithful normal CDF (the GPU's fast objective is within a few
              ulps of scipy's)?

The spread between such runs and the golden rows is the reference's own
reproducibility floor for these rows -- the yardstick for the GPU
deviations in tools/row_parity_report.py.

TEST / MEASUREMENT INFRASTRUCTURE ONLY (imports /root/reference).
Usage: python tools/ref_libm_floor.py MODE [workers] > profiles/r02/ref_floor_MODE_vehicle3d.json
"""
import json
import math
import multiprocessing
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from impact import abstraction as A  # noqa: E402
from impact import expr as E  # noqa: E402
from impact.config import load_config  # noqa: E402

import tests.golden_io as G  # noqa: E402


def _scalar(fn):
    uf = np.frompyfunc(fn, 1, 1)
    return lambda x: np.asarray(uf(x), dtype=float)


def _up(fn):
    return lambda x: np.nextafter(fn(x), np.inf)


MODE = sys.argv[1] if len(sys.argv) > 1 else "libm"
if MODE == "libm":
    E._FUNCS.update({"sin": (_scalar(math.sin), 1),
                     "cos": (_scalar(math.cos), 1),
                     "tan": (_scalar(math.tan), 1),
                     "atan": (_scalar(math.atan), 1)})
elif MODE == "trig":
    E._FUNCS.update({k: (_up(E._FUNCS[k][0]), 1)
                     for k in ("sin", "cos", "tan", "atan")})
elif MODE == "ndtr":
    from impact import noise as N
    N.ndtr = _up(N.ndtr)
else:
    raise SystemExit(f"unknown mode {MODE}")

_CTX = None


def _row(row):
    k, j, i = A.RowIndex(_CTX.n_u, _CTX.n_w).kji(row)
    return A._compute_one_row(_CTX, row, k, j, i)


def main():
    global _CTX
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    g = G.load("rows_vehicle3d")
    path = "/tmp/ref_libm_vehicle3d.cfg"
    with open(path, "w") as fh:
        fh.write(str(g["config"]))
    cfg = load_config(path)
    spaces = (cfg.state_space, cfg.input_space, cfg.disturb_space)
    _CTX = A._make_context(cfg.dynamics, cfg.noise, spaces, cfg.labels(),
                           cfg.abstraction_options())
    rows = [int(r) for r in g["rows"]]
    with multiprocessing.get_context("fork").Pool(workers) as pool:
        res = pool.map(_row, rows, chunksize=1)
    n = int(g["n_s"])
    out = dict(mode=MODE, rows=len(rows), entries=0, bitwise_rows=0, n_gt_1e12=0,
               n_gt_1e9=0, max_abs=0.0, per_row=[])
    for q, (row, r) in enumerate(zip(rows, res)):
        rm, rx = np.zeros(n), np.zeros(n)
        b, e = g["raw_ptr"][q], g["raw_ptr"][q + 1]
        rm[g["raw_col"][b:e]] = g["raw_lo"][b:e]
        rx[g["raw_col"][b:e]] = g["raw_hi"][b:e]
        d = np.maximum(np.abs(r[0] - rm), np.abs(r[1] - rx))
        out["entries"] += int(np.count_nonzero((rm != 0) | (rx != 0)))
        out["bitwise_rows"] += int(np.array_equal(r[0], rm) and
                                   np.array_equal(r[1], rx))
        out["n_gt_1e12"] += int(np.sum(d > 1e-12))
        out["n_gt_1e9"] += int(np.sum(d > 1e-9))
        out["max_abs"] = max(out["max_abs"], float(d.max()))
        if d.max() > 1e-12:
            out["per_row"].append(dict(row=row, n_gt_1e12=int(np.sum(d > 1e-12)),
                                       max_abs=float(d.max())))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
