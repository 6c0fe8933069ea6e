"""Deviation envelope of the GPU construction against the reference's seeded
row samples (tests/golden/rows_*.npz), as JSON -- the evidence behind the
tolerances in tests/test_construct_gpu.py.

Usage (GPU):  python tools/row_parity_report.py [name ...] > report.json
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import tests.golden_io as G  # noqa: E402
from paper_2401_03555_b200 import build_abstraction  # noqa: E402

NAMES = ("robot2d_reachavoid", "vehicle3d", "room5d", "bas7d_verify",
         "dim14_verify", "robot2d_reach")


def report(name):
    g = G.load("rows_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    per_k = int(g["n_u"]) * int(g["n_w"])
    n = int(g["n_s"])
    rows = [int(r) for r in g["rows"]]
    out = dict(rows=len(rows), entries=0, live_mismatch=0, bitwise_rows=0,
               t_max_abs=0.0, t_min_abs=0.0, vec_abs=0.0,
               n_gt_1e12=0, n_gt_1e9=0, n_gt_1e6=0, worst=[])
    built = {}
    for q, row in enumerate(rows):
        k, rel = divmod(row, per_k)
        if k not in built:
            built = {k: build_abstraction(
                cfg.dynamics, cfg.noise, cfg.spaces, labels,
                cfg.abstraction_options(), k_range=(k, 1)).csr()}
        sp, scol, slo, shi, r0, r1, a0, a1 = built[k]
        gm, gx, rm, rx = (np.zeros(n) for _ in range(4))
        b, e = sp[rel], sp[rel + 1]
        gm[scol[b:e]] = slo[b:e]
        gx[scol[b:e]] = shi[b:e]
        rb, re_ = g["ptr"][q], g["ptr"][q + 1]
        rm[g["col"][rb:re_]] = g["lo"][rb:re_]
        rx[g["col"][rb:re_]] = g["hi"][rb:re_]
        dm, dx = np.abs(gm - rm), np.abs(gx - rx)
        d = np.maximum(dm, dx)
        vec = max(abs(r0[rel] - g["r_min"][q]), abs(r1[rel] - g["r_max"][q]),
                  abs(a0[rel] - g["a_min"][q]), abs(a1[rel] - g["a_max"][q]))
        out["entries"] += int(np.count_nonzero((rm != 0) | (rx != 0)))
        out["live_mismatch"] += int(np.sum((gx > 1e-12) != (rx > 1e-12)))
        out["bitwise_rows"] += int(np.array_equal(gm, rm) and
                                   np.array_equal(gx, rx))
        out["t_min_abs"] = max(out["t_min_abs"], float(dm.max()))
        out["t_max_abs"] = max(out["t_max_abs"], float(dx.max()))
        out["vec_abs"] = max(out["vec_abs"], float(vec))
        out["n_gt_1e12"] += int(np.sum(d > 1e-12))
        out["n_gt_1e9"] += int(np.sum(d > 1e-9))
        out["n_gt_1e6"] += int(np.sum(d > 1e-6))
        if d.max() > 1e-12:
            c = int(np.argmax(d))
            out["worst"].append(dict(row=row, col=c, ref_min=rm[c],
                                     ref_max=rx[c], got_min=gm[c],
                                     got_max=gx[c], diff=float(d[c])))
    out["worst"] = sorted(out["worst"], key=lambda w: -w["diff"])[:10]
    return out


def main():
    names = sys.argv[1:] or NAMES
    res = {}
    for name in names:
        if G.have("rows_" + name):
            res[name] = report(name)
            print(name, {k: v for k, v in res[name].items() if k != "worst"},
                  file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
