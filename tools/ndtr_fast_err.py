"""Ulp error of the fast device CDF form against scipy's golden samples."""
import sys
import numpy as np
sys.path.insert(0, ".")
import tests.golden_io as G
from paper_2401_03555_b200.abstraction import device_ndtr
g = G.load("ndtr")
x, want = g["x"], g["y"]
got = device_ndtr(x, 2)
fin = np.isfinite(x) & (want > 0)
ulps = np.abs(got[fin] - want[fin]) / np.spacing(want[fin])
xf = x[fin]
for lo, hi in ((-40, -11.3), (-11.3, -1.5), (-1.5, -1), (-1, 0), (0, 1), (1, 1.5), (1.5, 11.3), (11.3, 40)):
    m = (xf >= lo) & (xf < hi)
    if m.any():
        i = np.argmax(ulps[m])
        print(f"x in [{lo}, {hi}): n={m.sum()} max ulps {ulps[m].max():.1f} at x={xf[m][i]!r} "
              f"abs {np.abs(got[fin] - want[fin])[m].max():.3g}")
