"""Compare two ab_stream.py dumps bit for bit."""
import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    same = np.array_equal(a[k], b[k])
    print(f"  {k}: {'bitwise equal' if same else 'DIFFER max ' + str(np.max(np.abs(a[k] - b[k])))}")
