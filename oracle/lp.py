"""Greedy feasible-distribution LP -- oracle restatement (TEST INFRASTRUCTURE).

Restates pkg/src/impact/feasible.py: stable weight order (:53-58), scalar
greedy fill (:61-77) and the row-batched Abel form used in every sweep
(RowsSolver, :80-111).
"""

import numpy as np

from paper_2401_03555_b200.errors import InfeasibleError


def order(weights, direction):
    """Stable argsort, descending for max, ties to the lower slot (:53-58)."""
    w = np.asarray(weights, dtype=float)
    return np.argsort(-w if direction == "max" else w, kind="stable")


def greedy(lower, upper, weights, direction, tol=1e-9):
    """Scalar greedy fill; returns (value, distribution) (:61-77)."""
    lower = np.asarray(lower, float)
    upper = np.asarray(upper, float)
    weights = np.asarray(weights, float)
    if float(np.sum(lower)) > 1 + tol or float(np.sum(upper)) < 1 - tol:
        raise InfeasibleError("no distribution fits the bounds")
    q = lower.copy()
    room = 1.0 - float(np.sum(q))
    for s in order(weights, direction):
        if room <= 0:
            break
        add = min(upper[s] - lower[s], room)
        q[s] += add
        room -= add
    return float(np.dot(weights, q)), q


class Rows:
    """Row-batched greedy values against one shared weight vector (:80-111)."""

    def __init__(self, lower, upper):
        self.lower = np.ascontiguousarray(lower, dtype=float)
        self.head = np.asarray(upper, dtype=float) - self.lower
        self.slack = np.maximum(0.0, 1.0 - self.lower.sum(axis=1))

    def values(self, weights, direction):
        w = np.asarray(weights, dtype=float)
        perm = order(w, direction)
        ws = w[perm]
        fill = np.minimum(np.cumsum(self.head[:, perm], axis=1),
                          self.slack[:, None])
        drop = np.append(ws[:-1] - ws[1:], ws[-1])
        return self.lower @ w + fill @ drop
