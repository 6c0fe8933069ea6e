"""Text writers of the reference's file formats -- oracle restatement.

TEST INFRASTRUCTURE.  Restates pkg/src/impact/fileio.py's writers in plain
Python: _fmt = format(x, ".17g") (:36-41), save_matrix (:94-101),
save_vector (:118-123), save_space (:138-143), save_labels (:164-169),
save_controller (:192-215) and save_abstraction (:285-299).  Each returns
the exact bytes the reference writes.  Pinned to the reference itself by
SHA-256 digests of its own output files on golden abstractions/controllers
(tests/golden/make_fileio_golden.py -> tests/golden/fileio_digests.json).
"""

import numpy as np


def fmt(x):
    return format(float(x), ".17g")


def row(values):
    return " ".join(fmt(v) for v in values)


def matrix_bytes(m):
    m = np.atleast_2d(np.asarray(m, dtype=float))
    lines = [f"imdpmat 1 {m.shape[0]} {m.shape[1]}"]
    lines += [row(r) for r in m]
    return ("\n".join(lines) + "\n").encode()


def vector_bytes(v):
    v = np.asarray(v, dtype=float).ravel()
    return ("\n".join([f"imdpvec 1 {len(v)}"] + [fmt(x) for x in v])
            + "\n").encode()


def space_bytes(space):
    return (f"imdpspace 1 {space.dim}\n" + "lb " + row(space.lb) + "\n"
            + "ub " + row(space.ub) + "\n" + "eta " + row(space.eta)
            + "\n").encode()


def labels_bytes(labels):
    out = f"imdplabels 1 {labels.total}\n"
    for key in ("safe", "target", "avoid"):
        out += key + " " + " ".join(str(int(i)) for i in getattr(labels, key))
        out += "\n"
    return out.encode()


def controller_bytes(states, coords, policy, inputs, p_min, p_max, meta):
    n = coords.shape[1]
    m = inputs.shape[1] if inputs is not None else 0
    it = meta.get("iterations", (0, 0))
    out = ["imdpctrl 1", f"spec {meta.get('spec', 'reach')}",
           f"mode {meta.get('mode', 'pessimistic')}",
           f"eps {fmt(meta.get('eps', 0.0))}",
           f"horizon {meta.get('horizon', 'infinite')}",
           f"iterations {int(it[0])} {int(it[1])}",
           f"policy {'inputs' if policy is not None else 'none'}",
           f"dims {n} {m}", f"states {len(states)}"]
    for k in range(len(states)):
        f = [str(int(states[k])), row(coords[k])]
        if policy is not None:
            f.append(str(int(policy[k])))
            if m:
                f.append(row(inputs[k]))
        f += [fmt(p_min[k]), fmt(p_max[k])]
        out.append(" ".join(f))
    return ("\n".join(out) + "\n").encode()
