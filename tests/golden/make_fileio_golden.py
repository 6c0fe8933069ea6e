"""Digests of the REFERENCE's own text files for the fileio parity tests.

TEST INFRASTRUCTURE ONLY.  Loads the golden abstractions / controllers
(tests/golden/full_*.npz, themselves produced by the reference), writes them
with the reference's fileio (/root/reference/pkg/src/impact/fileio.py:
save_abstraction :285-299, save_controller :192-215) into a temp directory,
and records the SHA-256 of every file in tests/golden/fileio_digests.json.
The tests check the oracle writer (oracle/fileio.py) and the GPU export
against these digests; nothing at run time reads /root/reference.

Usage:  python tests/golden/make_fileio_golden.py
"""

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from impact import abstraction as RA  # noqa: E402
from impact import fileio as RF  # noqa: E402
from impact import grid as RG  # noqa: E402
from impact import synthesis as RS  # noqa: E402
from impact.config import load_config  # noqa: E402

import tests.golden_io as G  # noqa: E402

NAMES = ("robot2d_ra_mini", "vehicle3d_mini", "bas7d_mini", "dim6_mini")


def ref_objects(name):
    g = G.load("full_" + name)
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as fh:
        fh.write(str(g["config"]))
    cfg = load_config(fh.name)
    os.unlink(fh.name)
    state, inp, dist = cfg.state_space, cfg.input_space, cfg.disturb_space
    labels = cfg.labels()
    t_min, t_max = G.dense(g)
    imdp = RA.Imdp(state, inp, dist, labels, t_min, t_max, g["r_min"],
                   g["r_max"], g["a_min"], g["a_max"])
    ctrl = None
    if str(g["error"]) == "":
        policy = g["policy"] if inp is not None else None
        it = tuple(int(x) for x in g["iterations"])
        ctrl = RS._make_controller(
            imdp, policy, g["p_min"], g["p_max"],
            "safety" if cfg.spec_type == "safety" else "reach",
            cfg.mode, cfg.eps, cfg.horizon, it,
            with_policy=inp is not None)
    return imdp, ctrl


def digest(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def main():
    out = {}
    for name in NAMES:
        imdp, ctrl = ref_objects(name)
        with tempfile.TemporaryDirectory() as d:
            RF.save_abstraction(d, imdp)
            files = {f: digest(os.path.join(d, f)) for f in sorted(os.listdir(d))}
            if ctrl is not None:
                RF.save_controller(os.path.join(d, "ctrl.txt"), ctrl)
                files["ctrl.txt"] = digest(os.path.join(d, "ctrl.txt"))
        out[name] = files
        print(name, len(files), "files")
    with open(os.path.join(HERE, "fileio_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
