"""Reference outputs of `impact simulate` for the simulation parity tests.

TEST INFRASTRUCTURE ONLY.  For a few golden mini systems (tests/golden/
full_*.npz, produced by the reference), writes the reference controller
with the reference's fileio, runs the REFERENCE CLI
(`impact simulate`, /root/reference/pkg/src/impact/cli.py:177-251) with
fixed seeds, rollouts and steps, and records the SHA-256 of its CSV plus
its printed summary in tests/golden/simulate_digests.json.  Nothing at run
time reads /root/reference.

Usage:  python tests/golden/make_simulate_golden.py
"""

import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from impact import cli as RC  # noqa: E402
from impact import fileio as RF  # noqa: E402

from tests.golden.make_fileio_golden import ref_objects  # noqa: E402
import tests.golden_io as G  # noqa: E402

# (name, seed, rollouts, steps, start_pmin)
CASES = [("robot2d_ra_mini", 0, 300, 25, None),
         ("robot2d_ra_mini", 77, 200, 40, 0.1),
         ("room5d_mini", 3, 200, 30, None),
         ("bas7d_mini", 11, 150, 20, None),
         ("dim6_mini", 5, 100, 30, None)]


def main():
    out = []
    for name, seed, rollouts, steps, pmin in CASES:
        g = G.load("full_" + name)
        imdp, ctrl = ref_objects(name)
        with tempfile.TemporaryDirectory() as d:
            cfgp = os.path.join(d, "sys.cfg")
            with open(cfgp, "w") as fh:
                fh.write(str(g["config"]))
            ctrlp = os.path.join(d, "ctrl.txt")
            RF.save_controller(ctrlp, ctrl)
            csvp = os.path.join(d, "out.csv")
            argv = ["simulate", "--config", cfgp, "--controller", ctrlp,
                    "--out", csvp, "--rollouts", str(rollouts), "--steps",
                    str(steps), "--seed", str(seed)]
            if pmin is not None:
                argv += ["--start-pmin", str(pmin)]
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = RC.main(argv)
            assert rc == 0, rc
            data = open(csvp, "rb").read()
        out.append(dict(name=name, seed=seed, rollouts=rollouts, steps=steps,
                        start_pmin=pmin, csv_sha256=hashlib.sha256(data).hexdigest(),
                        csv_lines=data.count(b"\n"), summary=buf.getvalue()))
        print(name, seed, rollouts, steps, data.count(b"\n"), "lines")
    with open(os.path.join(HERE, "simulate_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
