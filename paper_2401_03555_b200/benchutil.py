"""Measurement helpers shared by bench.py and the sharded bench step:
nvidia-smi clock / throttle sampling during a timed region, and the host
bytes the public API uploads per build (the e2e line's h2d count)."""

import os
import statistics
import subprocess
import tempfile



class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    INTERVAL_MS = 200

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None
        self.skip = 0

    def mark(self):
        """Start of the timed region: samples written so far (nvidia-smi's
        start-up, which stalls the driver for a second or more, is kept out
        of the timed region by starting the sampler one step earlier) are
        dropped from the summary."""
        if self.proc is None:
            return
        with open(self.path) as fh:
            self.skip = sum(1 for _ in fh)

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.INTERVAL_MS)], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-smi"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for q, line in enumerate(fh):
                if q < self.skip:
                    continue
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        load = [s for s in sm if s > 600] or sm
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap")
        for r in rows:
            for name, val in zip(names, r[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def h2d_bytes(cfg, labels):
    """Bytes the public API uploads per build (geometry, labels, folded
    constants) -- counted from the arrays build_abstraction hands over."""
    from paper_2401_03555_b200.abstraction import describe
    _, keep = describe(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                       cfg.abstraction_options())
    arrays = keep[0]
    return int(sum(a.nbytes for a in arrays.values()))
