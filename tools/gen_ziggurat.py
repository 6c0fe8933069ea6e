"""Extract numpy's ziggurat tables (Generator.normal) and verify them.

TOOLING (not product code at run time).  numpy's Generator.normal draws
with the 256-strip ziggurat of numpy/random/src/distributions/
ziggurat_constants.h (ki_double, wi_double, fi_double), compiled into
numpy/random/_generator*.so.  The tables are located in that binary by
ki_double[0] = 0x000EF33D8025EF6A and laid out fi | wi | ki.  They are
verified by replaying Generator.normal bit for bit from the raw Philox
stream with random_standard_normal's algorithm (distributions.c), then
written to paper_2401_03555_b200/csrc/ziggurat_tables.h.

    python tools/gen_ziggurat.py
"""
import glob
import math
import os
import struct

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2401_03555_b200", "csrc", "ziggurat_tables.h")
ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def tables():
    so = glob.glob(os.path.join(os.path.dirname(np.__file__), "random",
                                "_generator*.so"))[0]
    b = open(so, "rb").read()
    off = b.find(struct.pack("<Q", 0x000EF33D8025EF6A))
    assert off > 4096
    fi = np.frombuffer(b[off - 4096:off - 2048], dtype="<f8").copy()
    wi = np.frombuffer(b[off - 2048:off], dtype="<f8").copy()
    ki = np.frombuffer(b[off:off + 2048], dtype="<u8").copy()
    return ki, wi, fi


def normal_stream(raw, ki, wi, fi, count):
    """random_standard_normal (distributions.c) over a uint64 iterator."""
    out = []

    def next_double():
        return (next(raw) >> 11) * (1.0 / 9007199254740992.0)
    while len(out) < count:
        r = next(raw)
        idx = r & 0xff
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000fffffffffffff
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            out.append(x)
            continue
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-next_double())
                yy = -math.log1p(-next_double())
                if yy + yy > xx * xx:
                    out.append(-(ZIG_R + xx) if (rabs >> 8) & 1
                               else ZIG_R + xx)
                    break
        else:
            if (fi[idx - 1] - fi[idx]) * next_double() + fi[idx] < \
                    math.exp(-0.5 * x * x):
                out.append(x)
    return out


def verify(ki, wi, fi, n=400000):
    for seed in (1, 12345, 2**63 + 7):
        ss = np.random.SeedSequence(seed)
        g = np.random.Generator(np.random.Philox(ss))
        want = g.normal(0.0, 1.0, n)
        bg = np.random.Philox(np.random.SeedSequence(seed))
        raw = (int(v) for v in iter(lambda: bg.random_raw(), None))
        got = np.array(normal_stream(raw, ki, wi, fi, n))
        assert np.array_equal(got, want), (seed, np.flatnonzero(got != want)[:5])


def main():
    ki, wi, fi = tables()
    verify(ki, wi, fi)
    with open(OUT, "w") as fh:
        fh.write("// numpy's ziggurat tables for Generator.normal (256 strips):\n"
                 "// ki_double / wi_double / fi_double of numpy/random/src/\n"
                 "// distributions/ziggurat_constants.h, extracted from the\n"
                 f"// installed numpy {np.__version__} and verified bit for bit "
                 "by\n// tools/gen_ziggurat.py.  Generated file.\n#pragma once\n")
        fh.write("IMP_CONST unsigned long long imp_zig_ki[256] = {\n")
        fh.write(",\n".join(f"    0x{int(v):016x}ull" for v in ki) + "};\n")
        for name, arr in (("imp_zig_wi", wi), ("imp_zig_fi", fi)):
            fh.write(f"IMP_CONST unsigned long long {name}[256] = {{\n")
            fh.write(",\n".join(
                f"    0x{struct.unpack('<Q', struct.pack('<d', float(v)))[0]:016x}ull"
                for v in arr) + "};\n")
    print("verified; wrote", OUT)


if __name__ == "__main__":
    main()
