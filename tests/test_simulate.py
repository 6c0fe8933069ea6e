"""Closed-loop simulation against the reference CLI.

Pinning chain: `impact simulate` of the reference -> SHA-256 of its CSV and
its summary (tests/golden/simulate_digests.json) -> the oracle restatement
(oracle/simulate.py, numpy's own random streams) -> the GPU rollouts
(csrc/jit/simulate.cuh with numpy's SeedSequence / Philox / ziggurat normal
and glibc log1p restated in csrc/rng.h).  CPU: oracle vs digests, and the
rng.h source built for the host vs numpy on millions of draws.  GPU: CSV
bytes and summary vs the reference's.
"""

import ctypes
import hashlib
import json
import os
import random
import subprocess

import numpy as np
import pytest

from oracle import simulate as OS

from . import golden_io as G
from .test_fileio import controller_of

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2401_03555_b200", "csrc")


def cases():
    with open(os.path.join(G.GOLDEN, "simulate_digests.json")) as fh:
        return json.load(fh)


def setup_case(c):
    g = G.load("full_" + c["name"])
    cfg = G.config_of(g)
    cfg.seed = c["seed"]
    return cfg, controller_of(g, cfg, G.imdp(g))


@pytest.mark.parametrize("c", cases(), ids=lambda c: f"{c['name']}-{c['seed']}")
def test_oracle_matches_reference_cli(c):
    cfg, ctrl = setup_case(c)
    data, summary = OS.simulate(cfg, ctrl, c["rollouts"], c["steps"],
                                c["start_pmin"])
    assert hashlib.sha256(data).hexdigest() == c["csv_sha256"]
    assert summary == c["summary"]


@pytest.fixture(scope="module")
def rng_lib(tmp_path_factory):
    """Host build of csrc/rng.h (+ ndtr.h for glibc exp)."""
    d = tmp_path_factory.mktemp("rng")
    src = d / "rng_host.cpp"
    src.write_text(
        f'#include "{CSRC}/ndtr.h"\n#include "{CSRC}/rng.h"\n'
        'extern "C" void derive(unsigned long long b, long r, long d,'
        ' unsigned long long* o) { unsigned long long k[2] ='
        ' {(unsigned long long)r, (unsigned long long)d};'
        ' imp_seedseq(b, k, 2, o, 1); }\n'
        'extern "C" void normals(unsigned long long s, long n, double* o)'
        ' { ImpPhilox g; imp_philox_seed(&g, s);'
        ' for (long i = 0; i < n; ++i) o[i] = imp_std_normal(&g); }\n'
        'extern "C" void raws(unsigned long long s, long n,'
        ' unsigned long long* o) { ImpPhilox g; imp_philox_seed(&g, s);'
        ' for (long i = 0; i < n; ++i) o[i] = imp_philox_next(&g); }\n'
        'extern "C" void l1p(const double* x, long n, double* o)'
        ' { for (long i = 0; i < n; ++i) o[i] = imp_log1p(x[i]); }\n')
    so = d / "rng_host.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC",
                    str(src), "-o", str(so), "-lm"], check=True)
    return ctypes.CDLL(str(so))


def test_seedsequence_matches_numpy(rng_lib):
    out = (ctypes.c_ulonglong * 1)()
    rnd = random.Random(3)
    for _ in range(2000):
        b = rnd.getrandbits(64)
        r, d = rnd.randrange(0, 10**6), rnd.randrange(0, 4)
        rng_lib.derive(ctypes.c_ulonglong(b), r, d, out)
        assert out[0] == OS.derive_seed(b, r, d)


def test_philox_and_normal_streams_match_numpy(rng_lib):
    for seed in (0, 7, 2**64 - 1, OS.derive_seed(0, 5, 0)):
        raw = (ctypes.c_ulonglong * 64)()
        rng_lib.raws(ctypes.c_ulonglong(seed), 64, raw)
        bg = np.random.Philox(np.random.SeedSequence(seed))
        assert list(raw) == [int(bg.random_raw()) for _ in range(64)]
        n = 400000    # ~100 tail and ~4000 wedge draws
        y = np.empty(n)
        rng_lib.normals(ctypes.c_ulonglong(seed), n,
                        y.ctypes.data_as(ctypes.c_void_p))
        assert np.array_equal(y, OS.generator(seed).normal(0.0, 1.0, n))


def test_log1p_matches_glibc(rng_lib):
    import math
    rng = np.random.default_rng(2)
    x = np.concatenate([-rng.random(300000), rng.random(100000) * 10,
                        (rng.random(100000) - 0.5) * 1e-6,
                        -(rng.integers(0, 2**53, 100000) * 2.0**-53)])
    y = np.empty_like(x)
    rng_lib.l1p(x.ctypes.data_as(ctypes.c_void_p), len(x),
                y.ctypes.data_as(ctypes.c_void_p))
    want = np.array([math.log1p(v) for v in x])
    assert np.array_equal(y, want)


# --- GPU ---------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("c", cases(), ids=lambda c: f"{c['name']}-{c['seed']}")
def test_gpu_rollouts_match_reference_cli(c, tmp_path):
    from paper_2401_03555_b200.simulate import simulate
    cfg, ctrl = setup_case(c)
    res = simulate(cfg, ctrl, c["rollouts"], c["steps"], c["start_pmin"])
    res.write_csv(tmp_path / "out.csv")
    data = (tmp_path / "out.csv").read_bytes()
    assert hashlib.sha256(data).hexdigest() == c["csv_sha256"]
    assert res.summary(c["steps"]) + "\n" == c["summary"]


@pytest.mark.gpu
def test_gpu_rollouts_many_match_oracle():
    """10 000 rollouts (thousands of tail / wedge normal draws): every
    trace point bit-identical to the oracle's."""
    from paper_2401_03555_b200.simulate import simulate
    g = G.load("full_robot2d_ra_mini")
    cfg = G.config_of(g)
    cfg.seed = 12345
    ctrl = controller_of(g, cfg, G.imdp(g))
    res = simulate(cfg, ctrl, 10000, 30)
    want, _ = OS.simulate(cfg, ctrl, 10000, 30)
    assert res.csv_bytes() == want


@pytest.mark.gpu
def test_simulate_argument_errors():
    from paper_2401_03555_b200 import ConfigError
    from paper_2401_03555_b200.simulate import simulate
    g = G.load("full_robot2d_ra_mini")
    cfg = G.config_of(g)
    ctrl = controller_of(g, cfg, G.imdp(g))
    with pytest.raises(ConfigError, match="must be >= 1"):
        simulate(cfg, ctrl, 0, 10)
    with pytest.raises(ConfigError, match="no states with p_min"):
        simulate(cfg, ctrl, 5, 10, start_pmin=2.0)
