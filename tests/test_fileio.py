"""Text export in the reference's formats.

Pinning chain: the reference's own output files -> SHA-256 digests
(tests/golden/fileio_digests.json, made by make_fileio_golden.py) -> the
oracle writer (oracle/fileio.py) -> the GPU export (csrc/export.cu,
csrc/fmt17.h) through paper_2401_03555_b200.fileio.  Bytes must be
identical.  CPU tests: oracle vs digests, the device formatter source
compiled for the host vs Python's format(), and the host-side loaders.
GPU tests: save_abstraction / save_controller / save_matrix vs digests and
round trips.
"""

import ctypes
import hashlib
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import fileio as OF
from paper_2401_03555_b200 import FileFormatError
from paper_2401_03555_b200 import fileio as F

from . import golden_io as G

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2401_03555_b200", "csrc")
NAMES = ("robot2d_ra_mini", "vehicle3d_mini", "bas7d_mini", "dim6_mini")


def digests():
    with open(os.path.join(G.GOLDEN, "fileio_digests.json")) as fh:
        return json.load(fh)


def sha(b):
    return hashlib.sha256(b).hexdigest()


def fixture(name):
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    return g, cfg, G.imdp(g)


def controller_of(g, cfg, imdp):
    from paper_2401_03555_b200.synthesis import _make_controller
    policy = g["policy"] if imdp.input_space is not None else None
    kind = "safety" if cfg.spec_type == "safety" else "reach"

    class _Ph:
        def __init__(self, it):
            self.iterations, self.fallback, self.ms_device = it, False, 0.0
            self.ms_sweep = 0.0
    return _make_controller(imdp, policy, g["p_min"], g["p_max"], kind,
                            cfg.mode, cfg.eps, cfg.horizon,
                            tuple(_Ph(int(x)) for x in g["iterations"]),
                            with_policy=imdp.input_space is not None)


# --- CPU: the oracle writer is the reference's writer ------------------------

@pytest.mark.parametrize("name", NAMES)
def test_oracle_writer_matches_reference_digests(name):
    want = digests()[name]
    g, cfg, m = fixture(name)
    t_min, t_max = G.dense(g)
    got = {"t_min.txt": OF.matrix_bytes(t_min),
           "t_max.txt": OF.matrix_bytes(t_max),
           "state_space.txt": OF.space_bytes(m.state_space),
           "labels.txt": OF.labels_bytes(m.labels)}
    for k in ("r_min", "r_max", "a_min", "a_max"):
        got[k + ".txt"] = OF.vector_bytes(g[k])
    if m.input_space is not None:
        got["input_space.txt"] = OF.space_bytes(m.input_space)
    c = controller_of(g, cfg, m)
    got["ctrl.txt"] = OF.controller_bytes(c.states, c.coords, c.policy,
                                          c.inputs, c.p_min, c.p_max, c.meta)
    assert set(got) == set(want)
    for k, b in got.items():
        assert sha(b) == want[k], k


@pytest.fixture(scope="module")
def fmt_lib(tmp_path_factory):
    """Host build of csrc/fmt17.h (the device formatter's source)."""
    d = tmp_path_factory.mktemp("fmt17")
    src = d / "fmt_host.cpp"
    src.write_text(
        f'#include "{CSRC}/fmt17.h"\n'
        'extern "C" long fmt(const double* x, long n, char* out) {\n'
        '  long pos = 0;\n'
        '  for (long i = 0; i < n; ++i) { pos += imp_fmt17(x[i], out + pos);'
        ' out[pos++] = 10; }\n  return pos; }\n')
    so = d / "fmt_host.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", str(src), "-o",
                    str(so)], check=True)
    lib = ctypes.CDLL(str(so))
    lib.fmt.restype = ctypes.c_long
    return lib


def test_fmt17_matches_python_format(fmt_lib):
    rng = np.random.default_rng(11)
    edge = [0.0, -0.0, 1.0, 0.5, 0.1, 1e-4, 1e-5, 1e16, 1e17,
            9.999999999999999e16, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, np.inf, -np.inf, np.nan, 1 / 3,
            0.3829249225480262, 123456789012345678.0, 1e22, 1e23]
    x = np.concatenate([
        np.array(edge),
        rng.integers(0, 2**63, size=100000, dtype=np.int64).view(np.float64),
        rng.random(100000),
        rng.random(50000) * 10.0 ** rng.integers(-40, 3, 50000)])
    buf = ctypes.create_string_buffer(len(x) * 27)
    n = fmt_lib.fmt(x.ctypes.data_as(ctypes.c_void_p), len(x), buf)
    got = buf.raw[:n].decode().split("\n")[:-1]
    want = [format(float(v), ".17g") for v in x]
    bad = [(v, a, b) for v, a, b in zip(x, got, want) if a != b]
    assert not bad, bad[:5]


# --- CPU: loaders (host parsing) -----------------------------------------------

def test_loaders_round_trip_oracle_bytes(tmp_path):
    g, cfg, m = fixture("robot2d_ra_mini")
    t_min, _ = G.dense(g)
    (tmp_path / "m.txt").write_bytes(OF.matrix_bytes(t_min))
    assert np.array_equal(F.load_matrix(tmp_path / "m.txt"), t_min)
    (tmp_path / "v.txt").write_bytes(OF.vector_bytes(g["r_max"]))
    assert np.array_equal(F.load_vector(tmp_path / "v.txt"), g["r_max"])
    (tmp_path / "s.txt").write_bytes(OF.space_bytes(m.state_space))
    sp = F.load_space(tmp_path / "s.txt")
    assert np.array_equal(sp.lb, m.state_space.lb)
    (tmp_path / "l.txt").write_bytes(OF.labels_bytes(m.labels))
    lb = F.load_labels(tmp_path / "l.txt")
    assert np.array_equal(lb.safe, m.labels.safe)
    c = controller_of(g, cfg, m)
    (tmp_path / "c.txt").write_bytes(OF.controller_bytes(
        c.states, c.coords, c.policy, c.inputs, c.p_min, c.p_max, c.meta))
    back = F.load_controller(tmp_path / "c.txt")
    assert np.array_equal(back.p_min, c.p_min)
    assert np.array_equal(back.policy, c.policy)
    assert back.meta["iterations"] == tuple(int(i) for i in g["iterations"])


@pytest.mark.parametrize("text,msg", [
    ("imdpmat 2 1 1\n0\n", "bad header"),
    ("imdpmat 1 1 2\n0\n", "expected 2 values"),
    ("imdpmat 1 1 1\n0\n5\n", "trailing data"),
    ("imdpmat 1 2 1\n0\n", "unexpected end of file"),
    ("imdpmat 1 1 1\nx\n", "non-numeric"),
])
def test_load_matrix_errors(tmp_path, text, msg):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(FileFormatError, match=msg):
        F.load_matrix(p)


def test_load_controller_rejects_inverted_bounds(tmp_path):
    p = tmp_path / "c.txt"
    p.write_text("imdpctrl 1\nspec reach\nmode pessimistic\neps 1e-06\n"
                 "horizon infinite\niterations 1 1\npolicy none\ndims 1 0\n"
                 "states 1\n0 0 0.5 0.25\n")
    with pytest.raises(FileFormatError, match="p_min > p_max"):
        F.load_controller(p)


# --- GPU: device export -----------------------------------------------------------

def _dir_digests(d):
    return {f: sha(open(os.path.join(d, f), "rb").read())
            for f in sorted(os.listdir(d))}


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_save_abstraction_matches_reference_bytes(tmp_path, name):
    """Fixture bounds uploaded to the GPU, exported from the device rows."""
    g, cfg, m = fixture(name)
    m.device_handle()
    m._host.pop("t_min")      # force the device path for t
    m._host.pop("t_max")
    F.save_abstraction(tmp_path, m)
    c = controller_of(g, cfg, m)
    F.save_controller(tmp_path / "ctrl.txt", c)
    assert _dir_digests(tmp_path) == digests()[name]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["robot2d_ra_mini", "bas7d_mini",
                                  "dim6_mini"])
def test_gpu_built_abstraction_exports_reference_t_bytes(tmp_path, name):
    """Affine configs build bit-identical bounds, so the t files written
    straight from a GPU build equal the reference's bytes."""
    from paper_2401_03555_b200 import build_abstraction
    g, cfg, _ = fixture(name)
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                           cfg.abstraction_options(), exact=True)
    F.save_abstraction(tmp_path, im)
    want = digests()[name]
    got = _dir_digests(tmp_path)
    for k in ("t_min.txt", "t_max.txt", "labels.txt", "state_space.txt"):
        assert got[k] == want[k], k


@pytest.mark.gpu
def test_save_load_round_trip_bitwise(tmp_path):
    g, cfg, m = fixture("vehicle3d_mini")
    F.save_abstraction(tmp_path, m)
    back = F.load_abstraction(tmp_path)
    for k in ("t_min", "t_max", "r_min", "r_max", "a_min", "a_max"):
        assert np.array_equal(getattr(back, k), getattr(m, k)), k


@pytest.mark.gpu
def test_save_matrix_vector_random(tmp_path):
    rng = np.random.default_rng(5)
    a = rng.random((37, 11)) * 10.0 ** rng.integers(-30, 5, (37, 11))
    a[3] = 0.0
    F.save_matrix(tmp_path / "a.txt", a)
    assert (tmp_path / "a.txt").read_bytes() == OF.matrix_bytes(a)
    v = rng.standard_normal(1001)
    F.save_vector(tmp_path / "v.txt", v)
    assert (tmp_path / "v.txt").read_bytes() == OF.vector_bytes(v)


@pytest.mark.gpu
def test_save_abstraction_rejects_a_shard(tmp_path):
    from paper_2401_03555_b200 import build_abstraction
    g, cfg, _ = fixture("robot2d_ra_mini")
    shard = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                              cfg.labels(), k_range=(0, 3))
    with pytest.raises(ValueError, match="not a shard"):
        F.save_abstraction(tmp_path, shard)
