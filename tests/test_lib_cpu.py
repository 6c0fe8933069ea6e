"""The C-ABI library on a CPU-only host: it loads, exports every symbol the
header declares, NVRTC-compiles the construction module for the benchmark
systems, and product entry points fail loudly (no CPU fallback)."""

import os
import re

import pytest

from paper_2401_03555_b200 import _lib
from paper_2401_03555_b200.abstraction import jit_compile
from paper_2401_03555_b200.config import benchmark

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "impact_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|size_t|const char\*)\s+"
                                 r"(imp_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.imp_version().startswith(b"impact_b200")


@pytest.mark.parametrize("name", ["robot2d_reachavoid", "vehicle3d",
                                  "room5d"])
def test_nvrtc_compiles_construction_module(name, tmp_path):
    cfg = benchmark(name)
    out = tmp_path / f"{name}.cubin"
    jit_compile(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                cfg.abstraction_options(), cubin_path=out)
    blob = out.read_bytes()
    assert blob[:4] == b"\x7fELF" and len(blob) > 10000


def test_gpu_entry_points_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2401_03555_b200 import build_abstraction
    cfg = benchmark("robot2d_reach")
    with pytest.raises((RuntimeError, MemoryError)):
        build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels())
