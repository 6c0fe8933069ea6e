"""Build libimpact_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2401_03555_b200._build [--force]

Every translation unit is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and linked into paper_2401_03555_b200/libimpact_b200.so (git-ignored, but
shipped to the GPU box by gpurun).  The JIT construction source
(csrc/jit/*.cuh) is embedded into the library as a string so NVRTC can
specialise it per dynamics at run time.
"""

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libimpact_b200.so")
OBJ = os.path.join(HERE, "csrc", "_obj")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]
UNITS = ["imdp.cu", "sweep.cu", "build.cu", "export.cu"]
JIT_SOURCES = {"kJitPrelude": ["ndtr.h", "ziggurat_tables.h", "rng.h"],
               "kJitKernels": ["jit/construct.cuh", "jit/simulate.cuh"]}


def _embed_jit():
    """Write csrc/_jit_source.inc: the JIT sources as C++ raw strings
    (kJitPrelude = ndtr.h + numpy's random streams, kJitKernels = the
    construction and simulation kernels); the generated config + dynamics
    go between them at run time."""
    decls = []
    for name, rels in JIT_SOURCES.items():
        body = ""
        for rel in rels:
            with open(os.path.join(CSRC, rel)) as fh:
                text = fh.read().replace("#pragma once", "")
            body += "\n".join(line for line in text.split("\n")
                              if not line.startswith('#include "')) + "\n"
        chunks = [body[i:i + 12000] for i in range(0, len(body), 12000)]
        lit = "\n".join(f'R"IMPJIT({c})IMPJIT"' for c in chunks)
        decls.append(f"static const char {name}[] =\n{lit};\n")
    out = os.path.join(CSRC, "_jit_source.inc")
    new = "\n".join(decls)
    old = open(out).read() if os.path.exists(out) else None
    if old != new:
        with open(out, "w") as fh:
            fh.write(new)


def _digest():
    h = hashlib.sha256()
    for root, _, files in os.walk(CSRC):
        if "_obj" in root:
            continue
        for f in sorted(files):
            if f.endswith((".cu", ".h", ".cuh", ".inc")):
                with open(os.path.join(root, f), "rb") as fh:
                    h.update(f.encode() + fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    """Compile (if sources changed) and return the library path."""
    _embed_jit()
    stamp = os.path.join(OBJ, "stamp")
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) \
            and open(stamp).read() == dig:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    procs = []
    for unit in UNITS:
        obj = os.path.join(OBJ, unit.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((unit, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                             stderr=subprocess.STDOUT)))
        objs.append(obj)
    for unit, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {unit}")
    link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs,
            f"-L{CUDA}/lib64", f"-L{CUDA}/lib64/stubs", "-lcudart", "-lnvrtc", "-Xlinker", f"-rpath,{CUDA}/lib64"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
