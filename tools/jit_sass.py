"""Dump the NVRTC construction module of a benchmark (source + cubin) for
SASS inspection on a machine without a GPU:
    python tools/jit_sass.py vehicle3d /tmp/sass
    cuobjdump -sass /tmp/sass/vehicle3d.cubin"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_03555_b200 import abstraction, config  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
os.makedirs(out, exist_ok=True)
cfg = config.benchmark(name)
os.environ["IMPACT_DUMP_JIT"] = "1"
cwd = os.getcwd()
os.chdir(out)
try:
    abstraction.jit_compile(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                            cfg.abstraction_options(),
                            cubin_path=os.path.join(out, name + ".cubin"))
finally:
    os.chdir(cwd)
print(os.path.join(out, name + ".cubin"))
