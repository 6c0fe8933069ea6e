"""World-1 NCCL sharded phase 1 of a config: device ms with CUDA graphs of
G iterations vs eager, against the single-GPU loop (diagnostic)."""
import os
import sys
import time
sys.path.insert(0, ".")
import torch
import torch.distributed as dist
from paper_2401_03555_b200 import build_abstraction, sharded
from paper_2401_03555_b200.config import benchmark
from paper_2401_03555_b200.synthesis import run_phase as single_phase

name = sys.argv[1]
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("nccl", rank=0, world_size=1)
cfg = benchmark(name)
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                       cfg.abstraction_options())
spec = "safety" if cfg.spec_type == "safety" else "reach"
lp, u = ("max", "min") if spec == "safety" else ("min", "max")
for rep in range(2):
    t0 = time.perf_counter()
    r = single_phase(im, spec, lp, u, cfg.eps, cfg.horizon, 10**6)
    print(f"single: it {r.iterations} ms_device {r.ms_device:.1f} wall {1e3*(time.perf_counter()-t0):.1f}")
for G in (16, 2, 0, 64):
    eng = sharded.CudaShard(im, 0)
    for rep in range(2):
        torch.cuda.synchronize()
        e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e1.record()
        ph = sharded.run_phase(eng, dist, spec, lp, u, cfg.eps, cfg.horizon, 10**6, graph_iters=G)
        e2.record(); torch.cuda.synchronize()
        print(f"G={G}: it {ph.iterations} graphs {ph.graphs} device {e1.elapsed_time(e2):.1f} ms wall {1e3*(time.perf_counter()-t0):.1f} ms")
    eng.free()
dist.destroy_process_group()
