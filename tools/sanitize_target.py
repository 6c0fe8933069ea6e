"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
coupled (vehicle3d_mini, room5d_mini) and separable (robot2d_ra_mini)
builds in both construction modes, two-phase synthesis, a row-values call
on rows wider than 16 384 entries, and the device sharded loop with three
shards driven from one process."""
import sys
import numpy as np
sys.path.insert(0, ".")
import tests.golden_io as G  # noqa: E402
from paper_2401_03555_b200 import (build_abstraction, sharded,  # noqa: E402
                                   synthesize_reach, synthesize_safe)
from paper_2401_03555_b200.synthesis import row_values, run_phase  # noqa: E402

for name in ("robot2d_ra_mini", "vehicle3d_mini", "room5d_mini"):
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    for exact in (True, False):
        im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces,
                               cfg.labels(), cfg.abstraction_options(),
                               exact=exact)
    f = synthesize_safe if cfg.spec_type == "safety" else synthesize_reach
    c = f(im, mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon)
    print(name, c.meta["iterations"], flush=True)

rng = np.random.default_rng(1)
n_s, rows = 20000, 3
full = rng.dirichlet(np.ones(n_s + 2), size=rows)
lo, hi = full * 0.7, np.minimum(1.0, full * 1.3 + 1e-7)
w = np.concatenate([rng.uniform(0, 1, n_s), [1.0, 0.0]])
print("wide", row_values(lo[:, :n_s], hi[:, :n_s], lo[:, n_s], hi[:, n_s],
                         lo[:, n_s + 1], hi[:, n_s + 1], w, "min")[:2])

import torch  # noqa: E402
g = G.load("full_robot2d_ra_mini")
cfg = G.config_of(g)
labels = cfg.labels()
im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                       cfg.abstraction_options())
table = sharded.shard_table(im.n_s, 3)
engines = [sharded.CudaShard(build_abstraction(
    cfg.dynamics, cfg.noise, cfg.spaces, labels, cfg.abstraction_options(),
    k_range=(int(table[r]), int(table[r + 1] - table[r]))), 0, table)
    for r in range(3)]
for e in engines:
    e.begin(table, "reach", "min", "max", cfg.eps, None, 10**6)
it = 0
while True:
    it += 1
    for e in engines:
        e.sweep(it)
    chunks = [e.chunk(it).clone() for e in engines]
    st = torch.stack([e.stats for e in engines]).max(dim=0).values
    for e in engines:
        out = e.gathered(it)
        for r, ch in enumerate(chunks):
            out[r * ch.numel():(r + 1) * ch.numel()] = ch
        e.stats.copy_(st)
        e.control()
    if engines[0].poll()[0]:
        break
print("sharded loop iterations", it)
want = run_phase(im, "reach", "min", "max", cfg.eps, None, 10**6)
print("single loop iterations", want.iterations)
