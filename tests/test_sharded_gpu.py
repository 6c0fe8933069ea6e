"""The device-resident sharded phase loop (imp_shard_loop_*) on one B200.

* world 1 over NCCL (one process): sharded.synthesize -- device loop, NCCL
  in-place all-gather and all-reduce, CUDA graphs of 16 iterations -- equals
  the single-GPU synthesis bit for bit, with graphs and without;
* 2 / 3 / 4 / 8 shards of a cost-balanced table driven from one process, the
  collectives done by copies between the shards' packed buffers (no rank
  waits on another): the packed layout, uneven shards and the device
  control step give the single-GPU result bit for bit.
Multi-rank exchange logic over a real process group: tests/
test_sharded_gloo.py (gloo, CPU).
"""

import os
import socket

import numpy as np
import pytest

from paper_2401_03555_b200 import (build_abstraction, sharded,
                                   synthesize_reach, synthesize_safe)
from paper_2401_03555_b200.abstraction import state_costs

from . import golden_io as G

pytestmark = pytest.mark.gpu
NAMES = ("robot2d_ra_mini", "room5d_mini")


def _single(cfg, im):
    f = synthesize_safe if cfg.spec_type == "safety" else synthesize_reach
    return f(im, mode=cfg.mode, eps=cfg.eps, horizon=cfg.horizon)


@pytest.fixture(scope="module")
def nccl1():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("graph_iters", (16, 0))
@pytest.mark.parametrize("name", NAMES)
def test_world1_nccl_equals_single_gpu(nccl1, name, graph_iters):
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    im = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, cfg.labels(),
                           cfg.abstraction_options())
    want = _single(cfg, im)
    eng = sharded.CudaShard(im, 0)
    spec = G.spec_of(cfg)
    bound = sharded.LAUNCH_BOUND_MS
    sharded.LAUNCH_BOUND_MS = 1e9     # capture whenever graph_iters > 0
    try:
        p_min, p_max, policy, iters, fb = sharded.synthesize(
            eng, nccl1, spec, cfg.mode, cfg.eps, cfg.horizon,
            graph_iters=graph_iters)
    finally:
        sharded.LAUNCH_BOUND_MS = bound
    assert tuple(iters) == tuple(want.meta["iterations"])
    assert np.array_equal(p_min, want.p_min)
    assert np.array_equal(p_max, want.p_max)
    if want.policy is not None:
        assert np.array_equal(policy, want.policy)
    assert np.max(np.abs(p_min - g["p_min"])) <= 1e-9
    assert np.max(np.abs(p_max - g["p_max"])) <= 1e-9


def _drive(engines, spec, lp, u_obj, eps, horizon, table, fixed=None):
    """The sharded driver's iteration for several shards in one process:
    sweep every shard, 'all-gather' by copying chunks, 'all-reduce' by max,
    control every shard; poll after each iteration."""
    import torch
    for e in engines:
        local = None if fixed is None else \
            fixed[e.k_begin:e.k_begin + e.k_count]
        e.begin(table, spec, lp, u_obj, eps, horizon, 10**6, local)
    it = 0
    while True:
        it += 1
        for e in engines:
            e.sweep(it)
        chunks = [e.chunk(it).clone() for e in engines]
        stats = torch.stack([e.stats for e in engines]).max(dim=0).values
        for e in engines:
            out = e.gathered(it)
            for r, c in enumerate(chunks):
                out[r * c.numel():(r + 1) * c.numel()] = c
            e.stats.copy_(stats)
            e.control()
        done = [e.poll()[0] for e in engines]
        assert len(set(done)) == 1
        if done[0]:
            break
    res = []
    for e in engines:
        v0, v1 = np.empty(e.n_s), np.empty(e.n_s)
        pol = np.empty(max(e.k_count, 1), dtype=np.int64)
        _, out, st = e.poll((v0, v1, pol))
        assert st == 0
        res.append((v0, v1, pol[:e.k_count], out))
    return res


@pytest.mark.parametrize("n_shards", (2, 3, 4, 8))
@pytest.mark.parametrize("name", NAMES)
def test_balanced_shards_equal_single_gpu(name, n_shards):
    g = G.load("full_" + name)
    cfg = G.config_of(g)
    labels = cfg.labels()
    full = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                             cfg.abstraction_options())
    cost = state_costs(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                       cfg.abstraction_options())
    assert len(cost) == full.n_s and np.all(cost >= 1)
    table = sharded.balanced_shards(cost, n_shards)
    engines = []
    for r in range(n_shards):
        sh = build_abstraction(cfg.dynamics, cfg.noise, cfg.spaces, labels,
                               cfg.abstraction_options(),
                               k_range=(int(table[r]),
                                        int(table[r + 1] - table[r])))
        engines.append(sharded.CudaShard(sh, 0, table))
    spec = G.spec_of(cfg)
    if spec == "reach":
        lp1, u_obj = "min", "max"
    else:
        lp1, u_obj = "max", "min"
    from paper_2401_03555_b200.synthesis import run_phase
    want = run_phase(full, spec, lp1, u_obj, cfg.eps, cfg.horizon, 10**6)
    res = _drive(engines, spec, lp1, u_obj, cfg.eps, cfg.horizon, table)
    pol = np.concatenate([r[2] for r in res])
    for v0, v1, _, out in res:
        assert out.iterations == want.iterations
        assert np.array_equal(v0, want.pair.v0)
        assert np.array_equal(v1, want.pair.v1)
    assert np.array_equal(pol, want.policy)
    # phase 2 with the phase-1 policy fixed
    lp2 = "max" if lp1 == "min" else "min"
    want2 = run_phase(full, spec, lp2, u_obj, cfg.eps, cfg.horizon, 10**6,
                      fixed_policy=want.policy)
    res2 = _drive(engines, spec, lp2, u_obj, cfg.eps, cfg.horizon, table,
                  fixed=want.policy)
    for v0, v1, _, out in res2:
        assert out.iterations == want2.iterations
        assert np.array_equal(v0, want2.pair.v0)
        assert np.array_equal(v1, want2.pair.v1)
