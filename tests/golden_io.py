"""Helpers to load the reference-generated fixtures (tests/golden/*.npz)."""

import os

import numpy as np

from paper_2401_03555_b200.config import parse_config_text

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

MINIS = ("robot2d_ra_mini", "dim6_mini", "room5d_mini", "vehicle3d_mini",
         "bas4d_mini", "bas7d_mini")


def path(name):
    return os.path.join(GOLDEN, name + ".npz")


def have(name):
    return os.path.exists(path(name))


def load(name):
    return dict(np.load(path(name), allow_pickle=False))


def config_of(g):
    return parse_config_text(str(g["config"]))


def dense(g, prefix=""):
    """Dense (rows, n_s) t_min / t_max from a fixture's CSR."""
    ptr, col = g[prefix + "ptr"], g[prefix + "col"]
    lo, hi = g[prefix + "lo"], g[prefix + "hi"]
    n = len(ptr) - 1
    t_min = np.zeros((n, int(g["n_s"])))
    t_max = np.zeros_like(t_min)
    rows = np.repeat(np.arange(n), np.diff(ptr))
    t_min[rows, col] = lo
    t_max[rows, col] = hi
    return t_min, t_max


def model(g):
    """oracle.iterate.Model of a full_* fixture."""
    from oracle.iterate import Model
    t_min, t_max = dense(g)
    return Model(int(g["n_s"]), int(g["n_u"]), int(g["n_w"]), t_min, t_max,
                 g["r_min"], g["r_max"], g["a_min"], g["a_max"])


def imdp(g):
    """Product Imdp of a full_* fixture (uploaded to the GPU on first use)."""
    from paper_2401_03555_b200.abstraction import Imdp
    cfg = config_of(g)
    t_min, t_max = dense(g)
    return Imdp(cfg.state_space, cfg.input_space, cfg.disturb_space,
                cfg.labels(), t_min, t_max, g["r_min"], g["r_max"],
                g["a_min"], g["a_max"])


def spec_of(cfg):
    return "safety" if cfg.spec_type == "safety" else "reach"
