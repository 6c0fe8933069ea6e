import numpy as np, sys
sys.path.insert(0,'.')
import tests.golden_io as G
from paper_2401_03555_b200 import build_abstraction
for name in ["room5d_mini","vehicle3d_mini","bas4d_mini","bas7d_mini"]:
    g=G.load("full_"+name); cfg=G.config_of(g)
    im=build_abstraction(cfg.dynamics,cfg.noise,cfg.spaces,cfg.labels(),cfg.abstraction_options())
    rmin,rmax=G.dense(g)
    print(name, im.build_report)
    for k,got,ref in (("t_min",im.t_min,rmin),("t_max",im.t_max,rmax),("r_min",im.r_min,g["r_min"]),("r_max",im.r_max,g["r_max"]),("a_min",im.a_min,g["a_min"]),("a_max",im.a_max,g["a_max"])):
        d=np.abs(got-ref); rel=d/np.maximum(np.abs(ref),1e-300)
        print(f"  {k}: max {d.max():.3e} n>1e-15 {np.sum(d>1e-15)} n>1e-12 {np.sum(d>1e-12)} n>1e-9 {np.sum(d>1e-9)} maxrel {np.max(rel[ref!=0]) if np.any(ref!=0) else 0:.2e}")
    d=np.abs(im.t_max-rmax); i=np.unravel_index(np.argmax(d),d.shape); print("  worst", i, im.t_max[i], rmax[i], im.t_min[i], rmin[i])
    print("  live mismatch", np.sum((im.t_max>1e-12)!=(rmax>1e-12)))
