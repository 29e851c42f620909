import os, time, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_10089_b200 as bp
from synth import make_config
for c in [4, 5]:
    cfg = make_config(c)
    for mode in ["1", "0"]:
        os.environ["BPQN_NEAR_BRUTE"] = mode
        torch.cuda.synchronize(); t = time.time()
        g = bp.Geometry(cfg["centers"], cfg["p"])
        torch.cuda.synchronize(); ti = time.time() - t
        C1 = cfg["centers"] * 1.0005
        t = time.time(); bp.geometry_update(g, C1); torch.cuda.synchronize(); tu = time.time() - t
        t = time.time(); bp.geometry_update(g, cfg["centers"]); torch.cuda.synchronize(); tu2 = time.time() - t
        print("c%d brute=%s init %.3f s update %.3f / %.3f s n_inc %d" % (c, mode, ti, tu, tu2, g.n_incidences), flush=True)
        del g
    for p in [8, 4]:
        g = bp.Geometry(cfg["centers"], p)
        t = time.time(); bp.geometry_update(g, cfg["centers"] * 1.0005); torch.cuda.synchronize()
        print("c%d p=%d update %.3f s" % (c, p, time.time() - t), flush=True)
