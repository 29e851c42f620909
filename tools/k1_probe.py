"""K1/K2/K3 probe for ncu (development aid): layer applies on a BASELINE config.

  python tools/k1_probe.py [--config 4] [--mode d|s|sd] [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import layer_densities, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--mode", default="d")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--save", default="")
ap.add_argument("--p", type=int, default=0)
a = ap.parse_args()
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], a.p or cfg["p"], cfg["radius"], cfg["mu"])
f, q = layer_densities(a.config, g.N)
f = torch.tensor(f, device="cuda") if "s" in a.mode else None
q = torch.tensor(q, device="cuda") if "d" in a.mode else None
u = torch.empty((g.N, 3), dtype=torch.float64, device="cuda")
per, per2 = [], []
tot = dict(ms_allpairs=0.0, allpairs_gflop=0.0, ms_near=0.0, ms_self=0.0)
for _ in range(a.reps):
    bp.profile_reset(g, events=True)
    bp.layer_apply(g, f=f, q=q, out=u)
    pr1 = bp.profile_get(g)
    per.append(round(pr1["ms_allpairs"], 3))
    per2.append(round(pr1["ms_near"], 3))
    for k in tot:
        tot[k] += pr1[k]
torch.cuda.synchronize()
pr = tot
print("N", g.N, "mode", a.mode, "k1 ms/launch %.3f" % (pr["ms_allpairs"] / a.reps),
      "TFLOP/s %.2f" % (pr["allpairs_gflop"] / pr["ms_allpairs"]), "k2 %.3f k3 %.3f" % (pr["ms_near"] / a.reps,
                                                                                     pr["ms_self"] / a.reps),
      "per-launch", per, "k2 per-launch", per2)
if a.save:
    np.save(a.save, u.cpu().numpy())
