"""One FMM-mode D layer apply on a jittered n^3 lattice (ncu launch-list target; development aid).
  python tools/fmm_probe.py --n 16 --p 8 --order 10 --reps 2
  python tools/fmm_probe.py --config 4 --order 6"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--order", type=int, default=10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--config", type=int, default=0)   # > 0: a BASELINE config's spheres and p instead of the lattice
a = ap.parse_args()
rng = np.random.default_rng(20261000 + a.n)
if a.config:
    from synth.configs import make_config
    cfg = make_config(a.config)
    C, a.p = cfg["centers"], cfg["p"]
else:
    g1 = np.arange(a.n) * 2.02
    C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1]) + rng.uniform(-0.01, 0.01, (a.n ** 3, 3))
op = bp.default_disc_opts()
op.fmm_order = a.order
g = bp.Geometry(C, a.p, opts=op)
q = torch.tensor(rng.standard_normal((g.N, 3)), device="cuda")
for _ in range(a.reps):
    bp.layer_apply(g, None, q)
torch.cuda.synchronize()
print("ok N", g.N)
