"""GMRES settings study on one LCP MVP (development aid): iterations / ms / agreement.

  python tools/gmres_study.py [--config 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import lambda_test, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--restarts", default="50,100,200")
a = ap.parse_args()
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
bp.contacts(g, cfg["delta"])
lam = torch.tensor(lambda_test(a.config, g.nc, 0), device="cuda")
ref = None
for tol in (1e-8, 1e-12):
    for pre in (0, 1):
        for rs in [int(x) for x in a.restarts.split(",")]:
            w, st = bp.lcp_mvp(g, lam, gmres=bp.default_gmres_opts(tol=tol, restart=rs, precond=pre))
            w = w.cpu().numpy()
            if ref is None and tol == 1e-12:
                ref = w
            d = None if ref is None else float(np.linalg.norm(w - ref) / np.linalg.norm(ref))
            print(json.dumps(dict(config=a.config, tol=tol, precond=pre, restart=rs, iters=st.iters,
                                  restarts=st.restarts, ms=round(st.ms, 1), rel_resid=st.rel_resid,
                                  rel_diff_vs_first_1e12=d)), flush=True)
