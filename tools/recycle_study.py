"""GMRES recycling / deflation study (development aid): a sequence of MVPs on one
geometry with recycle=1, iterations per solve and agreement with cold solves.

  python tools/recycle_study.py --config 2 --n 6
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=6)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--max-iters", type=int, default=400)
a = ap.parse_args()
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], cfg["p"])
bp.contacts(g, 0.1)
rng = np.random.default_rng(1)
warm = bp.default_gmres_opts(tol=a.tol, recycle=1, max_iters=a.max_iters)
cold = bp.default_gmres_opts(tol=a.tol, max_iters=a.max_iters)
for k in range(a.n):
    lam = torch.tensor(rng.uniform(0, 1, g.nc), device="cuda")
    t = time.time()
    try:
        w, st = bp.lcp_mvp(g, lam, gmres=warm)
        rcw = 0
    except bp.BpqnError as e:
        rcw, st, w = e.code, None, None
    tw = time.time() - t
    wc, stc = bp.lcp_mvp(g, lam, gmres=cold)
    d = None if w is None else float(np.linalg.norm(w.cpu().numpy() - wc.cpu().numpy()) / np.linalg.norm(wc.cpu().numpy()))
    print(json.dumps(dict(k=k, rc=rcw, warm_iters=None if st is None else st.iters,
                          warm_resid=None if st is None else st.rel_resid, cold_iters=stc.iters,
                          rel_diff=d, warm_s=round(tw, 3))), flush=True)
