"""Per-iteration cost of device GMRES (K4) inside one LCP MVP: wall time per Arnoldi iteration with
the captured cycle graph (device-side stopping test, one host sync per restart cycle) against the
kernel time of the operator alone (K1 + K2 + K3 from the library's CUDA events).  The difference
is the per-iteration overhead (CGS2 / Givens kernels, launch gaps).
  python tools/gmres_overhead.py [configs...]   (1, 2, 4; "4lo" = c4 centres at p = 8; "4p4" = at p = 4)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_10089_b200 as bp  # noqa: E402
from synth import lambda_test, make_config  # noqa: E402


def run(tag):
    c = int(tag[0])
    cfg = make_config(c)
    p = cfg["p_lo"] if tag.endswith("lo") else (int(tag.split("p")[1]) if "p" in tag else cfg["p"])
    g = bp.Geometry(cfg["centers"], p)
    bp.contacts(g, cfg["delta"])
    lam = torch.tensor(lambda_test(c, g.nc, 0), device="cuda")
    gm = bp.default_gmres_opts(tol=1e-8)
    for _ in range(3):
        bp.lcp_mvp(g, lam, gmres=gm)
    torch.cuda.synchronize()
    reps = 10 if g.N < 50000 else 3
    t = time.perf_counter()
    for _ in range(reps):
        w, st = bp.lcp_mvp(g, lam, gmres=gm)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3 / reps
    # kernel time of the operator: library events (these MVPs run host-driven)
    bp.profile_reset(g, True)
    bp.lcp_mvp(g, lam, gmres=gm)
    pr = bp.profile_get(g)
    bp.profile_reset(g, False)
    apps = st.applies + 1   # + the single-layer RHS pass
    op_ms = (pr["ms_allpairs"] + pr["ms_near"] + pr["ms_self"]) / apps
    per_it = ms / max(st.iters, 1)
    out = dict(config=tag, N=g.N, iters=st.iters, ms_per_mvp=round(ms, 3), ms_per_iteration=round(per_it, 4),
               operator_ms_per_application=round(op_ms, 4),
               overhead_us_per_iteration=round((ms - op_ms * apps) / max(st.iters, 1) * 1e3, 1))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for tag in (sys.argv[1:] or ["1", "2", "4lo"]):
        run(tag)
