"""FMM-accelerated refinement (R39) at N = 589 824 (4 096 spheres, 16^3 lattice, p = 8): one LCP MVP to the DIRECT
1e-8 residual with order-`--order` FMM Krylov steps against the direct MVP (development aid; profiles/r02_fmm_m2l.md).
  python tools/fmm_refine_large.py --order 6"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--order", type=int, default=6)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--direct", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(20260099)
g1 = np.arange(a.n) * 2.02
C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1]) + rng.uniform(-0.01, 0.01, (a.n ** 3, 3))


def mvp(g, lam, gm):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w, st = bp.lcp_mvp(g, lam, gmres=gm)
    torch.cuda.synchronize()
    return w, st, (time.perf_counter() - t0) * 1e3


op = bp.default_disc_opts()
op.fmm_order = a.order
g = bp.Geometry(C, a.p, opts=op)
bp.contacts(g, 0.1)
lam = torch.tensor(np.random.default_rng(7).uniform(0, 1, g.nc), device="cuda")
gr = bp.default_gmres_opts(tol=a.tol, relax_fmm=1)
mvp(g, lam, gr)
w, st, ms = mvp(g, lam, gr)
out = {"N": g.N, "contacts": g.nc, "order": a.order,
       "refined": {"ms": ms, "fmm_steps": st.fmm_applies, "direct_residuals": st.applies - st.fmm_applies,
                   "final_direct_resid": st.rel_resid}}
del g
torch.cuda.empty_cache()
if a.direct:
    gd = bp.Geometry(C, a.p)
    bp.contacts(gd, 0.1)
    wd, std, msd = mvp(gd, lam, bp.default_gmres_opts(tol=a.tol))
    out["direct"] = {"ms": msd, "iters": std.iters}
    out["mvp_rel_diff"] = float(torch.linalg.norm(w - wd) / torch.linalg.norm(wd))
print(json.dumps(out))
