"""FMM-accelerated refinement (bpqn_gmres_opts.relax_fmm: Krylov steps with the FMM far field, cycles from the direct residual) against the
direct LCP MVP at a BASELINE config (development aid for profiles/r02_fmm_refine.md): per FMM order and tree depth,
the FMM D apply time and error against the direct one, then MVP time, GMRES steps (FMM) and direct residuals, the final
direct residual and the MVP's relative difference from the direct MVP.
  python tools/fmm_refine_probe.py --config 4 --orders 4,5,6,8 --levels 3 --deltas 0,1e-2,1e-3"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth.configs import make_config, lambda_test, layer_densities  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--orders", default="6,8,10")
ap.add_argument("--levels", default="2,3")
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--deltas", default="0", help="relax_delta values (0 = the library default)")
a = ap.parse_args()
cfg = make_config(a.config)
C, p = cfg["centers"], cfg["p"]


def ev_time(fn, reps):
    out, ts = None, []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return out, float(np.median(ts[1:] if len(ts) > 1 else ts))


gd = bp.Geometry(C, p)
N = gd.N
bp.contacts(gd, 0.1)
lam = torch.tensor(lambda_test(a.config, gd.nc), device="cuda")
_, q = layer_densities(a.config, N)
q = torch.tensor(q, device="cuda")
uD, msD = ev_time(lambda: bp.layer_apply(gd, None, q), a.reps)
gm = bp.default_gmres_opts(tol=a.tol)
(wD, stD), msmD = ev_time(lambda: bp.lcp_mvp(gd, lam, gmres=gm), a.reps)
print(json.dumps({"config": a.config, "N": N, "direct": {"d_apply_ms": msD, "mvp_ms": msmD, "iters": stD.iters,
                                                        "applies": stD.applies}}), flush=True)
for lv in [int(x) for x in a.levels.split(",")]:
    os.environ["BPQN_FMM_LEVELS"] = str(lv)
    for o in [int(x) for x in a.orders.split(",")]:
        op = bp.default_disc_opts()
        op.fmm_order = o
        g = bp.Geometry(C, p, opts=op)
        bp.contacts(g, 0.1)
        u, ms = ev_time(lambda: bp.layer_apply(g, None, q), a.reps)
        err = float(torch.linalg.norm(u - uD) / torch.linalg.norm(uD))
        r = {"levels": lv, "order": o, "fmm_d_apply_ms": ms, "d_rel_err": err}
        for dl in [float(x) for x in a.deltas.split(",")]:
            gr = bp.default_gmres_opts(tol=a.tol, relax_fmm=1, relax_delta=dl)
            r["relax_delta"] = dl
            (w, st), msm = ev_time(lambda: bp.lcp_mvp(g, lam, gmres=gr), a.reps)
            r.update(mvp_ms=msm, iters=st.iters, applies=st.applies, fmm_applies=st.fmm_applies,
                     restarts=st.restarts, final_resid=st.rel_resid,
                     mvp_rel_diff=float(torch.linalg.norm(w - wD) / torch.linalg.norm(wD)))
            print(json.dumps(r), flush=True)
        del g
        torch.cuda.empty_cache()
