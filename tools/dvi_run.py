"""Longer DVI time-stepping run (bpqn_dvi_step) of the 216-sphere Janus suspension (development aid).

  python tools/dvi_run.py [--steps 50] [--p 8 --p-lo 4] [--dt 1e-2]

Reports per-step contacts, active contacts, hi / lo MVPs, solve status and the minimum gap after the
step (non-negative up to the linearisation of the contact constraint), plus the mean step time.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--p-lo", type=int, default=4)
ap.add_argument("--dt", type=float, default=1e-2)
ap.add_argument("--lo-dense", type=int, default=2)   # R38: 2 = auto
ap.add_argument("--recycle", type=int, default=1)    # GMRES recycling (R33) inside each step's solves (C default)
ap.add_argument("--method", default="bi", choices=["bi", "mono", "bb"])   # LCP solver of each step
ap.add_argument("--gmres-tol", type=float, default=1e-8)   # hi-fidelity eps_gmres
ap.add_argument("--fmm-order", type=int, default=0)  # > 0: hi handle with an FMM, hi MVPs by FMM refinement (R39)
a = ap.parse_args()
cfg = make_config(4)
C = np.ascontiguousarray(cfg["centers"].copy())
A = np.ascontiguousarray(cfg["axes"].copy())
dop = bp.default_disc_opts()
dop.fmm_order = a.fmm_order
hi = bp.Geometry(C, a.p, opts=dop)
lo = bp.Geometry(C, a.p_lo) if a.method == "bi" else None
o = bp.default_solve_opts(method={"mono": 0, "bi": 1, "bb": 2}[a.method], eps_kkt_abs=1e-8, eps_kkt_rel=1e-8,
                          k_max=500, lo_dense=a.lo_dense if a.method == "bi" else 0)
o.gm_hi = bp.default_gmres_opts(tol=a.gmres_tol, recycle=a.recycle, relax_fmm=int(a.fmm_order > 0))
o.gm_lo = bp.default_gmres_opts(tol=1e-8, recycle=a.recycle)
t0 = time.perf_counter()
ms, gaps, bad = [], [], 0
for k in range(a.steps):
    _, r, rc = bp.dvi_step(hi, lo, C, A, cfg["F_nc"], slip_B=cfg["slip_B"], dt=a.dt, delta=cfg["delta"], opts=o)
    ms.append(r.ms_total)
    gaps.append(r.min_gap_after)
    bad += rc != 0
    print("step %3d rc %d contacts %3d active %3d hi %2d lo %3d GMRES its nc %3d c %3d min_gap %+.2e  %.0f ms" %
          (k, rc, r.n_contacts, r.active_contacts, r.lcp.hi_mvps, r.lcp.lo_mvps, r.gm_nc.iters, r.gm_c.iters,
           r.min_gap_after, r.ms_total),
          flush=True)
wall = time.perf_counter() - t0
print("steps %d  failed %d  mean %.0f ms/step  min gap over run %+.2e  wall %.1f s" %
      (a.steps, bad, np.mean(ms), min(gaps), wall))
