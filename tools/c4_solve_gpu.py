"""c4 Bi-PQN LCP solve on the GPU at parity settings (GMRES 1e-12 hi and lo, KKT 1e-10, R9/R12);
writes the solution lambda to gpurun_out/c4_lambda.npy (the candidate the oracle certifies with
tests/fixtures/make_fixtures.py --certify 4, R26 / DESIGN.md R35) and prints the report."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_10089_b200 as bp  # noqa: E402
from synth import make_config  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = make_config(c)
hi = bp.Geometry(cfg["centers"], cfg["p"])
lo = bp.Geometry(cfg["centers"], cfg["p_lo"])
pairs, nrm, gaps = bp.contacts(hi, cfg["delta"])
bp.set_contacts(lo, pairs, nrm, gaps)
gm = bp.default_gmres_opts(tol=1e-12)
slip = bp.janus_slip(hi, cfg["axes"], cfg["slip_B"])
b, _ = bp.lcp_b(hi, torch.tensor(cfg["F_nc"], device="cuda"), slip=slip, gmres=gm)
o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-10)
o.gm_hi.tol = o.gm_lo.tol = 1e-12
lam = torch.zeros(hi.nc, dtype=torch.float64, device="cuda")
t = time.time()
lam, rep, rc = bp.solve_lcp(hi, lo, b, lam, o)
torch.cuda.synchronize()
dt = time.time() - t
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/c%d_lambda.npy" % c, lam.cpu().numpy())
np.save("gpurun_out/c%d_b_gpu.npy" % c, b.cpu().numpy())
print(json.dumps(dict(config=c, rc=rc, s=dt, **rep.as_dict())), flush=True)
