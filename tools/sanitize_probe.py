"""Small end-to-end run for compute-sanitizer (development aid): contacts, layer
applies (S, D, S+D) and one MVP at c1 and c2, one Mono-PQN solve at c1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import lambda_test, layer_densities, make_config  # noqa: E402

for c in (1, 2):
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], cfg["p"])
    bp.contacts(g, 0.1)
    f, q = layer_densities(c, g.N)
    f, q = torch.tensor(f, device="cuda"), torch.tensor(q, device="cuda")
    for a, b in ((f, None), (None, q), (f, q)):
        bp.layer_apply(g, a, b)
    w, st = bp.lcp_mvp(g, torch.tensor(lambda_test(c, g.nc, 0), device="cuda"),
                       gmres=bp.default_gmres_opts(tol=1e-10, recycle=1))
    print("c%d mvp its %d" % (c, st.iters))
    if c == 1:
        b = torch.tensor(np.linspace(-0.05, 0.05, g.nc), device="cuda")
        lam, rep, rc = bp.solve_lcp(g, None, b, torch.zeros(g.nc, dtype=torch.float64, device="cuda"))
        print("solve rc", rc, rep.iterations)
torch.cuda.synchronize()
print("ok")
