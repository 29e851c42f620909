"""Near-contact accuracy of the discrete mobility (development aid).

Two unit spheres at gap h pushed together by F = (+1, 0, 0) and (-1, 0, 0): the
relative approach velocity U_rel = U_2x - U_1x from bpqn_mobility_apply at several p.
Reported: U_rel, the change against the previous p (discretisation error estimate) and
the ratio to the leading-order lubrication asymptote U_rel ~ 2 F h / (3 pi mu a^2)
(equal spheres, Reynolds lubrication; the ratio should tend to 1 as h -> 0).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402

FT = np.array([[1.0, 0, 0, 0, 0, 0], [-1.0, 0, 0, 0, 0, 0]])
out = []
for h in (0.1, 0.03, 0.01, 0.003):
    prev = None
    for p in (8, 12, 16, 20, 24):
        C = np.array([[0.0, 0.0, 0.0], [2.0 + h, 0.0, 0.0]])
        g = bp.Geometry(C, p)
        uo, st = bp.mobility_apply(g, torch.tensor(FT, device="cuda"),
                                   gmres=bp.default_gmres_opts(tol=1e-12, restart=200, max_iters=4000))
        uo = uo.cpu().numpy()
        urel = uo[1, 0] - uo[0, 0]
        row = dict(h=h, p=p, N=g.N, U_rel=urel, gmres_iters=st.iters,
                   change_vs_prev_p=None if prev is None else abs(urel - prev) / abs(urel),
                   ratio_to_lubrication=urel / (-2.0 * h / (3.0 * np.pi) * 1.0) if urel != 0 else None)
        prev = urel
        out.append(row)
        print(json.dumps(row), flush=True)
        del g
