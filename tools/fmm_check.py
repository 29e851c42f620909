"""FMM far field (bpqn_disc_opts.fmm_order) against the direct K1 sum on the GPU (development aid and
profiles/r02_fmm.md): relative L2 error of S, D and S+D layer applies and per-apply times, on jittered
cubic lattices of unit spheres (spacing 2.02, jitter +-0.01, the c4 recipe at other sizes).
  python tools/fmm_check.py --n 5 --p 8 --orders 6,8,10"""
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
ap.add_argument("--n", type=int, default=5)        # lattice n x n x n
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--orders", default="6,8,10")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--modes", default="s,d,sd")
a = ap.parse_args()
rng = np.random.default_rng(20261000 + a.n)
g1 = np.arange(a.n) * 2.02
C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1]) + rng.uniform(-0.01, 0.01, (a.n ** 3, 3))


def timed(g, f, q):
    out = None
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = bp.layer_apply(g, f, q)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return out, float(np.median(ts[1:] if len(ts) > 1 else ts))


t0 = time.time()
gd = bp.Geometry(C, a.p)
t_init_d = time.time() - t0
N = gd.N
f = torch.tensor(rng.standard_normal((N, 3)), device="cuda")
q = torch.tensor(rng.standard_normal((N, 3)), device="cuda")
args = {"s": (f, None), "d": (None, q), "sd": (f, q)}
ref = {}
res = {"spheres": len(C), "p": a.p, "N": N, "direct": {}}
for m in a.modes.split(","):
    ref[m], ms = timed(gd, *args[m])
    res["direct"][m] = {"ms": ms}
del gd
torch.cuda.empty_cache()
for o in [int(x) for x in a.orders.split(",")]:
    op = bp.default_disc_opts()
    op.fmm_order = o
    t0 = time.time()
    g = bp.Geometry(C, a.p, opts=op)
    torch.cuda.synchronize()
    r = {"init_s": round(time.time() - t0, 2)}
    for m in a.modes.split(","):
        u, ms = timed(g, *args[m])
        err = float(torch.linalg.norm(u - ref[m]) / torch.linalg.norm(ref[m]))
        r[m] = {"ms": ms, "rel_l2_vs_direct": err}
    res["fmm_%d" % o] = r
    print(json.dumps({"order": o, **r}), flush=True)
    del g
    torch.cuda.empty_cache()
print(json.dumps(res))
