"""Quick GPU-vs-oracle sanity run (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_10089_b200 as bp
from oracle.layer import Disc
from oracle import mobility as mob, lcp

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

rng = np.random.default_rng(0)
for (C, p) in [(np.array([[0.1, -0.2, 0.3], [2.15, 0.4, 0.1]]), 6), (np.array([[0., 0, 0]]), 5)]:
    t = time.time(); g = bp.Geometry(C, p); torch.cuda.synchronize(); tg = time.time() - t
    d = Disc(C, p)
    f = rng.standard_normal((d.N, 3)); q = rng.standard_normal((d.N, 3))
    fd = torch.tensor(f, device='cuda'); qd = torch.tensor(q, device='cuda')
    ref_s = d.apply_all(f=f); ref_d = d.apply_all(q=q)
    us = bp.layer_apply(g, f=fd).cpu().numpy(); ud = bp.layer_apply(g, q=qd).cpu().numpy()
    usd = bp.layer_apply(g, f=fd, q=qd).cpu().numpy()
    print('p', p, 'Np', len(C), 'init %.2fs' % tg, 'inc', g.n_incidences, len(d.inc), 'S rel %.2e D rel %.2e SD rel %.2e' % (rel(us, ref_s), rel(ud, ref_d), rel(usd, ref_s + ref_d)))
    FT = rng.standard_normal((len(C), 6))
    uo, st = bp.mobility_apply(g, torch.tensor(FT, device='cuda'))
    ref = mob.mobility(d, FT)
    print('  mobility rel %.2e iters %d (ms %.1f)' % (rel(uo.cpu().numpy(), ref), st.iters, st.ms))
