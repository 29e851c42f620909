"""Relative errors of the GPU LCP MVP and b against the oracle fixtures c1-c4 (GMRES 1e-12; development aid)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2604_10089_b200 as bp
from synth import lambda_test, make_config
for c in (1, 2, 3, 4):
    z = np.load(f'tests/fixtures/c{c}.npz')
    cfg = make_config(c)
    g = bp.Geometry(z['centers'], int(z['p']))
    bp.contacts(g, 0.1)
    gm = bp.default_gmres_opts(tol=1e-12)
    errs = []
    for k in range(z['w_test'].shape[0]):
        w, st = bp.lcp_mvp(g, torch.tensor(lambda_test(c, g.nc, k), device='cuda'), gmres=gm)
        errs.append(np.linalg.norm(w.cpu().numpy() - z['w_test'][k]) / np.linalg.norm(z['w_test'][k]))
    slip = bp.janus_slip(g, cfg['axes'], cfg['slip_B'])
    b, _ = bp.lcp_b(g, torch.tensor(cfg['F_nc'], device='cuda'), slip=slip, gmres=gm)
    eb = np.linalg.norm(b.cpu().numpy() - z['b']) / np.linalg.norm(z['b'])
    print(f"c{c} N={g.N} MVP rel err {max(errs):.2e} (GMRES {st.iters} its)  b rel err {eb:.2e}", flush=True)
