"""Correctness of every K1 launch shape (BPQN_K1_CFG) against the one-directional kernel (BPQN_K1=asym)
on a BASELINE config: relative L2 difference of S, D and S+D layer applies.  Run once per shape:
  for c in 0 1 ... ; do BPQN_K1_CFG=$c python tools/k1_cfg_check.py --config 1; done"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--save", default="")
ap.add_argument("--cfgs", default="")
a = ap.parse_args()
if a.cfgs:   # driver: reference (one-directional) then every shape in a fresh process
    ref = "/tmp/k1ref_%d.npz" % a.config
    env = dict(os.environ, BPQN_K1="asym")
    subprocess.check_call([sys.executable, __file__, "--config", str(a.config), "--save", ref], env=env)
    import numpy as np
    R = np.load(ref)
    for c in a.cfgs.split(","):
        out = "/tmp/k1cfg_%s_%d.npz" % (c, a.config)
        env = dict(os.environ, BPQN_K1_CFG=c)
        rc = subprocess.call([sys.executable, __file__, "--config", str(a.config), "--save", out], env=env)
        if rc:
            print("cfg", c, "FAILED rc", rc, flush=True)
            continue
        Z = np.load(out)
        errs = {k: float(np.linalg.norm(Z[k] - R[k]) / np.linalg.norm(R[k])) for k in R.files}
        print("cfg", c, {k: "%.2e" % v for k, v in errs.items()}, flush=True)
    sys.exit(0)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2604_10089_b200 as bp  # noqa: E402
from synth import layer_densities, make_config  # noqa: E402
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], cfg["p"])
f, q = layer_densities(a.config, g.N) if a.config == 5 else (np.random.default_rng(1).standard_normal((g.N, 3)),
                                                            np.random.default_rng(2).standard_normal((g.N, 3)))
f, q = torch.tensor(f, device="cuda"), torch.tensor(q, device="cuda")
res = dict(S=bp.layer_apply(g, f, None).cpu().numpy(), D=bp.layer_apply(g, None, q).cpu().numpy(),
           SD=bp.layer_apply(g, f, q).cpu().numpy())
np.savez(a.save, **res)
