"""Per-rank operator time of the sharded layer operator, one GPU (development aid).

  python tools/shard_probe.py [--config 4] [--worlds 2,4,8]

Runs rank 0 of `world` alone with local stand-ins for the collectives (the all-gather tiles
this rank's rows, the reduce-scatter keeps this rank's own partial sums), so the numbers are
this rank's kernel work only -- no NVLink traffic -- for the one-directional and the
symmetric K1 split (bpqn_geometry_shard / bpqn_geometry_shard_symmetric).  Output values are
not the operator (the other ranks' rows are missing).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_10089_b200 as bp  # noqa: E402
from synth import layer_densities, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
cfg = make_config(a.config)
g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
_, q = layer_densities(a.config, g.N)
q = torch.tensor(q, device="cuda")
u = torch.empty((g.N, 3), dtype=torch.float64, device="cuda")


def ag(send, recv):
    recv.view(-1, send.numel())[:] = send


def rs(send, recv):
    recv.copy_(send[:recv.numel()])


def run(label):
    bp.layer_apply(g, q=q, out=u)
    torch.cuda.synchronize()
    k1, k2, tot = [], [], []
    for _ in range(a.reps):
        bp.profile_reset(g, events=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bp.layer_apply(g, q=q, out=u)
        e1.record()
        torch.cuda.synchronize()
        pr = bp.profile_get(g)
        k1.append(pr["ms_allpairs"])
        k2.append(pr["ms_near"])
        tot.append(e0.elapsed_time(e1))
    print("%-32s K1 %.3f ms  K2 %.3f ms  apply %.3f ms" % (label, min(k1), min(k2), min(tot)), flush=True)


run("world 1")
for w in [int(x) for x in a.worlds.split(",")]:
    bp.geometry_shard(g, 0, w, allgather=ag)
    run("world %d one-directional K1" % w)
    bp.geometry_shard(g, 0, w, allgather=ag, symmetric=True, reduce_scatter=rs)
    run("world %d symmetric K1" % w)
    bp.geometry_shard(g, 0, 1)
