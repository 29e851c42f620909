"""Sharded operator (bpqn_geometry_shard, NEXT-4) -- two or three ranks, one GPU, gloo all-gather.

Each rank computes only its spheres' operator rows and the rows are all-gathered through
the host (gloo); with symmetric=True (bpqn_geometry_shard_symmetric) K1 is the symmetric
kernel over each rank's share of the units and its partial sums are reduce-scattered (gloo:
all-reduce of host copies) first.  No kernel waits on another process, so the ranks may
share the single GPU of the test box.  The sharded LCP MVP and mobility must equal the single-GPU result
(to GMRES tolerance: the sharded K1 is the one-directional kernel) and be bit-identical
on both ranks (replicated deterministic GMRES)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
import paper_2604_10089_b200 as bp
from synth import make_config, lambda_test
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
cfg = make_config({c})
g = bp.Geometry(cfg["centers"], cfg["p"])
bp.contacts(g, 0.1)
bp.geometry_shard(g, rank, world, symmetric={sym})
gm = bp.default_gmres_opts(tol=1e-12)
w, st = bp.lcp_mvp(g, torch.tensor(lambda_test({c}, g.nc, 0), device="cuda"), gmres=gm)
uo, st2 = bp.mobility_apply(g, torch.tensor(np.ones((g.np, 6)) * 0.3, device="cuda"), gmres=gm)
out = dict(rank=rank, w=w.cpu().numpy().tolist(), uo=uo.cpu().numpy().ravel().tolist(), iters=st.iters)
print(json.dumps(out), flush=True)
dist.destroy_process_group()
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("c,world,sym", [(1, 2, False), (2, 2, False), (1, 3, False),
                                         (1, 2, True), (2, 2, True), (2, 3, True)])
def test_sharded_mvp_two_ranks(c, world, sym, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10089_b200 as bp
    from synth import lambda_test, make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], cfg["p"])
    bp.contacts(g, 0.1)
    gm = bp.default_gmres_opts(tol=1e-12)
    w_ref, st_ref = bp.lcp_mvp(g, torch.tensor(lambda_test(c, g.nc, 0), device="cuda"), gmres=gm)
    uo_ref, _ = bp.mobility_apply(g, torch.tensor(np.ones((g.np, 6)) * 0.3, device="cuda"), gmres=gm)
    w_ref, uo_ref = w_ref.cpu().numpy(), uo_ref.cpu().numpy().ravel()
    del g
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, c=c, sym=sym))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), WORLD_SIZE=str(world))
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    w0 = np.array(res[0]["w"])
    for r in res[1:]:                                                  # replicated, deterministic
        assert np.array_equal(w0, np.array(r["w"]))
        assert np.array_equal(np.array(res[0]["uo"]), np.array(r["uo"]))
    assert np.linalg.norm(w0 - w_ref) / np.linalg.norm(w_ref) <= 1e-9
    uo = np.array(res[0]["uo"])
    assert np.linalg.norm(uo - uo_ref) / np.linalg.norm(uo_ref) <= 1e-9


@pytest.mark.parametrize("c,sym", [(1, True), (2, True), (2, False)])
def test_nccl_sharding_one_rank_equals_single_gpu(c, sym):
    """bpqn_geometry_shard_nccl with a one-rank NCCL communicator (the one GPU of the test box):
    the sharded code path -- K1 over the rank's units, NCCL reduce-scatter on the side stream
    overlapping K2, K3 on the owned spheres, NCCL all-gather, all enqueued on the handle's stream
    without host syncs -- gives the single-GPU operator and MVP.  (NCCL refuses two ranks on one
    GPU; the multi-rank split itself is covered by the callback tests above.)"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10089_b200 as bp
    from synth import lambda_test, make_config
    cfg = make_config(c)
    g = bp.Geometry(cfg["centers"], cfg["p"])
    bp.contacts(g, 0.1)
    gm = bp.default_gmres_opts(tol=1e-12)
    lam = torch.tensor(lambda_test(c, g.nc, 0), device="cuda")
    rng = np.random.default_rng(3)
    q = torch.tensor(rng.standard_normal((g.N, 3)), device="cuda")
    u_ref = bp.layer_apply(g, None, q).cpu().numpy()
    w_ref, _ = bp.lcp_mvp(g, lam, gmres=gm)
    w_ref = w_ref.cpu().numpy()
    bp.geometry_shard_nccl(g, 0, 1, bp.nccl_unique_id(), symmetric=sym)
    u = bp.layer_apply(g, None, q).cpu().numpy()
    w, _ = bp.lcp_mvp(g, lam, gmres=gm)       # host-driven steps (first cycle on the handle)
    w2, _ = bp.lcp_mvp(g, lam, gmres=gm)      # NCCL collectives inside the captured cycle graph
    assert np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref) <= 1e-13
    assert np.linalg.norm(w.cpu().numpy() - w_ref) / np.linalg.norm(w_ref) <= 1e-10
    assert np.array_equal(w.cpu().numpy(), w2.cpu().numpy())
    bp.geometry_shard(g, 0, 1)                # back to the single-GPU operator (frees the communicator)
    w3, _ = bp.lcp_mvp(g, lam, gmres=gm)
    assert np.array_equal(w3.cpu().numpy(), w_ref)
