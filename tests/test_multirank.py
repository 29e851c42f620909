"""World-size-2 checks of bench.py's multi-rank plumbing on CPU (gloo, 127.0.0.1).

DESIGN.md "Multi-GPU": N > 1 runs N independent replicas (weak scaling, no data-path
collective); the only cross-rank operations are the barriers around the timed region
and the max over ranks of the device time.  Here two gloo ranks check that max, that
the reported whole-job value divides by N, and that the reference arm prints on rank 0
only.
"""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import torch.distributed as dist
import bench
dist.init_process_group("gloo")
ws, rank = dist.get_world_size(), dist.get_rank()
bench.barrier(ws)
local_ms = 100.0 + 50.0 * rank          # rank 1 is the slow one
tot = bench.max_over_ranks(ws, local_ms, "cpu")
print(json.dumps({{"rank": rank, "max": tot, "value": tot / (ws * 2)}}), flush=True)
dist.destroy_process_group()
"""


def test_max_over_ranks_gloo(tmp_path):
    port = _free_port()
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=e, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    import json
    lines = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    assert all(l["max"] == 150.0 for l in lines)          # the slowest rank decides
    assert all(l["value"] == 150.0 / 4 for l in lines)    # K = 2 steps x N = 2 replicas


@pytest.mark.slow
def test_reference_arm_rank0_only(tmp_path):
    """torchrun-style launch of `bench.py --impl reference` with 2 gloo ranks: exactly one
    JSON line (rank 0), impl = reference, and both ranks exit 0."""
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2", OMP_NUM_THREADS="2")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                       "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "1"],
                                      env=e, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    import json
    lines = [l for o, _ in outs for l in o.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
