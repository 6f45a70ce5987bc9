"""One-sided peer-memory GPU tier: the sharded tier read directly from
each owner's HBM by the assembly kernel (dgnn_assemble_group_peer), no exchange round.

* loopback: every shard in one process, worlds 1 / 2 / 3 / 8;
* two processes on the one GPU of this box, shards exported / mapped with CUDA IPC and the
  handles all-gathered over a gloo group -- the production code path except for NVLink itself.
Every assembled batch equals the oracle's direct gather.
"""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

import oracle
from workload import make_workload

pytestmark = pytest.mark.gpu
RNG_SEED = 0x5EEDD15C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_05231_b200 as dg
    return dg


@pytest.mark.parametrize("world,window", [(1, 1), (2, 64), (3, 4), (8, 128)])
def test_peer_tier_loopback(dg, world, window):
    from paper_2405_05231_b200 import shard
    ctx = dg.Ctx(device=0)
    w = make_workload("tiny")
    dev = torch.device("cuda", 0)
    feats = w.features.to(dev)
    L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), feats, w.seeds.to(dev), [10, 5], 256, 500, 1000,
                          RNG_SEED, group_size=8)
    tier = shard.PeerTier.loopback(ctx, feats, L.plan, world)
    ref = oracle.sample(w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy(), 256, [10, 5], RNG_SEED)
    for b, out in L.assemble_epoch(host_window=window, peer_tier=tier, out_budget=600_000):
        got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(w.features.numpy(), ref[b].nodes)), f"batch {b}"
    ctx.sync()


WORKER = r'''
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["DGNN_ROOT"])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["PORT"], rank=rank, world_size=world)
import paper_2405_05231_b200 as dg
from paper_2405_05231_b200 import shard
import oracle
from workload import make_workload
ctx = dg.Ctx(device=0)
w = make_workload("tiny")
dev = torch.device("cuda", 0)
feats = w.features.to(dev)
# every rank derives the identical plan from the same epoch (counts would be all-reduced
# when ranks sample different batches; here each rank assembles every batch)
L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), feats, w.seeds.to(dev), [10, 5], 256, 500, 1000,
                      0x5EEDD15C, group_size=8)
tier = shard.PeerTier(ctx, feats, L.plan, rank, world, shard.all_gather_handles)
assert len(tier.maps) == world - 1
dist.barrier()  # every shard is mapped before anyone reads
ref = oracle.sample(w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy(), 256, [10, 5], 0x5EEDD15C)
bad = 0
for b, out in L.assemble_epoch(host_window=4, peer_tier=tier):
    got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
    bad += int(not np.array_equal(got, oracle.assemble(w.features.numpy(), ref[b].nodes)))
ctx.sync()
dist.barrier()  # nobody unmaps / frees a shard another rank may still read
print("RANK", rank, "BAD", bad, flush=True)
dist.destroy_process_group()
'''


def test_peer_tier_two_processes_ipc(dg):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = os.path.join(tempfile.mkdtemp(prefix="dgnn_peer_"), "worker.py")
    with open(path, "w") as f:
        f.write(WORKER)
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", PORT=str(port), DGNN_ROOT=ROOT)
        procs.append(subprocess.Popen([sys.executable, path], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True, cwd=ROOT))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, o[-3000:]
        assert f"RANK {r} BAD 0" in o, o[-3000:]
