"""The feature table partitioned by node range (the IGB-shaped case) against the
oracle (run on a B200 with -m gpu).

In one process the shards are separate device allocations (the same addressing the ranks use with
CUDA IPC mappings over NVLink): shard r holds rows [r * shard_rows, (r+1) * shard_rows).  The whole
offline layout reads its rows through that source -- GPU-tier and host-tier fills, the batched pack
-- and must equal the oracle byte for byte: tier buffers, every packed chunk, every assembled batch.
Two processes sharing the GPU (real IPC mappings, gloo) run the same through bench.py's Runner in
tests/test_gpu_bench_contract.py.
"""
import numpy as np
import pytest
import torch

import oracle
from workload import make_workload

pytestmark = pytest.mark.gpu
RNG_SEED = 0x5EEDD15C


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_05231_b200 as dg
    return dg


def _shards(dg, feats: torch.Tensor, world: int):
    N, dim = feats.shape
    shard_rows = (N + world - 1) // world
    bufs = []
    for r in range(world):
        lo, hi = min(N, r * shard_rows), min(N, (r + 1) * shard_rows)
        b = dg._abi.DeviceBuffer(0, max(hi - lo, 1) * feats.element_size() * dim)
        if hi > lo:
            b.view((hi - lo, dim), feats.dtype).copy_(feats[lo:hi])
        bufs.append(b)
    torch.cuda.synchronize()
    return dg._abi.ShardedFeatures.loopback(bufs, N, shard_rows, dim, feats.dtype)


@pytest.mark.parametrize("world,group,stage", [(2, 8, "pinned"), (3, 3, "hbm"), (8, 2, "pinned"), (1, 8, "pinned")])
def test_layout_from_partitioned_table(dg, world, group, stage):
    w = make_workload("tiny")
    dev = torch.device("cuda", 0)
    ctx = dg.Ctx(device=0)
    src = _shards(dg, w.features.to(dev), world)
    L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), src, w.seeds.to(dev), [10, 5], 256, 500, 1000,
                          RNG_SEED, group_size=group, stage=stage)
    ctx.sync()
    ref = oracle.offline_layout(w.indptr.numpy(), w.indices.numpy(), w.features.numpy(), w.seeds.numpy(), 256,
                                [10, 5], RNG_SEED, 500, 1000, group)
    assert np.array_equal(L.gpu_tier.cpu().numpy().reshape(-1), ref["gpu_buf"].reshape(-1))
    assert np.array_equal(L.host_tier.tensor.numpy(), ref["host_buf"].reshape(-1))
    arena = L.arena.tensor.numpy() if stage == "pinned" else L.arena_dev.cpu().numpy()
    for g, (buf, off) in zip(L.groups, ref["groups"]):
        assert np.array_equal(arena[g.arena_off:g.arena_off + g.group_bytes], buf)
    feats = w.features.numpy()
    for b, out in L.assemble_epoch(host_window=3):
        got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(feats, ref["samples"][b].nodes)), f"batch {b}"
    ctx.sync()


def test_igb_rows_through_shards(dg):
    """4 KiB rows (IGB's 1024-d fp32) gathered across shard boundaries equal the closed form."""
    from workload import feature_rows, feature_rows_np
    dev = torch.device("cuda", 0)
    N, dim, world = 10_000, 1024, 4
    feats = feature_rows(torch.arange(N, device=dev), dim)
    src = _shards(dg, feats, world)
    ctx = dg.Ctx(device=0)
    ids = torch.tensor([0, 2499, 2500, 2501, 4999, 5000, 7499, 7500, 9999, 1, 9998, 5000], dtype=torch.int32,
                       device=dev)
    out = torch.empty((ids.numel(), dim), dtype=torch.float32, device=dev)
    dg.dgnn_gather_rows(ctx, src, ids, out)
    ctx.sync()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), feature_rows_np(ids.cpu().numpy(), dim).view(np.uint32))
