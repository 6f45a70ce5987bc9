"""The multi-GPU product path over NCCL (runs when >= 2 GPUs are visible; skipped otherwise).

One process per GPU, backend "nccl".  The ranks split one epoch of the tiny config into
contiguous batch blocks (batch ids are global, so placement never changes an output),
all-reduce the access counts over NCCL (a4) and derive the tier plan (a5).  Then:
  * counts and tier map equal the single-process oracle over the whole epoch (G-invariance);
  * every rank's packed chunks equal the oracle's pack of its batches;
  * every batch is assembled three ways and must equal the oracle's direct gather:
    the replicated GPU tier; the GPU tier sharded over the ranks with remote rows fetched by
    the NCCL all-to-all exchange (shard.fetch_remote_rows); and the sharded tier read one-sided
    through CUDA IPC peer mappings over NVLink (shard.PeerTier).
The same checks run with gloo and both ranks on one GPU in test_gpu_multirank.py /
test_gpu_peer_tier.py; this file is the NCCL / multi-device half.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

RNG_SEED = 0x5EEDD15C
FAN, B, GPU_ROWS, HOST_ROWS, GROUP = [10, 5], 256, 500, 1000, 2


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        import oracle
        import paper_2405_05231_b200 as dg
        from paper_2405_05231_b200 import shard
        from paper_2405_05231_b200.layout import batch_range
        from workload import make_workload
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        w = make_workload("tiny")
        ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
        feats = w.features.numpy()
        nb = oracle.num_batches(len(sd), B)
        lo, hi = batch_range(nb, rank, world)
        my_seeds = w.seeds[lo * B:min(hi * B, len(sd))]
        ctx = dg.Ctx(device=dev)
        fdev = w.features.to(dev)
        L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), fdev, my_seeds.to(dev), FAN, B,
                              GPU_ROWS, HOST_ROWS, RNG_SEED, group_size=GROUP, batch_id_base=lo)
        ref = oracle.sample(ip, ix, sd, B, FAN, RNG_SEED)
        counts = oracle.count_frequencies(ref, len(ip) - 1)
        tier_map, _, _ = oracle.select_tiers(counts, GPU_ROWS, HOST_ROWS)
        assert np.array_equal(L.counts.cpu().numpy().view(np.uint32), counts), "counts differ"
        assert np.array_equal(L.plan.tier_map.cpu().numpy().view(np.uint32), tier_map), "tier map differs"
        mine = ref[lo:hi]
        plists = [oracle.classify(s.nodes, tier_map)[1] for s in mine]
        arena = L.arena.tensor.numpy()
        for gi, g in enumerate(L.groups):
            want = oracle.pack(feats, plists[g.b_lo:g.b_hi])
            assert np.array_equal(arena[g.arena_off:g.arena_off + g.group_bytes], want[0]), f"group {gi}"

        def check(it, how):
            n = 0
            for b, out in it:
                got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
                assert np.array_equal(got, oracle.assemble(feats, mine[b].nodes)), f"{how}: rank {rank} batch {b}"
                n += 1
            assert n == hi - lo, how

        check(L.assemble_epoch(), "replicated")
        tier = shard.ShardedTier(ctx, fdev, L.plan, rank, world)
        a2a = shard.nccl_all_to_all()

        def remote(c, addr, out):
            shard.fetch_remote_rows(c, tier, addr, out, a2a)
        # the exchange is collective per run: every rank assembles its block as one run here
        assert len(L.assembly_groups()) == 1
        check(L.assemble_epoch(sharded_tier=tier, remote=remote), "nccl all-to-all")
        peer = shard.PeerTier(ctx, fdev, L.plan, rank, world, shard.all_gather_handles)
        dist.barrier()
        check(L.assemble_epoch(host_window=3, peer_tier=peer), "peer (NVLink, one-sided)")
        ctx.sync()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


def test_nccl_ranks_split_one_epoch_and_equal_the_oracle():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU over NCCL)")
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res
