"""World-size-2 parity of the product path on the box's one GPU (gloo stands in for NCCL).

Each rank runs offline_layout on its own epoch (batch ids rank*nb ..), the layout all-reduces
the access counts (a4) and derives the tier plan (a5) from all ranks' batches; every
rank's counts, tier map, packed chunks and assembled batches must equal the oracle run over the
union of both ranks' batches (outputs at G = 2 byte-identical to the single oracle).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

RNG_SEED = 0x5EEDD15C
FAN, B, GPU_ROWS, HOST_ROWS, GROUP = [10, 5], 256, 500, 1000, 8


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        import oracle
        import paper_2405_05231_b200 as dg
        from workload import make_workload
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        w = make_workload("tiny")
        ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
        feats = w.features.numpy()
        nb = oracle.num_batches(len(sd), B)
        ctx = dg.Ctx(device=dev)
        L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), w.features.to(dev), w.seeds.to(dev), FAN,
                              B, GPU_ROWS, HOST_ROWS, RNG_SEED, group_size=GROUP, batch_id_base=rank * nb)
        # the oracle over the union of both ranks' epochs
        samples = [oracle.sample(ip, ix, sd, B, FAN, RNG_SEED, batch_id_base=r * nb) for r in range(world)]
        counts = np.zeros(len(ip) - 1, np.uint32)
        for s in samples:
            oracle.count_frequencies(s, len(ip) - 1, counts)
        tier_map, _, _ = oracle.select_tiers(counts, GPU_ROWS, HOST_ROWS)
        assert np.array_equal(L.counts.cpu().numpy().view(np.uint32), counts), "counts differ"
        assert np.array_equal(L.plan.tier_map.cpu().numpy().view(np.uint32), tier_map), "tier map differs"
        mine = samples[rank]
        plists = [oracle.classify(s.nodes, tier_map)[1] for s in mine]
        arena = L.arena.tensor.numpy()
        for gi, g in enumerate(L.groups):
            ref = oracle.pack(feats, plists[gi * GROUP:(gi + 1) * GROUP])
            assert np.array_equal(arena[g.arena_off:g.arena_off + g.group_bytes], ref[0]), f"group {gi}"
        n = 0
        for b, out in L.assemble_epoch():
            got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
            assert np.array_equal(got, oracle.assemble(feats, mine[b].nodes)), f"rank {rank} batch {b}"
            n += 1
        assert n == nb
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_ranks_equal_the_union_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
