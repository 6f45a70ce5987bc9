"""World-size-2 checks of the sharded path's host logic on CPU (gloo backend).

The product path shards mini-batches across ranks (rank r samples epoch r, i.e.
batch ids r*nb .. (r+1)*nb-1, reading c9) and exchanges exactly one thing: the
access counts, all-reduced between a3 and a5 so that every rank derives the same
cache plan.  Here each rank plays its part with the oracle and gloo; the plan every
rank derives must equal the single-process oracle over both epochs (G-invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workload import make_workload

RNG_SEED = 0x5EEDD15C


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import oracle
    from paper_2405_05231_b200.layout import batch_range, _dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = make_workload("tiny", features=False)
        ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
        nb = oracle.num_batches(len(sd), 256)
        # this rank's epoch
        S = oracle.sample(ip, ix, sd, 256, [10, 5], RNG_SEED, batch_id_base=rank * nb)
        counts = torch.from_numpy(oracle.count_frequencies(S, w.num_nodes).astype(np.int64))
        assert _dist() is dist  # the layout driver sees the process group and all-reduces
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
        tm, g, h = oracle.select_tiers(counts.numpy().astype(np.uint32), 500, 1000)
        # contiguous batch blocks partition [0, n) (the within-epoch sharding helper)
        spans = [batch_range(nb * world, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == nb * world
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        q.put((rank, counts.numpy(), tm, g, h))
    finally:
        dist.destroy_process_group()


def _exchange_worker(rank, world, port, q):
    """The sharded-tier all-to-all choreography (shard.exchange_remote_rows) with numpy
    stand-ins for the CUDA request / gather kernels."""
    from paper_2405_05231_b200.shard import exchange_remote_rows, shard_of
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rb, k_gpu = 16, 101
        table = np.arange(k_gpu * rb, dtype=np.uint8).reshape(k_gpu, rb) ^ 0x5A  # GPU tier rows by slot
        my_shard = table[rank::world]                                              # slot s on rank s % world
        rng = np.random.default_rng(rank)
        want = rng.integers(0, k_gpu, 300)
        remote = [int(s) for s in want if shard_of(int(s), world)[0] != rank]
        by_owner = [[s for s in remote if s % world == o] for o in range(world)]
        send_counts = np.array([len(x) for x in by_owner], np.int64)
        req = torch.tensor([shard_of(s, world)[1] for o in range(world) for s in by_owner[o]], dtype=torch.int32)

        def serve(ids):
            return torch.from_numpy(my_shard[ids.numpy()].copy())

        def a2a(x, send_splits, recv_splits):
            out = torch.empty(sum(recv_splits), dtype=x.dtype)
            dist.all_to_all_single(out, x.contiguous(), output_split_sizes=list(recv_splits),
                                   input_split_sizes=list(send_splits))
            return out

        back = exchange_remote_rows(send_counts, req, serve, a2a, world, rb).numpy().reshape(-1, rb)
        expect = np.concatenate([table[by_owner[o]] for o in range(world)] or [np.zeros((0, rb), np.uint8)])
        q.put((rank, bool(np.array_equal(back, expect)), len(remote)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_tier_all_to_all_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res) and all(n > 0 for _, _, n in res)


def test_count_allreduce_gives_the_single_process_plan():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # single process: both epochs in one offline pass
    w = make_workload("tiny", features=False)
    sd = w.seeds.numpy()
    S = oracle.sample(w.indptr.numpy(), w.indices.numpy(), np.concatenate([sd, sd]), 256, [10, 5], RNG_SEED)
    counts = oracle.count_frequencies(S, w.num_nodes)
    tm, g, h = oracle.select_tiers(counts, 500, 1000)
    for _, c, tm_r, g_r, h_r in res:
        assert np.array_equal(c.astype(np.uint32), counts)
        assert np.array_equal(tm_r, tm) and np.array_equal(g_r, g) and np.array_equal(h_r, h)
