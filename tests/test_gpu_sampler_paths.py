"""Both a3 dedup paths of dgnn_sample against the oracle (run on a B200 with -m gpu).

The sampler has two implementations of "new = distinct(cand) minus nodes-so-far, ordered by ID,
edges remapped" (readings c10/c11): the default partitioned path (candidates bucketed by
(batch, ID range), deduplicated in shared memory) and the per-batch global hash-set path, which
also serves as its fallback when a bucket overflows.  DGNN_SAMPLE_DEDUP=table selects the second.
The partitioned path orders a bucket's new IDs by counting (sub-range counts, rank within the
sub-range) up to 2048 of them and by a bitonic sort above; DGNN_SAMPLE_ORDER=sort sorts every
bucket, so both orderings are compared.
Every case is compared byte for byte with the oracle, including inputs built so that one ID range
holds more distinct IDs than a shared-memory bucket (the fallback must give the same bytes).
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import csr_from_adj, random_csr, random_csr_fast
from workload import make_workload

pytestmark = pytest.mark.gpu

RNG_SEED = 0x5EEDD15C


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_05231_b200 as dg
    return dg


@pytest.fixture(scope="module")
def ctx(dg):
    return dg.Ctx(device=0)


@pytest.fixture(params=["part", "part-sort", "table"])
def path(request, monkeypatch):
    monkeypatch.delenv("DGNN_SAMPLE_ORDER", raising=False)
    if request.param == "table":
        monkeypatch.setenv("DGNN_SAMPLE_DEDUP", "table")
    else:
        monkeypatch.delenv("DGNN_SAMPLE_DEDUP", raising=False)
    if request.param == "part-sort":  # every bucket's new IDs ordered by the bitonic sort
        monkeypatch.setenv("DGNN_SAMPLE_ORDER", "sort")
    return request.param


def _run(dg, ctx, indptr, indices, seeds, B, fan, seed, base=0, group=0, blocks=False):
    dev = torch.device("cuda", 0)
    ip = torch.as_tensor(np.asarray(indptr, np.int64)).to(dev)
    ix = torch.as_tensor(np.asarray(indices, np.int32)).to(dev)
    sd = torch.as_tensor(np.asarray(seeds, np.int32)).to(dev)
    counts = torch.zeros(len(indptr) - 1, dtype=torch.int32, device=dev)
    ctx.set_sample_group(group)
    ctx.set_sample_mode(blocks)
    try:
        S = dg.dgnn_sample(ctx, ip, ix, sd, B, fan, seed, base, counts)
    finally:
        ctx.set_sample_group(0)
        ctx.set_sample_mode(False)
    return S, counts


def _check(S, counts, ref, n):
    assert S.num_batches == len(ref)
    nodes, eptr, src = S.nodes.cpu().numpy(), S.eptr.cpu().numpy(), S.src_local.cpu().numpy()
    for b, r in enumerate(ref):
        assert np.array_equal(nodes[S.node_off_host[b]:S.node_off_host[b + 1]], r.nodes), f"batch {b}: nodes"
        assert np.array_equal(S.hop_off_host[b], r.hop_off), f"batch {b}: hop_off"
        assert np.array_equal(eptr[S.eptr_off_host[b]:S.eptr_off_host[b + 1]], r.eptr), f"batch {b}: eptr"
        assert np.array_equal(src[S.edge_off_host[b]:S.edge_off_host[b + 1]], r.src_local), f"batch {b}: src_local"
    assert np.array_equal(counts.cpu().numpy().view(np.uint32), oracle.count_frequencies(ref, n))


@pytest.mark.parametrize("trial", range(16))
def test_random_graphs_both_paths(dg, ctx, path, trial):
    rng = np.random.default_rng(7000 + trial)
    n = int(rng.integers(30, 20000))
    indptr, indices = random_csr_fast(rng, n, max_deg=int(rng.integers(1, 60)))
    H = int(rng.integers(1, 4))
    fan = [int(x) for x in rng.choice([0, 1, 2, 3, 5, 10, 15, 31, 32, 33, 40], size=H)]
    seeds = rng.permutation(n)[:int(rng.integers(1, n))].astype(np.int32)
    B = int(rng.integers(1, 1500))
    base = int(rng.integers(0, 1 << 40))
    seed = int(rng.integers(0, 1 << 63))
    blocks = bool(trial % 4 == 3)
    ref = oracle.sample(indptr, indices, seeds, B, fan, seed, batch_id_base=base, blocks=blocks)
    S, counts = _run(dg, ctx, indptr, indices, seeds, B, fan, seed, base, int(rng.choice([0, 1, 3, 7])), blocks)
    _check(S, counts, ref, n)


def test_tiny_both_paths(dg, ctx, path):
    w = make_workload("tiny")
    ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
    ref = oracle.sample(ip, ix, sd, 256, [10, 5], RNG_SEED)
    for group in (0, 3):
        S, counts = _run(dg, ctx, ip, ix, sd, 256, [10, 5], RNG_SEED, group=group)
        _check(S, counts, ref, 10_000)


def test_concentrated_ids_fall_back(dg, ctx, path):
    """A hub whose 6000 neighbours sit in the lowest IDs of a 2^20-node graph: at the partition count
    the node bound asks for, one (batch, ID range) bucket holds all 6000 distinct IDs, more than a
    shared-memory table takes, so the partitioned path must hand the group to the hash-set path."""
    n = 1 << 20
    hub = n - 1
    adj = {hub: list(range(6000)), 5: [hub, 7, 900_000], 900_000: list(range(100, 4100))}
    ip, ix = csr_from_adj(n, adj)
    seeds = np.array([hub, 5, 900_000, 17, 123_456], np.int32)
    for fan, B in (([6000, 3], 5), ([5000, 4000], 2), ([6000], 1)):
        ref = oracle.sample(ip, ix, seeds, B, fan, RNG_SEED)
        S, counts = _run(dg, ctx, ip, ix, seeds, B, fan, RNG_SEED)
        _check(S, counts, ref, n)


def test_large_batch_uses_table_path(dg, ctx, path):
    """batch_size above the partitioned path's seed-sort limit (4096) still samples bit-exactly."""
    rng = np.random.default_rng(99)
    n = 30000
    indptr, indices = random_csr_fast(rng, n, max_deg=12)
    seeds = rng.permutation(n)[:12000].astype(np.int32)
    ref = oracle.sample(indptr, indices, seeds, 5000, [4, 3], RNG_SEED)
    S, counts = _run(dg, ctx, indptr, indices, seeds, 5000, [4, 3], RNG_SEED)
    _check(S, counts, ref, n)


def test_duplicate_seed_rejected_on_both_paths(dg, ctx, path):
    ip, ix = csr_from_adj(40, {0: [1], 1: [2]})
    with pytest.raises(dg.DgnnError) as e:
        _run(dg, ctx, ip, ix, [3, 9, 3], 3, [1], 0)
    assert e.value.status == 1


@pytest.mark.parametrize("mode", ["range", "group"])
@pytest.mark.parametrize("trial", range(4))
def test_access_counter_modes(dg, ctx, monkeypatch, mode, trial):
    """a4: the range-major epoch counter (default: shared-memory counters per 2^14-ID
    range over every batch's ID-ascending hop slices, one RED per seed) and the per-group
    counter (DGNN_SAMPLE_COUNT=group) both equal the oracle's batch-membership counts; counts
    accumulate across calls (+=), including N not a multiple of the range size."""
    if mode == "group":
        monkeypatch.setenv("DGNN_SAMPLE_COUNT", "group")
    else:
        monkeypatch.delenv("DGNN_SAMPLE_COUNT", raising=False)
    rng = np.random.default_rng(9100 + trial)
    n = int(rng.integers(100, 70000))
    indptr, indices = random_csr_fast(rng, n, max_deg=int(rng.integers(1, 30)))
    fan = [int(x) for x in rng.choice([1, 2, 5, 10, 15], size=int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[:int(rng.integers(1, min(n, 5000)))].astype(np.int32)
    B = int(rng.integers(1, 700))
    ref = oracle.sample(indptr, indices, seeds, B, fan, 5, blocks=bool(trial % 2))
    want = oracle.count_frequencies(ref, n)
    dev = torch.device("cuda", 0)
    ip = torch.as_tensor(indptr).to(dev)
    ix = torch.as_tensor(indices).to(dev)
    sd = torch.as_tensor(seeds).to(dev)
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    ctx.set_sample_mode(bool(trial % 2))
    try:
        dg.dgnn_sample(ctx, ip, ix, sd, B, fan, 5, 0, counts)
        assert np.array_equal(counts.cpu().numpy().view(np.uint32), want)
        dg.dgnn_sample(ctx, ip, ix, sd, B, fan, 5, 0, counts)  # accumulates
        assert np.array_equal(counts.cpu().numpy().view(np.uint32), 2 * want)
    finally:
        ctx.set_sample_mode(False)
