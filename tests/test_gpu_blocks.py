"""DGL-block sampling variant (reading c27): GPU vs oracle, bit-exact.

Samples (nodes, hop_off, the per-hop eptr arrays, src_local), access counts, the trainer stub
over blocks, and the offline layout + assembly of block samples.
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import random_csr
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
    c = dg.Ctx(device=0)
    c.set_sample_mode(True)
    return c


def _gpu(dg, ctx, indptr, indices, seeds, B, fan, seed, group=0, base=0):
    dev = torch.device("cuda", 0)
    counts = torch.zeros(len(indptr) - 1, dtype=torch.int32, device=dev)
    ctx.set_sample_group(group)
    S = dg.dgnn_sample(ctx, torch.as_tensor(np.asarray(indptr, np.int64)).to(dev),
                       torch.as_tensor(np.asarray(indices, np.int32)).to(dev),
                       torch.as_tensor(np.asarray(seeds, np.int32)).to(dev), B, fan, seed, base, counts)
    ctx.set_sample_group(0)
    return S, counts


def _compare(S, ref):
    assert S.blocks and S.num_batches == len(ref)
    nodes, eptr, src = S.nodes.cpu().numpy(), S.eptr.cpu().numpy(), S.src_local.cpu().numpy()
    for b, r in enumerate(ref):
        assert np.array_equal(nodes[S.node_off_host[b]:S.node_off_host[b + 1]], r.nodes), f"batch {b} nodes"
        assert np.array_equal(S.hop_off_host[b], r.hop_off), f"batch {b} hop_off"
        assert np.array_equal(eptr[S.eptr_off_host[b]:S.eptr_off_host[b + 1]], r.eptr), f"batch {b} eptr"
        assert np.array_equal(src[S.edge_off_host[b]:S.edge_off_host[b + 1]], r.src_local), f"batch {b} src"


@pytest.mark.parametrize("trial", range(10))
def test_block_sampling_random(dg, ctx, trial):
    rng = np.random.default_rng(1200 + trial)
    n = int(rng.integers(30, 600))
    indptr, indices = random_csr(rng, n, int(rng.integers(1, 45)))
    fan = [int(rng.choice([0, 1, 2, 5, 10, 33])) for _ in range(int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[: int(rng.integers(1, min(n, 200)))].astype(np.int32)
    B = int(rng.integers(1, 40))
    ref = oracle.sample(indptr, indices, seeds, B, fan, trial * 7 + 1, batch_id_base=trial * 1000, blocks=True)
    for group in (0, 3):
        S, counts = _gpu(dg, ctx, indptr, indices, seeds, B, fan, trial * 7 + 1, group, trial * 1000)
        _compare(S, ref)
        assert np.array_equal(counts.cpu().numpy().view(np.uint32), oracle.count_frequencies(ref, n))


def test_block_sampling_tiny_and_trainer(dg, ctx):
    w = make_workload("tiny")
    ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
    ref = oracle.sample(ip, ix, sd, 256, [10, 5], RNG_SEED, blocks=True)
    S, _ = _gpu(dg, ctx, ip, ix, sd, 256, [10, 5], RNG_SEED)
    _compare(S, ref)
    feats = w.features.numpy()
    x = torch.as_tensor(feats[S.nodes.cpu().numpy().astype(np.int64)]).cuda().contiguous()
    dg.dgnn_train_stub(ctx, S, 0, S.num_batches, x)
    xs = x.cpu().numpy()
    for b, s in enumerate(ref):
        exp = oracle.train_stub(s, feats[s.nodes.astype(np.int64)])
        n0 = S.node_off_host[b]
        assert np.array_equal(xs[n0:n0 + len(exp)].view(np.uint32), exp.view(np.uint32)), f"batch {b}"


@pytest.mark.parametrize("trial", range(4))
def test_block_trainer_random(dg, ctx, trial):
    rng = np.random.default_rng(1300 + trial)
    n = int(rng.integers(40, 300))
    indptr, indices = random_csr(rng, n, 20)
    fan = [int(rng.choice([0, 3, 8, 40])) for _ in range(int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[:50].astype(np.int32)
    dim = int(rng.choice([4, 100, 128, 7]))
    ref = oracle.sample(indptr, indices, seeds, 6, fan, trial, blocks=True)
    S, _ = _gpu(dg, ctx, indptr, indices, seeds, 6, fan, trial)
    feats = (rng.random((n, dim)) * 2 - 1).astype(np.float32)
    x = torch.as_tensor(feats[S.nodes.cpu().numpy().astype(np.int64)]).cuda().contiguous()
    dg.dgnn_train_stub(ctx, S, 0, S.num_batches, x)
    xs = x.cpu().numpy()
    for b, s in enumerate(ref):
        exp = oracle.train_stub(s, feats[s.nodes.astype(np.int64)])
        n0 = S.node_off_host[b]
        assert np.array_equal(xs[n0:n0 + len(exp)].view(np.uint32), exp.view(np.uint32)), f"batch {b}"


def test_block_layout_and_assembly(dg, ctx):
    """The offline layout only reads the samples' node lists, so block samples flow through a4-a9
    unchanged: counts, tiers and every assembled batch equal the oracle's."""
    w = make_workload("tiny")
    feats = w.features.numpy()
    ref = oracle.sample(w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy(), 256, [10, 5], RNG_SEED, blocks=True)
    counts = oracle.count_frequencies(ref, 10_000)
    tm, _, _ = oracle.select_tiers(counts, 500, 1000)
    dev = torch.device("cuda", 0)
    L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), w.features.to(dev), w.seeds.to(dev), [10, 5],
                          256, 500, 1000, RNG_SEED, group_size=8)
    ctx.sync()
    assert np.array_equal(L.counts.cpu().numpy().view(np.uint32), counts)
    assert np.array_equal(L.plan.tier_map.cpu().numpy().view(np.uint32), tm)
    for b, out in L.assemble_epoch(host_window=4):
        got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(feats, ref[b].nodes)), f"batch {b}"
