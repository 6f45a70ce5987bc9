"""Trainer stub (reading t1; surrogate of Eq. 1) and the training
pipeline (queues of depth 2): GPU vs oracle, bit-exact fp32.

The oracle side samples, tiers, classifies and assembles with oracle/ only, then runs
oracle.train_stub on each batch's direct-gather rows; the GPU side runs the whole path through
the C ABI and the trainer on its own stream.
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import random_csr
from workload import make_workload, feature_rows_np

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


@pytest.mark.parametrize("trial", range(8))
def test_train_stub_random(dg, ctx, trial):
    """Standalone: random graphs, 1-3 hops incl. fanout 0 and > 32, dims 4 to 260 (float4 and
    scalar paths), several batches per call."""
    rng = np.random.default_rng(700 + trial)
    n = int(rng.integers(50, 400))
    indptr, indices = random_csr(rng, n, int(rng.integers(1, 50)))
    H = int(rng.integers(1, 4))
    fan = [int(rng.choice([0, 1, 3, 10, 40])) for _ in range(H)]
    dim = int(rng.choice([4, 12, 100, 128, 7, 260]))
    seeds = rng.permutation(n)[: int(rng.integers(1, 60))].astype(np.int32)
    B = int(rng.integers(1, 20))
    ref = oracle.sample(indptr, indices, seeds, B, fan, trial)
    feats = (rng.random((n, dim)) * 4 - 2).astype(np.float32)
    dev = torch.device("cuda", 0)
    S = dg.dgnn_sample(ctx, torch.as_tensor(indptr).to(dev), torch.as_tensor(indices).to(dev),
                       torch.as_tensor(seeds).to(dev), B, fan, trial, 0, None)
    nodes = S.nodes.cpu().numpy()
    x = torch.as_tensor(feats[nodes.astype(np.int64)]).to(dev).contiguous()  # direct gather (input)
    b_mid = S.num_batches // 2
    dg.dgnn_train_stub(ctx, S, 0, b_mid, x[:S.node_off_host[b_mid]])
    dg.dgnn_train_stub(ctx, S, b_mid, S.num_batches, x[S.node_off_host[b_mid]:])
    xs = x.cpu().numpy()
    for b, s in enumerate(ref):
        n0 = S.node_off_host[b]
        exp = oracle.train_stub(s, feats[s.nodes.astype(np.int64)])
        got = xs[n0:n0 + len(exp)]
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), f"batch {b}"


@pytest.mark.parametrize("window,separate", [(64, True), (1, False)])
def test_train_epoch_tiny(dg, ctx, window, separate):
    w = make_workload("tiny")
    feats = w.features.numpy()
    ref = oracle.sample(w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy(), 256, [10, 5], RNG_SEED)
    dev = torch.device("cuda", 0)
    L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), w.features.to(dev), w.seeds.to(dev), [10, 5],
                          256, 500, 1000, RNG_SEED, group_size=8)
    tctx = dg.Ctx(device=0, stream=torch.cuda.Stream(dev)) if separate else None
    got = {}
    for b0, b1, x in L.train_epoch(train_ctx=tctx, host_window=window, out_budget=256 * 7 * 512):
        s = tctx.stream if tctx is not None else ctx.stream
        with torch.cuda.stream(s):
            for b in range(b0, b1):
                r0 = int(L.samples.node_off_host[b] - L.samples.node_off_host[b0])
                got[b] = x[r0:r0 + int(L.samples.hop_off_host[b][1])].clone()
    torch.cuda.synchronize()
    assert len(got) == len(ref)
    for b, s in enumerate(ref):
        exp = oracle.train_stub(s, oracle.assemble(feats, s.nodes).view(np.float32))
        assert np.array_equal(got[b].cpu().numpy().view(np.uint32), exp.view(np.uint32)), f"batch {b}"


def test_train_epoch_products_sampled(dg, ctx):
    from workload import CONFIGS, config_rows
    w = make_workload("products", device="cuda")
    cfg = CONFIGS["products"]
    gr, hr = config_rows(cfg)
    L = dg.offline_layout(ctx, w.indptr, w.indices, w.features, w.seeds, cfg["fanout"], cfg["batch_size"], gr, hr,
                          RNG_SEED, group_size=cfg["group_size"])
    check = [0, 57, L.num_batches - 1]
    ref = oracle.sample(w.indptr.cpu().numpy(), w.indices.cpu().numpy(), w.seeds.cpu().numpy(), cfg["batch_size"],
                        cfg["fanout"], RNG_SEED, batches=check)
    tctx = dg.Ctx(device=0, stream=torch.cuda.Stream(torch.device("cuda", 0)))
    got = {}
    for b0, b1, x in L.train_epoch(train_ctx=tctx):
        with torch.cuda.stream(tctx.stream):
            for b in check:
                if b0 <= b < b1:
                    r0 = int(L.samples.node_off_host[b] - L.samples.node_off_host[b0])
                    got[b] = x[r0:r0 + int(L.samples.hop_off_host[b][1])].clone()
    torch.cuda.synchronize()
    for b, s in zip(check, ref):
        rows = feature_rows_np(s.nodes, cfg["dim"], 1)
        exp = oracle.train_stub(s, rows)
        assert np.array_equal(got[b].cpu().numpy().view(np.uint32), exp.view(np.uint32)), f"batch {b}"
