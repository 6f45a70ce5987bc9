"""The window-ordered host tier against the oracle (run on a B200 with -m gpu).

offline_layout(host_order=W) lays the host tier out physically in (window mask, slot) order so that
the assembler's host-row windows of W batches are a few contiguous ranges (copy-engine copies).
Slots, tier map and addresses stay the oracle's; checked here: the masks equal a numpy
recomputation from the oracle's address tables, the physical order is the (reversed mask, slot) sort, the
physical tier rows are the oracle's host-tier rows permuted, every window's ranges cover exactly
its slots, and every batch assembled through every reader -- the ordered windows, other window
sizes (slot list remapped), per-batch UVA reads and Layout.assemble -- equals the direct gather.
"""
import numpy as np
import pytest
import torch

import oracle
from workload import make_workload

pytestmark = pytest.mark.gpu
RNG_SEED = 0x5EEDD15C
FAN, B, GPU_ROWS, HOST_ROWS = [10, 5], 256, 500, 1000


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_05231_b200 as dg
    return dg


@pytest.fixture(scope="module")
def tiny():
    return make_workload("tiny")


@pytest.fixture(scope="module")
def ref(tiny):
    return oracle.offline_layout(tiny.indptr.numpy(), tiny.indices.numpy(), tiny.features.numpy(),
                                 tiny.seeds.numpy(), B, FAN, RNG_SEED, GPU_ROWS, HOST_ROWS, 8)


@pytest.mark.parametrize("W,budget,group", [(2, 1 << 30, 8), (3, 1 << 30, 3), (1, 1 << 30, 8), (4, 600_000, 2)])
def test_window_ordered_host_tier(dg, tiny, ref, W, budget, group):
    ctx = dg.Ctx(device=0)
    dev = torch.device("cuda", 0)
    gctx = dg.Ctx(device=0, stream=torch.cuda.Stream())
    L = dg.offline_layout(ctx, tiny.indptr.to(dev), tiny.indices.to(dev), tiny.features.to(dev), tiny.seeds.to(dev),
                          FAN, B, GPU_ROWS, HOST_ROWS, RNG_SEED, group_size=group, host_order=W)
    ctx.sync()
    feats = tiny.features.numpy()
    kh = L.plan.k_host
    if W == 1:
        assert L.host_order is None  # one batch per window: nothing to order
        return
    ho = L.host_order
    assert ho is not None and L.host_order_key == (W, 1 << 30)
    # masks from the oracle's address tables and the windows of the default assembly plan
    groups, wins = L.host_windows(W)
    want = np.zeros(kh, np.uint32)
    for w, (r0, r1) in enumerate(wins):
        for b in range(groups[r0][0], groups[r1 - 1][1]):
            a = ref["addr"][b]
            host = a[(a >> 30) == 1] & ((1 << 30) - 1)
            want[host] |= np.uint32(1 << w)
    mask = ho.slot_mask[:kh].cpu().numpy().view(np.uint32)
    assert np.array_equal(mask, want)
    rev = np.zeros(kh, np.uint32)  # the sort key: the mask's window bits reversed (window 0 most significant)
    for w in range(ho.nwin):
        rev |= ((want >> w) & 1) << (ho.nwin - 1 - w)
    order = np.lexsort((np.arange(kh), rev))  # by reversed mask, then slot
    phys_of_slot = ho.phys_of_slot[:kh].cpu().numpy()
    assert np.array_equal(phys_of_slot[order], np.arange(kh))
    host_rows = L.host_tier.tensor.numpy().reshape(kh, -1)
    assert np.array_equal(host_rows[phys_of_slot], ref["host_buf"])
    assert len(ho.ranges[0]) == 3  # window 0's rows: one contiguous range (the most significant key bit)
    for w in range(ho.nwin):
        rg = ho.ranges[w].reshape(-1, 3)
        covered = np.concatenate([np.arange(lo, hi) for lo, hi, _ in rg]) if len(rg) else np.zeros(0, np.int64)
        assert np.array_equal(np.sort(covered), np.sort(phys_of_slot[(want >> w) & 1 == 1]))
        assert ho.rows[w] == len(covered)
    nodes = ref["samples"]
    for hw in (W, W + 3, 1):
        n = 0
        for b, out in L.assemble_epoch(host_window=hw, gather_ctx=gctx, out_budget=budget):
            got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
            assert np.array_equal(got, oracle.assemble(feats, nodes[b].nodes)), f"window {hw} batch {b}"
            n += 1
        assert n == len(nodes)
    for b in (0, len(nodes) - 1):
        n_b = len(nodes[b].nodes)
        with torch.cuda.stream(ctx.stream):
            out = torch.empty((n_b, 128), dtype=torch.float32, device=dev)
        L.assemble(b, out)
        ctx.sync()
        assert np.array_equal(out.view(torch.uint8).reshape(n_b, -1).cpu().numpy(), oracle.assemble(feats, nodes[b].nodes))
    ctx.sync()
    gctx.sync()


@pytest.mark.parametrize("W,budget,group,early", [(2, 1 << 30, 8, False), (3, 600_000, 3, True)])
def test_host_tier_read_from_the_table(dg, tiny, ref, W, budget, group, early):
    """host_from_table (the feature table in pinned host memory, bench.py's e2e mode): no host-tier
    copy is built; the windows' scheduled rows are gathered from the table (dgnn_gather_ranges) into
    the same staging positions, so every assembled batch still equals the direct gather -- also with
    window 0 staged ahead through early_host_prefetch."""
    from paper_2405_05231_b200.layout import Workspace
    ctx = dg.Ctx(device=0)
    dev = torch.device("cuda", 0)
    gctx = dg.Ctx(device=0, stream=torch.cuda.Stream())
    hb = dg.HostBuffer(tiny.features.numel() * tiny.features.element_size())
    f_host = hb.tensor.view(tiny.features.dtype).view(tiny.features.shape)
    f_host.copy_(tiny.features)
    L = dg.offline_layout(ctx, tiny.indptr.to(dev), tiny.indices.to(dev), f_host, tiny.seeds.to(dev), FAN, B,
                          GPU_ROWS, HOST_ROWS, RNG_SEED, group_size=group, host_order=W, asm_out_budget=budget,
                          host_from_table=True)
    ctx.sync()
    assert L.host_tier is None and L.host_table is not None and L.host_order is not None
    feats = tiny.features.numpy()
    nodes = ref["samples"]
    ws = Workspace()
    ev = L.early_host_prefetch(gctx, ws, W, budget, "_t") if early else None
    assert (ev is not None) == early
    n = 0
    for b, out in L.assemble_epoch(host_window=W, gather_ctx=gctx, out_budget=budget, ws=ws, arena_tag="_t",
                                   early=ev):
        got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(feats, nodes[b].nodes)), f"batch {b}"
        n += 1
    assert n == len(nodes)
    with pytest.raises(ValueError):  # no host-tier copy: other windows cannot read it
        for _ in L.assemble_epoch(host_window=W + 3, gather_ctx=gctx, out_budget=budget):
            pass
    ctx.sync()
    gctx.sync()
    del hb


@pytest.mark.slow
def test_host_tier_read_from_the_table_products_scale(dg):
    """The e2e leg's layout at products scale (192 batches, 2.4 M nodes, 400-byte rows, two windows
    of 128 batches, 64 MB stage pieces, window 0 staged early): the table in pinned host memory,
    the host tier read from it; every assembled batch equals the source rows of its nodes (the
    generator's closed form on the GPU)."""
    from paper_2405_05231_b200.layout import Workspace
    from workload import CONFIGS, config_rows, feature_rows, make_features, make_graph, make_seeds
    dev = torch.device("cuda", 0)
    cfg = dict(CONFIGS["products"])
    indptr, indices = make_graph(cfg["num_nodes"], cfg["num_edges"], cfg["degree"], cfg["skew"], 0, dev)
    seeds = make_seeds(cfg["num_nodes"], cfg["num_seeds"], 0, dev)
    feats = make_features(cfg["num_nodes"], cfg["dim"], dev, fseed=1)
    hb = dg.HostBuffer(feats.numel() * 4)
    f_host = hb.tensor.view(torch.float32).view(feats.shape)
    f_host.copy_(feats.cpu())
    del feats
    gpu_rows, host_rows = config_rows(cfg)
    ctx = dg.Ctx(device=0)
    gctx = dg.Ctx(device=0, stream=torch.cuda.Stream())
    budget = 256 << 20
    L = dg.offline_layout(ctx, indptr, indices, f_host, seeds, cfg["fanout"], cfg["batch_size"], gpu_rows, host_rows,
                          RNG_SEED, group_size=0, host_order=128, asm_out_budget=budget, host_from_table=True,
                          stage_piece=64 << 20)
    assert L.host_tier is None and L.host_order is not None and L.host_order.nwin == 2
    ws = Workspace()
    ev = L.early_host_prefetch(gctx, ws, 128, budget, "_p")
    assert ev is not None
    S = L.samples
    n, bad = 0, []
    for b, out in L.assemble_epoch(host_window=128, gather_ctx=gctx, out_budget=budget, ws=ws, arena_tag="_p",
                                   early=ev):
        n0, n1 = int(S.node_off_host[b]), int(S.node_off_host[b + 1])
        exp = feature_rows(S.nodes[n0:n1].to(torch.int64), cfg["dim"], 1)
        if not torch.equal(out.reshape(-1).view(torch.int32), exp.reshape(-1).view(torch.int32)):
            bad.append(b)
        n += 1
    ctx.sync()
    gctx.sync()
    assert n == S.num_batches and bad == []
    del hb
