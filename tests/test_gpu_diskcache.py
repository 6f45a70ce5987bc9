"""Segmented disk cache (Sec. 5.1; readings d1-d8): GPU vs oracle through the C ABI.

Inputs are seeded packed lists (workload.make_packed_lists, or the oracle's own offline layout
of the tiny configuration); both sides consume the same arrays.  Everything compared here is
integer / index / byte work, so the bar is bit-exact: V_r of every segment, the reduced packed
lists, the merged page requests, the d8 addresses, Eq. 2 space and I/O totals, the heuristic's s,
the materialized cache pages and the partial inputs.
"""
import numpy as np
import pytest
import torch

import oracle
from workload import feature_rows_np, make_features, make_packed_lists, make_workload

pytestmark = pytest.mark.gpu
PAGE = 4096


@pytest.fixture(scope="module")
def dg():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_05231_b200 as dg
    return dg


@pytest.fixture(scope="module")
def ctx(dg):
    return dg.Ctx(device=0)


def _lists(ids, off):
    return [ids[off[b]:off[b + 1]] for b in range(len(off) - 1)]


def _index(dg, ctx, ids, off, N):
    dev = torch.device("cuda", 0)
    return dg.DiskIndex(ctx, torch.as_tensor(ids).to(dev), torch.as_tensor(off).to(dev), off, N)


def _compare(P, ref, R):
    assert P.nseg == len(ref.seg_off) - 1
    assert np.array_equal(P.seg_off.cpu().numpy(), ref.seg_off)
    assert np.array_equal(P.seg_page_off.cpu().numpy(), ref.seg_page_off)
    assert np.array_equal(P.cache_ids.cpu().numpy(), ref.cache_ids)
    assert np.array_equal(P.pk_off.cpu().numpy(), ref.pk_off)
    assert np.array_equal(P.pk_ids.cpu().numpy(), ref.pk_ids)
    assert np.array_equal(P.req_off.cpu().numpy(), ref.req_off)
    assert np.array_equal(P.req_pages.cpu().numpy().astype(np.int64), ref.req_pages)
    assert np.array_equal(P.dc_addr.cpu().numpy().view(np.uint32), ref.dc_addr[:R])
    assert (P.space_pages, P.io_pages, P.cache_pages, P.chunk_pages) == \
        (ref.space_pages, ref.io_pages, ref.cache_pages, ref.chunk_pages)
    assert np.array_equal(P.pk_off_host, ref.pk_off) and np.array_equal(P.req_off_host, ref.req_off)


CASES = [
    # nb, N, rows/batch, alpha, row_bytes, s, m, k, reorder
    (1, 50, 20, 2.0, 512, 1, 0, 4, True),
    (7, 300, 60, 3.0, 400, 3, 1, 2, True),
    (13, 2000, 300, 4.0, 512, 4, 1, 4, True),
    (13, 2000, 300, 4.0, 512, 4, 1, 4, False),
    (40, 5000, 700, 5.0, 1024, 40, 0, 8, True),
    (40, 5000, 700, 5.0, 1024, 41, 2, 1, True),
    (64, 20000, 3000, 6.0, 4096, 5, 1, 16, True),
    (9, 100, 0, 2.0, 512, 2, 1, 4, True),       # every packed list empty
    (2500, 30000, 40, 3.0, 512, 7, 1, 3, True),  # nb > 2048: global-memory counters
]


@pytest.mark.parametrize("case", CASES)
def test_plan_parity(dg, ctx, case):
    nb, N, rows, alpha, rb, s, m, k, reorder = case
    ids, off = make_packed_lists(nb, N, rows, alpha, seed=nb * 31 + s)
    seed = 0xD15C0000 + nb
    ref = oracle.disk_plan(_lists(ids, off), N, rb, s, m, k, seed, reorder)
    idx = _index(dg, ctx, ids, off, N)
    P = dg.dgnn_disk_plan_build(ctx, idx, rb, s, m, k, seed, reorder)
    _compare(P, ref, int(off[-1]))


@pytest.mark.parametrize("case", [c for c in CASES if c[8]][:6])
def test_plan_parity_literal_algorithm1(dg, ctx, case):
    """Algorithm 1 line 8 as printed (one scalar MinHash value, the minimum over the k functions,
    P:368): the kernels' plan equals the oracle's literal plan."""
    nb, N, rows, alpha, rb, s, m, k, _ = case
    ids, off = make_packed_lists(nb, N, rows, alpha, seed=nb * 31 + s)
    seed = 0xD15C0000 + nb
    ref = oracle.disk_plan(_lists(ids, off), N, rb, s, m, k, seed, True, literal=True)
    idx = _index(dg, ctx, ids, off, N)
    P = dg.dgnn_disk_plan_build(ctx, idx, rb, s, m, k, seed, True, literal=True)
    _compare(P, ref, int(off[-1]))


@pytest.mark.parametrize("m", [0, 1, 3])
def test_space_and_search(dg, ctx, m):
    ids, off = make_packed_lists(70, 4000, 400, 5.0, seed=5 + m)
    pl = _lists(ids, off)
    idx = _index(dg, ctx, ids, off, 4000)
    s_list = list(range(1, 71)) + [100]
    got = dg.dgnn_disk_space(ctx, idx, 512, s_list, m)
    assert got.tolist() == [oracle.disk_space(pl, 4000, 512, s, m) for s in s_list]
    for budget in (got.min() - 1, got.min(), int(np.median(got)), got.max(), got[0]):
        assert dg.dgnn_disk_search(ctx, idx, 512, int(budget), m) == oracle.disk_search(pl, 4000, 512, int(budget), m)


def test_tiny_offline_layout(dg, ctx):
    """The oracle's own packed lists of the tiny configuration (every node reused by several batches)."""
    w = make_workload("tiny")
    lay = oracle.offline_layout(w.indptr.numpy(), w.indices.numpy(), w.features.numpy(), w.seeds.numpy(), 256,
                                [10, 5], 0x5EEDD15C, 500, 1000, 8)
    pl = lay["packed"]
    off = np.concatenate([[0], np.cumsum([len(p) for p in pl])]).astype(np.int64)
    ids = np.concatenate(pl).astype(np.int32)
    idx = _index(dg, ctx, ids, off, 10_000)
    for s, m in ((1, 1), (2, 1), (3, 1), (8, 1), (4, 0), (8, 5)):
        ref = oracle.disk_plan(pl, 10_000, 512, s, m, 4, 99)
        _compare(dg.dgnn_disk_plan_build(ctx, idx, 512, s, m, 4, 99), ref, len(ids))
    budget = oracle.disk_space(pl, 10_000, 512, 3, 1)
    assert dg.dgnn_disk_search(ctx, idx, 512, budget, 1) == oracle.disk_search(pl, 10_000, 512, budget, 1)


@pytest.mark.parametrize("dim", [128, 100, 1024])
def test_cache_fill_and_partial_input(dg, ctx, dim):
    """Cache pages == oracle pages; partial input (pages + reduced chunks) == the batches' DISK rows."""
    dev = torch.device("cuda", 0)
    N, nb = 3000, 11
    ids, off = make_packed_lists(nb, N, 250, 4.0, seed=dim)
    pl = _lists(ids, off)
    rb = dim * 4
    feats = make_features(N, dim, dev)
    ref = oracle.disk_plan(pl, N, rb, 3, 1, 4, 7)
    idx = _index(dg, ctx, ids, off, N)
    P = dg.dgnn_disk_plan_build(ctx, idx, rb, 3, 1, 4, 7)
    cache = torch.full((P.cache_pages * PAGE,), 0xAB, dtype=torch.uint8, device=dev)
    dg.dgnn_disk_cache_fill(ctx, P, feats, cache)
    fnp = feature_rows_np(np.arange(N), dim, 1)
    assert np.array_equal(cache.cpu().numpy(), oracle.disk_cache_fill(fnp, ref))
    # reduced chunks (c20 layout of P_b') packed by the existing a7 kernel
    ch_off = dg.dgnn_chunk_layout(P.pk_off_host, rb)
    chunks = torch.zeros(max(int(ch_off[-1]), 16), dtype=torch.uint8, device=dev)
    dg.dgnn_pack(ctx, feats, P.pk_ids, P.pk_off, torch.as_tensor(ch_off).to(dev), P.n_packed, int(ch_off[-1]), chunks)
    out_off = dg.dgnn_chunk_layout(off, rb)
    for (b_lo, b_hi) in ((0, nb), (2, 7), (10, 11)):
        q0, q1 = P.req_off_host[b_lo], P.req_off_host[b_hi]
        pages = cache.view(-1, PAGE)[P.req_pages[q0:q1].long()].reshape(-1).contiguous()
        c_off = torch.as_tensor(ch_off[b_lo:b_hi + 1] - ch_off[b_lo]).to(dev)
        o_off = torch.as_tensor(out_off[b_lo:b_hi + 1] - out_off[b_lo]).to(dev)
        out = torch.zeros(int(out_off[b_hi] - out_off[b_lo]), dtype=torch.uint8, device=dev)
        dg.dgnn_disk_partial(ctx, P, b_lo, b_hi, pages if pages.numel() else None,
                             chunks[int(ch_off[b_lo]):], c_off, out, o_off)
        o = out.cpu().numpy()
        for b in range(b_lo, b_hi):
            base = out_off[b] - out_off[b_lo]
            n = off[b + 1] - off[b]
            got = o[base:base + n * rb].reshape(n, rb)
            assert np.array_equal(got, oracle.gather_rows(fnp, pl[b])), f"batch {b}"


def test_papers_scale_plan(dg, ctx):
    """Full papers-shaped epoch (1172 batches, ~41 M packed rows over 111 M nodes): the whole
    plan equals the oracle's at the heuristic's s and at s = 50 (the paper's Fig. 5 segment)."""
    N, nb = 111_059_956, 1172
    ids, off = make_packed_lists(nb, N, 35_000, 2.0, seed=1172)
    pl = _lists(ids, off)
    idx = _index(dg, ctx, ids, off, N)
    row_bytes = 512
    budget = oracle.disk_space(pl, N, row_bytes, 20, 1)  # keeps the oracle's linear search short
    s_h, pages = dg.dgnn_disk_search(ctx, idx, row_bytes, budget, 1)
    assert (s_h, pages) == oracle.disk_search(pl, N, row_bytes, budget, 1)
    assert 1 <= s_h <= 20
    for s in sorted({max(s_h, 1), 50}):
        ref = oracle.disk_plan(pl, N, row_bytes, s, 1, 4, 2024)
        _compare(dg.dgnn_disk_plan_build(ctx, idx, row_bytes, s, 1, 4, 2024), ref, len(ids))


# ------------------------------------------ the four-level store end to end ----
RNG_SEED = 0x5EEDD15C


@pytest.mark.parametrize("stage,frac,window", [("pinned", 0.8, 64), ("hbm", 0.6, 1), ("pinned", 1.0, 128),
                                               ("file", 0.7, 4)])
def test_layout_with_disk_cache_tiny(dg, ctx, stage, frac, window):
    """offline_layout with a disk budget: the heuristic's s, the segment caches, the reduced
    chunks and every assembled batch equal the oracle's (assembly == direct gather)."""
    w = make_workload("tiny")
    feats = w.features.numpy()
    ref = oracle.offline_layout(w.indptr.numpy(), w.indices.numpy(), feats, w.seeds.numpy(), 256, [10, 5],
                                RNG_SEED, 500, 1000, 8)
    pl = ref["packed"]
    rb = w.row_bytes
    packed_only = sum((len(p) * rb + 4095) // 4096 for p in pl)
    s_ref, _ = oracle.disk_search(pl, 10_000, rb, int(frac * packed_only), 1)
    assert s_ref >= 1
    dplan = oracle.disk_plan(pl, 10_000, rb, s_ref, 1, 4, RNG_SEED)
    dev = torch.device("cuda", 0)
    import os
    import tempfile
    path = os.path.join(tempfile.mkdtemp(prefix="dgnn_dc_"), "disk.bin") if stage == "file" else None
    L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), w.features.to(dev), w.seeds.to(dev), [10, 5],
                          256, 500, 1000, RNG_SEED, group_size=8, stage=stage, disk_budget_frac=frac, file_path=path)
    ctx.sync()
    assert L.disk_plan.s == s_ref
    assert L.stats["disk_cache"]["space_pages"] == dplan.space_pages
    if stage == "file":
        arena = np.fromfile(path, dtype=np.uint8)
    else:
        arena = L.arena.tensor.numpy() if L.arena is not None else L.arena_dev.cpu().numpy()
    cache = arena[L.cache_off:L.cache_off + dplan.cache_pages * PAGE]
    assert np.array_equal(cache, oracle.disk_cache_fill(feats, dplan))
    # reduced chunks: the oracle's pack of P_b'
    red = [dplan.pk_ids[dplan.pk_off[b]:dplan.pk_off[b + 1]] for b in range(len(pl))]
    for g in L.groups:
        buf, off = oracle.pack(feats, red[g.b_lo:g.b_hi])
        assert np.array_equal(arena[g.arena_off:g.arena_off + g.group_bytes], buf)
    # the assembly on its own ctx / stream, as bench.py runs it (the partial input must be built
    # on the assembling stream, ordered with its staged chunks)
    actx = dg.Ctx(device=0, stream=torch.cuda.Stream(dev))
    seen = 0
    for b, out in L.assemble_epoch(ctx=actx, host_window=window, out_budget=256 * 7 * 512):
        with torch.cuda.stream(actx.stream):
            got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(feats, ref["samples"][b].nodes)), f"batch {b}"
        seen += 1
    assert seen == len(pl)
    for b in ((0, len(pl) - 1) if stage != "file" else ()):  # single-batch path (memory-resident tiers)
        n = len(ref["samples"][b].nodes)
        out = torch.empty((n, w.features.shape[1]), dtype=w.features.dtype, device=dev)
        L.assemble(b, out)
        ctx.sync()
        got = out.view(torch.uint8).reshape(n, -1).cpu().numpy()
        assert np.array_equal(got, oracle.assemble(feats, ref["samples"][b].nodes))


def test_layout_with_disk_cache_products(dg, ctx):
    """products-shaped epoch (193 batches, 400-byte rows: pages with a 96-byte tail) at 80 % of
    the packed-only space: the plan's Eq. 2 space fits, the I/O beats identity order, and sampled
    batches assemble to the direct gather."""
    w = make_workload("products", device="cuda")
    dev = torch.device("cuda", 0)
    from workload import config_rows, CONFIGS
    cfg = CONFIGS["products"]
    gr, hr = config_rows(cfg)
    L = dg.offline_layout(ctx, w.indptr, w.indices, w.features, w.seeds, cfg["fanout"], cfg["batch_size"], gr, hr,
                          RNG_SEED, group_size=cfg["group_size"], disk_budget_frac=0.8)
    ctx.sync()
    dc = L.stats["disk_cache"]
    assert dc["space_pages"] <= dc["budget_pages"] and L.disk_plan.s > 1
    nodes = L.samples.nodes.cpu().numpy()
    check = {0, 1, 96, L.num_batches - 1}
    for b, out in L.assemble_epoch():
        if b in check:
            n0, n1 = L.samples.node_off_host[b], L.samples.node_off_host[b + 1]
            ids = nodes[n0:n1]
            exp = feature_rows_np(ids, cfg["dim"], 1).view(np.uint8).reshape(len(ids), -1)
            got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
            assert np.array_equal(got, exp), f"batch {b}"
