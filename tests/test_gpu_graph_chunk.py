"""The graph sample kept in the chunk and the graph-loader stage (reading c22b),
against the oracle (run on a B200 with -m gpu).

offline_layout(embed_graph=True) packs every batch's sample into its chunk and then frees the
samples' device arrays, so training can only get the graph back through the loader
(dgnn_samples_load over the staged chunks).  Checked: every packing group's bytes equal
oracle.pack_embedded; the loader's samples equal the oracle's; the trainer stub over the loaded
samples equals oracle.train_stub for every batch; for the pinned, HBM and O_DIRECT-file disk
tiers, runs of one and several batches, both sampling variants.
"""
import os
import tempfile

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
    out = {}
    for blocks in (False, True):
        s = oracle.sample(tiny.indptr.numpy(), tiny.indices.numpy(), tiny.seeds.numpy(), B, FAN, RNG_SEED,
                          blocks=blocks)
        counts = oracle.count_frequencies(s, 10_000)
        tm, _, _ = oracle.select_tiers(counts, GPU_ROWS, HOST_ROWS)
        out[blocks] = (s, [oracle.classify(x.nodes, tm)[1] for x in s])
    return out


def _layout(dg, ctx, tiny, stage, group, td):
    dev = torch.device("cuda", 0)
    return dg.offline_layout(ctx, tiny.indptr.to(dev), tiny.indices.to(dev), tiny.features.to(dev),
                             tiny.seeds.to(dev), FAN, B, GPU_ROWS, HOST_ROWS, RNG_SEED, group_size=group,
                             stage=stage, file_path=os.path.join(td, "disk.bin"), embed_graph=True)


@pytest.mark.parametrize("stage,group,blocks", [("pinned", 8, False), ("pinned", 3, True), ("hbm", 2, False),
                                                ("file", 3, False)])
def test_embedded_chunks_loader_and_trainer(dg, tiny, ref, stage, group, blocks):
    ctx = dg.Ctx(device=0)
    ctx.set_sample_mode(blocks)
    samples, plists = ref[blocks]
    feats = tiny.features.numpy()
    with tempfile.TemporaryDirectory() as td:
        L = _layout(dg, ctx, tiny, stage, group, td)
        ctx.sync()
        assert L.samples.nodes is None, "the samples' device arrays must be dropped"
        # packed bytes: every group equals the oracle's embedded pack of its batches
        if stage == "pinned":
            arena = L.arena.tensor.numpy()
        elif stage == "hbm":
            arena = L.arena_dev.cpu().numpy()
        else:
            with open(os.path.join(td, "disk.bin"), "rb") as f:
                arena = np.frombuffer(f.read(), np.uint8)
        for g in L.groups:
            buf, off, sec = oracle.pack_embedded(feats, plists[g.b_lo:g.b_hi], samples[g.b_lo:g.b_hi])
            assert np.array_equal(arena[g.arena_off:g.arena_off + g.group_bytes], buf), f"group {g.b_lo}"
            assert np.array_equal(g.sec_off, sec)
        # the loader over the whole arena on the device
        if stage != "file":
            dev_arena = torch.as_tensor(arena).to("cuda")
            sec = torch.as_tensor(L.sec_abs).to("cuda")
            S = dg.dgnn_samples_load(ctx, L.samples, 0, L.num_batches, dev_arena, sec)
            ctx.sync()
            nodes, eptr, src = S.nodes.cpu().numpy(), S.eptr.cpu().numpy(), S.src_local.cpu().numpy()
            for b, r in enumerate(samples):
                assert np.array_equal(nodes[S.node_off_host[b]:S.node_off_host[b + 1]], r.nodes)
                assert np.array_equal(eptr[S.eptr_off_host[b]:S.eptr_off_host[b + 1]], r.eptr)
                assert np.array_equal(src[S.edge_off_host[b]:S.edge_off_host[b + 1]], r.src_local)
                assert np.array_equal(S.hop_off_host[b], r.hop_off)
            assert np.array_equal(S.node_off.cpu().numpy(), np.asarray(S.node_off_host))
        # training through the loader stage: seed embeddings equal the oracle's
        tctx = dg.Ctx(device=0, stream=torch.cuda.Stream())
        seen = 0
        for b0, b1, x in L.train_epoch(train_ctx=tctx, out_budget=600_000 if group == 2 else 1 << 30,
                                       host_window=2):
            tctx.sync()
            no = L.samples.node_off_host
            for b in range(b0, b1):
                r = samples[b]
                got = x[int(no[b] - no[b0]):int(no[b] - no[b0]) + int(r.hop_off[1])].cpu().numpy()
                want = oracle.train_stub(r, oracle.assemble(feats, r.nodes).view(np.float32))
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"batch {b}"
                seen += 1
        ctx.sync()
        assert seen == L.num_batches
    ctx.set_sample_mode(False)


def test_loader_rejects_a_misplaced_section(dg, tiny, ref):
    ctx = dg.Ctx(device=0)
    with tempfile.TemporaryDirectory() as td:
        L = _layout(dg, ctx, tiny, "pinned", 8, td)
        ctx.sync()
        dev_arena = L.arena.tensor.to("cuda")
        bad = torch.as_tensor(L.sec_abs + 4).to("cuda")  # one word off
        with pytest.raises(dg.DgnnError):
            dg.dgnn_samples_load(ctx, L.samples, 0, L.num_batches, dev_arena, bad)
            ctx.sync()
