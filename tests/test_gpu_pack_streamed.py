"""Batched packing from partitions (Sec. 5.2, Fig. 6; NEXT #3): GPU vs oracle.

The chunks produced partition by partition, from a pinned host table or an O_DIRECT feature
file, are byte-identical to the oracle's pack of the oracle's own packed lists (and so to the
one-launch HBM pack); the source pages read equal the oracle's batched page count.
"""
import os
import tempfile

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_lines
from workload import make_packed_lists, make_workload, feature_rows_np

pytestmark = pytest.mark.gpu
RNG_SEED = 0x5EEDD15C
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


def _run(dg, ctx, pl, feats_np, part_rows, source_kind):
    from paper_2405_05231_b200 import packing
    from paper_2405_05231_b200.layout import HostBuffer
    dev = torch.device("cuda", 0)
    N, rb = feats_np.shape[0], feats_np.reshape(feats_np.shape[0], -1).view(np.uint8).shape[1]
    off = np.concatenate([[0], np.cumsum([len(p) for p in pl])]).astype(np.int64)
    ids = np.concatenate([np.asarray(p, np.int32) for p in pl]) if len(pl) else np.zeros(0, np.int32)
    idx = dg.DiskIndex(ctx, torch.as_tensor(ids).to(dev), torch.as_tensor(off).to(dev), off, N)
    co = dg.dgnn_chunk_layout(off, rb)
    group = torch.full((max(int(co[-1]), 16),), 0xCD, dtype=torch.uint8, device=dev)
    ft = torch.as_tensor(feats_np)
    keep = None
    if source_kind == "file":
        path = os.path.join(tempfile.mkdtemp(prefix="dgnn_feat_"), "features.bin")
        size = packing.write_feature_file(path, ft)
        src = dg._abi.DiskFile(path, size, direct=True, create=False)
    else:
        hb = HostBuffer(N * rb)
        hb.tensor.copy_(ft.contiguous().view(torch.uint8).reshape(-1))
        src = keep = hb
    rep = packing.pack_streamed(ctx, idx, src, N, rb, torch.as_tensor(co).to(dev), group, part_rows)
    ctx.sync()
    del keep
    return group.cpu().numpy()[:int(co[-1])], rep


def test_fig6_on_the_gpu(dg, ctx):
    g = {"batch": []}
    for line in golden_lines("fig6_packing.txt"):
        k, *rest = line.split()
        if k == "batch":
            g["batch"].append([int(x) for x in rest])
        else:
            g[k] = int(rest[0])
    feats = feature_rows_np(np.arange(g["num_nodes"]), g["row_bytes"] // 4, 1)
    got, rep = _run(dg, ctx, g["batch"], feats, g["partition_rows"], "pinned")
    buf, _ = oracle.pack(feats, g["batch"])
    assert np.array_equal(got, buf)
    assert rep["pages"] == g["batched_pages"] == oracle.pack_pages(g["batch"], 4, g["row_bytes"], 4)[1]


@pytest.mark.parametrize("source", ["pinned", "file"])
@pytest.mark.parametrize("dim,part", [(128, 64), (100, 1024), (128, 8), (1024, 3)])
def test_streamed_equals_oracle(dg, ctx, source, dim, part):
    N, nb = 3000, 23
    ids, off = make_packed_lists(nb, N, 200, 3.0, seed=dim + part)
    pl = [ids[off[b]:off[b + 1]] for b in range(nb)]
    pl[5] = pl[5][:0]  # an empty chunk
    feats = feature_rows_np(np.arange(N), dim, 1)
    rb = dim * 4
    step = PAGE // int(np.gcd(PAGE, rb))
    part_rows = step * part
    got, rep = _run(dg, ctx, pl, feats, part_rows, source)
    buf, _ = oracle.pack(feats, pl)
    assert np.array_equal(got, buf)
    assert rep["pages"] == oracle.pack_pages(pl, N, rb, part_rows)[1]


def test_streamed_tiny_layout(dg, ctx):
    """The oracle's own offline layout of the tiny configuration: every packed group rebuilt
    partition by partition equals the oracle's groups."""
    w = make_workload("tiny")
    feats = w.features.numpy()
    ref = oracle.offline_layout(w.indptr.numpy(), w.indices.numpy(), feats, w.seeds.numpy(), 256, [10, 5],
                                RNG_SEED, 500, 1000, 8)
    got, rep = _run(dg, ctx, ref["packed"], feats, 512, "file")
    assert np.array_equal(got, ref["groups"][0][0])
    assert rep["pages"] == oracle.pack_pages(ref["packed"], 10_000, 512, 512)[1]
