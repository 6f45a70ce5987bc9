"""Pins of oracle.pack_embedded: the graph sample kept in the chunk (reading c22b).

The section is parsed back here with struct (independently of the oracle's numpy serialization)
and must reproduce the oracle's own sample arrays; the rows must be exactly ``pack``'s rows, every
chunk must start on a 4096-byte boundary, the section on a 16-byte boundary right after the rows,
and every other byte must be zero.
"""
import struct

import numpy as np
import pytest

import oracle
from conftest import random_csr


def _parse(buf, off):
    H, n, m, e = struct.unpack_from("<4i", buf, off)
    p = off + 16
    hop = list(struct.unpack_from(f"<{H + 2}i", buf, p)); p += 4 * (H + 2)
    nodes = list(struct.unpack_from(f"<{n}i", buf, p)); p += 4 * n
    eptr = list(struct.unpack_from(f"<{m}i", buf, p)); p += 4 * m
    src = list(struct.unpack_from(f"<{e}i", buf, p)); p += 4 * e
    return H, hop, nodes, eptr, src, p


@pytest.mark.parametrize("trial", range(8))
@pytest.mark.parametrize("blocks", [False, True])
def test_sections_parse_back_to_the_samples(trial, blocks):
    rng = np.random.default_rng(500 + trial)
    n = int(rng.integers(20, 400))
    indptr, indices = random_csr(rng, n, max_deg=int(rng.integers(1, 20)))
    fan = [int(x) for x in rng.choice([0, 1, 3, 5, 10], size=int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[:int(rng.integers(1, n))].astype(np.int32)
    B = int(rng.integers(1, 40))
    samples = oracle.sample(indptr, indices, seeds, B, fan, 11, blocks=blocks)
    dim = int(rng.choice([1, 3, 32, 100]))
    feats = rng.standard_normal((n, dim)).astype(np.float32)
    counts = oracle.count_frequencies(samples, n)
    tm, _, _ = oracle.select_tiers(counts, n // 10, n // 5)
    plists = [oracle.classify(s.nodes, tm)[1] for s in samples]
    buf, off, sec = oracle.pack_embedded(feats, plists, samples)
    plain, _ = oracle.pack(feats, plists)
    rb = 4 * dim
    assert len(buf) == off[-1] and np.all(off % 4096 == 0) and np.all(np.diff(off) > 0)
    used = np.zeros(len(buf), bool)
    for i, (s, p) in enumerate(zip(samples, plists)):
        rows_end = off[i] + len(p) * rb
        assert np.array_equal(buf[off[i]:rows_end], feats[p].view(np.uint8).reshape(-1))
        assert sec[i] == off[i] + (len(p) * rb + 15) // 16 * 16
        H, hop, nodes, eptr, src, end = _parse(buf.tobytes(), int(sec[i]))
        assert H == len(fan) and hop == list(s.hop_off) and nodes == list(s.nodes)
        assert eptr == list(s.eptr) and src == list(s.src_local)
        assert end <= off[i + 1]
        used[off[i]:rows_end] = True
        used[sec[i]:end] = True
    assert not np.any(buf[~used]), "padding must be zero"
    # the rows part of every chunk is pack()'s chunk rows
    _, poff = oracle.pack(feats, plists)
    for i, p in enumerate(plists):
        assert np.array_equal(buf[off[i]:off[i] + len(p) * rb], plain[poff[i]:poff[i] + len(p) * rb])


def test_fig1_section_words():
    """Fig. 1: the forcing graph's one batch serializes as the hand-derived words."""
    adj = {0: [3, 5], 3: [2, 7], 5: [9, 11]}
    from conftest import csr_from_adj
    ip, ix = csr_from_adj(12, adj)
    s = oracle.sample(ip, ix, np.array([0], np.int32), 1, [2, 2], 7)
    feats = np.zeros((12, 1), np.float32)
    buf, off, sec = oracle.pack_embedded(feats, [np.array([], np.int32)], s)
    words = np.frombuffer(buf.tobytes(), "<i4")
    # H=2, n=7, m=hop_off[2]+1=4 (nodes 0,3,5 expand), e=6; hop_off [0,1,3,7];
    # nodes [0,3,5,2,7,9,11]; eptr [0,2,4,6]; src [1,2,3,4,5,6]
    want = [2, 7, 4, 6, 0, 1, 3, 7, 0, 3, 5, 2, 7, 9, 11, 0, 2, 4, 6, 1, 2, 3, 4, 5, 6]
    assert sec[0] == 0 and list(words[:len(want)]) == want and not words[len(want):].any()
    assert off[-1] == 4096
