"""Pins for the oracle's DGL-block sampling variant (reading c27) and its
trainer stub.

* Fig. 1 in block form: the seed resamples at hop 2 (degree = fanout: both edges again),
  the node set is unchanged -- derived by hand from the definition.
* Full fanout: hop h's edges are exactly every CSR edge of every node within distance <= h of
  the seeds (brute-force BFS), the node set is the BFS ball -- the same as node-wise.
* Draw keying: a node expanding at hop h in both variants (hop 0: the seeds; hop 1: the nodes
  found at hop 0, identical in both) draws the same positions (Philox key (seed, v, bid, h, s)).
* Structure on random graphs: per hop and node, min(k, d) distinct real edges in ascending CSR
  position; eptr per hop covers every node of the sample so far.
* Trainer stub: float64 dense recomputation over the block adjacency, within 1e-5.
"""
from collections import deque

import numpy as np
import pytest

import oracle
from conftest import csr_from_adj, random_csr
from conftest import golden_lines


def _fig1_graph():
    g = {}
    for line in golden_lines("fig1_sampling.txt"):
        key, *rest = line.split()
        g[key] = rest
    adj = {}
    for tok in g["edges"]:
        v, nb = tok.split(":")
        adj[int(v)] = [int(x) for x in nb.split(",")]
    return csr_from_adj(int(g["num_nodes"][0]), adj), g


def hop_edges(s, h):
    """[(dst_local, src_local)] of hop h of a block-mode sample."""
    base = sum(int(s.hop_off[i + 1]) + 1 for i in range(h))
    ep = s.eptr[base:base + int(s.hop_off[h + 1]) + 1]
    return [(j, int(s.src_local[e])) for j in range(int(s.hop_off[h + 1])) for e in range(ep[j], ep[j + 1])]


def test_fig1_blocks():
    (indptr, indices), g = _fig1_graph()
    (s,) = oracle.sample(indptr, indices, [0], 1, [2, 2], 0, blocks=True)
    assert s.nodes.tolist() == [int(x) for x in g["nodes"]]
    assert hop_edges(s, 0) == [(0, 1), (0, 2)]
    assert hop_edges(s, 1) == [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5), (2, 6)]
    assert s.eptr.tolist() == [0, 2, 2, 4, 6, 8]


def _dist(indptr, indices, seeds, hops):
    dist = {int(v): 0 for v in seeds}
    q = deque(int(v) for v in seeds)
    while q:
        v = q.popleft()
        if dist[v] == hops:
            continue
        for u in indices[indptr[v]:indptr[v + 1]]:
            if int(u) not in dist:
                dist[int(u)] = dist[v] + 1
                q.append(int(u))
    return dist


@pytest.mark.parametrize("trial", range(15))
def test_full_fanout_is_every_edge_of_the_ball(trial):
    rng = np.random.default_rng(300 + trial)
    n = int(rng.integers(10, 80))
    indptr, indices = random_csr(rng, n, 6)
    H = int(rng.integers(1, 4))
    seeds = rng.permutation(n)[: int(rng.integers(1, 5))].astype(np.int32)
    (s,) = oracle.sample(indptr, indices, seeds, len(seeds), [100] * H, trial, blocks=True)
    (w,) = oracle.sample(indptr, indices, seeds, len(seeds), [100] * H, trial)
    assert s.nodes.tolist() == w.nodes.tolist() and s.hop_off.tolist() == w.hop_off.tolist()
    dist = _dist(indptr, indices, seeds, H)
    nodes = s.nodes.tolist()
    for h in range(H):
        got = sorted((nodes[j], nodes[u]) for j, u in hop_edges(s, h))
        exp = sorted((v, int(u)) for v, d in dist.items() if d <= h for u in indices[indptr[v]:indptr[v + 1]])
        assert got == exp


@pytest.mark.parametrize("trial", range(10))
def test_structure_and_shared_draw_keys(trial):
    rng = np.random.default_rng(500 + trial)
    n = int(rng.integers(30, 200))
    indptr, indices = random_csr(rng, n, 12)
    fan = [int(rng.integers(0, 8)) for _ in range(int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[:20].astype(np.int32)
    S = oracle.sample(indptr, indices, seeds, 7, fan, trial, blocks=True)
    W = oracle.sample(indptr, indices, seeds, 7, fan, trial)
    for s, w in zip(S, W):
        nodes = s.nodes
        assert len(set(nodes.tolist())) == len(nodes)
        for h, k in enumerate(fan):
            per = {}
            for j, u in hop_edges(s, h):
                per.setdefault(j, []).append(int(nodes[u]))
            for j in range(int(s.hop_off[h + 1])):
                v = int(nodes[j])
                nb = indices[indptr[v]:indptr[v + 1]].tolist()
                got = per.get(j, [])
                assert len(got) == min(k, len(nb))
                pos = [nb.index(x) for x in got]  # graphs have no multi-edges
                assert pos == sorted(set(pos))
        # hop 0 (the seeds) and hop 1 (the nodes found at hop 0) expand in both variants with
        # the same keys, so they draw the same neighbours
        for h in range(min(2, len(fan))):
            wmap = {}
            lo, hi = int(w.hop_off[h]), int(w.hop_off[h + 1])
            for j in range(lo, hi):
                wmap[int(w.nodes[j])] = [int(w.nodes[w.src_local[e]]) for e in range(w.eptr[j], w.eptr[j + 1])]
            bmap = {}
            for j, u in hop_edges(s, h):
                bmap.setdefault(int(nodes[j]), []).append(int(nodes[u]))
            for v, nb in wmap.items():
                assert bmap.get(v, []) == nb


def dense_blocks(s, x):
    n = len(s.nodes)
    X = x.astype(np.float64)
    H = len(s.hop_off) - 2
    for k in range(1, H + 1):
        h = H - k
        M = np.zeros((n, n))
        for j, u in hop_edges(s, h):
            M[j, u] += 1.0
        deg = M.sum(axis=1, keepdims=True)
        M = np.divide(M, deg, out=np.zeros_like(M), where=deg > 0)
        X = X + M @ X
    return X[: s.hop_off[1]]


@pytest.mark.parametrize("trial", range(8))
def test_trainer_blocks_dense(trial):
    rng = np.random.default_rng(900 + trial)
    n = int(rng.integers(20, 100))
    indptr, indices = random_csr(rng, n, 7)
    H = int(rng.integers(1, 4))
    fan = [int(rng.integers(0, 5)) for _ in range(H)]
    seeds = rng.permutation(n)[:9].astype(np.int32)
    for s in oracle.sample(indptr, indices, seeds, 4, fan, trial, blocks=True):
        x = (rng.random((len(s.nodes), 10)) * 2 - 1).astype(np.float32)
        assert np.allclose(oracle.train_stub(s, x), dense_blocks(s, x), rtol=1e-5, atol=1e-5)
