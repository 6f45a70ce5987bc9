"""Pins for the oracle's trainer stub (surrogate of Eq. 1; reading t1).

* Fig. 1 with all-ones features: hop-1 nodes become 1 + 1 = 2 after layer 1, the seed
  1 + mean(2, 2) = 3 after layer 2 -- exact in fp32 (hand derivation of the recurrence).
* A seed without sampled edges keeps its own feature; fanout [0] leaves every seed as is.
* Dense recomputation: the recurrence written as per-hop row-normalised adjacency matrices in
  float64 numpy (a different formulation: no loops over edges) agrees within 1e-5 on random
  samples -- a wrong hop order, a dropped self term or a wrong neighbour index fails it.
* Order independence: with integer-valued features every partial sum is exact, so
  permuting each node's edge list gives bit-identical embeddings.
"""
import numpy as np
import pytest

import oracle
from conftest import csr_from_adj, golden_lines, random_csr


def _fig1_sample():
    g = {}
    for line in golden_lines("fig1_sampling.txt"):
        key, *rest = line.split()
        g[key] = rest
    adj = {}
    for tok in g["edges"]:
        v, nb = tok.split(":")
        adj[int(v)] = [int(x) for x in nb.split(",")]
    indptr, indices = csr_from_adj(int(g["num_nodes"][0]), adj)
    (s,) = oracle.sample(indptr, indices, [int(x) for x in g["seeds"]], 1, [int(x) for x in g["fanout"]], 0)
    return s


def test_fig1_all_ones():
    s = _fig1_sample()
    x = np.ones((len(s.nodes), 16), np.float32)
    out = oracle.train_stub(s, x)
    assert out.shape == (1, 16) and np.all(out == 3.0)


def test_seed_without_edges_keeps_its_feature():
    indptr, indices = csr_from_adj(4, {0: [1, 2], 1: [2]})  # node 3 isolated
    rng = np.random.default_rng(0)
    samples = oracle.sample(indptr, indices, [3, 0], 2, [2, 1], 5)
    x = rng.random((len(samples[0].nodes), 8)).astype(np.float32)
    out = oracle.train_stub(samples[0], x)
    assert np.array_equal(out[0], x[0])  # seed 3 has no neighbours
    assert not np.array_equal(out[1], x[1])
    (s0,) = oracle.sample(indptr, indices, [0, 1], 2, [0], 5)
    x = rng.random((len(s0.nodes), 8)).astype(np.float32)
    assert np.array_equal(oracle.train_stub(s0, x), x[:2])


def dense_reference(s, x):
    """float64: X <- X + M_h X with M_h[j, u] = (edges j->u) / deg_h(j) for j in hop h, deepest hop first."""
    n = len(s.nodes)
    X = x.astype(np.float64)
    H = len(s.hop_off) - 2
    for k in range(1, H + 1):
        h = H - k
        M = np.zeros((n, n))
        for j in range(s.hop_off[h], s.hop_off[h + 1]):
            e0, e1 = s.eptr[j], s.eptr[j + 1]
            if e1 > e0:
                np.add.at(M[j], s.src_local[e0:e1], 1.0 / (e1 - e0))
        X = X + M @ X
    return X[: s.hop_off[1]]


@pytest.mark.parametrize("trial", range(12))
def test_dense_recomputation(trial):
    rng = np.random.default_rng(40 + trial)
    n = int(rng.integers(20, 120))
    indptr, indices = random_csr(rng, n, int(rng.integers(1, 9)))
    H = int(rng.integers(1, 4))
    fan = [int(rng.integers(0, 6)) for _ in range(H)]
    seeds = rng.permutation(n)[: int(rng.integers(1, 12))].astype(np.int32)
    for s in oracle.sample(indptr, indices, seeds, 5, fan, trial):
        x = (rng.random((len(s.nodes), 12)) * 2 - 1).astype(np.float32)
        got = oracle.train_stub(s, x)
        assert np.allclose(got, dense_reference(s, x), rtol=1e-5, atol=1e-5)


def test_edge_order_independence_on_exact_values():
    """One hop over integer-valued features: every partial sum is exact, so only the final
    division rounds -- identically for any order of a node's edges."""
    rng = np.random.default_rng(9)
    indptr, indices = random_csr(rng, 80, 8)
    for s in oracle.sample(indptr, indices, np.arange(0, 80, 7, dtype=np.int32), 4, [6], 3):
        x = rng.integers(-8, 9, size=(len(s.nodes), 6)).astype(np.float32)
        base = oracle.train_stub(s, x)
        perm = s.src_local.copy()
        for j in range(len(s.eptr) - 1):
            seg = perm[s.eptr[j]:s.eptr[j + 1]]
            perm[s.eptr[j]:s.eptr[j + 1]] = seg[rng.permutation(len(seg))]
        s2 = oracle.Sample(s.bid, s.nodes, s.hop_off, s.eptr, perm)
        assert np.array_equal(oracle.train_stub(s2, x), base)
