"""Pins for the oracle's node-wise K-hop sampler.

* Fig. 1 worked example with a forcing graph.
* Full fanout equals the K-hop BFS ball, layer by layer, by brute force.
* Star graph, fanout [0], partition arithmetic,
  empty seeds, duplicate seeds rejected (reading c12).
* Structural invariants on random graphs: real edges, min(k, d) per node,
  distinct nodes, seeds first, per-hop blocks ascending (c10), determinism.
"""
from collections import deque

import numpy as np
import pytest

import oracle
from conftest import csr_from_adj, golden_lines, random_csr


def _fig1():
    g = {}
    for line in golden_lines("fig1_sampling.txt"):
        key, *rest = line.split()
        g[key] = rest
    n = int(g["num_nodes"][0])
    adj = {}
    for tok in g["edges"]:
        v, nb = tok.split(":")
        adj[int(v)] = [int(x) for x in nb.split(",")]
    return n, adj, g


def test_fig1_worked_example():
    n, adj, g = _fig1()
    indptr, indices = csr_from_adj(n, adj)
    fan = [int(x) for x in g["fanout"]]
    seeds = [int(x) for x in g["seeds"]]
    for rng_seed in (0, 1, 0xDEADBEEF):  # degree == fanout: no draw can matter
        (s,) = oracle.sample(indptr, indices, seeds, 1, fan, rng_seed)
        assert s.nodes.tolist() == [int(x) for x in g["nodes"]]
        for h in range(2):
            exp = [tuple(int(x) for x in e.split("<-")) for e in g[f"hop{h}"]]
            got = []
            for j in range(s.hop_off[h], s.hop_off[h + 1]):
                for e in range(s.eptr[j], s.eptr[j + 1]):
                    got.append((j, int(s.src_local[e])))
            assert got == exp


def _bfs_layers(indptr, indices, seeds, hops):
    dist = {int(v): 0 for v in seeds}
    q = deque(int(v) for v in seeds)
    while q:
        v = q.popleft()
        if dist[v] == hops:
            continue
        for u in indices[indptr[v]:indptr[v + 1]]:
            u = int(u)
            if u not in dist:
                dist[u] = dist[v] + 1
                q.append(u)
    return [sorted(v for v, d in dist.items() if d == h) for h in range(1, hops + 1)]


@pytest.mark.parametrize("trial", range(40))
def test_full_fanout_equals_bfs_layers(trial):
    rng = np.random.default_rng(trial)
    n = int(rng.integers(2, 300))
    indptr, indices = random_csr(rng, n, max_deg=int(rng.integers(1, 9)))
    hops = int(rng.integers(1, 4))
    maxd = int((indptr[1:] - indptr[:-1]).max())
    ns = int(rng.integers(1, min(n, 20) + 1))
    seeds = rng.choice(n, ns, replace=False).astype(np.int32)
    (s,) = oracle.sample(indptr, indices, seeds, ns, [maxd + int(rng.integers(0, 3))] * hops, trial)
    layers = _bfs_layers(indptr, indices, seeds, hops)
    assert s.nodes[:ns].tolist() == seeds.tolist()
    for h in range(hops):
        assert s.nodes[s.hop_off[h + 1]:s.hop_off[h + 2]].tolist() == layers[h]
    # every out-edge of every frontier node is present, in CSR order
    for j in range(int(s.hop_off[hops])):
        v = s.nodes[j]
        got = s.nodes[s.src_local[s.eptr[j]:s.eptr[j + 1]]].tolist()
        assert got == indices[indptr[v]:indptr[v + 1]].tolist()


def test_star_graph():
    indptr, indices = csr_from_adj(6, {0: [1, 2, 3, 4, 5]})
    for seed in range(5):
        (s,) = oracle.sample(indptr, indices, [0], 1, [5], seed)
        assert s.nodes.tolist() == [0, 1, 2, 3, 4, 5]


def test_zero_fanout_gives_seeds_only():
    rng = np.random.default_rng(5)
    indptr, indices = random_csr(rng, 100, 8)
    seeds = np.arange(0, 100, 3, dtype=np.int32)
    for s in oracle.sample(indptr, indices, seeds, 7, [0], 1):
        assert s.nodes.tolist() == seeds[(s.bid) * 7:(s.bid + 1) * 7].tolist()
        assert len(s.src_local) == 0 and s.hop_off.tolist() == [0, len(s.nodes), len(s.nodes)]


def test_partition_arithmetic_and_empty():
    rng = np.random.default_rng(0)
    indptr, indices = random_csr(rng, 3000, 4)
    seeds = rng.permutation(3000)[:2049].astype(np.int32)
    S = oracle.sample(indptr, indices, seeds, 1024, [2], 3)
    assert [len(s.nodes[:s.hop_off[1]]) for s in S] == [1024, 1024, 1]
    assert [s.bid for s in S] == [0, 1, 2]
    assert oracle.sample(indptr, indices, np.zeros(0, np.int32), 1024, [2], 3) == []
    S2 = oracle.sample(indptr, indices, seeds, 1024, [2], 3, batch_id_base=100)
    assert [s.bid for s in S2] == [100, 101, 102]


def test_duplicate_or_invalid_seeds_rejected():
    indptr, indices = csr_from_adj(4, {0: [1], 1: [2]})
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample(indptr, indices, [1, 1], 2, [1], 0)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError):
        oracle.sample(indptr, indices, [7], 1, [1], 0)
    # across batches duplicates are fine (c12)
    assert len(oracle.sample(indptr, indices, [1, 1], 1, [1], 0)) == 2


@pytest.mark.parametrize("trial", range(15))
def test_structural_invariants_random(trial):
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(50, 2000))
    indptr, indices = random_csr(rng, n, max_deg=int(rng.integers(1, 40)))
    fan = [int(x) for x in rng.integers(0, 12, size=int(rng.integers(1, 4)))]
    seeds = rng.permutation(n)[: int(rng.integers(1, n))].astype(np.int32)
    B = int(rng.integers(1, 200))
    S = oracle.sample(indptr, indices, seeds, B, fan, trial * 7 + 1, threads=4)
    S1 = oracle.sample(indptr, indices, seeds, B, fan, trial * 7 + 1, threads=1)
    for s, s1 in zip(S, S1):  # determinism across thread counts
        assert np.array_equal(s.nodes, s1.nodes) and np.array_equal(s.src_local, s1.src_local)
    for s in S:
        nodes = s.nodes
        assert len(set(nodes.tolist())) == len(nodes)
        ns = int(s.hop_off[1])
        assert nodes[:ns].tolist() == seeds[s.bid * B:s.bid * B + ns].tolist()
        for h in range(len(fan)):
            blk = nodes[s.hop_off[h + 1]:s.hop_off[h + 2]]
            assert np.all(np.diff(blk) > 0)
            for j in range(int(s.hop_off[h]), int(s.hop_off[h + 1])):
                v = int(nodes[j])
                d = int(indptr[v + 1] - indptr[v])
                e0, e1 = int(s.eptr[j]), int(s.eptr[j + 1])
                assert e1 - e0 == min(fan[h], d)
                nb = nodes[s.src_local[e0:e1]]
                row = indices[indptr[v]:indptr[v + 1]]
                assert set(nb.tolist()) <= set(row.tolist())   # every sampled neighbour is a real edge
                pos = [int(np.nonzero(row == u)[0][0]) for u in nb]
                assert pos == sorted(pos) and len(set(pos)) == len(pos)  # distinct CSR positions, ascending
                # every src is a node discovered no later than this hop
                assert np.all(s.src_local[e0:e1] < s.hop_off[h + 2])


def test_neighbour_inclusion_is_uniform():
    """Over many batch ids a degree-20 node includes each neighbour w.p. 5/20."""
    adj = {0: list(range(1, 21))}
    indptr, indices = csr_from_adj(21, adj)
    trials = 3000
    seeds = np.zeros(trials, np.int32)
    hits = np.zeros(21)
    for s in oracle.sample(indptr, indices, seeds, 1, [5], 77):
        hits[s.nodes[1:]] += 1
    expect = trials * 5 / 20
    chi2 = float(((hits[1:] - expect) ** 2 / expect).sum())
    assert chi2 < 50, chi2  # 19 dof


def test_sampled_neighbours_depend_on_bid_not_position():
    """Reading c8: draws are keyed by the global node ID, not its local index."""
    rng = np.random.default_rng(9)
    indptr, indices = random_csr(rng, 500, 30, allow_empty=False)
    a = oracle.sample(indptr, indices, [10, 20], 2, [3], 5)[0]
    b = oracle.sample(indptr, indices, [20, 10], 2, [3], 5)[0]
    def nbrs(s, v):
        j = s.nodes.tolist().index(v)
        return sorted(s.nodes[s.src_local[s.eptr[j]:s.eptr[j + 1]]].tolist())
    assert nbrs(a, 10) == nbrs(b, 10) and nbrs(a, 20) == nbrs(b, 20)
