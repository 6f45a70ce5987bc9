"""Pins for the oracle's counting, tier selection, classify, pack and assemble.

* counts: S:128 ({0,1},{1,2} -> [1,2,1]) and conservation S:129.
* tiers: Fig. 3, capacity edge cases, the partition
  invariant (c19), and the optimality statement of P:226 -- the GPU tier holds
  the K_g largest counts and GPU+HOST the K_g+K_h largest -- which holds for
  ANY tie-break; plus the ordering invariant of S:106.
* classify: Fig. 3 address table (S:294 adapted to reading c18).
* pack / assemble: rows equal the closed-form features (an independent
  numpy transcription, workload.feature_rows_np), 4 KiB chunk alignment and
  zero padding (c20), three-source reconstruction == direct gather,
  SPEC acceptance #1 fixture.
"""
import numpy as np
import pytest

import oracle
from conftest import golden_lines, random_csr
from workload import feature_rows_np, make_workload


class _S:
    def __init__(self, nodes):
        self.nodes = np.asarray(nodes, np.int32)


def test_counts_spec_example_and_conservation():
    c = oracle.count_frequencies([_S([0, 1]), _S([1, 2])], 3)
    assert c.tolist() == [1, 2, 1]
    assert oracle.count_frequencies([], 4).tolist() == [0, 0, 0, 0]
    rng = np.random.default_rng(1)
    indptr, indices = random_csr(rng, 400, 6)
    S = oracle.sample(indptr, indices, rng.permutation(400)[:300].astype(np.int32), 37, [4, 3], 11)
    c = oracle.count_frequencies(S, 400)
    assert int(c.sum()) == sum(len(s.nodes) for s in S)
    for v in rng.integers(0, 400, 50):
        assert c[v] == sum(int(v in set(s.nodes.tolist())) for s in S)


def _fig3():
    g = {}
    for line in golden_lines("fig3_assembly.txt"):
        key, *rest = line.split()
        g[key] = rest
    return g


def test_fig3_tiers_and_address_table():
    g = _fig3()
    n = int(g["num_nodes"][0])
    counts = np.zeros(n, np.uint32)
    for tok in g["counts"]:
        v, c = tok.split(":")
        counts[int(v)] = int(c)
    tm, gpu, host = oracle.select_tiers(counts, *[int(x) for x in g["capacities"]])
    assert gpu.tolist() == [int(x) for x in g["gpu"]]
    assert host.tolist() == [int(x) for x in g["host"]]
    addr, P = oracle.classify([int(x) for x in g["batch"]], tm)
    code = {"G": 0, "H": 1, "D": 2}
    exp = [(code[a.split(":")[0]] << 30) | int(a.split(":")[1]) for a in g["addr"]]
    assert addr.tolist() == exp
    assert P.tolist() == [int(x) for x in g["packed"]]


def test_capacity_edge_cases():
    counts = np.array([0, 3, 1, 0, 2, 2], np.uint32)
    tm, gpu, host = oracle.select_tiers(counts, 0, 0)
    assert len(gpu) == 0 and len(host) == 0 and np.all(tm >> 30 == 2)
    tm, gpu, host = oracle.select_tiers(counts, 10, 10)
    assert sorted(gpu.tolist() + host.tolist()) == [1, 2, 4, 5]   # every accessed node cached
    assert gpu.tolist() == [1, 2, 4, 5] and len(host) == 0
    assert (tm[[0, 3]] >> 30).tolist() == [2, 2]                  # zero counts never cached
    tm, gpu, host = oracle.select_tiers(counts, 1, 2)
    assert gpu.tolist() == [1] and host.tolist() == [4, 5]        # tie 2,2 both fit


@pytest.mark.parametrize("trial", range(30))
def test_tier_optimality_partition_and_order(trial):
    rng = np.random.default_rng(trial)
    n = int(rng.integers(1, 3000))
    counts = rng.integers(0, int(rng.integers(1, 12)), n).astype(np.uint32)
    kg = int(rng.integers(0, n + 2))
    kh = int(rng.integers(0, n + 2))
    tm, gpu, host = oracle.select_tiers(counts, kg, kh)
    nnz = int((counts > 0).sum())
    assert len(gpu) == min(kg, nnz) and len(host) == min(kh, nnz - len(gpu))
    top = np.sort(counts)[::-1]
    # P:226 optimality, independent of the tie-break
    assert int(counts[gpu].sum()) == int(top[:len(gpu)].sum())
    assert int(counts[gpu].sum() + counts[host].sum()) == int(top[:len(gpu) + len(host)].sum())
    # partition (c19) and slots ascending by ID (c17)
    tiers = tm >> 30
    assert set(np.unique(tiers).tolist()) <= {0, 1, 2}
    assert np.array_equal(np.nonzero(tiers == 0)[0], gpu) and np.array_equal(np.nonzero(tiers == 1)[0], host)
    assert np.array_equal(tm[gpu] & oracle.SLOT_MASK, np.arange(len(gpu)))
    assert np.array_equal(tm[host] & oracle.SLOT_MASK, np.arange(len(host)))
    assert np.all(tm[tiers == 2] & oracle.SLOT_MASK == 0)
    # gpu >= host >= uncached, ties broken by ascending node ID
    def key(v):
        return (-int(counts[v]), int(v))
    disk = np.nonzero((tiers == 2) & (counts > 0))[0]
    if len(gpu) and len(host):
        assert max(key(v) for v in gpu) < min(key(v) for v in host)
    if len(host) and len(disk):
        assert max(key(v) for v in host) < min(key(v) for v in disk)
    if len(gpu) and len(disk) and not len(host):
        assert max(key(v) for v in gpu) < min(key(v) for v in disk)
    assert np.all(counts[tiers != 2] > 0)


def test_classify_every_node_resolves_once():
    rng = np.random.default_rng(3)
    n = 500
    counts = rng.integers(0, 5, n).astype(np.uint32)
    tm, gpu, host = oracle.select_tiers(counts, 40, 60)
    nodes = rng.permutation(n)[:200].astype(np.int32)
    addr, P = oracle.classify(nodes, tm)
    t = addr >> 30
    assert np.array_equal(P, nodes[t == 2])
    assert np.array_equal(addr[t == 2] & oracle.SLOT_MASK, np.arange(len(P)))
    assert np.array_equal(addr[t != 2], tm[nodes[t != 2]])


def test_chunk_offsets_alignment_and_empty_chunks():
    off = oracle.chunk_offsets([3, 0, 9, 0, 1], 400)
    assert off.tolist() == [0, 4096, 4096, 8192, 8192, 12288]
    assert oracle.chunk_offsets([], 512).tolist() == [0]
    assert oracle.chunk_offsets([8, 8], 512).tolist() == [0, 4096, 8192]


def test_pack_rows_equal_closed_form_features_and_zero_padding():
    dim = 100  # 400-byte rows: 4096 % 400 != 0 (reading c20)
    n = 300
    feats = feature_rows_np(np.arange(n), dim, fseed=3)
    rng = np.random.default_rng(4)
    plists = [rng.choice(n, int(rng.integers(0, 40)), replace=False).astype(np.int32) for _ in range(6)]
    plists[2] = np.zeros(0, np.int32)
    buf, off = oracle.pack(feats, plists)
    assert np.all(off % 4096 == 0) and len(buf) == off[-1]
    for i, P in enumerate(plists):
        chunk = buf[off[i]:off[i + 1]]
        body = chunk[:len(P) * 400].view(np.float32).reshape(len(P), dim)
        exp = feature_rows_np(P, dim, fseed=3)
        assert np.array_equal(body.view(np.uint32), exp.view(np.uint32))
        assert not chunk[len(P) * 400:].any()


def test_spec_acceptance_fixture_assembly_bit_exact():
    """1000 nodes, dim 128, 100 batches, fanout [5,5], tiers 5% / 10%."""
    w = make_workload("tiny", num_nodes=1000, num_edges=10_000, num_seeds=100 * 8, batch_size=8,
                      fanout=(5, 5))
    feats = w.features.numpy()
    L = oracle.offline_layout(w.indptr.numpy(), w.indices.numpy(), feats, w.seeds.numpy(), 8, [5, 5],
                              0x5EED, 50, 100, group_size=16, threads=4)
    assert len(L["samples"]) == 100
    for i, s in enumerate(L["samples"]):
        g, r = divmod(i, 16)
        buf, off = L["groups"][g]
        chunk = buf[off[r]:off[r + 1]]
        rec = oracle.assemble_tiers(L["addr"][i], L["gpu_buf"], L["host_buf"], chunk, 512)
        direct = feature_rows_np(s.nodes, 128, fseed=1).view(np.uint8).reshape(-1, 512)
        assert np.array_equal(rec, direct)
        assert np.array_equal(oracle.assemble(feats, s.nodes), direct)


def test_assemble_tiers_rejects_unresolvable_address():
    with pytest.raises(oracle.OracleError) as e:
        oracle.assemble_tiers(np.array([(2 << 30) | 5], np.uint32), np.zeros(0, np.uint8),
                              np.zeros(0, np.uint8), np.zeros(512, np.uint8), 512)
    assert e.value.code == 2


def test_tiny_config_shape_matches_survey():
    """Sanity: the tiny config yields ~75% of N per batch and tier boundaries inside count ties."""
    w = make_workload("tiny", features=False)
    S = oracle.sample(w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy(), 256, [10, 5], 0x5EED)
    assert len(S) == 8
    n = np.mean([len(s.nodes) for s in S])
    assert 6000 < n < 9000
    c = oracle.count_frequencies(S, 10_000)
    tm, gpu, host = oracle.select_tiers(c, 500, 1000)
    assert c[gpu].min() == c[gpu].max() or len(set(c[gpu].tolist())) <= 3
