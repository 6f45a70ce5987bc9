"""CPU oracle for the DiskGNN offline hot path -- TEST INFRASTRUCTURE ONLY.

This package is the parity oracle: a plain, slow, obviously correct CPU
implementation of what the path computes, written from the paper
(``/root/reference/PAPER.md``, cited as ``P:n``) and the readings listed in
DESIGN.md.  It shares no code with ``paper_2405_05231_b200`` and neither
imports the other.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may use it.

The arithmetic lives in ``dgnn_oracle.c`` (plain C, compiled with gcc); this
module only marshals numpy arrays through ctypes.

Functions and the passage each follows:

* ``philox4x32_10``, ``draw64``, ``floyd``  -- the RNG and subset draw
  (readings c5-c8; Salmon et al. SC'11; Bentley & Floyd 1987).
* ``sample``            -- node-wise K-hop sampling, P:205 / S:50-62.
* ``count_frequencies`` -- P:271.
* ``select_tiers``      -- P:226.
* ``classify``          -- address tables.
* ``chunk_offsets``, ``pack`` -- batched packing.
* ``gather_rows``       -- tier buffers and direct-gather assembly.
* ``assemble_tiers``    -- three-source reconstruction.
* ``disk_space``, ``disk_search``, ``disk_perm``, ``disk_plan``,
  ``disk_cache_fill``   -- segmented disk cache, Eq. 2 and Algorithm 1,
  P:311-414 (readings d1-d8 in dgnn_oracle.c and DESIGN.md).
* ``train_stub``        -- the trainer's surrogate of Eq. 1, reading t1.
* ``pack_pages``        -- source pages read by individual vs batched packing (Fig. 6).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dgnn_oracle.c")
_LIB = os.path.join(_HERE, "libdgnn_oracle.so")
_lock = threading.Lock()
_lib = None

TIER_GPU, TIER_HOST, TIER_DISK = 0, 1, 2
TIER_SHIFT = 30
SLOT_MASK = (1 << TIER_SHIFT) - 1


def build(force: bool = False) -> str:
    """Compile dgnn_oracle.c into libdgnn_oracle.so (gcc, OpenMP across batches)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Batch(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("num_hops", ctypes.c_int32),
        ("num_nodes", ctypes.c_int64),
        ("nodes", ctypes.POINTER(ctypes.c_int32)),
        ("hop_off", ctypes.POINTER(ctypes.c_int32)),
        ("num_edges", ctypes.c_int64),
        ("eptr", ctypes.POINTER(ctypes.c_int32)),
        ("src_local", ctypes.POINTER(ctypes.c_int32)),
    ]


def _L():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i64, i32, u64, u32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint32
            lib.oracle_philox4x32_10.argtypes = [P, P, P]
            lib.oracle_draw64.argtypes = [u64, u32, u64, u32, u32]
            lib.oracle_draw64.restype = u64
            lib.oracle_floyd.argtypes = [i64, i32, u64, u32, u64, u32, P]
            lib.oracle_floyd_core.argtypes = [i64, i32, P, P]
            lib.oracle_sample_range.argtypes = [P, P, i64, P, i64, i32, i64, P, i32, u64, i64, i64, i32, P, i32]
            lib.oracle_sample_range.restype = ctypes.c_int
            lib.oracle_batch_free.argtypes = [ctypes.POINTER(_Batch)]
            lib.oracle_count_add.argtypes = [P, i64, P]
            lib.oracle_select_tiers.argtypes = [P, i64, i64, i64, P, P, P, P, P]
            lib.oracle_select_tiers.restype = ctypes.c_int
            lib.oracle_classify.argtypes = [P, i64, P, P, P]
            lib.oracle_classify.restype = i64
            lib.oracle_chunk_offsets.argtypes = [P, i64, i64, P]
            lib.oracle_pack.argtypes = [P, i64, P, P, i64, P, P]
            lib.oracle_gather_rows.argtypes = [P, i64, P, i64, P]
            lib.oracle_assemble_tiers.argtypes = [P, i64, P, i64, P, i64, P, i64, i64, P]
            lib.oracle_assemble_tiers.restype = ctypes.c_int
            lib.oracle_disk_space.argtypes = [P, P, i64, i64, i64, i64, i64, P]
            lib.oracle_disk_search.argtypes = [P, P, i64, i64, i64, i64, i64, P, P]
            lib.oracle_disk_perm.argtypes = [u64, i64, i64, i64, P]
            lib.oracle_disk_plan.argtypes = [P, P, i64, i64, i64, i64, i64, i32, u64, i32,
                                             P, P, P, P, P, P, P, P, P]
            lib.oracle_disk_cache_fill.argtypes = [P, i64, P, P, P, i64, P]
            lib.oracle_train_stub.argtypes = [P, i64, i64, P, i32, P, P, i32]
            lib.oracle_train_stub.restype = ctypes.c_int
            lib.oracle_pack_pages.argtypes = [P, P, i64, i64, i64, i64, P, P]
            lib.oracle_pack_pages.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


# ---------------------------------------------------------------- RNG ----
def philox4x32_10(ctr, key):
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _L().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return tuple(int(x) for x in out)


def draw64(rng_seed: int, v: int, bid: int, h: int, s: int) -> int:
    return int(_L().oracle_draw64(rng_seed, v, bid, h, s))


def floyd(d: int, k: int, rng_seed: int, v: int, bid: int, h: int) -> list:
    out = np.zeros(max(k, 1), np.int64)
    _L().oracle_floyd(d, k, rng_seed, v, bid, h, _p(out))
    return [int(x) for x in out[:k]]


def floyd_core(d: int, k: int, draws) -> list:
    """Floyd's subset map for explicit draws t[s] in [0, d-k+s] (exhaustive tests)."""
    t = _c(draws, np.int64)
    out = np.zeros(max(k, 1), np.int64)
    _L().oracle_floyd_core(d, k, _p(t), _p(out))
    return [int(x) for x in out[:k]]


# ------------------------------------------------------------ sampling ----
@dataclass
class Sample:
    """One graph sample: nodes = seeds then per-hop new nodes."""
    bid: int
    nodes: np.ndarray      # int32 [n]
    hop_off: np.ndarray    # int32 [H+2]
    eptr: np.ndarray       # int32 [hop_off[H]+1]; blocks: per hop h, hop_off[h+1]+1 entries, concatenated
    src_local: np.ndarray  # int32 [num_edges]
    blocks: bool = False   # the DGL-block variant (reading c27)


def num_batches(num_seeds: int, batch_size: int) -> int:
    return (num_seeds + batch_size - 1) // batch_size


def sample(indptr, indices, seeds, batch_size: int, fanout, rng_seed: int,
           batch_id_base: int = 0, batches=None, threads: int = 1, blocks: bool = False) -> list:
    """Sample batches t (default: all ceil(S/B)); returns a list of Sample.

    ``blocks``: the DGL-block variant (reading c27): every node of the sample so far is
    resampled at each hop, and each hop has its own eptr array.

    ``batches`` may be a range/list of batch ordinals t to sample (each keyed
    by bid = batch_id_base + t); they are processed as contiguous runs.
    """
    indptr = _c(indptr, np.int64)
    indices = _c(indices, np.int32)
    seeds = _c(seeds, np.int32)
    fan = _c(fanout, np.int32)
    nb = num_batches(len(seeds), batch_size)
    ts = list(range(nb)) if batches is None else [int(t) for t in batches]
    L = _L()
    out = []
    i = 0
    while i < len(ts):
        j = i
        while j + 1 < len(ts) and ts[j + 1] == ts[j] + 1:
            j += 1
        t_lo, t_hi = ts[i], ts[j] + 1
        arr = (ctypes.POINTER(_Batch) * (t_hi - t_lo))()
        rc = L.oracle_sample_range(_p(indptr), _p(indices), len(indptr) - 1, _p(seeds), len(seeds),
                                   batch_size, batch_id_base, _p(fan), len(fan), rng_seed, t_lo, t_hi,
                                   threads, ctypes.cast(arr, ctypes.c_void_p), int(bool(blocks)))
        try:
            if rc != 0:
                raise OracleError(rc, "sample")
            for t in range(t_lo, t_hi):
                b = arr[t - t_lo].contents
                H = b.num_hops
                n = b.num_nodes
                hop = np.ctypeslib.as_array(b.hop_off, (H + 2,)).copy()
                n_eptr = int(sum(int(hop[h + 1]) + 1 for h in range(H))) if blocks else int(hop[H]) + 1
                out.append(Sample(
                    bid=batch_id_base + t,
                    nodes=np.ctypeslib.as_array(b.nodes, (n,)).copy() if n else np.zeros(0, np.int32),
                    hop_off=hop,
                    eptr=np.ctypeslib.as_array(b.eptr, (n_eptr,)).copy(),
                    src_local=(np.ctypeslib.as_array(b.src_local, (b.num_edges,)).copy()
                               if b.num_edges else np.zeros(0, np.int32)),
                    blocks=bool(blocks),
                ))
        finally:
            for t in range(t_lo, t_hi):
                if arr[t - t_lo]:
                    L.oracle_batch_free(arr[t - t_lo])
        i = j + 1
    return out


def count_frequencies(samples, num_nodes: int, counts=None) -> np.ndarray:
    """counts[v] = number of batches whose node set contains v."""
    c = np.zeros(num_nodes, np.uint32) if counts is None else counts
    for s in samples:
        nodes = _c(s.nodes, np.int32)
        _L().oracle_count_add(_p(nodes), len(nodes), _p(c))
    return c


def select_tiers(counts, gpu_rows: int, host_rows: int):
    """Rank by (count desc, ID asc), zero counts never cached.

    Returns (tier_map uint32[N], gpu_ids int32[K_g], host_ids int32[K_h]).
    """
    counts = _c(counts, np.uint32)
    N = len(counts)
    tier_map = np.zeros(N, np.uint32)
    g = np.zeros(max(min(gpu_rows, N), 1), np.int32)
    h = np.zeros(max(min(host_rows, N), 1), np.int32)
    kg = np.zeros(1, np.int64)
    kh = np.zeros(1, np.int64)
    rc = _L().oracle_select_tiers(_p(counts), N, gpu_rows, host_rows, _p(tier_map), _p(g), _p(h),
                                  _p(kg), _p(kh))
    if rc != 0:
        raise OracleError(rc, "select_tiers")
    return tier_map, g[: int(kg[0])].copy(), h[: int(kh[0])].copy()


def classify(nodes, tier_map):
    """Address table of one batch: returns (addr uint32[n], P int32[p])."""
    nodes = _c(nodes, np.int32)
    tier_map = _c(tier_map, np.uint32)
    addr = np.zeros(len(nodes), np.uint32)
    packed = np.zeros(max(len(nodes), 1), np.int32)
    p = _L().oracle_classify(_p(nodes), len(nodes), _p(tier_map), _p(addr), _p(packed))
    return addr, packed[:p].copy()


def chunk_offsets(packed_rows, row_bytes: int) -> np.ndarray:
    pr = _c(packed_rows, np.int64)
    off = np.zeros(len(pr) + 1, np.int64)
    _L().oracle_chunk_offsets(_p(pr), len(pr), row_bytes, _p(off))
    return off


def _rows_u8(features) -> np.ndarray:
    f = np.ascontiguousarray(features)
    return f.reshape(f.shape[0], -1).view(np.uint8)


def pack(features, packed_lists):
    """Batched packing of one group: returns (group_buf uint8, chunk_off int64[nb+1])."""
    f = _rows_u8(features)
    row_bytes = f.shape[1]
    rows = np.array([len(p) for p in packed_lists], np.int64)
    cat = _c(np.concatenate([np.asarray(p, np.int32) for p in packed_lists]) if len(packed_lists)
             else np.zeros(0, np.int32), np.int32)
    off = chunk_offsets(rows, row_bytes)
    buf = np.zeros(int(off[-1]), np.uint8)
    _L().oracle_pack(_p(f), row_bytes, _p(cat), _p(rows), len(rows), _p(off), _p(buf))
    return buf, off


def pack_embedded(features, packed_lists, samples):
    """Batched packing with the graph sample kept in each chunk (Sec. 4: "the graph sample
    of the mini-batch is also kept in the chunk"; byte layout = reading c22b of DESIGN.md):
    chunk i = its |P_i| rows (as ``pack``), then at roundup(|P_i| * row_bytes, 16) the int32 words
    H, n_i, m_i, e_i, hop_off[H+2], nodes[n_i], eptr[m_i], src_local[e_i], then zeros up to a
    4096-byte boundary.  Returns (group_buf uint8, chunk_off int64[nb+1], sec_off int64[nb])."""
    f = _rows_u8(features)
    row_bytes = f.shape[1]
    chunks, off, sec = [], [0], []
    for p, s in zip(packed_lists, samples):
        rows = gather_rows(f, np.asarray(p, np.int32)).reshape(-1)
        H = len(s.hop_off) - 2
        words = np.concatenate([np.array([H, len(s.nodes), len(s.eptr), len(s.src_local)], np.int64),
                                np.asarray(s.hop_off, np.int64), np.asarray(s.nodes, np.int64),
                                np.asarray(s.eptr, np.int64), np.asarray(s.src_local, np.int64)])
        sec_bytes = words.astype("<i4").view(np.uint8)
        a = (len(rows) + 15) // 16 * 16
        size = (a + len(sec_bytes) + 4095) // 4096 * 4096
        chunk = np.zeros(size, np.uint8)
        chunk[:len(rows)] = rows
        chunk[a:a + len(sec_bytes)] = sec_bytes
        chunks.append(chunk)
        sec.append(off[-1] + a)
        off.append(off[-1] + size)
    buf = np.concatenate(chunks) if chunks else np.zeros(0, np.uint8)
    return buf, np.array(off, np.int64), np.array(sec, np.int64)


def gather_rows(features, ids) -> np.ndarray:
    """out[s] = features[ids[s]] as raw bytes (row_bytes per row)."""
    f = _rows_u8(features)
    ids = _c(ids, np.int32)
    out = np.zeros((len(ids), f.shape[1]), np.uint8)
    _L().oracle_gather_rows(_p(f), f.shape[1], _p(ids), len(ids), _p(out))
    return out


def assemble(features, nodes) -> np.ndarray:
    """Direct-gather assembly: out[j] = features[nodes[j]]."""
    return gather_rows(features, nodes)


def assemble_tiers(addr, gpu_buf, host_buf, chunk, row_bytes: int) -> np.ndarray:
    """Three-source reconstruction from the address table."""
    addr = _c(addr, np.uint32)
    g = np.ascontiguousarray(gpu_buf, np.uint8).reshape(-1)
    h = np.ascontiguousarray(host_buf, np.uint8).reshape(-1)
    c = np.ascontiguousarray(chunk, np.uint8).reshape(-1)
    out = np.zeros((len(addr), row_bytes), np.uint8)
    rc = _L().oracle_assemble_tiers(_p(addr), len(addr), _p(g), len(g) // row_bytes, _p(h),
                                    len(h) // row_bytes, _p(c), len(c) // row_bytes, row_bytes, _p(out))
    if rc != 0:
        raise OracleError(rc, "assemble_tiers")
    return out


def offline_layout(indptr, indices, features, seeds, batch_size, fanout, rng_seed, gpu_rows, host_rows,
                   group_size, batch_id_base=0, threads=1):
    """The whole offline pass of the oracle, in the paper's order (P:508-511 analogue).

    Returns a dict with samples, counts, tiers, per-batch addr/P, packed groups,
    tier buffers.  Small configurations only (everything is held in memory).
    """
    samples = sample(indptr, indices, seeds, batch_size, fanout, rng_seed, batch_id_base, threads=threads)
    N = len(indptr) - 1
    counts = count_frequencies(samples, N)
    tier_map, gpu_ids, host_ids = select_tiers(counts, gpu_rows, host_rows)
    addrs, plists = [], []
    for s in samples:
        a, p = classify(s.nodes, tier_map)
        addrs.append(a)
        plists.append(p)
    groups = []
    for g0 in range(0, len(samples), group_size):
        groups.append(pack(features, plists[g0:g0 + group_size]))
    return dict(samples=samples, counts=counts, tier_map=tier_map, gpu_ids=gpu_ids, host_ids=host_ids,
                addr=addrs, packed=plists, groups=groups,
                gpu_buf=gather_rows(features, gpu_ids), host_buf=gather_rows(features, host_ids))


# ------------------------------------------------- segmented disk cache ----
PAGE = 4096


def _packed_concat(packed_lists):
    rows = np.array([len(p) for p in packed_lists], np.int64)
    off = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(rows, out=off[1:])
    cat = (np.concatenate([np.asarray(p, np.int32) for p in packed_lists]) if len(packed_lists)
           else np.zeros(0, np.int32))
    return _c(cat, np.int32), off


def disk_space(packed_lists, num_nodes: int, row_bytes: int, s: int, m: int) -> int:
    """Eq. 2 space of (s, m) in 4096-byte pages (readings d1-d3)."""
    cat, off = _packed_concat(packed_lists)
    out = np.zeros(1, np.int64)
    rc = _L().oracle_disk_space(_p(cat), _p(off), len(off) - 1, num_nodes, row_bytes, s, m, _p(out))
    if rc != 0:
        raise OracleError(rc, "disk_space")
    return int(out[0])


def disk_search(packed_lists, num_nodes: int, row_bytes: int, budget_pages: int, m: int = 1):
    """Heuristic of P:410-413: (minimum s with space <= budget or 0, its space)."""
    cat, off = _packed_concat(packed_lists)
    s_out = np.zeros(1, np.int64)
    pg = np.zeros(1, np.int64)
    rc = _L().oracle_disk_search(_p(cat), _p(off), len(off) - 1, num_nodes, row_bytes, m, budget_pages,
                                 _p(s_out), _p(pg))
    if rc != 0:
        raise OracleError(rc, "disk_search")
    return int(s_out[0]), int(pg[0])


def disk_perm(seed: int, g: int, t: int, n: int) -> np.ndarray:
    """Permutation H_t of the n local batch indices of segment g (reading d5)."""
    H = np.zeros(max(n, 1), np.int64)
    rc = _L().oracle_disk_perm(seed, g, t, n, _p(H))
    if rc != 0:
        raise OracleError(rc, "disk_perm")
    return H[:n].copy()


@dataclass
class DiskPlan:
    s: int
    m: int
    seg_off: np.ndarray        # int64 [nseg+1]
    cache_ids: np.ndarray      # int32 [seg_off[-1]] (V_r of every segment)
    seg_page_off: np.ndarray   # int64 [nseg+1]
    pk_ids: np.ndarray         # int32 (P_b' concatenated)
    pk_off: np.ndarray         # int64 [nb+1]
    req_pages: np.ndarray      # int64 (merged page requests)
    req_off: np.ndarray        # int64 [nb+1]
    dc_addr: np.ndarray        # uint32 [R] (reading d8)
    space_pages: int
    io_pages: int
    cache_pages: int
    chunk_pages: int


def disk_plan(packed_lists, num_nodes: int, row_bytes: int, s: int, m: int, k: int = 4, seed: int = 0,
              reorder: bool = True, literal: bool = False) -> DiskPlan:
    """Segments, V_d, Algorithm 1 order, P_b', merged requests (d1-d8).

    ``literal``: Algorithm 1 line 8 as printed: one scalar MinHash value per node,
    the minimum over the k hash functions, instead of reading d6's per-function signature."""
    cat, off = _packed_concat(packed_lists)
    nb = len(off) - 1
    R = int(off[-1])
    nseg = (nb + s - 1) // s if s >= 1 else 0
    cap = max(R, 1)
    seg_off = np.zeros(nseg + 1, np.int64)
    seg_page_off = np.zeros(nseg + 1, np.int64)
    cache_ids = np.zeros(cap, np.int32)
    pk_ids = np.zeros(cap, np.int32)
    pk_off = np.zeros(nb + 1, np.int64)
    req_pages = np.zeros(cap, np.int64)
    req_off = np.zeros(nb + 1, np.int64)
    dc_addr = np.zeros(cap, np.uint32)
    tot = np.zeros(4, np.int64)
    rc = _L().oracle_disk_plan(_p(cat), _p(off), nb, num_nodes, row_bytes, s, m, k, seed,
                               (2 if literal else 1) if reorder else 0,
                               _p(seg_off), _p(cache_ids), _p(seg_page_off), _p(pk_ids), _p(pk_off),
                               _p(req_pages), _p(req_off), _p(dc_addr), _p(tot))
    if rc != 0:
        raise OracleError(rc, "disk_plan")
    return DiskPlan(s=s, m=m, seg_off=seg_off, cache_ids=cache_ids[: seg_off[-1]].copy(),
                    seg_page_off=seg_page_off, pk_ids=pk_ids[: pk_off[-1]].copy(), pk_off=pk_off,
                    req_pages=req_pages[: req_off[-1]].copy(), req_off=req_off, dc_addr=dc_addr[:R].copy(),
                    space_pages=int(tot[0]), io_pages=int(tot[1]), cache_pages=int(tot[2]),
                    chunk_pages=int(tot[3]))


def disk_cache_fill(features, plan: DiskPlan) -> np.ndarray:
    """The segment caches as bytes: V_r rows, fpp per 4096-byte page, zero tails."""
    f = _rows_u8(features)
    row_bytes = f.shape[1]
    nseg = len(plan.seg_off) - 1
    out = np.zeros(int(plan.seg_page_off[-1]) * PAGE, np.uint8)
    ids = _c(plan.cache_ids, np.int32)
    _L().oracle_disk_cache_fill(_p(f), row_bytes, _p(ids), _p(_c(plan.seg_off, np.int64)),
                                _p(_c(plan.seg_page_off, np.int64)), nseg, _p(out))
    return out


def disk_partial_input(chunk: np.ndarray, pages: np.ndarray, dc_addr_b: np.ndarray, row_bytes: int) -> np.ndarray:
    """Partial input of one batch: its DISK rows in local order, read from its
    packed chunk (dc_addr < 2^31: chunk row) or its fetched cache pages (d8)."""
    fpp = PAGE // row_bytes
    out = np.zeros((len(dc_addr_b), row_bytes), np.uint8)
    for r, a in enumerate(np.asarray(dc_addr_b, np.uint64)):
        a = int(a)
        if a >> 31:
            q, slot = divmod(a & 0x7FFFFFFF, fpp)
            out[r] = pages[q * PAGE + slot * row_bytes: q * PAGE + (slot + 1) * row_bytes]
        else:
            out[r] = chunk[a * row_bytes:(a + 1) * row_bytes]
    return out


# --------------------------------------------------------- trainer stub ----
def train_stub(sample: Sample, feats) -> np.ndarray:
    """Seed embeddings h^H of one batch (reading t1) from its assembled rows (fp32 [n, dim])."""
    x = np.array(feats, dtype=np.float32, copy=True, order="C").reshape(len(sample.nodes), -1)
    H = len(sample.hop_off) - 2
    hop = _c(sample.hop_off, np.int32)
    ep = _c(sample.eptr, np.int32)
    src = _c(sample.src_local, np.int32)
    rc = _L().oracle_train_stub(_p(x), x.shape[0], x.shape[1], _p(hop), H, _p(ep), _p(src),
                                int(bool(getattr(sample, "blocks", False))))
    if rc != 0:
        raise OracleError(rc, "train_stub")
    return x[: int(hop[1])].copy()


# ------------------------------------------------- packing page accounting ----
def pack_pages(packed_lists, num_nodes: int, row_bytes: int, part_rows: int):
    """(individual, batched) 4096-byte source pages read to pack ``packed_lists`` (Fig. 6)."""
    cat, off = _packed_concat(packed_lists)
    ind = np.zeros(1, np.int64)
    bat = np.zeros(1, np.int64)
    rc = _L().oracle_pack_pages(_p(cat), _p(off), len(off) - 1, num_nodes, row_bytes, part_rows, _p(ind), _p(bat))
    if rc != 0:
        raise OracleError(rc, "pack_pages")
    return int(ind[0]), int(bat[0])
