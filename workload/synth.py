"""Synthetic workloads shaped like the paper's datasets (inputs only).

Recipe:

* Out-degrees: ``uniform`` (every node E/N), ``lognormal`` (sigma=1) or
  ``pareto`` (alpha=2) weights w_v, d_v = floor(E * w_v / sum w) plus one
  extra edge for a seeded subset so sum d_v = E exactly; capped at N-1.
* Destinations: the bucketed popularity law of ``tab:access_skewness``
  (PAPER.md:543-546): the nodes are permuted by a seeded permutation pi and
  split into rank buckets [0,1%), [1,5%), [5,10%), [10,100%); each edge picks
  a bucket with the table's share, then a node uniformly inside it.
* Clean-up: self-loops and duplicate (row, dst) pairs are dropped, rows are
  sorted ascending; the realized E is what the CSR holds.
* Features: closed form f(v, j) = as_float(0x3F800000 | (fmix64((v*dim+j) ^
  fseed*0x9E3779B97F4A7C15) >> 41)) - 1.0f, an exact fp32 in [0, 1).
* Seeds: a seeded random sample of the node IDs, shuffled.

The graph is generated with torch's seeded generators on whichever device is
given; the output is deterministic per (config, seed, device type), which is
all the tests need: both the oracle and the CUDA path are fed the SAME arrays.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

# tab:access_skewness: share of accesses by node-rank bucket
SKEW = {
    "PS": (0.432, 0.365, 0.112, 0.091),
    "FS": (0.141, 0.255, 0.182, 0.421),
    "MG": (0.564, 0.323, 0.073, 0.040),
    "IG": (0.225, 0.300, 0.208, 0.267),
}
BUCKET_EDGES = (0.0, 0.01, 0.05, 0.10, 1.0)

CONFIGS = {
    # BASELINE.json configs[0]: the parity case the oracle finishes in seconds
    "tiny": dict(num_nodes=10_000, num_edges=100_000, degree="uniform", skew=None, dim=128,
                 fanout=(10, 5), batch_size=256, num_seeds=2048, group_size=8,
                 gpu_frac=0.05, host_frac=0.10),
    # configs[1]
    "products": dict(num_nodes=2_400_000, num_edges=62_000_000, degree="lognormal", skew="PS", dim=100,
                     fanout=(15, 10, 5), batch_size=1024, num_seeds=196_615, group_size=0,
                     gpu_frac=0.05, host_frac=0.10),
    # configs[2]: the north_star's scaling workload
    "papers": dict(num_nodes=111_000_000, num_edges=1_600_000_000, degree="lognormal", skew="PS", dim=128,
                   fanout=(10, 10, 10), batch_size=1024, num_seeds=1_200_000, group_size=0,
                   gpu_frac=0.05, host_frac=0.10),
    # configs[3]
    "friendster": dict(num_nodes=65_600_000, num_edges=1_800_000_000, degree="pareto", skew="FS", dim=256,
                       fanout=(10, 10, 10), batch_size=1024, num_seeds=656_000, group_size=0,
                       gpu_frac=0.05, host_frac=0.10),
    # configs[4] (features exceed one GPU: needs the sharded tier, not run at N=1)
    "igb": dict(num_nodes=100_000_000, num_edges=1_200_000_000, degree="lognormal", skew="IG", dim=1024,
                fanout=(10, 10, 10), batch_size=1024, num_seeds=1_000_000, group_size=0,
                gpu_frac=0.05, host_frac=0.10),
}

M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """uint64 constant -> the int64 with the same bits (torch has no uint64 math)."""
    x &= M64
    return x - (1 << 64) if x >= (1 << 63) else x


_FM1 = _s64(0xFF51AFD7ED558CCD)
_FM2 = _s64(0xC4CEB9FE1A85EC53)
_GOLD = 0x9E3779B97F4A7C15


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bits."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def _fmix64_t(h: torch.Tensor) -> torch.Tensor:
    h = h ^ _lsr(h, 33)
    h = h * _FM1
    h = h ^ _lsr(h, 33)
    h = h * _FM2
    h = h ^ _lsr(h, 33)
    return h


def feature_rows(ids: torch.Tensor, dim: int, fseed: int = 1) -> torch.Tensor:
    """Closed-form fp32 feature rows f(v, j) for node IDs ``ids`` (any device)."""
    ids = ids.to(torch.int64)
    j = torch.arange(dim, device=ids.device, dtype=torch.int64)
    x = ids[:, None] * dim + j[None, :]
    x = x ^ _s64(fseed * _GOLD)
    h = _fmix64_t(x)
    bits = (_lsr(h, 41) | 0x3F800000).to(torch.int32)
    return bits.view(torch.float32) - 1.0


def feature_rows_np(ids, dim: int, fseed: int = 1) -> np.ndarray:
    """The same closed form in numpy uint64 (an independent transcription for checks)."""
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = ids[:, None] * np.uint64(dim) + np.arange(dim, dtype=np.uint64)[None, :]
        x ^= np.uint64((fseed * _GOLD) & M64)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xFF51AFD7ED558CCD)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xC4CEB9FE1A85EC53)
        x ^= x >> np.uint64(33)
    bits = ((x >> np.uint64(41)) | np.uint64(0x3F800000)).astype(np.uint32)
    return bits.view(np.float32) - np.float32(1.0)


def make_features(num_nodes: int, dim: int, device, fseed: int = 1, out: torch.Tensor | None = None,
                  chunk_rows: int = 1 << 22) -> torch.Tensor:
    """Materialize the whole [N, dim] fp32 table (chunked)."""
    if out is None:
        out = torch.empty((num_nodes, dim), dtype=torch.float32, device=device)
    for r0 in range(0, num_nodes, chunk_rows):
        r1 = min(num_nodes, r0 + chunk_rows)
        ids = torch.arange(r0, r1, device=out.device, dtype=torch.int64)
        out[r0:r1] = feature_rows(ids, dim, fseed).to(out.device)
    return out


def _degrees(N: int, E: int, law: str, gen: torch.Generator, device) -> torch.Tensor:
    if law == "uniform":
        d = torch.full((N,), E // N, dtype=torch.int64, device=device)
        rem = E - int(d.sum())
    else:
        if law == "lognormal":
            w = torch.exp(torch.randn(N, generator=gen, device=device, dtype=torch.float64))
        elif law == "pareto":
            u = torch.rand(N, generator=gen, device=device, dtype=torch.float64).clamp_min(1e-12)
            w = u.pow(-1.0 / 2.0)  # alpha = 2
        else:
            raise ValueError(law)
        d = torch.floor(w * (E / float(w.sum()))).to(torch.int64)
        rem = E - int(d.sum())
    if rem > 0:
        extra = torch.randperm(N, generator=gen, device=device)[:rem]
        d[extra] += 1
    return d.clamp_(max=max(N - 1, 0))


def make_graph(num_nodes: int, num_edges: int, degree: str = "uniform", skew: str | None = None,
               seed: int = 0, device="cpu", chunk_nodes: int = 1 << 22):
    """CSR (indptr int64 [N+1], indices int32 [E']) on ``device``; see module doc."""
    N, E = int(num_nodes), int(num_edges)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 1000003 + 17)
    deg = _degrees(N, E, degree, gen, device)
    perm = torch.randperm(N, generator=gen, device=device) if skew else None
    if skew:
        shares = torch.tensor(SKEW[skew], dtype=torch.float64, device=device)
        cum = torch.cumsum(shares, 0)
        cum[-1] = 1.0
        bounds = [int(round(b * N)) for b in BUCKET_EDGES]
        lo = torch.tensor(bounds[:-1], dtype=torch.int64, device=device)
        size = torch.tensor([max(bounds[i + 1] - bounds[i], 1) for i in range(4)], dtype=torch.int64,
                            device=device)
    rows_out, cols_out, counts = [], [], torch.zeros(N, dtype=torch.int64, device=device)
    for v0 in range(0, N, chunk_nodes):
        v1 = min(N, v0 + chunk_nodes)
        d = deg[v0:v1]
        m = int(d.sum())
        if m == 0:
            continue
        row = torch.repeat_interleave(torch.arange(v0, v1, device=device, dtype=torch.int64), d)
        if skew:
            u = torch.rand(m, generator=gen, device=device, dtype=torch.float64)
            b = torch.searchsorted(cum, u, right=True).clamp_(max=3)
            r = torch.rand(m, generator=gen, device=device, dtype=torch.float64)
            pos = lo[b] + torch.minimum((r * size[b].to(torch.float64)).to(torch.int64), size[b] - 1)
            dst = perm[pos.clamp_(max=N - 1)]
        else:
            dst = torch.randint(0, N, (m,), generator=gen, device=device, dtype=torch.int64)
        keep = dst != row
        key = torch.unique(row[keep] * N + dst[keep])  # sorted, de-duplicated (row, dst)
        r_ = key // N
        rows_out.append(r_)
        cols_out.append((key - r_ * N).to(torch.int32))
    if rows_out:
        rows = torch.cat(rows_out)
        indices = torch.cat(cols_out)
        counts = torch.bincount(rows, minlength=N)
    else:
        indices = torch.zeros(0, dtype=torch.int32, device=device)
    indptr = torch.zeros(N + 1, dtype=torch.int64, device=device)
    indptr[1:] = torch.cumsum(counts, 0)
    return indptr, indices


def make_seeds(num_nodes: int, num_seeds: int, seed: int = 0, device="cpu") -> torch.Tensor:
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 7919 + 5)
    return torch.randperm(num_nodes, generator=gen, device=device)[:num_seeds].to(torch.int32)


def config_rows(cfg: dict) -> tuple:
    """GPU / host tier capacities in rows: floor(frac * N) (reading c16)."""
    N = cfg["num_nodes"]
    return int(cfg["gpu_frac"] * N), int(cfg["host_frac"] * N)


@dataclass
class Workload:
    name: str
    cfg: dict
    indptr: torch.Tensor
    indices: torch.Tensor
    seeds: torch.Tensor
    features: torch.Tensor | None
    seed: int = 0
    fseed: int = 1
    extra: dict = field(default_factory=dict)

    @property
    def num_nodes(self) -> int:
        return int(self.indptr.numel() - 1)

    @property
    def row_bytes(self) -> int:
        return int(self.cfg["dim"]) * 4


def make_workload(name: str, device="cpu", seed: int = 0, fseed: int = 1, features: bool = True,
                  **overrides) -> Workload:
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    indptr, indices = make_graph(cfg["num_nodes"], cfg["num_edges"], cfg["degree"], cfg["skew"], seed,
                                 device)
    seeds = make_seeds(cfg["num_nodes"], cfg["num_seeds"], seed, device)
    feats = make_features(cfg["num_nodes"], cfg["dim"], device, fseed) if features else None
    return Workload(name, cfg, indptr, indices, seeds, feats, seed, fseed)


def make_packed_lists(nb: int, num_nodes: int, rows_per_batch: int, alpha: float = 2.0, seed: int = 0,
                      jitter: float = 0.25):
    """Seeded stand-in for an epoch's packed lists (the DISK rows of each batch) -- an INPUT
    for the segmented-disk-cache parity tests, not a product of the method.

    Each batch draws about rows_per_batch node IDs as floor(N * u**alpha) through a seeded
    permutation (alpha > 1: a few IDs are popular, as the cold tail of a sampled epoch),
    drops duplicates and keeps them in a shuffled local order.  Returns (ids int32 [R],
    off int64 [nb+1]).
    """
    rng = np.random.default_rng(seed)
    perm = rng.permutation(num_nodes).astype(np.int32)
    parts, off = [], np.zeros(nb + 1, np.int64)
    for b in range(nb):
        n = max(0, int(rows_per_batch * (1.0 + jitter * (2.0 * rng.random() - 1.0))))
        raw = np.minimum((num_nodes * rng.random(n) ** alpha).astype(np.int64), num_nodes - 1)
        ids = perm[np.unique(raw)]
        rng.shuffle(ids)
        parts.append(ids)
        off[b + 1] = off[b] + len(ids)
    ids = np.concatenate(parts) if parts else np.zeros(0, np.int32)
    return ids.astype(np.int32), off
