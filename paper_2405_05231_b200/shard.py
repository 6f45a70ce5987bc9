"""Sharded GPU tier (north_star "the GPU feature cache is partitioned
across the GPUs' HBM, and remote rows are fetched with NCCL all-to-all over NVLink").

When the GPU tier does not fit replicated (IGB-shaped features, or forced), slot s of the
tier lives on rank s % world at local row s // world.  Assembling a run of batches then
needs, per rank, the GPU-tier rows other ranks own:

    1. dgnn_shard_requests    -> requests grouped by owner (owner-local rows + out positions)
    2. all_to_all  (counts)   -> how many rows every peer asks of me
    3. all_to_all  (rows ids) -> the local rows every peer asks of me
    4. dgnn_gather_rows       -> I gather them from my shard (HBM)
    5. all_to_all  (rows)     -> the rows travel back over NVLink
    6. dgnn_scatter_rows      -> they land at their positions in the output
    and dgnn_assemble_group_sharded fills every other row locally.

The collective choreography (steps 2-5) is ``exchange_remote_rows``; it is written against
three small local callbacks so that the same code drives the CUDA kernels with NCCL in
production and plain numpy with gloo in the CPU test of the protocol.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _abi as A


def shard_of(slot: int, world: int):
    """(owner rank, owner-local row) of a GPU-tier slot."""
    return slot % world, slot // world


class ShardedTier:
    """This rank's shard of the GPU tier, gathered from the features (a7 "special mini-batch")."""

    def __init__(self, ctx: A.Ctx, features: torch.Tensor, plan: A.CachePlan, rank: int, world: int):
        self.ctx, self.rank, self.world = ctx, rank, world
        self.k_gpu = plan.k_gpu
        self.row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
        ids = A.dgnn_tier_shard_ids(ctx, plan.gpu_ids, plan.k_gpu, rank, world)
        with torch.cuda.stream(ctx.stream):
            self.rows = torch.empty((ids.numel(), self.row_bytes), dtype=torch.uint8, device=ctx.device)
        A.dgnn_gather_rows(ctx, features, ids, self.rows)


def exchange_remote_rows(send_counts: np.ndarray, req_rows, serve, all_to_all, world: int, row_bytes: int):
    """Steps 2-5.  ``send_counts[o]``: rows I request from owner o (grouped in ``req_rows``);
    ``serve(ids)``: my shard's rows for the ids peers sent me; ``all_to_all(x, send_splits,
    recv_splits)``: the process group's all-to-all on a flat tensor.  Returns the requested
    rows grouped by owner, in request order."""
    recv_counts = all_to_all(torch.as_tensor(send_counts, dtype=torch.int64), [1] * world, [1] * world)
    recv_counts = [int(x) for x in recv_counts.cpu().tolist()]
    send_counts = [int(x) for x in send_counts]
    asked = all_to_all(req_rows, send_counts, recv_counts)           # ids peers want from my shard
    served = serve(asked)                                            # [sum(recv_counts), row_bytes] uint8
    back = all_to_all(served.reshape(-1), [c * row_bytes for c in recv_counts],
                      [c * row_bytes for c in send_counts])
    return back


def nccl_all_to_all(group=None):
    import torch.distributed as dist

    def a2a(x: torch.Tensor, send_splits, recv_splits):
        out = torch.empty(sum(recv_splits), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x.contiguous(), output_split_sizes=list(recv_splits),
                               input_split_sizes=list(send_splits), group=group)
        return out
    return a2a


def fetch_remote_rows(ctx: A.Ctx, tier: ShardedTier, addr: torch.Tensor, out: torch.Tensor, all_to_all):
    """Deliver the remote GPU-tier rows of one run into ``out`` (collective: every rank calls it
    once per run, in the same order)."""
    off, req_slot, req_pos = A.dgnn_shard_requests(ctx, addr, tier.k_gpu, tier.rank, tier.world)

    def serve(ids: torch.Tensor) -> torch.Tensor:
        with torch.cuda.stream(ctx.stream):
            rows = torch.empty((ids.numel(), tier.row_bytes), dtype=torch.uint8, device=ctx.device)
        A.dgnn_gather_rows(ctx, tier.rows, ids.to(torch.int32), rows)
        return rows

    with torch.cuda.stream(ctx.stream):
        back = exchange_remote_rows(np.diff(off), req_slot, serve, all_to_all, tier.world, tier.row_bytes)
    if int(off[-1]):  # (an empty call only serves the peers' requests)
        A.dgnn_scatter_rows(ctx, back, int(off[-1]), tier.row_bytes, req_pos, out)


def fetch_remote_rows_loopback(ctx: A.Ctx, tiers: list, rank: int, addr: torch.Tensor, out: torch.Tensor):
    """Single-process stand-in for the exchange (all shards local): owner o answers rank
    ``rank``'s requests directly from its shard.  Used to test the kernels on one GPU."""
    t = tiers[rank]
    off, req_slot, req_pos = A.dgnn_shard_requests(ctx, addr, t.k_gpu, rank, t.world)
    for o in range(t.world):
        n = int(off[o + 1] - off[o])
        if o == rank or n == 0:
            continue
        with torch.cuda.stream(ctx.stream):
            rows = torch.empty((n, t.row_bytes), dtype=torch.uint8, device=ctx.device)
        A.dgnn_gather_rows(ctx, tiers[o].rows, req_slot[int(off[o]):int(off[o + 1])], rows)
        A.dgnn_scatter_rows(ctx, rows, n, t.row_bytes, req_pos[int(off[o]):int(off[o + 1])], out)


class PeerTier:
    """The sharded GPU tier read one-sided through peer memory.

    Each rank fills its shard (slot s on rank s % world at row s // world) in a plain device
    allocation, exports its CUDA IPC handle, and maps every other rank's shard; the assembly
    kernel (dgnn_assemble_group_peer) then loads a remote GPU-tier row straight from its
    owner's HBM over NVLink / NVSwitch.  The request / all-to-all / scatter round of
    ``exchange_remote_rows`` disappears into the gather: one kernel, no collective on the
    data path after the one-time handle exchange.

    ``exchange(handle_bytes) -> [handle of rank 0, ..., rank world-1]`` is the process
    group's all-gather of the 64-byte handles (``all_gather_handles``).
    """

    def __init__(self, ctx: A.Ctx, features: torch.Tensor, plan: A.CachePlan, rank: int, world: int, exchange):
        self.ctx, self.rank, self.world, self.k_gpu = ctx, rank, world, plan.k_gpu
        self.row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
        dev = ctx.device.index if ctx.device.index is not None else 0
        self.shard = _fill_shard(ctx, features, plan, rank, world, self.row_bytes)
        ctx.sync()  # the shard is complete before anyone maps it
        handles = exchange(self.shard.ipc_handle())
        self.maps, ptrs = [], []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(self.shard.ptr)
            else:
                m = A.IpcMapping(dev, h)
                self.maps.append(m)
                ptrs.append(m.ptr)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=ctx.device)

    @classmethod
    def loopback(cls, ctx: A.Ctx, features: torch.Tensor, plan: A.CachePlan, world: int):
        """All world shards in this process (the single-GPU test of the kernel path)."""
        self = cls.__new__(cls)
        self.ctx, self.rank, self.world, self.k_gpu = ctx, 0, world, plan.k_gpu
        self.row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
        self.shards = [_fill_shard(ctx, features, plan, r, world, self.row_bytes) for r in range(world)]
        self.maps = []
        self.peers = torch.tensor([s.ptr for s in self.shards], dtype=torch.int64, device=ctx.device)
        ctx.sync()
        return self


def _fill_shard(ctx, features, plan, rank, world, row_bytes):
    ids = A.dgnn_tier_shard_ids(ctx, plan.gpu_ids, plan.k_gpu, rank, world)
    dev = ctx.device.index if ctx.device.index is not None else 0
    buf = A.DeviceBuffer(dev, max(ids.numel(), 1) * row_bytes)
    if ids.numel():
        A.dgnn_gather_rows(ctx, features, ids, buf.view((ids.numel(), row_bytes)))
    return buf


def all_gather_handles(handle: bytes, group=None) -> list:
    """The process group's all-gather of this rank's 64-byte IPC handle (any backend)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


class PeerSlots:
    """The partitioned GPU tier of a pipelined multi-pass run (bench.py --gpu-tier peer|nccl).

    Two passes are in flight, so every rank keeps two shard buffers (slot = pass % 2), each a
    plain cudaMalloc allocation of ``ceil(gpu_rows / world)`` rows.  Their CUDA IPC handles are
    all-gathered once; ``view(slot)`` then hands the assembly a peer table (this rank's shard plus
    the mapped shards of every other rank) for dgnn_assemble_group_peer, and ``sharded(slot, k_gpu)``
    the same shard for the NCCL exchange path.  Filling a slot and reading it are separated by
    the Runner's two cross-rank barriers per pass (filled everywhere before any assembly reads it;
    read everywhere before the pass after next refills it)."""

    class _View:
        def __init__(self, peers, world):
            self.peers, self.world = peers, world

    def __init__(self, device: int, gpu_rows: int, row_bytes: int, rank: int, world: int, exchange):
        self.rank, self.world, self.row_bytes = rank, world, row_bytes
        self.rows_cap = max(1, (gpu_rows + world - 1) // world)
        self.bufs = [A.DeviceBuffer(device, self.rows_cap * row_bytes) for _ in range(2)]
        self.maps, self.views = [], []
        dev = torch.device("cuda", device)
        for b in self.bufs:
            handles = exchange(b.ipc_handle())
            ptrs = []
            for r, h in enumerate(handles):
                if r == rank:
                    ptrs.append(b.ptr)
                else:
                    m = A.IpcMapping(device, h)
                    self.maps.append(m)
                    ptrs.append(m.ptr)
            self.views.append(self._View(torch.tensor(ptrs, dtype=torch.int64, device=dev), world))

    def shard(self, slot: int) -> torch.Tensor:
        return self.bufs[slot].view((self.rows_cap, self.row_bytes))

    def view(self, slot: int):
        return self.views[slot]

    def sharded(self, slot: int, k_gpu: int):
        t = ShardedTier.__new__(ShardedTier)
        t.ctx, t.rank, t.world, t.k_gpu, t.row_bytes = None, self.rank, self.world, k_gpu, self.row_bytes
        n_local = max(0, (k_gpu - self.rank + self.world - 1) // self.world)
        t.rows = self.shard(slot)[:n_local]
        return t


def gloo_all_to_all(group=None):
    """all_to_all through host memory (gloo has no CUDA all-to-all): the test stand-in for
    nccl_all_to_all when several ranks share one GPU."""
    import torch.distributed as dist

    def a2a(x: torch.Tensor, send_splits, recv_splits):
        xc = x.contiguous().cpu()
        out = torch.empty(sum(recv_splits), dtype=x.dtype)
        dist.all_to_all_single(out, xc, output_split_sizes=list(recv_splits), input_split_sizes=list(send_splits),
                               group=group)
        return out.to(x.device)
    return a2a
