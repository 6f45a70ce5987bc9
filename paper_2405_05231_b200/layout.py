"""The offline-layout driver: DiskGNN's layout half (P:508-511 ``DiskGNN_train``)
over the C ABI, plus the training-time assembler.

    layout = offline_layout(ctx, indptr, indices, features, seeds, fanout, batch_size,
                            gpu_rows, host_rows, rng_seed, group_size)
    for b, feats in layout.assemble_epoch():   # feats: [n_b, dim] on the GPU
        ...

Every step runs in libdgnn.so kernels; this module only sequences the calls,
owns buffers (torch device tensors, pinned host buffers) and, when
torch.distributed is initialized with world size > 1, all-reduces the access
counts (the one exchange step of the path).

Data placement:
  * CSR, features: HBM (inputs).
  * GPU tier: HBM buffer [K_g, row_bytes]; host tier: pinned host [K_h, row_bytes]
    read by the assemble kernel over PCIe through UVA.
  * Disk tier: a pinned host arena holding every batch's 4 KiB-aligned chunk
    (the "packed feature chunks" of P:283); chunks are staged to HBM on the side
    stream, double-buffered, while the previous batch is being assembled.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi as A


FILE_CHUNK = 64 << 20  # bounce-buffer piece for file staging (4096-aligned for O_DIRECT)


class HostBuffer:
    """Pinned, device-mapped host memory (dgnn_host_alloc) viewed as a CPU uint8 tensor."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        A._check(A.load_library().dgnn_host_alloc(self.nbytes, ctypes.byref(p)), "dgnn_host_alloc")
        self.ptr = int(p.value or 0)
        import weakref
        self._fin = weakref.finalize(self, A.load_library().dgnn_host_free, ctypes.c_void_p(self.ptr))
        buf = (ctypes.c_uint8 * max(self.nbytes, 1)).from_address(self.ptr)
        self.tensor = torch.frombuffer(buf, dtype=torch.uint8, count=self.nbytes) if self.nbytes else \
            torch.empty(0, dtype=torch.uint8)

    def free(self):
        self._fin()


class Workspace:
    """Grow-only buffers reused across offline passes (pinning tens of GB per pass would
    dominate the step otherwise)."""

    def __init__(self):
        self._host = {}
        self._dev = {}
        # buffer name -> (ctx, stage ticket) of the last side-stream copy reading it: the next pass
        # that rewrites the buffer waits for exactly that copy (wait_reader / set_reader)
        self._readers = {}

    def wait_reader(self, ctx: A.Ctx, name: str):
        """Make ``ctx``'s stream wait until the side-stream copies that last read buffer ``name``
        are done."""
        r = self._readers.get(name)
        if r is None:
            return
        rctx, ticket = r
        if rctx is ctx:
            A.dgnn_stage_wait(ctx, ticket)
        else:  # another ctx's side stream: wait for all of it
            ctx.stream.wait_stream(torch.cuda.ExternalStream(rctx.side_stream_ptr, device=ctx.device))

    def set_reader(self, ctx: A.Ctx, name: str, ticket):
        if ticket is not None:
            self._readers[name] = (ctx, ticket)

    def host(self, name: str, nbytes: int) -> "HostBuffer":
        b = self._host.get(name)
        if b is None or b.nbytes < nbytes:
            # the old buffer is only dropped here: a Layout built earlier may still hold it, and
            # its finalizer frees it when the last holder lets go
            b = HostBuffer(int(nbytes * 1.05) + 4096 if b is not None else nbytes)
            self._host[name] = b
        return b

    def dev(self, name: str, nbytes: int, device) -> torch.Tensor:
        t = self._dev.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
            self._dev[name] = t
        return t


def _dist():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


def batch_range(num_batches: int, rank: int, world: int):
    """Contiguous batch block of one rank (batches shard with no exchange)."""
    lo = num_batches * rank // world
    hi = num_batches * (rank + 1) // world
    return lo, hi


@dataclass
class Group:
    b_lo: int
    b_hi: int
    rows: np.ndarray          # packed rows per batch
    chunk_off: np.ndarray     # group-relative chunk offsets (bytes), nb+1
    arena_off: int            # where the group's chunks start in the disk arena
    group_bytes: int
    sec_off: np.ndarray = None  # group-relative byte offset of each batch's graph section (embed_graph)


@dataclass
class Layout:
    ctx: A.Ctx
    samples: A.Samples
    plan: A.CachePlan
    counts: torch.Tensor
    row_bytes: int
    dim: int
    dtype: torch.dtype
    addr: torch.Tensor              # uint32 (as int32) address table of every node of every batch
    gpu_tier: torch.Tensor          # [K_g, row_bytes] uint8, HBM
    host_tier: HostBuffer           # [K_h * row_bytes] pinned (None when read from the table itself)
    arena: HostBuffer | None        # disk tier (pinned), or None when kept in HBM
    arena_dev: torch.Tensor | None  # disk tier kept in HBM (stage="hbm")
    groups: list = field(default_factory=list)
    batch_chunk: np.ndarray = None  # [nb, 2]: (arena byte offset, packed rows)
    stats: dict = field(default_factory=dict)
    _asm_plans: dict = field(default_factory=dict)
    stage_pieces: list = field(default_factory=list)  # (b_lo, b_hi, ticket) of each stage-out copy
    _pinned_srcs: list = field(default_factory=list)  # pinned sources of async H2D table uploads
    disk: A.DiskFile | None = None  # the disk tier as a file (stage="file")
    batch_tiers: np.ndarray = None  # [nb, 3] rows per tier (GPU, HOST, DISK) of each batch
    disk_plan: A.DiskPlan | None = None  # segmented disk cache (Sec. 5.1), when a disk budget is set
    cache_off: int = 0              # byte offset of the segment caches in the disk tier
    sec_abs: np.ndarray = None      # [nb] disk-tier byte offset of each batch's graph section
    host_order: A.HostOrder | None = None  # window-ordered host tier (physical rows permuted)
    host_order_key: tuple = None    # (host_window, out_budget) the ordering was built for
    host_w0_event: object = None    # the layout stream's event once window 0's host rows are filled
    host_table: object = None       # (host_from_table) the host-resident feature table the tier's rows are read from
    host_w0_ticket: int = None      # (fill through HBM) the side-stream ticket of window 0's rows
    host_fill_ticket: int = None    # (fill through HBM) the ticket after which the whole tier is filled

    def phase_ms(self) -> dict:
        """Device time of the layout's phases (after the stream has passed them)."""
        ev = self.stats.get("_events", [])
        return {ev[i][0]: ev[i - 1][1].elapsed_time(ev[i][1]) for i in range(1, len(ev))}

    def wait_chunks(self, stream, b_hi: int, _done=None):
        """Make ``stream`` wait for the stage-out copies holding batches < b_hi."""
        for pi, (b_lo, _, ticket) in enumerate(self.stage_pieces):
            if b_lo >= b_hi:
                break
            if _done is None or pi not in _done:
                A.dgnn_stage_wait_stream(self.ctx, ticket, stream)
                if _done is not None:
                    _done.add(pi)

    @property
    def num_batches(self) -> int:
        return self.samples.num_batches

    # ------------------------------------------------------------ a9
    def tier_mix(self) -> dict:
        """Rows of all batches by source tier (measurement only, torch ops outside the path)."""
        t = (self.addr[:self.samples.total_nodes].view(torch.int32) >> 30) & 3
        c = torch.bincount(t.to(torch.int64), minlength=3).cpu().tolist()
        return {"gpu_rows": c[0], "host_rows": c[1], "disk_rows": c[2]}

    def assemble(self, b: int, out: torch.Tensor, chunk_dev: torch.Tensor | None = None) -> torch.Tensor:
        """Assemble batch b into ``out`` ([n_b, dim]) reading the chunk from ``chunk_dev`` if given
        (already staged to HBM), else directly from the arena (UVA over PCIe).  With a disk cache
        the batch's partial input (chunk rows + its cache pages) is built first."""
        if self.host_tier is None:
            raise ValueError("the host tier is read from the feature table (host_from_table): assemble through "
                             "assemble_epoch with the layout's host windows")
        n0, n1 = int(self.samples.node_off_host[b]), int(self.samples.node_off_host[b + 1])
        off, rows = int(self.batch_chunk[b, 0]), int(self.batch_chunk[b, 1])
        if chunk_dev is not None:
            chunk = chunk_dev
        elif self.arena_dev is not None:
            chunk = self.arena_dev.data_ptr() + off
        else:
            chunk = self.arena.ptr + off
        if self.disk_plan is not None:
            dev = self.ctx.device
            dp = self.disk_plan
            rows = int(self.batch_tiers[b, 2])
            with torch.cuda.stream(self.ctx.stream):
                q = int(dp.req_off_host[b + 1] - dp.req_off_host[b])
                pages = torch.empty(max(q, 1) * 4096, dtype=torch.uint8, device=dev)
                part = torch.empty(max(rows * self.row_bytes, 16), dtype=torch.uint8, device=dev)
                zero = torch.zeros(2, dtype=torch.int64, device=dev)
                chunk = self._partial(self.ctx, b, b + 1, chunk, zero, zero, pages, part)
        if self.host_fill_ticket is not None:
            A.dgnn_stage_wait(self.ctx, self.host_fill_ticket)
        if self.host_order is None:
            A.dgnn_assemble(self.ctx, self.addr[n0:n1], self.gpu_tier, self.plan.k_gpu, self.host_tier.ptr,
                            self.plan.k_host, chunk, rows, self.row_bytes, out)
        else:  # window-ordered host tier: slot s is physical row phys_of_slot[s]
            with torch.cuda.stream(self.ctx.stream):
                t = torch.tensor([0, n1 - n0, 0, 1 << 62, 0, rows], dtype=torch.int64).to(self.ctx.device,
                                                                                          non_blocking=False)
            A.dgnn_assemble_group(self.ctx, self.addr[n0:n1], t[0:2], n1 - n0, self.gpu_tier, self.plan.k_gpu,
                                  self.host_tier.ptr, self.plan.k_host, chunk, t[2:4], t[4:6], self.row_bytes, out,
                                  host_map=self.host_order.phys_of_slot)
        return out

    def early_host_prefetch(self, gctx: A.Ctx, ws: "Workspace", host_window: int, out_budget: int,
                            arena_tag: str, after=()):
        """Stage window 0's host rows (one contiguous physical range) into this epoch's staging arena
        ahead of its assembly, on ``gctx``'s stream once that part of the tier is filled and the
        ``after`` events (the arena's previous user done) have passed -> the event to hand to
        assemble_epoch(early=...), or None when the assembly would not use the ordering."""
        ho = self.host_order
        if ho is None or self.host_order_key != (host_window, int(out_budget)) or \
                (self.host_w0_event is None and self.host_w0_ticket is None):
            return None
        with torch.cuda.stream(gctx.stream):
            nbytes = max(ho.capacity, 1) * self.row_bytes
            arena = ws.dev("staging0" + arena_tag, nbytes, gctx.device)[:nbytes]
        if self.host_w0_ticket is not None:
            A.dgnn_stage_wait_stream(self.ctx, self.host_w0_ticket, gctx.stream)
        else:
            gctx.stream.wait_event(self.host_w0_event)
        for ev in after:
            gctx.stream.wait_event(ev)
        if os.environ.get("DGNN_ASM_TRACE") == "1":  # (measurement only) the copy's own start
            self._early_start = torch.cuda.Event(enable_timing=True)
            self._early_start.record(gctx.stream)
        self._stage_window(gctx, arena, 0)
        ev = torch.cuda.Event()
        ev.record(gctx.stream)
        return ev

    def _stage_window(self, gctx: A.Ctx, dst, w: int):
        """Window w's scheduled host rows into the staging arena ``dst``: the copy engine's ranges of the
        pinned tier, or (host_from_table) the same rows gathered from the host-resident table."""
        ho = self.host_order
        if self.host_table is None:
            A.dgnn_copy_ranges(gctx, dst, self.host_tier.ptr, ho.copies[w], self.row_bytes)
            return
        tri, pre, nr, rows = ho.copies_dev(self.ctx)[w]
        A.dgnn_gather_ranges(gctx, self.host_table, self.row_bytes, ho.phys_ids, tri, pre, nr, rows, dst)

    def host_windows(self, host_window: int, out_budget: int = 1 << 30):
        """The assembler's host-row windows: (first run, last run + 1) over assembly_groups(out_budget),
        each spanning fewer than ``host_window`` batches past its first run's start."""
        groups = self.assembly_groups(out_budget)
        windows = []
        if host_window > 1 and self.plan.k_host > 0:
            r0 = 0
            while r0 < len(groups):
                r1 = r0 + 1
                while r1 < len(groups) and groups[r1 - 1][1] - groups[r0][0] < host_window:
                    r1 += 1
                windows.append((r0, r1))
                r0 = r1
        return groups, windows

    def _cache_rows(self) -> torch.Tensor:
        """The segment caches as [pages, 4096] (pinned host through UVA, or HBM)."""
        dp = self.disk_plan
        src = self.arena.tensor if self.arena is not None else self.arena_dev
        return src[self.cache_off:self.cache_off + max(dp.cache_pages, 1) * 4096].view(-1, 4096)

    def _partial(self, ctx: A.Ctx, b0: int, b1: int, chunk, chunk_off: torch.Tensor, out_off: torch.Tensor, pages,
                 out, bounce=None):
        """Partial input of batches [b0, b1), enqueued on ``ctx``: fetch their merged
        cache-page requests into ``pages`` (a UVA gather from the pinned / HBM cache region, or
        page preads from the disk-tier file through ``bounce``) and interleave them with the
        (reduced) chunk rows into ``out``: dense DISK rows in local order at ``out_off``."""
        dp = self.disk_plan
        q0, q1 = int(dp.req_off_host[b0]), int(dp.req_off_host[b1])
        if q1 > q0:
            if self.disk is not None:
                t = A.dgnn_stage_file_read_pages(ctx, self.disk, self.cache_off, self._req_pages_host[q0:q1], pages,
                                                 bounce.ptr, FILE_CHUNK)
                A.dgnn_stage_wait(ctx, t)
            else:
                A.dgnn_gather_rows(ctx, self._cache_rows(), dp.req_pages[q0:q1], pages)
        A.dgnn_disk_partial(ctx, dp, b0, b1, pages, chunk, chunk_off, out, out_off)
        return out

    def assembly_groups(self, out_budget: int = 1 << 30):
        """Runs of consecutive batches assembled per launch: the output of a run fits
        ``out_budget`` bytes and its chunks are one contiguous span of the disk tier."""
        # (dgnn_assembly_runs: the last b1 with no[b1] - no[b0] <= max_rows, at least one batch, at
        # most 1024, cached per budget)
        key = ("runs", int(out_budget))
        runs = self._asm_plans.get(key)
        if runs is None:
            runs = A.dgnn_assembly_runs(self.samples.node_off_host, max(1, out_budget // self.row_bytes), 1024)
            self._asm_plans[key] = runs
        return runs

    def assembly_plan(self, out_budget: int = 1 << 30):
        """Per-run device tables (node offsets, chunk byte offsets, packed-row prefix, all
        relative to the run), built once on the layout's stream and cached."""
        key = int(out_budget)
        plan = self._asm_plans.get(key)
        if plan is not None:
            return plan
        groups = self.assembly_groups(out_budget)
        # node offsets, chunk byte offsets and packed-row prefix of every run, relative to the run
        # (chunks of consecutive batches are contiguous, 4 KiB-aligned, in the disk tier); with the
        # segmented disk cache the dense partial-input offsets instead (dgnn_assembly_tables)
        tab, offs, spans = A.dgnn_assembly_tables(
            self.samples.node_off_host, self.batch_chunk[:, 0], self.batch_chunk[:, 1],
            self.batch_tiers[:, 2] if self.disk_plan is not None else None,
            self.sec_abs if self.disk_plan is None else None, int(self.stats["chunk_bytes"]), self.row_bytes, groups)
        # kernel-parameter upload (dgnn_upload): the host never waits for the layout's stream, and
        # the tables do not queue on a copy engine behind the window / stage copies in flight
        flat = A.dgnn_upload(self.ctx, tab)
        with torch.cuda.stream(self.ctx.stream):
            ready = torch.cuda.Event()
            ready.record(self.ctx.stream)  # tiers, address tables and these tables are in place
        plan = (groups, spans, flat, offs, ready)
        self._asm_plans[key] = plan
        return plan

    def assemble_epoch(self, ctx: A.Ctx | None = None, out_budget: int = 1 << 30, host_window: int = 128,
                       gather_ctx: A.Ctx | None = None, sharded_tier=None, remote=None, runs: bool = False,
                       ring_wait: dict | None = None, ws: Workspace | None = None, peer_tier=None,
                       pcie_rows: torch.Tensor | None = None, on_run=None, arena_tag: str = "", early=None):
        """Pipelined assembly: the chunks of the next run of batches are staged H2D
        on the side stream while the current run is assembled on the ctx stream (one
        dgnn_assemble_group launch per run).  Yields (b, features[n_b, dim]) per batch; a
        yielded view stays valid until two runs later.  Enqueueing never blocks the host.

        ``host_window`` > 1 merges host-tier reads over windows of that many batches
        (dgnn_host_window): each CPU-cache row crosses PCIe once per window into an HBM
        staging buffer instead of once per batch.  ``host_window=1`` is the
        paper's per-batch UVA read of the CPU cache.  The outputs are identical.  With a
        ``gather_ctx`` (a ctx on another stream) the next window's PCIe gather runs there,
        double-buffered, overlapping the current window's HBM-bound runs.

        ``sharded_tier`` (a shard.ShardedTier) + ``remote(ctx, addr_run, out)`` assemble with
        the GPU tier partitioned over ranks: local GPU-tier rows from this rank's shard,
        remote ones delivered by ``remote`` (shard.fetch_remote_rows over NCCL, or the
        single-process loopback).

        ``runs=True`` yields (b0, b1, out_run) once per run instead; with ``ring_wait`` (run index
        -> event) the run that reuses run i's output slot first waits for ring_wait[i] (a
        consumer on another stream, e.g. the trainer: a queue of depth 2).

        ``ws``: a Workspace for the rings and staging buffers, reused by every epoch assembled
        on the same stream (keeps tens of GB out of the caching allocator's churn).

        ``peer_tier`` (a shard.PeerTier): the GPU tier sharded over ranks and read one-sided
        through peer memory (dgnn_assemble_group_peer), no exchange round.

        ``pcie_rows`` (device int64 [1], measurement only): accumulates the host-tier rows the
        window gathers move over PCIe.

        ``arena_tag`` names this epoch's staging arena in ``ws`` (epochs in flight at once use
        different tags); ``early`` = the event of early_host_prefetch: window 0's host rows are
        already in that arena.

        ``on_run(i, b0, b1, chunk, sec_off)``: called on the ctx stream after run i is assembled,
        with the run's staged chunks (device tensor or pointer) and, when the chunks keep their
        graph samples (embed_graph), the device offsets of the batches' graph sections in it."""
        ctx = ctx or self.ctx
        gctx = gather_ctx or ctx
        nb = self.num_batches
        if nb == 0:
            return
        groups, spans, flat, offs, ready = self.assembly_plan(out_budget)
        if ctx is not self.ctx:
            if self.disk_plan is None and (self.arena is not None or self.disk is not None):
                # the tables were uploaded on the layout's stream after the tiers and address
                # tables; staged chunks are waited for run by run (wait_chunks, stage-out
                # tickets), so the assembly need not wait for the packs of later groups
                ctx.stream.wait_event(ready)
            else:  # chunks packed straight into HBM, or segment caches written after the packs
                ctx.stream.wait_stream(self.ctx.stream)
        no = self.samples.node_off_host
        dev = ctx.device
        kh = self.plan.k_host
        windows = self.host_windows(host_window, out_budget)[1]  # (first run, last run + 1)
        ho = self.host_order
        ordered = ho is not None and bool(windows) and self.host_order_key == (host_window, int(out_budget))
        if self.host_tier is None and not ordered and kh > 0:
            raise ValueError("the host tier is read from the feature table (host_from_table): assemble with the "
                             "layout's host windows (host_window and out_budget of offline_layout's host_order)")
        def buf(name, n, dtype=torch.uint8, shape=None):
            """n elements of dtype, from the workspace when there is one (grow-only, >= 16 bytes)."""
            esz = torch.empty(0, dtype=dtype).element_size()
            nbytes = max(int(n) * esz, 16)
            raw = torch.empty(nbytes, dtype=torch.uint8, device=dev) if ws is None else ws.dev(name, nbytes, dev)
            t = raw[:int(n) * esz].view(dtype)
            return t.view(shape) if shape is not None else t

        with torch.cuda.stream(ctx.stream):
            max_rows = max(s[1] - s[0] for s in spans)
            max_c = max(s[3] - s[2] for s in spans)
            out_ring = [buf(f"out{i}", max_rows * self.dim, self.dtype, (max_rows, self.dim)) for i in range(2)]
            staged = self.arena is not None or self.disk is not None
            bounce_r = HostBuffer(FILE_CHUNK) if self.disk is not None else None
            chunk_ring = [buf(f"chunk{i}", max_c) for i in range(2)] if staged else None
            dp = self.disk_plan
            if dp is not None:  # per run: its cache pages and its partial input (dense DISK rows)
                dpre = np.concatenate([[0], np.cumsum(self.batch_tiers[:, 2])])
                max_pg = max(int(dp.req_off_host[b1] - dp.req_off_host[b0]) for b0, b1 in groups)
                max_pi = max(int(dpre[b1] - dpre[b0]) for b0, b1 in groups)
                page_ring = [buf(f"pages{i}", max(max_pg, 1) * 4096) for i in range(2)]
                part_ring = [buf(f"partial{i}", max_pi * self.row_bytes) for i in range(2)]
            if windows:
                # staging rows: the window's host-row accesses bound its distinct host rows
                hpre = np.concatenate([[0], np.cumsum(self.batch_tiers[:, 1])])
                cap = min(kh, max(int(hpre[groups[r1 - 1][1]] - hpre[groups[r0][0]]) for r0, r1 in windows))
                if ordered:
                    cap = max(ho.rows)  # exact: the rows of each window's physical ranges
                    arena_rows = ho.capacity  # the scheduled staging arena (two windows' rows)
                stamp = buf("stamp", kh, torch.int32)
                stamp.fill_(-1)  # window ids restart at 0 every epoch
                nbuf = 2 if gctx is not ctx else 1
                smap = [buf(f"smap{i}", kh, torch.int32) for i in range(nbuf)]
                wlist = [buf(f"wlist{i}", max(cap, 1), torch.int32) for i in range(nbuf)]
                wcount = [buf(f"wcount{i}", 1, torch.int64) for i in range(nbuf)]
                use_runs = self.row_bytes % 16 == 0 and os.environ.get("DGNN_GATHER_RUNS", "0") == "1" and ho is None
                if use_runs:  # runs of consecutive host slots: one contiguous copy each
                    wruns = [buf(f"wruns{i}", max(cap, 1), torch.int32) for i in range(nbuf)]
                    wnruns = [buf(f"wnruns{i}", 1, torch.int64) for i in range(nbuf)]
                if ordered:  # one arena; each window's rows sit where the schedule put them
                    arena = buf("staging0" + arena_tag, max(arena_rows, 1) * self.row_bytes)
                    staging = [arena, arena]
                else:
                    staging = [buf(f"staging{i}", max(cap, 1) * self.row_bytes) for i in range(nbuf)]
            # ordered windows over a pinned disk tier: each window's chunk span (contiguous) is staged
            # with its host rows in one copy on the gather stream, so a run never waits for a copy of
            # its own (the runs then chain at HBM speed); spans above the budget keep per-run staging
            wspan = []
            if ordered and self.arena is not None and self.disk_plan is None and gctx is not ctx:
                wspan = [(spans[r0][2], spans[r1 - 1][3]) for r0, r1 in windows]
                if max(hi - lo for lo, hi in wspan) > int(os.environ.get("DGNN_WIN_CHUNK_BUDGET", str(4 << 30))):
                    wspan = []
            if wspan:
                wchunk = [buf(f"wchunk{i}", max(hi - lo for lo, hi in wspan)) for i in range(2)]
        if self.host_fill_ticket is not None:  # the host tier is filled on the layout's side stream
            A.dgnn_stage_wait_stream(self.ctx, self.host_fill_ticket, ctx.stream)
        if gctx is not ctx:
            gctx.stream.wait_stream(ctx.stream)  # stamp / buffers were created on the ctx stream
        run_window = {r0: wi for wi, (r0, _) in enumerate(windows)}
        last_run = {r1 - 1: wi for wi, (_, r1) in enumerate(windows)}
        ev_ready, ev_done = {}, {}
        # DGNN_ASM_TRACE=1 (measurement only): per window, timing events of its copy and its runs
        trace = {} if os.environ.get("DGNN_ASM_TRACE") == "1" else None
        self._asm_trace = trace

        def _tev(stream):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e

        def prefetch(w):
            # window w's distinct host rows -> staging[w % nbuf] (PCIe), on the gather stream
            s = w % nbuf
            if w >= nbuf and gctx is not ctx:
                gctx.stream.wait_event(ev_done[w - nbuf])  # the runs that used this buffer are done
            w0, w1 = windows[w]
            if trace is not None:
                trace.setdefault(w, {})["copy0"] = _tev(gctx.stream)
            if ordered:
                # window-ordered host tier: the window's rows are a few physical ranges -> copy engine
                A.dgnn_host_window_ranges(gctx, ho, w, smap[s])
                if w == 0 and early is not None:  # (staged ahead: early_host_prefetch)
                    gctx.stream.wait_event(early)
                else:
                    self._stage_window(gctx, staging[s], w)
                if wspan:  # and the window's chunks: each stage-out piece of the span is copied in as
                    # soon as that piece is in the arena (the round trip pipelines piece by piece)
                    lo, hi = wspan[w]
                    for pi, (pb, pe, ticket) in enumerate(self.stage_pieces):
                        plo = int(self.batch_chunk[pb, 0])
                        phi = int(self.batch_chunk[pe, 0]) if pe < nb else int(self.stats["chunk_bytes"])
                        a, z = max(lo, plo), min(hi, phi)
                        if a >= z:
                            continue
                        if pi not in waited_g:
                            A.dgnn_stage_wait_stream(self.ctx, ticket, gctx.stream)
                            waited_g.add(pi)
                        A.dgnn_copy_ranges(gctx, wchunk[w % 2], self.arena.ptr, [a, z, a - lo], 1)
                if pcie_rows is not None:
                    with torch.cuda.stream(gctx.stream):
                        pcie_rows.add_(ho.copy_rows[w])
                ev = torch.cuda.Event(enable_timing=trace is not None)
                ev.record(gctx.stream)
                ev_ready[w] = ev
                if trace is not None:
                    trace[w]["copy1"] = ev
                return
            A.dgnn_host_window(gctx, self.addr[spans[w0][0]:spans[w1 - 1][1]], w, stamp, kh, wlist[s], smap[s],
                               wcount[s])
            if ho is not None:  # (windows other than the ordering's) slot list -> physical rows
                A.dgnn_remap_ids_dev(gctx, wlist[s], wcount[s], ho.phys_of_slot)
            if use_runs:
                A.dgnn_host_window_runs(gctx, stamp, kh, w, smap[s], wruns[s], wnruns[s])
                A.dgnn_gather_runs_dev(gctx, self.host_tier.ptr, self.row_bytes, wlist[s], wcount[s], wruns[s],
                                       wnruns[s], cap, staging[s])
            else:
                A.dgnn_gather_rows_dev(gctx, self.host_tier.ptr, kh, self.row_bytes, wlist[s], wcount[s],
                                       staging[s])
            if pcie_rows is not None:
                with torch.cuda.stream(gctx.stream):
                    pcie_rows.add_(wcount[s])
            ev = torch.cuda.Event()
            ev.record(gctx.stream)
            ev_ready[w] = ev

        tickets = {}

        waited = set()
        waited_g = set()

        def stage(i):
            n0, n1, c_lo, c_hi = spans[i]
            self.wait_chunks(ctx.stream, groups[i][1], waited)  # the run's chunks have been staged out
            if self.disk is not None:  # pread (O_DIRECT) of the run's chunk span, then H2D
                tickets[i] = A.dgnn_stage_file_read(ctx, self.disk, c_lo, chunk_ring[i % 2], c_hi - c_lo,
                                                    bounce_r.ptr, FILE_CHUNK)
            else:
                tickets[i] = A.dgnn_stage_copy(ctx, chunk_ring[i % 2], self.arena.ptr + c_lo, c_hi - c_lo, 1)

        run_win = {}
        for wi, (r0, r1) in enumerate(windows):
            for r in range(r0, r1):
                run_win[r] = wi
        if staged and not wspan:
            stage(0)
        for i, (b0, b1) in enumerate(groups):
            n0, n1, c_lo, c_hi = spans[i]
            if wspan:  # the window's chunks were staged with its host rows
                w_i = run_win[i]
                chunk = wchunk[w_i % 2].data_ptr() + (c_lo - wspan[w_i][0])
            elif staged:
                if i + 1 < len(groups):
                    stage(i + 1)
                A.dgnn_stage_wait(ctx, tickets.pop(i))
                chunk = chunk_ring[i % 2]
            else:
                chunk = self.arena_dev.data_ptr() + c_lo
            if i in run_window:  # first run of a host window: its host rows must be staged
                w = run_window[i]
                if w not in ev_ready:
                    prefetch(w)
                if gctx is not ctx:
                    ctx.stream.wait_event(ev_ready[w])
                    if w + 1 < len(windows):
                        prefetch(w + 1)  # overlaps this window's (HBM-bound) runs
                if trace is not None:
                    trace.setdefault(w, {})["runs0"] = _tev(ctx.stream)
                cur = w % nbuf
            k = b1 - b0
            t = flat[int(offs[i]):int(offs[i + 1])]
            out = out_ring[i % 2]
            if ring_wait is not None and (i - 2) in ring_wait:
                ctx.stream.wait_event(ring_wait.pop(i - 2))  # the consumer of run i-2 released the slot
            if dp is not None:
                chunk = self._partial(ctx, b0, b1, chunk, t[3 * k + 3:4 * k + 4], t[k + 1:2 * k + 2],
                                      page_ring[i % 2], part_ring[i % 2], bounce_r)
            if windows:
                host_src, host_map = staging[cur], smap[cur]
            else:
                host_src, host_map = self.host_tier.ptr, (ho.phys_of_slot if ho is not None else None)
            if peer_tier is not None:
                A.dgnn_assemble_group_peer(ctx, self.addr[n0:n1], t[:k + 1], n1 - n0, peer_tier.peers,
                                           self.plan.k_gpu, peer_tier.world, host_src, kh, chunk, t[k + 1:2 * k + 2],
                                           t[2 * k + 2:3 * k + 3], self.row_bytes, out, host_map=host_map)
            elif sharded_tier is None:
                A.dgnn_assemble_group(ctx, self.addr[n0:n1], t[:k + 1], n1 - n0, self.gpu_tier, self.plan.k_gpu,
                                      host_src, kh, chunk, t[k + 1:2 * k + 2], t[2 * k + 2:3 * k + 3], self.row_bytes,
                                      out, host_map=host_map)
            else:  # GPU tier sharded over ranks: local rows here, remote rows over the exchange
                A.dgnn_assemble_group_sharded(ctx, self.addr[n0:n1], t[:k + 1], n1 - n0, sharded_tier.rows,
                                              self.plan.k_gpu, sharded_tier.rank, sharded_tier.world, host_src, kh,
                                              chunk, t[k + 1:2 * k + 2], t[2 * k + 2:3 * k + 3], self.row_bytes,
                                              out, host_map=host_map)
                remote(ctx, self.addr[n0:n1], out)
            if on_run is not None:
                on_run(i, b0, b1, chunk, t[3 * k + 3:4 * k + 3] if self.sec_abs is not None else None)
            if i in last_run:
                ev = torch.cuda.Event(enable_timing=trace is not None)
                ev.record(ctx.stream)
                ev_done[last_run[i]] = ev
                if trace is not None:
                    trace[last_run[i]]["runs1"] = ev
            if runs:
                yield b0, b1, out[:n1 - n0]
            else:
                for b in range(b0, b1):
                    yield b, out[int(no[b] - n0):int(no[b + 1] - n0)]

    def train_epoch(self, ctx: A.Ctx | None = None, train_ctx: A.Ctx | None = None, **kw):
        """The training pipeline over this layout: feature loading (chunk staging on
        the side stream) -> feature assembling (ctx) -> model training (the trainer stub,
        dgnn_train_stub, on ``train_ctx``'s stream), stages linked by queues of depth 2.
        Graph loading is free here: the graph samples stay in HBM (reading c22).  Yields
        (b0, b1, x_run) per run after its trainer launch; each batch's seed rows of x_run hold
        its seed embeddings once ``train_ctx``'s stream has passed that point."""
        ctx = ctx or self.ctx
        tctx = train_ctx or ctx
        ring_wait = {}
        loaded = {}
        if self.sec_abs is not None:
            # the graph loader: each run's graph samples come out of its staged chunks
            def on_run(i, b0, b1, chunk, sec):
                loaded[i] = A.dgnn_samples_load(ctx, self.samples, b0, b1, chunk, sec)
            kw["on_run"] = on_run
        for i, (b0, b1, x) in enumerate(self.assemble_epoch(ctx, runs=True, ring_wait=ring_wait, **kw)):
            if tctx is not ctx:
                ev = torch.cuda.Event()
                ev.record(ctx.stream)
                tctx.stream.wait_event(ev)
            if self.sec_abs is not None:
                # run i-2's samples: the ctx stream has waited for its trainer (the ring), so their
                # stream-ordered release on the ctx stream is safe
                loaded.pop(i - 2, None)
                A.dgnn_train_stub(tctx, loaded[i], 0, b1 - b0, x)
            else:
                A.dgnn_train_stub(tctx, self.samples, b0, b1, x)
            yield b0, b1, x
            if tctx is not ctx:
                ev = torch.cuda.Event()
                ev.record(tctx.stream)
                ring_wait[i] = ev


def offline_layout(ctx: A.Ctx, indptr: torch.Tensor, indices: torch.Tensor, features: torch.Tensor,
                   seeds: torch.Tensor, fanout, batch_size: int, gpu_rows: int, host_rows: int, rng_seed: int,
                   group_size: int = 64, batch_id_base: int = 0, stage: str = "pinned",
                   counts: torch.Tensor | None = None, ws: Workspace | None = None,
                   group_budget: int = 4 << 30, stage_piece: int = 1 << 40, file_path: str | None = None,
                   direct_io: bool = True, disk_budget: int | None = None, disk_m: int = 1,
                   disk_k: int = 4, disk_budget_frac: float | None = None, after_sample=None,
                   scratch_ws: Workspace | None = None, before_pack=None, gpu_shard=None,
                   embed_graph: bool = False, host_order: int | None = None,
                   asm_out_budget: int = 1 << 30, host_from_table: bool = False) -> Layout:
    """Run a1-a8 on this rank's batches.

    ``seeds`` are this rank's seeds (batch t of them gets bid = batch_id_base + t).
    With torch.distributed initialized (world > 1) the counts are all-reduced so that
    every rank derives the identical cache plan from all ranks' batches.
    ``stage``: "pinned" (disk tier in a pinned host arena, the default) or "hbm".
    ``disk_budget`` (bytes): activate the segmented disk cache (Sec. 5.1) when
    the packed chunks exceed it -- the heuristic of P:410-413 picks the smallest segment
    size s whose Eq. 2 space fits (threshold ``disk_m``, MinHash with ``disk_k`` hashes).
    ``disk_budget_frac`` states the budget as a fraction of the packed-only space instead.
    ``scratch_ws``: a Workspace for buffers that do not outlive this call (the packed lists and
    the pack group buffers), shared by consecutive passes on the same ctx: before reusing them
    the ctx stream waits for the previous pass's stage-out on the ctx side stream.
    ``before_pack``: called right before a7 is enqueued (a scheduling hook: bench.py makes the
    layout stream wait there for the previous pass's assembly, so the HBM-bound pack runs alone).
    ``gpu_shard`` = (rank, world, buffer [>= ceil(gpu_rows / world), row_bytes] uint8): the GPU tier is
    partitioned over the ranks (slot s on rank s % world at row s // world) and this
    rank fills only its shard into ``buffer`` (Layout.gpu_tier is then the shard); the assembly
    reads the other shards through peer memory (shard.PeerTier) or the NCCL exchange.
    ``embed_graph``: keep each batch's graph sample in its chunk (reading c22b) and free the
    samples' device arrays once packed: training then reads the graph through the loader stage
    (Layout.train_epoch, dgnn_samples_load); the host-side offsets stay as the layout's metadata.
    ``host_order`` = W: lay the host tier out in window order (dgnn_host_order) for an assembly with
    host_window=W and out_budget=``asm_out_budget``: each window's host rows become a few contiguous
    ranges that the copy engine moves; outputs are unchanged (every reader maps slot -> physical row).
    ``after_sample``: called once the samples are complete (dgnn_sample returns when they are),
    before the rest of the pass is enqueued -- a scheduling hook (bench.py starts the previous
    pass's assembly there, so that sampling never shares the GPU with it).
    """
    dev = ctx.device
    N = indptr.numel() - 1
    if isinstance(features, A.ShardedFeatures):  # the table partitioned by node range over ranks
        row_bytes, dim = features.row_bytes, features.dim
        if disk_budget is not None or disk_budget_frac is not None:
            raise ValueError("the segmented disk cache reads an unpartitioned feature table")
    else:
        row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
        dim = features.numel() // max(features.shape[0], 1)
    stats = {"_events": []}

    import time as _time
    stats["_host"] = []

    def mark(name):  # phase boundaries on the layout's stream + host clock (measurement only)
        e = torch.cuda.Event(enable_timing=True)
        e.record(ctx.stream)
        stats["_events"].append((name, e))
        stats["_host"].append((name, _time.perf_counter()))

    fine_marks = os.environ.get("DGNN_LAYOUT_TRACE") == "1"

    def fine(name):  # (DGNN_LAYOUT_TRACE=1) finer marks inside the classify phase
        if fine_marks:
            mark(name)

    def side_mark(name):  # (DGNN_LAYOUT_TRACE=1) where the side stream's copies have got to
        if fine_marks:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.ExternalStream(ctx.side_stream_ptr, device=dev))
            stats.setdefault("_side", []).append((name, e))

    mark("start")
    if counts is None:
        counts = torch.zeros(N, dtype=torch.int32, device=dev)
    # a1-a3 (+ the fused access counter)
    samples = A.dgnn_sample(ctx, indptr, indices, seeds, batch_size, fanout, rng_seed, batch_id_base, counts)
    mark("sample")
    if after_sample is not None:
        after_sample()
    # a4: global histogram across ranks
    d = _dist()
    if d is not None:
        with torch.cuda.stream(ctx.stream):
            d.all_reduce(counts, op=d.ReduceOp.SUM)
    # a5
    plan = A.dgnn_build_cache(ctx, counts, gpu_rows, host_rows)
    mark("plan")
    # tier buffers as special mini-batches
    def buf(name, n, dtype, shape=None):  # per-pass buffers from the workspace (no allocator churn)
        nbytes = max(int(n), 1) * torch.empty(0, dtype=dtype).element_size()
        t = ws.dev(name, nbytes, dev)[:nbytes].view(dtype) if ws is not None else \
            torch.empty(max(int(n), 1), dtype=dtype, device=dev)
        return t[:int(n)].view(shape) if shape is not None else t

    if gpu_shard is None:
        gpu_tier = buf("gpu_tier", plan.k_gpu * row_bytes, torch.uint8, (plan.k_gpu, row_bytes))
        A.dgnn_gather_rows(ctx, features, plan.gpu_ids, gpu_tier)
    else:  # this rank's shard of the partitioned GPU tier
        rank, world, shard_buf = gpu_shard
        ids = A.dgnn_tier_shard_ids(ctx, plan.gpu_ids, plan.k_gpu, rank, world)
        if ids.numel() > shard_buf.shape[0]:
            raise ValueError(f"GPU-tier shard of {ids.numel()} rows exceeds its buffer ({shard_buf.shape[0]})")
        gpu_tier = shard_buf[:ids.numel()]
        if ids.numel():
            A.dgnn_gather_rows(ctx, features, ids, gpu_tier)
    # host_from_table: the feature table is host-resident (pinned), so the tier's rows need no copy of
    # their own -- the assembler's window staging gathers them from the table (dgnn_gather_ranges)
    table_host = bool(host_from_table and host_order and plan.k_host > 0 and
                      not isinstance(features, A.ShardedFeatures) and not features.is_cuda)
    host_tier = None if table_host else (ws.host("host_tier", plan.k_host * row_bytes) if ws is not None else
                                         HostBuffer(plan.k_host * row_bytes))
    if not host_order:
        A.dgnn_gather_rows(ctx, features, plan.host_ids, host_tier.ptr)
    mark("tiers")
    # a6 for every batch of this rank at once
    nb = samples.num_batches
    total_nodes = samples.total_nodes
    addr = buf("addr", total_nodes, torch.int32)
    if scratch_ws is not None:
        # (the scratch buffers a side-stream copy of the previous pass still reads -- the host-fill
        # staging and the pack group buffers -- are waited for right before they are rewritten)
        nbytes = max(int(total_nodes), 1) * 4
        packed_ids = scratch_ws.dev("packed_ids", nbytes, dev)[:nbytes].view(torch.int32)
    else:
        packed_ids = buf("packed_ids", total_nodes, torch.int32)
    packed_off = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    po = A.dgnn_classify(ctx, plan, samples, 0, nb, addr, packed_ids, packed_off) if nb else np.zeros(1, np.int64)
    batch_tiers = A.dgnn_batch_tier_counts(ctx, samples, 0, nb, addr) if nb else np.zeros((0, 3), np.int64)
    fine("c_classify")
    dplan = None
    if disk_budget_frac is not None and nb:
        disk_budget = int(disk_budget_frac * int(((np.diff(po) * row_bytes + 4095) // 4096).sum())) * 4096
    if disk_budget is not None and nb:
        idx = A.DiskIndex(ctx, packed_ids[:int(po[-1])], packed_off, po, N)
        s_seg, pages = A.dgnn_disk_search(ctx, idx, row_bytes, int(disk_budget) // 4096, disk_m)
        if s_seg == 0:
            raise ValueError(f"disk budget {disk_budget} B is below the smallest Eq. 2 space ({pages * 4096} B)")
        dplan = A.dgnn_disk_plan_build(ctx, idx, row_bytes, s_seg, disk_m, disk_k, rng_seed)
        del idx
        po = dplan.pk_off_host  # the chunks now hold the reduced packed lists P_b'
        packed_ids = dplan.pk_ids
    rows = np.diff(po)
    # a7 layout: groups of `group_size` batches, each a contiguous run of 4 KiB-aligned chunks
    groups = []
    batch_chunk = np.zeros((nb, 2), np.int64)
    arena_off = 0
    if embed_graph and (disk_budget is not None or dplan is not None):
        raise ValueError("embed_graph with the segmented disk cache is not supported")
    # packing groups: at most `group_size` batches (0 = unbounded) whose chunks fit the group-buffer
    # budget (the analogue of P:439's "C - 4N" partition sizing; dgnn_packing_groups)
    for g0, g1 in (A.dgnn_packing_groups(po, row_bytes, group_size, group_budget) if nb else []):
        rel = po[g0:g1 + 1] - po[g0]
        so = None
        if embed_graph:
            co, so = A.dgnn_chunk_layout_graph(samples, g0, rel, row_bytes)
        else:
            co = A.dgnn_chunk_layout(rel, row_bytes)
        groups.append(Group(g0, g1, rows[g0:g1], co, arena_off, int(co[-1]), so))
        batch_chunk[g0:g1, 0] = arena_off + co[:-1]
        batch_chunk[g0:g1, 1] = rows[g0:g1]
        arena_off += int(co[-1])
    chunk_bytes = arena_off
    cache_off = arena_off
    if dplan is not None:
        arena_off += dplan.cache_pages * 4096
    arena = arena_dev = disk = None
    if stage == "pinned":
        arena = ws.host("arena", arena_off) if ws is not None else HostBuffer(arena_off)
    elif stage == "hbm":
        arena_dev = torch.empty(max(arena_off, 16), dtype=torch.uint8, device=dev)
    elif stage == "file":
        if not file_path:
            raise ValueError("stage='file' needs file_path")
        disk = A.DiskFile(file_path, max(arena_off, 4096), direct=direct_io)
    else:
        raise ValueError(stage)
    fine("c_arena")
    L = Layout(ctx, samples, plan, counts, row_bytes, dim, features.dtype, addr, gpu_tier, host_tier, arena,
               arena_dev, groups, batch_chunk, stats)
    L.batch_tiers = batch_tiers
    L.disk_plan = dplan
    L.cache_off = cache_off
    if embed_graph and nb:
        L.sec_abs = np.concatenate([g.arena_off + g.sec_off for g in groups]).astype(np.int64)
    if dplan is not None:
        stats.update(disk_cache={"s": dplan.s, "m": dplan.m, "k": disk_k, "budget_pages": int(disk_budget) // 4096,
                                 "space_pages": dplan.space_pages, "io_pages": dplan.io_pages,
                                 "cache_pages": dplan.cache_pages, "chunk_pages": dplan.chunk_pages,
                                 "cache_rows": dplan.n_cache, "requests": dplan.n_req})
    stats.update(row_bytes=row_bytes, groups=len(groups), packed_rows=int(po[-1]),
                 packed_bytes=int(po[-1]) * row_bytes, arena_bytes=arena_off, chunk_bytes=chunk_bytes,
                 k_gpu=plan.k_gpu, k_host=plan.k_host, total_nodes=total_nodes, total_edges=samples.total_edges)
    if host_order and plan.k_host > 0:
        # window-ordered host tier (needs the address tables): fill it in physical order
        ho = None
        if nb:
            groups_a, wins = L.host_windows(int(host_order), int(asm_out_budget))
            if 0 < len(wins) <= 32:
                no = samples.node_off_host
                wo = [int(no[groups_a[r0][0]]) for r0, _ in wins] + [int(no[groups_a[wins[-1][1] - 1][1]])]
                try:
                    ho = A.HostOrder(ctx, addr, wo, plan.host_ids, plan.k_host)
                except A.DgnnError:  # too many distinct window masks: keep the slot order
                    ho = None
        fine("c_hostorder")
        if ho is None and table_host:  # no window ordering after all: the tier is materialized
            host_tier = L.host_tier = ws.host("host_tier", plan.k_host * row_bytes) if ws is not None else \
                HostBuffer(plan.k_host * row_bytes)
            table_host = False
        if ho is not None and table_host:
            L.host_order, L.host_order_key = ho, (int(host_order), int(asm_out_budget))
            L.host_table = features
            ho.copies_dev(ctx)  # every window's copy list on the device (uploaded on the layout's stream)
            ev = torch.cuda.Event()
            ev.record(ctx.stream)  # phys_ids and the lists are in place: window 0 may be staged
            L.host_w0_event = ev
            stats["host_order"] = {"windows": ho.nwin, "groups": ho.n_groups, "source": "feature table",
                                   "ranges_per_window": [len(r) // 3 for r in ho.ranges], "rows": ho.rows,
                                   "rows_copied": ho.copy_rows, "arena_rows": ho.capacity}
        elif ho is not None:
            L.host_order, L.host_order_key = ho, (int(host_order), int(asm_out_budget))
            # window 0's rows first (one contiguous range of the physical order), then the rest: the
            # assembler may stage window 0 as soon as its part is filled (Layout.early_host_prefetch)
            kh, rb = plan.k_host, row_bytes
            first = ho.ranges[0].reshape(-1, 3)[:, :2] if len(ho.ranges[0]) else np.zeros((0, 2), np.int64)
            rest, cur = [], 0  # the complement of window 0's ranges in [0, kh): the runs of unfilled rows
            for lo, hi in sorted((int(a), int(b)) for a, b in first):
                if lo > cur:
                    rest.append((cur, lo))
                cur = max(cur, hi)
            if cur < kh:
                rest.append((cur, kh))
            fws = scratch_ws if scratch_ws is not None else ws
            if fws is not None and not isinstance(features, A.ShardedFeatures):
                # through HBM: the rows gathered in physical order on the layout's stream (HBM-bound,
                # milliseconds), then copied to the pinned tier by the copy engine on the side stream
                # (window 0's range first), so the layout's stream does not spend the D2H time.  The
                # buffer is scratch: the next pass on this ctx reuses it after waiting for the side
                # stream (the wait before classify)
                with torch.cuda.stream(ctx.stream):
                    hbuf = fws.dev("host_fill", kh * rb, dev)[:kh * rb]
                fws.wait_reader(ctx, "host_fill")  # the previous pass's fill copies read it
                A.dgnn_gather_rows(ctx, features, ho.phys_ids[:kh], hbuf)
                t = None
                for lo, hi in first:
                    t = A.dgnn_stage_copy(ctx, host_tier.ptr + int(lo) * rb, hbuf.data_ptr() + int(lo) * rb,
                                          (int(hi) - int(lo)) * rb, 0)
                L.host_w0_ticket = t
                side_mark("fill_w0_done")
                for lo, hi in rest:
                    t = A.dgnn_stage_copy(ctx, host_tier.ptr + int(lo) * rb, hbuf.data_ptr() + int(lo) * rb,
                                          (int(hi) - int(lo)) * rb, 0)
                L.host_fill_ticket = t
                side_mark("fill_done")
                fws.set_reader(ctx, "host_fill", t)
            else:  # SM stores into the pinned tier, window 0's range first
                for lo, hi in first:
                    A.dgnn_gather_rows(ctx, features, ho.phys_ids[int(lo):int(hi)], host_tier.ptr + int(lo) * rb)
                ev = torch.cuda.Event()
                ev.record(ctx.stream)
                L.host_w0_event = ev
                for lo, hi in rest:
                    A.dgnn_gather_rows(ctx, features, ho.phys_ids[int(lo):int(hi)], host_tier.ptr + int(lo) * rb)
            stats["host_order"] = {"windows": ho.nwin, "groups": ho.n_groups,
                                   "ranges_per_window": [len(r) // 3 for r in ho.ranges], "rows": ho.rows,
                                   "rows_copied": ho.copy_rows, "arena_rows": ho.capacity}
        else:
            A.dgnn_gather_rows(ctx, features, plan.host_ids, host_tier.ptr)
    fine("c_fill")
    if nb:
        L.assembly_plan(int(asm_out_budget))  # a9's per-run tables, uploaded here on the layout's stream
    fine("c_asmplan")
    # a7's tables go up before the pack's wait (before_pack): an H2D copy queued between that wait
    # and the pack would sit behind whatever the copy engines are moving for the assembly then
    # (kernel-parameter uploads, dgnn_upload: a blocking copy would hold the host until this stream
    # passes the wait for the previous pass's assembly, and an async copy-engine copy would queue
    # behind the window copies -- and the pack behind it)
    rel_all = A.dgnn_upload(ctx, np.concatenate(
        [np.concatenate([po[g.b_lo:g.b_hi + 1] - po[g.b_lo], g.chunk_off]) for g in groups]
        or [np.zeros(0, np.int64)]).astype(np.int64))
    sec_dev = None
    if embed_graph and nb:  # group-relative graph-section offsets of every batch
        sec_dev = A.dgnn_upload(ctx, np.concatenate([g.sec_off for g in groups]).astype(np.int64))
    mark("classify")
    if before_pack is not None:
        before_pack()
        mark("pack_wait")  # (measurement: where the pack's wait for the previous assembly ended)
    # a7 pack + a8 stage-out, double-buffered group buffers; every group's stage-out
    # ticket is kept so the assembler waits for exactly the chunks it reads
    with torch.cuda.stream(ctx.stream):
        max_gb = max([g.group_bytes for g in groups], default=0)
        staged = arena is not None or disk is not None
        # group buffers come from the workspace when there is one: re-allocating GBs every
        # pass can force the caching allocator to map memory inside the timed region
        gws = scratch_ws if scratch_ws is not None else ws
        L._group_bufs = [(gws.dev(f"group_buf{i}", max(max_gb, 16), dev)[:max(max_gb, 16)] if gws is not None
                          else torch.empty(max(max_gb, 16), dtype=torch.uint8, device=dev))
                         for i in range(min(2, len(groups)))] if staged else []
    if disk is not None:
        L.disk = disk
        L._bounce_w = ws.host("bounce_w", FILE_CHUNK) if ws is not None else HostBuffer(FILE_CHUNK)
    bufs = L._group_bufs
    if bufs and gws is not None:
        gws.wait_reader(ctx, "group_buf")  # the previous pass's stage-out copies read them
    group_last_ticket = []
    off = 0
    for gi, g in enumerate(groups):
        k = g.b_hi - g.b_lo
        rel_po, rel_co = rel_all[off:off + k + 1], rel_all[off + k + 1:off + 2 * k + 2]
        off += 2 * k + 2
        ids = packed_ids[int(po[g.b_lo]):int(po[g.b_hi])]
        total = int(po[g.b_hi] - po[g.b_lo])
        if disk is not None:  # a8 to a file: pwrite of the whole group through the bounce buffer
            if gi >= 2:
                A.dgnn_stage_wait(ctx, group_last_ticket[gi - 2])
            dst = bufs[gi % 2]
            A.dgnn_pack(ctx, features, ids, rel_po, rel_co, total, g.group_bytes, dst)
            if sec_dev is not None:
                A.dgnn_pack_graph(ctx, samples, g.b_lo, k, sec_dev[g.b_lo:g.b_hi], dst)
            t = A.dgnn_stage_file_write(ctx, disk, g.arena_off, dst, g.group_bytes, L._bounce_w.ptr, FILE_CHUNK)
            L.stage_pieces.append((g.b_lo, g.b_hi, t))
            group_last_ticket.append(t)
        elif arena is not None:
            if gi >= 2:
                A.dgnn_stage_wait(ctx, group_last_ticket[gi - 2])  # its buffer is being reused
            dst = bufs[gi % 2]
            A.dgnn_pack(ctx, features, ids, rel_po, rel_co, total, g.group_bytes, dst)
            if sec_dev is not None:
                A.dgnn_pack_graph(ctx, samples, g.b_lo, k, sec_dev[g.b_lo:g.b_hi], dst)
            # stage-out in pieces of <= stage_piece bytes on batch boundaries, so the assembler
            # can start on the first batches while the rest is still crossing PCIe
            # (at least 8 pieces per group, >= 64 MB each: the assembly stages each window's chunks in
            # piece by piece, so smaller groups need finer pieces to pipeline the round trip)
            piece = stage_piece if stage_piece >= (1 << 40) else min(stage_piece, max(64 << 20, g.group_bytes // 8))
            b = g.b_lo
            while b < g.b_hi:
                e = b + 1
                while e < g.b_hi and g.chunk_off[e + 1 - g.b_lo] - g.chunk_off[b - g.b_lo] <= piece:
                    e += 1
                lo, hi = int(g.chunk_off[b - g.b_lo]), int(g.chunk_off[e - g.b_lo])
                t = A.dgnn_stage_copy(ctx, arena.ptr + g.arena_off + lo, dst.data_ptr() + lo, hi - lo, 0)
                L.stage_pieces.append((b, e, t))
                b = e
            group_last_ticket.append(L.stage_pieces[-1][2])
            side_mark(f"stage_out_g{gi}_done")
        else:
            dst = arena_dev[g.arena_off:g.arena_off + max(g.group_bytes, 0)]
            A.dgnn_pack(ctx, features, ids, rel_po, rel_co, total, g.group_bytes, dst)
            if sec_dev is not None:
                A.dgnn_pack_graph(ctx, samples, g.b_lo, k, sec_dev[g.b_lo:g.b_hi], dst)
    if group_last_ticket and gws is not None:
        gws.set_reader(ctx, "group_buf", group_last_ticket[-1])
    if dplan is not None:
        L._req_pages_host = dplan.req_pages.cpu().numpy() if disk is not None else None
    if dplan is not None and dplan.cache_pages:
        # the segment caches, MinHash-ordered, after the chunks
        if disk is not None:  # through HBM into the disk-tier file
            with torch.cuda.stream(ctx.stream):
                cache_dev = torch.empty(dplan.cache_pages * 4096, dtype=torch.uint8, device=dev)
            A.dgnn_disk_cache_fill(ctx, dplan, features, cache_dev)
            t = A.dgnn_stage_file_write(ctx, disk, cache_off, cache_dev, cache_dev.numel(), L._bounce_w.ptr,
                                        FILE_CHUNK)
            A.dgnn_stage_sync(ctx, t)  # on disk before the layout returns (cache_dev is released)
        else:
            A.dgnn_disk_cache_fill(ctx, dplan, features, L._cache_rows())
    if embed_graph and nb:
        samples.drop_device()  # from here on the graph samples live in the chunks only
    mark("pack")
    L._rel_all = rel_all
    # packed_ids is only read by the pack kernels on this stream: releasing it now is
    # stream-ordered, so later allocations on the stream reuse it after the packs
    return L
