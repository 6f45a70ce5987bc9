"""Batched packing from a partitioned feature source (Sec. 5.2).

When the feature table does not fit in HBM (IGB-scale), it is read in partitions of
consecutive node IDs -- each partition once, sequentially, from a pinned host buffer or an
O_DIRECT file -- and every packed row of every batch is routed from the partition holding it
(``dgnn_pack_partition``).  Partition i+1 is staged on the ctx side stream while partition i is
routed (two partition buffers).  The partition size follows P:439: of a memory budget C, every
batch keeps a 4 KiB buffer, so partitions get C - 4 KiB x N (rounded down to whole pages and rows).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _abi as A
from .layout import FILE_CHUNK, HostBuffer

PAGE = 4096


def partition_rows(budget_bytes: int, num_batches: int, row_bytes: int) -> int:
    """partition bytes = C - 4 KiB x N, as a row count whose bytes are whole pages."""
    avail = int(budget_bytes) - PAGE * int(num_batches)
    if avail <= 0:
        raise ValueError(f"budget {budget_bytes} B leaves no room for partitions next to {num_batches} 4 KiB buffers")
    step = PAGE // int(np.gcd(PAGE, int(row_bytes)))  # rows per whole number of pages
    rows = (avail // row_bytes) // step * step
    if rows == 0:
        raise ValueError("budget below one page-aligned partition")
    return int(rows)


def pack_streamed(ctx: A.Ctx, idx: A.DiskIndex, source, num_rows: int, row_bytes: int, chunk_off: torch.Tensor,
                  group_buf, part_rows: int, ring: list | None = None) -> dict:
    """Fill ``group_buf`` (chunk layout ``chunk_off``, device int64 [nb+1]) with the packed rows of
    ``idx`` read partition by partition from ``source``: a ``DiskFile`` holding the feature table
    (row v at v * row_bytes, padded to whole pages) or a pinned ``HostBuffer``.  Only partitions
    holding at least one packed row are read.  Returns {"parts", "pages", "bytes"} read."""
    if (part_rows * row_bytes) % PAGE:
        raise ValueError("partitions must not split a page")
    dev = ctx.device
    nparts = -(-int(num_rows) // int(part_rows))
    counts = A.dgnn_disk_index_partition_counts(ctx, idx, part_rows, nparts)
    parts = [int(p) for p in np.nonzero(counts)[0]]
    part_bytes = part_rows * row_bytes
    with torch.cuda.stream(ctx.stream):
        bufs = ring or [torch.empty(part_bytes, dtype=torch.uint8, device=dev) for _ in range(min(2, len(parts)))]
    is_file = isinstance(source, A.DiskFile)
    bounce = HostBuffer(FILE_CHUNK) if is_file else None
    src_ptr = None if is_file else (source.ptr if isinstance(source, HostBuffer) else int(source.data_ptr()))
    tickets = {}
    read = 0

    def span(i):
        p0 = parts[i] * part_rows
        return p0, min(p0 + part_rows, int(num_rows))

    def stage(i):
        nonlocal read
        p0, p1 = span(i)
        nbytes = (p1 - p0) * row_bytes
        if is_file:
            nbytes = -(-nbytes // PAGE) * PAGE  # O_DIRECT: whole pages (the file is padded)
            tickets[i] = A.dgnn_stage_file_read(ctx, source, p0 * row_bytes, bufs[i % 2], nbytes, bounce.ptr,
                                                FILE_CHUNK)
        else:
            tickets[i] = A.dgnn_stage_copy(ctx, bufs[i % 2], src_ptr + p0 * row_bytes, nbytes, 1)
        read += nbytes

    if parts:
        stage(0)
    for i in range(len(parts)):
        if i + 1 < len(parts):
            stage(i + 1)  # ordered after partition i-1's routing, which used this buffer
        A.dgnn_stage_wait(ctx, tickets.pop(i))
        p0, p1 = span(i)
        A.dgnn_pack_partition(ctx, idx, bufs[i % 2], p0, p1, row_bytes, chunk_off, group_buf)
    A.dgnn_pack_tails(ctx, idx, row_bytes, chunk_off, group_buf)
    pages = sum(-(-(span(i)[1] - span(i)[0]) * row_bytes // PAGE) for i in range(len(parts)))
    return {"parts": len(parts), "pages": int(pages), "bytes": int(read), "_keep": (bufs, bounce)}


def write_feature_file(path: str, features: torch.Tensor) -> int:
    """The feature table as a file for ``pack_streamed``: rows back to back, zero-padded to a
    whole page (O_DIRECT reads whole pages).  Returns the file size."""
    raw = features.contiguous().view(torch.uint8).reshape(-1).cpu().numpy()
    size = -(-raw.size // PAGE) * PAGE
    with open(path, "wb") as f:
        f.write(raw.tobytes())
        f.write(b"\0" * (size - raw.size))
    return size
