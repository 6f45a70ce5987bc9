"""ctypes binding of libdgnn.so (include/dgnn.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls and does no
computation of its own: torch tensors are turned into raw pointers and sizes,
the status is checked, library-owned results are wrapped so that they are
freed with the matching ``*_free``.  If the shared library is missing or
cannot be loaded the import fails loudly; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading
import weakref

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGNN_LIB") or os.path.join(_PKG, "libdgnn.so")  # DGNN_LIB: A/B builds

P = ctypes.c_void_p
i32, i64, u32, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64

DGNN_OK, DGNN_EINVAL, DGNN_ERANGE, DGNN_ENOMEM, DGNN_ECUDA, DGNN_ECOMM, DGNN_EIO, DGNN_EUNSUPPORTED = range(8)
STATUS_NAMES = ["OK", "EINVAL", "ERANGE", "ENOMEM", "ECUDA", "ECOMM", "EIO", "EUNSUPPORTED"]
TIER_GPU, TIER_HOST, TIER_DISK = 0, 1, 2
TIER_SHIFT = 30
SLOT_MASK = (1 << TIER_SHIFT) - 1
KERNELS = ["scan", "sample_seed", "sample_hop", "sample_order", "sample_remap", "sample_compact", "sample_setup",
           "cache_hist", "cache_select", "classify", "pack_gather", "tier_gather", "assemble", "misc", "sort", "disk_plan", "disk_gather", "train",
           "host_window", "host_gather", "tier_gather_pcie", "graph_io", "sample_dedup", "sample_count"]
K = {name: i for i, name in enumerate(KERNELS)}
CALLBACKS = [0]  # allocator callbacks from the library into Python (each needs the GIL)

# every symbol include/dgnn.h declares (checked by tests/test_abi_symbols.py)
EXPORTS = [
    "dgnn_ctx_create", "dgnn_ctx_destroy", "dgnn_ctx_set_stream", "dgnn_ctx_stream", "dgnn_ctx_side_stream",
    "dgnn_ctx_sync", "dgnn_last_error", "dgnn_ctx_set_sample_group", "dgnn_ctx_launches", "dgnn_ctx_set_timing", "dgnn_ctx_set_timing_mask",
    "dgnn_ctx_kernel_stats", "dgnn_ctx_reset_stats", "dgnn_kernel_name", "dgnn_sample", "dgnn_samples_get_info",
    "dgnn_samples_free", "dgnn_build_cache", "dgnn_cache_plan_get_info", "dgnn_cache_plan_free", "dgnn_classify",
    "dgnn_chunk_layout", "dgnn_pack", "dgnn_gather_rows", "dgnn_stage_copy", "dgnn_stage_wait", "dgnn_stage_sync",
    "dgnn_host_alloc", "dgnn_host_free", "dgnn_assemble", "dgnn_assemble_group", "dgnn_ctx_set_assemble_occupancy",
    "dgnn_host_window", "dgnn_gather_rows_dev", "dgnn_stage_wait_stream", "dgnn_tier_shard_ids",
    "dgnn_shard_requests", "dgnn_scatter_rows", "dgnn_assemble_group_sharded", "dgnn_batch_tier_counts",
    "dgnn_file_open", "dgnn_file_close", "dgnn_stage_file_write", "dgnn_stage_file_read",
    "dgnn_disk_index_build", "dgnn_disk_index_free", "dgnn_disk_space", "dgnn_disk_search", "dgnn_disk_plan_build",
    "dgnn_disk_plan_get_info", "dgnn_disk_plan_free", "dgnn_disk_cache_fill", "dgnn_disk_partial",
    "dgnn_train_stub", "dgnn_stage_file_read_pages", "dgnn_host_window_runs", "dgnn_gather_runs_dev", "dgnn_ctx_set_sample_mode", "dgnn_ctx_set_grid_cap", "dgnn_assemble_group_peer", "dgnn_device_alloc",
    "dgnn_device_free", "dgnn_ipc_handle", "dgnn_ipc_open", "dgnn_ipc_close", "dgnn_disk_index_partition_counts", "dgnn_pack_partition", "dgnn_pack_tails",
    "dgnn_ctx_set_keep_limit", "dgnn_ctx_kept_bytes", "dgnn_ctx_set_sample_budget", "dgnn_file_set_queues",
    "dgnn_chunk_layout_graph", "dgnn_pack_graph", "dgnn_samples_load", "dgnn_samples_drop_device",
    "dgnn_host_order", "dgnn_host_order_ranges", "dgnn_host_window_ranges", "dgnn_copy_ranges", "dgnn_remap_ids_dev",
    "dgnn_pack_sharded", "dgnn_gather_rows_sharded", "dgnn_host_order_schedule", "dgnn_upload",
    "dgnn_gather_ranges", "dgnn_packing_groups", "dgnn_assembly_runs", "dgnn_assembly_tables",
]


class DgnnError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{fn} -> DGNN_{name}: {msg}")
        self.status = status


class _CSR(ctypes.Structure):
    _fields_ = [("num_nodes", i64), ("num_edges", i64), ("indptr", P), ("indices", P)]


class _SamplesInfo(ctypes.Structure):
    _fields_ = [("num_batches", i64), ("num_hops", i32), ("batch_id_base", i64), ("total_nodes", i64),
                ("total_edges", i64), ("total_eptr", i64), ("node_off", P), ("nodes", P), ("hop_off", P),
                ("eptr_off", P), ("eptr", P), ("edge_off", P), ("src_local", P), ("node_off_host", P),
                ("edge_off_host", P), ("eptr_off_host", P), ("hop_off_host", P), ("mode", i32)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("num_nodes", i64), ("k_gpu", i64), ("k_host", i64), ("tier_map", P), ("gpu_ids", P),
                ("host_ids", P), ("gpu_min_count", u32), ("host_min_count", u32)]


class _DiskPlanInfo(ctypes.Structure):
    _fields_ = [(n, i64) for n in ("nb", "nseg", "s", "m", "fpp", "row_bytes", "n_cache", "n_packed", "n_req",
                                   "space_pages", "io_pages", "cache_pages", "chunk_pages")] + \
               [(n, P) for n in ("seg_off", "cache_ids", "seg_page_off", "pk_ids", "pk_off", "req_pages", "req_off",
                                 "dc_addr", "pk_off_host", "req_off_host", "seg_off_host", "seg_page_off_host")]


class _KStat(ctypes.Structure):
    _fields_ = [("launches", i64), ("ms", ctypes.c_double), ("bytes", ctypes.c_double)]


_ALLOC_FN = ctypes.CFUNCTYPE(P, ctypes.c_size_t, P, P)
_FREE_FN = ctypes.CFUNCTYPE(None, P, ctypes.c_size_t, P, P)


class _Allocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("user", P)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libdgnn.so and declare its signatures (no GPU needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `python paper_2405_05231_b200/build.py` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        sig = {
            "dgnn_ctx_create": (i32, [ctypes.c_int, P, P, ctypes.POINTER(P)]),
            "dgnn_ctx_destroy": (None, [P]),
            "dgnn_ctx_set_stream": (i32, [P, P]),
            "dgnn_ctx_stream": (P, [P]),
            "dgnn_ctx_side_stream": (P, [P]),
            "dgnn_ctx_sync": (i32, [P]),
            "dgnn_last_error": (ctypes.c_char_p, []),
            "dgnn_ctx_set_sample_group": (i32, [P, i32]),
            "dgnn_ctx_set_keep_limit": (i32, [P, i64]),
            "dgnn_ctx_kept_bytes": (i64, [P]),
            "dgnn_ctx_set_sample_budget": (i32, [P, i64]),
            "dgnn_ctx_launches": (i64, [P]),
            "dgnn_ctx_set_timing": (i32, [P, ctypes.c_int]),
            "dgnn_ctx_set_timing_mask": (i32, [P, u64]),
            "dgnn_ctx_kernel_stats": (i32, [P, i32, ctypes.POINTER(_KStat)]),
            "dgnn_ctx_reset_stats": (i32, [P]),
            "dgnn_kernel_name": (ctypes.c_char_p, [i32]),
            "dgnn_sample": (i32, [P, ctypes.POINTER(_CSR), P, i64, i32, i64, P, i32, u64, P, ctypes.POINTER(P)]),
            "dgnn_samples_get_info": (i32, [P, ctypes.POINTER(_SamplesInfo)]),
            "dgnn_samples_free": (None, [P]),
            "dgnn_build_cache": (i32, [P, P, i64, i64, i64, ctypes.POINTER(P)]),
            "dgnn_cache_plan_get_info": (i32, [P, ctypes.POINTER(_PlanInfo)]),
            "dgnn_cache_plan_free": (None, [P]),
            "dgnn_classify": (i32, [P, P, P, i64, i64, P, P, P, P]),
            "dgnn_chunk_layout": (i32, [P, i64, i64, P]),
            "dgnn_batch_tier_counts": (i32, [P, P, i64, i64, P, P]),
            "dgnn_file_open": (i32, [ctypes.c_char_p, i32, i32, i64, ctypes.POINTER(P)]),
            "dgnn_file_close": (i32, [P]),
            "dgnn_file_set_queues": (i32, [P, i32]),
            "dgnn_chunk_layout_graph": (i32, [P, i64, P, i64, i64, P, P]),
            "dgnn_pack_graph": (i32, [P, P, i64, i64, P, P]),
            "dgnn_samples_load": (i32, [P, P, i64, i64, P, P, ctypes.POINTER(P)]),
            "dgnn_samples_drop_device": (i32, [P]),
            "dgnn_host_order": (i32, [P, P, P, i32, P, i64, P, P, P, i64, P, P, ctypes.POINTER(i64)]),
            "dgnn_host_order_ranges": (i32, [P, P, i64, i64, i32, P, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
            "dgnn_host_window_ranges": (i32, [P, P, P, i64, i32, P, i64, P]),
            "dgnn_copy_ranges": (i32, [P, P, P, P, i64, i64]),
            "dgnn_upload": (i32, [P, P, P, i64]),
            "dgnn_packing_groups": (i32, [P, i64, i64, i64, i64, P, ctypes.POINTER(i64)]),
            "dgnn_assembly_runs": (i32, [P, i64, i64, i64, P, ctypes.POINTER(i64)]),
            "dgnn_assembly_tables": (i32, [P, P, P, P, P, i64, i64, i64, P, i64, P, i64, P, P]),
            "dgnn_gather_ranges": (i32, [P, P, i64, P, P, P, i64, i64, P]),
            "dgnn_remap_ids_dev": (i32, [P, P, P, i64, P]),
            "dgnn_host_order_schedule": (i32, [P, P, i64, i64, i32, i64, P, i64, P, P, i64, P,
                                                ctypes.POINTER(i64)]),
            "dgnn_pack_sharded": (i32, [P, P, i64, i32, i64, P, P, P, i64, i64, i64, P]),
            "dgnn_gather_rows_sharded": (i32, [P, P, i64, i32, i64, P, i64, P]),
            "dgnn_stage_file_write": (i32, [P, P, i64, P, i64, P, i64, ctypes.POINTER(i64)]),
            "dgnn_stage_file_read": (i32, [P, P, i64, P, i64, P, i64, ctypes.POINTER(i64)]),
            "dgnn_pack": (i32, [P, P, i64, i64, P, P, P, i64, i64, i64, P]),
            "dgnn_gather_rows": (i32, [P, P, i64, i64, P, i64, P]),
            "dgnn_stage_copy": (i32, [P, P, P, i64, i32, ctypes.POINTER(i64)]),
            "dgnn_stage_wait": (i32, [P, i64]),
            "dgnn_stage_wait_stream": (i32, [P, i64, P]),
            "dgnn_stage_sync": (i32, [P, i64]),
            "dgnn_host_alloc": (i32, [i64, ctypes.POINTER(P)]),
            "dgnn_host_free": (i32, [P]),
            "dgnn_assemble": (i32, [P, P, i64, P, i64, P, i64, P, i64, i64, P]),
            "dgnn_assemble_group": (i32, [P, P, P, i64, i64, P, i64, P, i64, P, P, P, P, i64, P]),
            "dgnn_host_window": (i32, [P, P, i64, i32, P, i64, P, i64, P, P]),
            "dgnn_tier_shard_ids": (i32, [P, P, i64, i32, i32, P, ctypes.POINTER(i64)]),
            "dgnn_shard_requests": (i32, [P, P, i64, i64, i32, i32, P, P, P]),
            "dgnn_scatter_rows": (i32, [P, P, i64, i64, P, P]),
            "dgnn_assemble_group_sharded": (i32, [P, P, P, i64, i64, P, i64, i32, i32, P, i64, P, P, P, P, i64, P]),
            "dgnn_gather_rows_dev": (i32, [P, P, i64, i64, P, P, i64, P]),
            "dgnn_ctx_set_assemble_occupancy": (i32, [P, i32]),
            "dgnn_disk_index_build": (i32, [P, P, P, P, i64, i64, ctypes.POINTER(P)]),
            "dgnn_disk_index_free": (None, [P]),
            "dgnn_disk_space": (i32, [P, P, i64, P, i64, i64, P]),
            "dgnn_disk_search": (i32, [P, P, i64, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
            "dgnn_disk_plan_build": (i32, [P, P, i64, i64, i64, i32, u64, i32, ctypes.POINTER(P)]),
            "dgnn_disk_plan_get_info": (i32, [P, ctypes.POINTER(_DiskPlanInfo)]),
            "dgnn_disk_plan_free": (None, [P]),
            "dgnn_disk_cache_fill": (i32, [P, P, P, i64, P]),
            "dgnn_disk_partial": (i32, [P, P, i64, i64, P, P, P, P, P]),
            "dgnn_train_stub": (i32, [P, P, i64, i64, P, i64]),
            "dgnn_ctx_set_sample_mode": (i32, [P, i32]),
            "dgnn_host_window_runs": (i32, [P, P, i64, i32, P, P, P]),
            "dgnn_gather_runs_dev": (i32, [P, P, i64, P, P, P, P, i64, P]),
            "dgnn_stage_file_read_pages": (i32, [P, P, i64, P, i64, P, P, i64, i32, ctypes.POINTER(i64)]),
            "dgnn_ctx_set_grid_cap": (i32, [P, i32]),
            "dgnn_assemble_group_peer": (i32, [P, P, P, i64, i64, P, i64, i32, P, i64, P, P, P, P, i64, P]),
            "dgnn_device_alloc": (i32, [i32, i64, ctypes.POINTER(P)]),
            "dgnn_device_free": (i32, [P]),
            "dgnn_ipc_handle": (i32, [P, P]),
            "dgnn_ipc_open": (i32, [i32, P, ctypes.POINTER(P)]),
            "dgnn_ipc_close": (i32, [P]),
            "dgnn_disk_index_partition_counts": (i32, [P, P, i64, i64, P]),
            "dgnn_pack_partition": (i32, [P, P, P, i64, i64, i64, P, P]),
            "dgnn_pack_tails": (i32, [P, P, i64, P, P]),
        }
        # Enqueue-only entry points (kernel launches, async copies, stream waits: they never wait
        # for the device or another thread) are called through a PyDLL handle, which keeps the
        # GIL across the call.  Releasing it for a few microseconds would make the calling thread
        # queue for it again behind the other host thread (the layout and the assembly are
        # enqueued by two threads): up to a switch interval per call, hundreds of calls per pass.
        # Calls that synchronize (sizes read back, dgnn_sample, ...) keep releasing the GIL.
        LP = ctypes.PyDLL(path) if os.environ.get("DGNN_PYDLL", "1") == "1" else None
        for name, (res, args) in sig.items():
            f = getattr(LP if (LP is not None and name in _ENQUEUE_ONLY) else L, name)
            f.restype = res
            f.argtypes = args
            setattr(L, name, f)
        _lib = L
        return L


# entry points that only enqueue work on streams (no synchronization, no host waits); see load_library
_ENQUEUE_ONLY = frozenset([
    "dgnn_assemble_group", "dgnn_assemble_group_peer", "dgnn_assemble_group_sharded", "dgnn_copy_ranges", "dgnn_upload",
    "dgnn_gather_ranges",
    "dgnn_host_window_ranges", "dgnn_host_window", "dgnn_remap_ids_dev", "dgnn_stage_wait",
    "dgnn_stage_wait_stream", "dgnn_stage_copy", "dgnn_gather_rows", "dgnn_gather_rows_dev", "dgnn_pack",
    "dgnn_ctx_launches", "dgnn_ctx_stream", "dgnn_ctx_side_stream", "dgnn_last_error", "dgnn_kernel_name",
])


def _check(status: int, fn: str):
    if status != DGNN_OK:
        msg = load_library().dgnn_last_error()
        raise DgnnError(status, fn, msg.decode() if msg else "")


def _ptr(t) -> P:
    if t is None:
        return P(0)
    if isinstance(t, int):
        return P(t)
    if isinstance(t, torch.Tensor):
        if t.numel() and not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return P(t.data_ptr() if t.numel() else 0)
    raise TypeError(type(t))


def _need_cuda(t: torch.Tensor, name: str, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


# ---------------------------------------------------------------- views
class _DevView:
    """Zero-copy __cuda_array_interface__ over library-owned memory; keeps the owner alive."""

    _TYPESTR = {torch.int32: "<i4", torch.int64: "<i8", torch.uint32: "<u4", torch.uint8: "|u1"}

    def __init__(self, ptr: int, n: int, dtype, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": self._TYPESTR[dtype],
                                         "data": (int(ptr) if n else 0, False), "version": 3, "strides": None,
                                         "stream": None}


class _Handle:
    """Owns one library handle.  The zero-copy views of a result reference this object, not the
    Python wrapper that stores them: wrapper -> views -> handle has no reference cycle, so the
    library memory is released as soon as the wrapper and its views are dropped, not at the next
    full cyclic garbage collection (which let whole epochs of samples pile up in HBM)."""

    def __init__(self, free_fn, handle, ctx=None):
        self.handle = handle
        # the ctx is an argument of the finalizer: it outlives every result allocated through it
        self.free = weakref.finalize(self, free_fn, handle) if ctx is None else \
            weakref.finalize(self, _free_with_ctx, free_fn, handle, ctx)


def _free_with_ctx(free_fn, handle, ctx):
    free_fn(handle)


def _view(ptr: int, n: int, dtype, owner, device) -> torch.Tensor:
    if n == 0:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_DevView(ptr, n, dtype, owner), device=device)


def _host_array(ptr: int, n: int, ctype):
    import numpy as np
    if n == 0:
        return np.zeros(0, dtype=np.dtype(ctype))
    return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), (n,)).copy()


# ------------------------------------------------------------------ context
class Ctx:
    """A dgnn_ctx bound to one device and a CUDA stream (default: torch's current stream).

    Library-owned buffers are allocated from torch's caching allocator unless
    ``torch_allocator=False`` (then cudaMallocAsync).
    """

    def __init__(self, device=None, stream: torch.cuda.Stream | None = None, torch_allocator: bool = True):
        L = load_library()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._alloc = None
        alloc_p = P(0)
        if torch_allocator:
            dev = self.device.index

            def _a(nbytes, stream, user):
                CALLBACKS[0] += 1
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0))
                except Exception:
                    return None

            def _f(ptr, nbytes, stream, user):
                CALLBACKS[0] += 1
                try:
                    torch.cuda.caching_allocator_delete(int(ptr))
                except Exception:
                    pass

            self._alloc = _Allocator(_ALLOC_FN(_a), _FREE_FN(_f), P(0))
            alloc_p = ctypes.cast(ctypes.pointer(self._alloc), P)
        h = P()
        _check(L.dgnn_ctx_create(self.device.index, P(self.stream.cuda_stream), alloc_p, ctypes.byref(h)),
               "dgnn_ctx_create")
        self.handle = h
        self._finalizer = weakref.finalize(self, L.dgnn_ctx_destroy, h)

    def close(self):
        self._finalizer()

    # statistics -------------------------------------------------------
    def launches(self) -> int:
        return int(load_library().dgnn_ctx_launches(self.handle))

    def set_timing(self, on: bool):
        _check(load_library().dgnn_ctx_set_timing(self.handle, int(bool(on))), "dgnn_ctx_set_timing")

    def set_timing_mask(self, kinds=None):
        """Time only these kernel families (names of KERNELS) when timing is on; None = all."""
        mask = (1 << 64) - 1 if kinds is None else sum(1 << K[k] for k in kinds)
        _check(load_library().dgnn_ctx_set_timing_mask(self.handle, mask), "dgnn_ctx_set_timing_mask")

    def kernel_stats(self) -> dict:
        out = {}
        for name, kid in K.items():
            s = _KStat()
            _check(load_library().dgnn_ctx_kernel_stats(self.handle, kid, ctypes.byref(s)), "dgnn_ctx_kernel_stats")
            out[name] = {"launches": int(s.launches), "ms": float(s.ms), "bytes": float(s.bytes)}
        return out

    def reset_stats(self):
        _check(load_library().dgnn_ctx_reset_stats(self.handle), "dgnn_ctx_reset_stats")

    def sync(self):
        _check(load_library().dgnn_ctx_sync(self.handle), "dgnn_ctx_sync")

    def set_assemble_occupancy(self, blocks_per_sm: int):
        _check(load_library().dgnn_ctx_set_assemble_occupancy(self.handle, int(blocks_per_sm)),
               "dgnn_ctx_set_assemble_occupancy")

    def set_sample_group(self, batches: int):
        _check(load_library().dgnn_ctx_set_sample_group(self.handle, int(batches)), "dgnn_ctx_set_sample_group")

    def set_keep_limit(self, nbytes: int):
        """Bytes of recycled sample arenas / sampler scratch the ctx may keep (dgnn_ctx_set_keep_limit)."""
        _check(load_library().dgnn_ctx_set_keep_limit(self.handle, int(nbytes)), "dgnn_ctx_set_keep_limit")

    def kept_bytes(self) -> int:
        return int(load_library().dgnn_ctx_kept_bytes(self.handle))

    def set_sample_budget(self, nbytes: int):
        """Scratch budget of one sampling group (dgnn_ctx_set_sample_budget)."""
        _check(load_library().dgnn_ctx_set_sample_budget(self.handle, int(nbytes)), "dgnn_ctx_set_sample_budget")

    def set_grid_cap(self, max_blocks: int):
        """Cap every grid this ctx launches (0 = none); see dgnn_ctx_set_grid_cap."""
        _check(load_library().dgnn_ctx_set_grid_cap(self.handle, int(max_blocks)), "dgnn_ctx_set_grid_cap")

    def set_sample_mode(self, blocks: bool):
        """False: node-wise (reading c4, default); True: the DGL-block variant (reading c27)."""
        _check(load_library().dgnn_ctx_set_sample_mode(self.handle, int(bool(blocks))), "dgnn_ctx_set_sample_mode")

    @property
    def side_stream_ptr(self) -> int:
        return int(load_library().dgnn_ctx_side_stream(self.handle) or 0)


# ------------------------------------------------------------------ samples
class Samples:
    """Library-owned result of dgnn_sample (batch-major concatenated layout)."""

    def __init__(self, ctx: Ctx, handle):
        L = load_library()
        self.ctx = ctx
        self.handle = handle
        self._owner = _Handle(L.dgnn_samples_free, handle, ctx)
        self._finalizer = self._owner.free
        info = _SamplesInfo()
        _check(L.dgnn_samples_get_info(handle, ctypes.byref(info)), "dgnn_samples_get_info")
        self.num_batches = int(info.num_batches)
        self.num_hops = int(info.num_hops)
        self.batch_id_base = int(info.batch_id_base)
        self.total_nodes = int(info.total_nodes)
        self.total_edges = int(info.total_edges)
        nb, H = self.num_batches, self.num_hops
        dev = ctx.device
        self.node_off = _view(info.node_off, nb + 1, torch.int64, self._owner, dev)
        self.nodes = _view(info.nodes, self.total_nodes, torch.int32, self._owner, dev)
        self.hop_off = _view(info.hop_off, nb * (H + 2), torch.int32, self._owner, dev)
        self.eptr_off = _view(info.eptr_off, nb + 1, torch.int64, self._owner, dev)
        self.eptr = _view(info.eptr, int(info.total_eptr), torch.int32, self._owner, dev)
        self.edge_off = _view(info.edge_off, nb + 1, torch.int64, self._owner, dev)
        self.src_local = _view(info.src_local, self.total_edges, torch.int32, self._owner, dev)
        self.node_off_host = _host_array(info.node_off_host, nb + 1, ctypes.c_int64)
        self.edge_off_host = _host_array(info.edge_off_host, nb + 1, ctypes.c_int64)
        self.eptr_off_host = _host_array(info.eptr_off_host, nb + 1, ctypes.c_int64)
        self.hop_off_host = _host_array(info.hop_off_host, nb * (H + 2), ctypes.c_int32).reshape(nb, H + 2)
        self.blocks = bool(info.mode)

    def drop_device(self):
        """Free the nodes / eptr / src_local device arrays (dgnn_samples_drop_device); the host-side
        offsets stay (the layout's metadata, e.g. for the graph loader)."""
        _check(load_library().dgnn_samples_drop_device(self.handle), "dgnn_samples_drop_device")
        self.nodes = self.eptr = self.src_local = None

    def batch(self, b: int) -> dict:
        """Device views of batch b: nodes, hop_off (host), eptr, src_local."""
        n0, n1 = int(self.node_off_host[b]), int(self.node_off_host[b + 1])
        e0, e1 = int(self.edge_off_host[b]), int(self.edge_off_host[b + 1])
        p0, p1 = int(self.eptr_off_host[b]), int(self.eptr_off_host[b + 1])
        return {"bid": self.batch_id_base + b, "nodes": self.nodes[n0:n1], "hop_off": self.hop_off_host[b],
                "eptr": self.eptr[p0:p1], "src_local": self.src_local[e0:e1]}


def dgnn_sample(ctx: Ctx, indptr: torch.Tensor, indices: torch.Tensor, seeds: torch.Tensor, batch_size: int,
                fanout, rng_seed: int, batch_id_base: int = 0, counts: torch.Tensor | None = None) -> Samples:
    _need_cuda(indptr, "indptr", torch.int64)
    _need_cuda(indices, "indices", torch.int32)
    _need_cuda(seeds, "seeds", torch.int32)
    if counts is not None:
        _need_cuda(counts, "counts")
        if counts.dtype not in (torch.int32, torch.uint32) or counts.numel() != indptr.numel() - 1:
            raise ValueError("counts must be a 32-bit tensor of length num_nodes")
    fan = (ctypes.c_int32 * max(len(fanout), 1))(*[int(k) for k in fanout])
    csr = _CSR(indptr.numel() - 1, indices.numel(), _ptr(indptr), _ptr(indices))
    h = P()
    _check(load_library().dgnn_sample(ctx.handle, ctypes.byref(csr), _ptr(seeds), seeds.numel(), int(batch_size),
                                      int(batch_id_base), fan, len(fanout), int(rng_seed) & ((1 << 64) - 1),
                                      _ptr(counts), ctypes.byref(h)), "dgnn_sample")
    return Samples(ctx, h)


# --------------------------------------------------------------- cache plan
class CachePlan:
    def __init__(self, ctx: Ctx, handle):
        L = load_library()
        self.ctx = ctx
        self.handle = handle
        self._owner = _Handle(L.dgnn_cache_plan_free, handle, ctx)
        self._finalizer = self._owner.free
        info = _PlanInfo()
        _check(L.dgnn_cache_plan_get_info(handle, ctypes.byref(info)), "dgnn_cache_plan_get_info")
        self.num_nodes = int(info.num_nodes)
        self.k_gpu = int(info.k_gpu)
        self.k_host = int(info.k_host)
        self.gpu_min_count = int(info.gpu_min_count)
        self.host_min_count = int(info.host_min_count)
        dev = ctx.device
        self.tier_map = _view(info.tier_map, self.num_nodes, torch.int32, self._owner, dev)
        self.gpu_ids = _view(info.gpu_ids, self.k_gpu, torch.int32, self._owner, dev)
        self.host_ids = _view(info.host_ids, self.k_host, torch.int32, self._owner, dev)


def dgnn_build_cache(ctx: Ctx, counts: torch.Tensor, gpu_rows: int, host_rows: int) -> CachePlan:
    _need_cuda(counts, "counts")
    h = P()
    _check(load_library().dgnn_build_cache(ctx.handle, _ptr(counts), counts.numel(), int(gpu_rows), int(host_rows),
                                           ctypes.byref(h)), "dgnn_build_cache")
    return CachePlan(ctx, h)


# ------------------------------------------------------------ classify / pack
def dgnn_classify(ctx: Ctx, plan: CachePlan, samples: Samples, b_lo: int, b_hi: int, addr: torch.Tensor,
                  packed_ids: torch.Tensor, packed_off: torch.Tensor, want_host: bool = True):
    import numpy as np
    n = int(samples.node_off_host[b_hi] - samples.node_off_host[b_lo])
    _need_cuda(addr, "addr")
    _need_cuda(packed_ids, "packed_ids", torch.int32)
    _need_cuda(packed_off, "packed_off", torch.int64)
    if addr.numel() < n or packed_ids.numel() < n or packed_off.numel() < b_hi - b_lo + 1:
        raise ValueError("dgnn_classify: output buffers too small")
    host = np.zeros(b_hi - b_lo + 1, np.int64) if want_host else None
    _check(load_library().dgnn_classify(ctx.handle, plan.handle, samples.handle, b_lo, b_hi, _ptr(addr),
                                        _ptr(packed_ids), _ptr(packed_off),
                                        P(host.ctypes.data) if host is not None else P(0)), "dgnn_classify")
    return host


def dgnn_batch_tier_counts(ctx: Ctx, samples: Samples, b_lo: int, b_hi: int, addr: torch.Tensor):
    """-> int64 [b_hi-b_lo, 3]: rows of each tier (GPU, HOST, DISK) per batch."""
    import numpy as np
    out = np.zeros((max(b_hi - b_lo, 0), 3), np.int64)
    _check(load_library().dgnn_batch_tier_counts(ctx.handle, samples.handle, int(b_lo), int(b_hi), _ptr(addr),
                                                 P(out.ctypes.data) if out.size else P(0)), "dgnn_batch_tier_counts")
    return out


def dgnn_packing_groups(packed_off_host, row_bytes: int, group_size: int, group_budget: int):
    """-> [(b_lo, b_hi)] packing groups of consecutive batches (host arithmetic in the library)."""
    import numpy as np
    po = np.ascontiguousarray(packed_off_host, dtype=np.int64)
    nb = len(po) - 1
    lo = np.zeros(nb + 1, np.int64)
    n = i64()
    _check(load_library().dgnn_packing_groups(P(po.ctypes.data), nb, int(row_bytes), int(group_size),
                                              int(group_budget), P(lo.ctypes.data), ctypes.byref(n)),
           "dgnn_packing_groups")
    k = int(n.value)
    return [(int(lo[i]), int(lo[i + 1]) if i + 1 < k else nb) for i in range(k)]


def dgnn_assembly_runs(node_off_host, max_rows: int, max_batches: int = 1024):
    """-> [(b_lo, b_hi)] assembler runs of consecutive batches (host arithmetic in the library)."""
    import numpy as np
    no = np.ascontiguousarray(node_off_host, dtype=np.int64)
    nb = len(no) - 1
    lo = np.zeros(nb + 1, np.int64)
    n = i64()
    _check(load_library().dgnn_assembly_runs(P(no.ctypes.data), nb, int(max_rows), int(max_batches),
                                             P(lo.ctypes.data), ctypes.byref(n)), "dgnn_assembly_runs")
    k = int(n.value)
    return [(int(lo[i]), int(lo[i + 1]) if i + 1 < k else nb) for i in range(k)]


def dgnn_assembly_tables(node_off, chunk_start, chunk_rows, disk_rows, sec_abs, chunk_bytes: int, row_bytes: int,
                         runs):
    """-> (flat int64 tables back to back, their offsets [n_runs+1], spans [(n0, n1, c_lo, c_hi)]) of
    the assembler's runs (host arithmetic in the library; see dgnn.h)."""
    import numpy as np

    def arr(x):
        return None if x is None else np.ascontiguousarray(x, dtype=np.int64)
    no, cs, cr, dr, sc = arr(node_off), arr(chunk_start), arr(chunk_rows), arr(disk_rows), arr(sec_abs)
    nb = len(no) - 1
    lo = np.array([r[0] for r in runs] + ([runs[-1][1]] if runs else [0]), np.int64)
    k_tot = sum(b1 - b0 for b0, b1 in runs)
    cap = 4 * (k_tot + len(runs)) + 16
    tab = np.zeros(cap, np.int64)
    offs = np.zeros(len(runs) + 1, np.int64)
    spans = np.zeros(4 * max(len(runs), 1), np.int64)
    p = lambda a: P(a.ctypes.data) if a is not None else P(0)
    _check(load_library().dgnn_assembly_tables(p(no), p(cs), p(cr), p(dr), p(sc), nb, int(chunk_bytes),
                                               int(row_bytes), P(lo.ctypes.data), len(runs), P(tab.ctypes.data), cap,
                                               P(offs.ctypes.data), P(spans.ctypes.data)), "dgnn_assembly_tables")
    return tab[:int(offs[-1])].copy(), offs, [tuple(int(v) for v in spans[4 * r:4 * r + 4]) for r in range(len(runs))]


def dgnn_chunk_layout(packed_off_host, row_bytes: int):
    import numpy as np
    po = np.ascontiguousarray(packed_off_host, dtype=np.int64)
    out = np.zeros(len(po), np.int64)
    _check(load_library().dgnn_chunk_layout(P(po.ctypes.data), len(po) - 1, int(row_bytes), P(out.ctypes.data)),
           "dgnn_chunk_layout")
    return out


def dgnn_chunk_layout_graph(samples: Samples, b_lo: int, packed_off_host, row_bytes: int):
    """-> (chunk_off int64 [nb+1], sec_off int64 [nb]) with graph sections (reading c22b)."""
    import numpy as np
    po = np.ascontiguousarray(packed_off_host, dtype=np.int64)
    nb = len(po) - 1
    co = np.zeros(nb + 1, np.int64)
    so = np.zeros(max(nb, 1), np.int64)
    _check(load_library().dgnn_chunk_layout_graph(samples.handle, int(b_lo), P(po.ctypes.data), nb, int(row_bytes),
                                                  P(co.ctypes.data), P(so.ctypes.data)), "dgnn_chunk_layout_graph")
    return co, so[:nb]


def dgnn_pack_graph(ctx: Ctx, samples: Samples, b_lo: int, nb: int, sec_off_dev: torch.Tensor, group_buf):
    _check(load_library().dgnn_pack_graph(ctx.handle, samples.handle, int(b_lo), int(nb), _ptr(sec_off_dev),
                                          _ptr(group_buf)), "dgnn_pack_graph")


def dgnn_samples_load(ctx: Ctx, meta: Samples, b_lo: int, b_hi: int, base, sec_off_dev: torch.Tensor) -> Samples:
    """The graph loader: batches [b_lo, b_hi) of ``meta`` read back from staged chunks."""
    h = P()
    _check(load_library().dgnn_samples_load(ctx.handle, meta.handle, int(b_lo), int(b_hi), _ptr(base),
                                            _ptr(sec_off_dev), ctypes.byref(h)), "dgnn_samples_load")
    return Samples(ctx, h)


def dgnn_upload(ctx: Ctx, src, dtype=torch.int64) -> torch.Tensor:
    """A small host array (numpy) -> a new device tensor on ctx's stream, through kernel
    parameters (dgnn_upload), not the copy engines."""
    import numpy as np
    a = np.ascontiguousarray(src)
    with torch.cuda.stream(ctx.stream):
        out = torch.empty(a.size, dtype=dtype, device=ctx.device)
    if out.element_size() != a.itemsize:
        raise ValueError("dgnn_upload: dtype size mismatch")
    _check(load_library().dgnn_upload(ctx.handle, _ptr(out), P(a.ctypes.data), a.nbytes), "dgnn_upload")
    return out


def dgnn_gather_ranges(ctx: Ctx, table, row_bytes: int, ids: torch.Tensor, ranges_dev: torch.Tensor,
                       prefix_dev: torch.Tensor, nr: int, total_rows: int, dst):
    _check(load_library().dgnn_gather_ranges(ctx.handle, _ptr(table), int(row_bytes), _ptr(ids), _ptr(ranges_dev),
                                             _ptr(prefix_dev), int(nr), int(total_rows), _ptr(dst)),
           "dgnn_gather_ranges")


class HostOrder:
    """The window-ordered host tier of one layout (dgnn_host_order): device slot_mask / phys_of_slot
    / phys_ids, and per window its physical ranges (host triples + device copy)."""

    def __init__(self, ctx: Ctx, addr: torch.Tensor, win_node_off, host_ids: torch.Tensor, k_host: int,
                 max_groups: int = 4096):
        import numpy as np
        wo = np.ascontiguousarray(win_node_off, dtype=np.int64)
        self.nwin, self.k_host = len(wo) - 1, int(k_host)
        dev = ctx.device
        with torch.cuda.stream(ctx.stream):
            self.slot_mask = torch.empty(max(self.k_host, 1), dtype=torch.int32, device=dev)
            self.phys_of_slot = torch.empty(max(self.k_host, 1), dtype=torch.int32, device=dev)
            self.phys_ids = torch.empty(max(self.k_host, 1), dtype=torch.int32, device=dev)
        gs = np.zeros(max_groups, np.int64)
        gm = np.zeros(max_groups, np.uint32)
        ng = i64()
        _check(load_library().dgnn_host_order(ctx.handle, _ptr(addr), P(wo.ctypes.data), self.nwin, _ptr(host_ids),
                                              self.k_host, _ptr(self.phys_ids), _ptr(self.phys_of_slot),
                                              _ptr(self.slot_mask), int(max_groups), P(gs.ctypes.data),
                                              P(gm.ctypes.data), ctypes.byref(ng)), "dgnn_host_order")
        self.n_groups = int(ng.value)
        self.ranges, self.rows = [], []
        cap = max(self.n_groups, 1)
        for w in range(self.nwin):
            rg = np.zeros(3 * cap, np.int64)
            nr, rows = i64(), i64()
            _check(load_library().dgnn_host_order_ranges(P(gs.ctypes.data), P(gm.ctypes.data), self.n_groups,
                                                         self.k_host, w, P(rg.ctypes.data), cap, ctypes.byref(nr),
                                                         ctypes.byref(rows)), "dgnn_host_order_ranges")
            self.ranges.append(rg[:3 * int(nr.value)].copy())
            self.rows.append(int(rows.value))
        # the staging schedule: one arena of two windows' rows, but never more than the tier (the
        # rows resident at a prefetch are those windows w-1 and w need, each group once, so k_host
        # always fits); rows shared by consecutive windows are copied once, and spare room bridges the
        # gaps between a group's runs (dgnn_host_order_schedule)
        self.capacity = min(2 * max(self.rows), self.k_host) if self.rows else 0
        cap_t = 4 * cap * (self.nwin + 1) + 16
        co, mo = np.zeros(3 * cap_t, np.int64), np.zeros(3 * cap_t, np.int64)
        coff, moff = np.zeros(self.nwin + 1, np.int64), np.zeros(self.nwin + 1, np.int64)
        copied = i64()
        _check(load_library().dgnn_host_order_schedule(P(gs.ctypes.data), P(gm.ctypes.data), self.n_groups,
                                                       self.k_host, self.nwin, self.capacity, P(co.ctypes.data),
                                                       cap_t, P(coff.ctypes.data), P(mo.ctypes.data), cap_t,
                                                       P(moff.ctypes.data), ctypes.byref(copied)),
               "dgnn_host_order_schedule")
        self.rows_copied = int(copied.value)
        self._copies_dev = None
        self.copies = [co[3 * coff[w]:3 * coff[w + 1]].copy() for w in range(self.nwin)]
        self.copy_rows = [int((c[1::3] - c[0::3]).sum()) for c in self.copies]
        maps = [mo[3 * moff[w]:3 * moff[w + 1]].copy() for w in range(self.nwin)]
        self.map_len = [len(m) // 3 for m in maps]
        cat = np.concatenate(self.ranges + maps + [np.zeros(1, np.int64)]).astype(np.int64)
        flat = dgnn_upload(ctx, cat)
        offs = np.concatenate([[0], np.cumsum([len(r) for r in self.ranges + maps])])
        self.ranges_dev = [flat[int(offs[w]):int(offs[w + 1])] for w in range(self.nwin)]
        self.map_dev = [flat[int(offs[self.nwin + w]):int(offs[self.nwin + w + 1])] for w in range(self.nwin)]

    def copies_dev(self, ctx: Ctx):
        """Per window: (triples_dev, prefix_dev, n_triples, rows) of its scheduled copy list, for
        dgnn_gather_ranges (the tier read from the feature table); uploaded once, on ctx's stream."""
        import numpy as np
        if self._copies_dev is None:
            parts, meta = [], []
            for c in self.copies:
                c = np.ascontiguousarray(c, dtype=np.int64)
                pre = np.concatenate([[0], np.cumsum(c[1::3] - c[0::3])]).astype(np.int64)
                meta.append((len(c), len(pre), len(c) // 3, int(pre[-1])))
                parts += [c, pre]
            flat = dgnn_upload(ctx, np.concatenate(parts + [np.zeros(1, np.int64)]))
            out, o = [], 0
            for nc, npre, nr, rows in meta:
                out.append((flat[o:o + nc], flat[o + nc:o + nc + npre], nr, rows))
                o += nc + npre
            self._copies_dev = out
        return self._copies_dev


def dgnn_host_window_ranges(ctx: Ctx, ho: HostOrder, window: int, smap: torch.Tensor, scheduled: bool = True):
    """smap of window ``window``: into the scheduled arena (default) or the per-window ranges."""
    rg, n = (ho.map_dev[window], ho.map_len[window]) if scheduled else \
        (ho.ranges_dev[window], len(ho.ranges[window]) // 3)
    _check(load_library().dgnn_host_window_ranges(ctx.handle, _ptr(ho.slot_mask), _ptr(ho.phys_of_slot), ho.k_host,
                                                  int(window), _ptr(rg), n, _ptr(smap)), "dgnn_host_window_ranges")


def dgnn_copy_ranges(ctx: Ctx, dst, src_host_ptr: int, ranges, row_bytes: int):
    import numpy as np
    rg = np.ascontiguousarray(ranges, dtype=np.int64)
    _check(load_library().dgnn_copy_ranges(ctx.handle, _ptr(dst), P(src_host_ptr), P(rg.ctypes.data) if rg.size
                                           else P(0), len(rg) // 3, int(row_bytes)), "dgnn_copy_ranges")


def dgnn_remap_ids_dev(ctx: Ctx, ids: torch.Tensor, n_dev: torch.Tensor, table: torch.Tensor):
    _check(load_library().dgnn_remap_ids_dev(ctx.handle, _ptr(ids), _ptr(n_dev), ids.numel(), _ptr(table)),
           "dgnn_remap_ids_dev")


class ShardedFeatures:
    """A feature table partitioned by node range over ranks: rank r holds rows
    [r * shard_rows, min((r + 1) * shard_rows, num_rows)) in a DeviceBuffer; ``peers`` (device
    int64 [world]) points at every shard (this rank's own, the others' CUDA IPC mappings).  Passed as
    ``features`` to offline_layout / dgnn_pack / dgnn_gather_rows, which then read rows through it."""

    def __init__(self, shard: "DeviceBuffer", num_rows: int, shard_rows: int, dim: int, dtype, rank: int,
                 world: int, exchange):
        self.shard, self.num_rows, self.shard_rows, self.dim, self.dtype = shard, int(num_rows), int(shard_rows), \
            int(dim), dtype
        self.rank, self.world = rank, world
        self.row_bytes = torch.empty(0, dtype=dtype).element_size() * self.dim
        dev = torch.device("cuda", shard.device)
        handles = exchange(shard.ipc_handle())
        self.maps, ptrs = [], []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(shard.ptr)
            else:
                m = IpcMapping(shard.device, h)
                self.maps.append(m)
                ptrs.append(m.ptr)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        self.shape = (self.num_rows, self.dim)

    @classmethod
    def loopback(cls, shards: list, num_rows: int, shard_rows: int, dim: int, dtype):
        """Every shard in this process (the single-GPU test of the sharded source)."""
        self = cls.__new__(cls)
        self.shard, self.shards, self.num_rows, self.shard_rows, self.dim, self.dtype = shards[0], shards, \
            int(num_rows), int(shard_rows), int(dim), dtype
        self.rank, self.world, self.maps = 0, len(shards), []
        self.row_bytes = torch.empty(0, dtype=dtype).element_size() * self.dim
        self.peers = torch.tensor([s.ptr for s in shards], dtype=torch.int64, device=torch.device("cuda", shards[0].device))
        self.shape = (self.num_rows, self.dim)
        return self


def dgnn_pack(ctx: Ctx, features, packed_ids: torch.Tensor, packed_off: torch.Tensor,
              chunk_off: torch.Tensor, total_rows: int, group_bytes: int, group_buf: torch.Tensor):
    if isinstance(features, ShardedFeatures):
        f = features
        _check(load_library().dgnn_pack_sharded(ctx.handle, _ptr(f.peers), f.shard_rows, f.world, f.row_bytes,
                                                _ptr(packed_ids), _ptr(packed_off), _ptr(chunk_off),
                                                chunk_off.numel() - 1, int(total_rows), int(group_bytes),
                                                _ptr(group_buf)), "dgnn_pack_sharded")
        return
    row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
    nb = chunk_off.numel() - 1
    _check(load_library().dgnn_pack(ctx.handle, _ptr(features), features.shape[0], row_bytes, _ptr(packed_ids),
                                    _ptr(packed_off), _ptr(chunk_off), nb, int(total_rows), int(group_bytes),
                                    _ptr(group_buf)), "dgnn_pack")


def dgnn_gather_rows(ctx: Ctx, features, ids: torch.Tensor, out):
    if isinstance(features, ShardedFeatures):
        f = features
        _check(load_library().dgnn_gather_rows_sharded(ctx.handle, _ptr(f.peers), f.shard_rows, f.world, f.row_bytes,
                                                       _ptr(ids), ids.numel(), _ptr(out)), "dgnn_gather_rows_sharded")
        return
    row_bytes = features.element_size() * (features.numel() // max(features.shape[0], 1))
    _check(load_library().dgnn_gather_rows(ctx.handle, _ptr(features), features.shape[0], row_bytes, _ptr(ids),
                                           ids.numel(), _ptr(out)), "dgnn_gather_rows")


# ------------------------------------------------------------------ staging
def dgnn_stage_copy(ctx: Ctx, dst, src, nbytes: int, kind: int) -> int:
    t = i64()
    _check(load_library().dgnn_stage_copy(ctx.handle, _ptr(dst), _ptr(src), int(nbytes), int(kind), ctypes.byref(t)),
           "dgnn_stage_copy")
    return int(t.value)


class DiskFile:
    """The disk tier as a file (dgnn_file_open); O_DIRECT by default."""

    def __init__(self, path: str, size: int, direct: bool = True, create: bool = True):
        h = P()
        _check(load_library().dgnn_file_open(path.encode(), int(direct), int(create), int(size), ctypes.byref(h)),
               "dgnn_file_open")
        self.handle, self.path, self.direct, self.size = h, path, direct, size
        self._finalizer = weakref.finalize(self, load_library().dgnn_file_close, h)

    def set_queues(self, queues: int):
        """I/O queues (worker threads) of the file's engine, before its first transfer."""
        _check(load_library().dgnn_file_set_queues(self.handle, int(queues)), "dgnn_file_set_queues")

    def close(self):
        self._finalizer()


def dgnn_stage_file_write(ctx: Ctx, f: DiskFile, file_off: int, dev_src, nbytes: int, bounce, chunk_bytes: int):
    t = i64()
    _check(load_library().dgnn_stage_file_write(ctx.handle, f.handle, int(file_off), _ptr(dev_src), int(nbytes),
                                                _ptr(bounce), int(chunk_bytes), ctypes.byref(t)),
           "dgnn_stage_file_write")
    return int(t.value)


def dgnn_stage_file_read(ctx: Ctx, f: DiskFile, file_off: int, dev_dst, nbytes: int, bounce, chunk_bytes: int):
    t = i64()
    _check(load_library().dgnn_stage_file_read(ctx.handle, f.handle, int(file_off), _ptr(dev_dst), int(nbytes),
                                               _ptr(bounce), int(chunk_bytes), ctypes.byref(t)),
           "dgnn_stage_file_read")
    return int(t.value)


def dgnn_stage_wait(ctx: Ctx, ticket: int):
    _check(load_library().dgnn_stage_wait(ctx.handle, int(ticket)), "dgnn_stage_wait")


def dgnn_stage_wait_stream(ctx: Ctx, ticket: int, stream: torch.cuda.Stream):
    _check(load_library().dgnn_stage_wait_stream(ctx.handle, int(ticket), P(stream.cuda_stream)),
           "dgnn_stage_wait_stream")


def dgnn_stage_sync(ctx: Ctx, ticket: int):
    _check(load_library().dgnn_stage_sync(ctx.handle, int(ticket)), "dgnn_stage_sync")


# ----------------------------------------------------------------- assemble
def dgnn_assemble(ctx: Ctx, addr: torch.Tensor, gpu_tier, k_gpu: int, host_tier, k_host: int, chunk,
                  chunk_rows: int, row_bytes: int, out: torch.Tensor):
    _check(load_library().dgnn_assemble(ctx.handle, _ptr(addr), addr.numel(), _ptr(gpu_tier), int(k_gpu),
                                        _ptr(host_tier), int(k_host), _ptr(chunk), int(chunk_rows), int(row_bytes),
                                        _ptr(out)), "dgnn_assemble")


def dgnn_assemble_group(ctx: Ctx, addr: torch.Tensor, node_off: torch.Tensor, n: int, gpu_tier, k_gpu: int,
                        host_tier, k_host: int, chunk_base, chunk_off: torch.Tensor, chunk_rows: torch.Tensor,
                        row_bytes: int, out, host_map=None):
    _check(load_library().dgnn_assemble_group(ctx.handle, _ptr(addr), _ptr(node_off), node_off.numel() - 1, int(n),
                                              _ptr(gpu_tier), int(k_gpu), _ptr(host_tier), int(k_host),
                                              _ptr(host_map), _ptr(chunk_base), _ptr(chunk_off), _ptr(chunk_rows),
                                              int(row_bytes), _ptr(out)), "dgnn_assemble_group")


def dgnn_assemble_group_sharded(ctx: Ctx, addr: torch.Tensor, node_off: torch.Tensor, n: int, gpu_shard, k_gpu: int,
                                rank: int, world: int, host_tier, k_host: int, chunk_base, chunk_off: torch.Tensor,
                                chunk_rows: torch.Tensor, row_bytes: int, out, host_map=None):
    _check(load_library().dgnn_assemble_group_sharded(
        ctx.handle, _ptr(addr), _ptr(node_off), node_off.numel() - 1, int(n), _ptr(gpu_shard), int(k_gpu), int(rank),
        int(world), _ptr(host_tier), int(k_host), _ptr(host_map), _ptr(chunk_base), _ptr(chunk_off),
        _ptr(chunk_rows), int(row_bytes), _ptr(out)), "dgnn_assemble_group_sharded")


def dgnn_tier_shard_ids(ctx: Ctx, gpu_ids: torch.Tensor, k_gpu: int, rank: int, world: int) -> torch.Tensor:
    n_local = max(0, (k_gpu - rank + world - 1) // world) if k_gpu > rank else 0
    with torch.cuda.stream(ctx.stream):
        ids = torch.empty(max(n_local, 1), dtype=torch.int32, device=ctx.device)
    nl = i64()
    _check(load_library().dgnn_tier_shard_ids(ctx.handle, _ptr(gpu_ids), int(k_gpu), int(rank), int(world),
                                              _ptr(ids), ctypes.byref(nl)), "dgnn_tier_shard_ids")
    return ids[:int(nl.value)]


def dgnn_shard_requests(ctx: Ctx, addr: torch.Tensor, k_gpu: int, rank: int, world: int):
    """-> (req_off_host int64 [world+1], req_slot, req_pos) grouped by owner rank."""
    import numpy as np
    n = addr.numel()
    with torch.cuda.stream(ctx.stream):
        req_slot = torch.empty(max(n, 1), dtype=torch.int32, device=ctx.device)
        req_pos = torch.empty(max(n, 1), dtype=torch.int32, device=ctx.device)
    off = np.zeros(world + 1, np.int64)
    _check(load_library().dgnn_shard_requests(ctx.handle, _ptr(addr), n, int(k_gpu), int(rank), int(world),
                                              P(off.ctypes.data), _ptr(req_slot), _ptr(req_pos)),
           "dgnn_shard_requests")
    return off, req_slot[:int(off[-1])], req_pos[:int(off[-1])]


def dgnn_scatter_rows(ctx: Ctx, rows, n: int, row_bytes: int, pos: torch.Tensor, out):
    _check(load_library().dgnn_scatter_rows(ctx.handle, _ptr(rows), int(n), int(row_bytes), _ptr(pos), _ptr(out)),
           "dgnn_scatter_rows")


def dgnn_host_window(ctx: Ctx, addr: torch.Tensor, window_id: int, stamp: torch.Tensor, k_host: int,
                     list_: torch.Tensor, smap: torch.Tensor, count: torch.Tensor):
    _check(load_library().dgnn_host_window(ctx.handle, _ptr(addr), addr.numel(), int(window_id), _ptr(stamp),
                                           int(k_host), _ptr(list_), list_.numel(), _ptr(smap), _ptr(count)),
           "dgnn_host_window")


def dgnn_gather_rows_dev(ctx: Ctx, features, num_rows: int, row_bytes: int, ids: torch.Tensor, n_dev: torch.Tensor,
                         out):
    _check(load_library().dgnn_gather_rows_dev(ctx.handle, _ptr(features), int(num_rows), int(row_bytes), _ptr(ids),
                                               _ptr(n_dev), ids.numel(), _ptr(out)), "dgnn_gather_rows_dev")


# ------------------------------------------------- segmented disk cache ----
class DiskIndex:
    """An epoch's packed lists sorted by (node, batch) on the device (dgnn_disk_index_build)."""

    def __init__(self, ctx: Ctx, packed_ids: torch.Tensor, packed_off: torch.Tensor, packed_off_host, num_nodes: int):
        import numpy as np
        L = load_library()
        _need_cuda(packed_ids, "packed_ids", torch.int32)
        _need_cuda(packed_off, "packed_off", torch.int64)
        po = np.ascontiguousarray(packed_off_host, dtype=np.int64)
        self.ctx = ctx
        self.nb = len(po) - 1
        self.packed_off_host = po.copy()
        h = P()
        _check(L.dgnn_disk_index_build(ctx.handle, _ptr(packed_ids), _ptr(packed_off), P(po.ctypes.data), self.nb,
                                       int(num_nodes), ctypes.byref(h)), "dgnn_disk_index_build")
        self.handle = h
        self._finalizer = weakref.finalize(self, L.dgnn_disk_index_free, h)


def dgnn_disk_space(ctx: Ctx, idx: DiskIndex, row_bytes: int, s_list, m: int):
    import numpy as np
    sl = np.ascontiguousarray(s_list, dtype=np.int64)
    out = np.zeros(len(sl), np.int64)
    _check(load_library().dgnn_disk_space(ctx.handle, idx.handle, int(row_bytes), P(sl.ctypes.data) if sl.size else P(0),
                                          len(sl), int(m), P(out.ctypes.data) if out.size else P(0)),
           "dgnn_disk_space")
    return out


def dgnn_disk_search(ctx: Ctx, idx: DiskIndex, row_bytes: int, budget_pages: int, m: int = 1):
    s = i64()
    pg = i64()
    _check(load_library().dgnn_disk_search(ctx.handle, idx.handle, int(row_bytes), int(m), int(budget_pages),
                                           ctypes.byref(s), ctypes.byref(pg)), "dgnn_disk_search")
    return int(s.value), int(pg.value)


class DiskPlan:
    """Segmented disk cache plan (readings d1-d8); zero-copy device views + host offsets."""

    def __init__(self, ctx: Ctx, handle, R: int):
        L = load_library()
        self.ctx = ctx
        self.handle = handle
        self._owner = _Handle(L.dgnn_disk_plan_free, handle, ctx)
        self._finalizer = self._owner.free
        info = _DiskPlanInfo()
        _check(L.dgnn_disk_plan_get_info(handle, ctypes.byref(info)), "dgnn_disk_plan_get_info")
        for n in ("nb", "nseg", "s", "m", "fpp", "row_bytes", "n_cache", "n_packed", "n_req", "space_pages",
                  "io_pages", "cache_pages", "chunk_pages"):
            setattr(self, n, int(getattr(info, n)))
        dev = ctx.device
        nb, nseg = self.nb, self.nseg
        self.seg_off = _view(info.seg_off, nseg + 1, torch.int64, self._owner, dev)
        self.cache_ids = _view(info.cache_ids, self.n_cache, torch.int32, self._owner, dev)
        self.seg_page_off = _view(info.seg_page_off, nseg + 1, torch.int64, self._owner, dev)
        self.pk_ids = _view(info.pk_ids, self.n_packed, torch.int32, self._owner, dev)
        self.pk_off = _view(info.pk_off, nb + 1, torch.int64, self._owner, dev)
        self.req_pages = _view(info.req_pages, self.n_req, torch.int32, self._owner, dev)
        self.req_off = _view(info.req_off, nb + 1, torch.int64, self._owner, dev)
        self.dc_addr = _view(info.dc_addr, R, torch.uint32, self._owner, dev)
        self.pk_off_host = _host_array(info.pk_off_host, nb + 1, ctypes.c_int64)
        self.req_off_host = _host_array(info.req_off_host, nb + 1, ctypes.c_int64)
        self.seg_off_host = _host_array(info.seg_off_host, nseg + 1, ctypes.c_int64)
        self.seg_page_off_host = _host_array(info.seg_page_off_host, nseg + 1, ctypes.c_int64)


def dgnn_disk_plan_build(ctx: Ctx, idx: DiskIndex, row_bytes: int, s: int, m: int, k: int = 4, seed: int = 0,
                         reorder: bool = True, literal: bool = False) -> DiskPlan:
    """``literal``: Algorithm 1 line 8 as printed (scalar MinHash over the k functions)."""
    h = P()
    _check(load_library().dgnn_disk_plan_build(ctx.handle, idx.handle, int(row_bytes), int(s), int(m), int(k),
                                               int(seed) & (2**64 - 1), (2 if literal else 1) if reorder else 0,
                                               ctypes.byref(h)),
           "dgnn_disk_plan_build")
    return DiskPlan(ctx, h, int(idx.packed_off_host[-1]))


def dgnn_disk_cache_fill(ctx: Ctx, plan: DiskPlan, features: torch.Tensor, out):
    _check(load_library().dgnn_disk_cache_fill(ctx.handle, plan.handle, _ptr(features), features.shape[0], _ptr(out)),
           "dgnn_disk_cache_fill")


def dgnn_disk_partial(ctx: Ctx, plan: DiskPlan, b_lo: int, b_hi: int, pages, chunks, chunk_off: torch.Tensor, out,
                      out_off: torch.Tensor):
    _check(load_library().dgnn_disk_partial(ctx.handle, plan.handle, int(b_lo), int(b_hi), _ptr(pages), _ptr(chunks),
                                            _ptr(chunk_off), _ptr(out), _ptr(out_off)), "dgnn_disk_partial")


# ------------------------------------------------------------ trainer stub ----
def dgnn_train_stub(ctx: Ctx, samples: Samples, b_lo: int, b_hi: int, x: torch.Tensor):
    """In place: x = the assembled fp32 rows of batches [b_lo, b_hi) ([n, dim]); afterwards each
    batch's seed rows hold h^H (reading t1)."""
    _need_cuda(x, "x", torch.float32)
    dim = x.shape[-1] if x.dim() > 1 else 1
    _check(load_library().dgnn_train_stub(ctx.handle, samples.handle, int(b_lo), int(b_hi), _ptr(x), int(dim)),
           "dgnn_train_stub")


# ------------------------------------------ batched packing from partitions ----
def dgnn_disk_index_partition_counts(ctx: Ctx, idx: DiskIndex, part_rows: int, nparts: int):
    import numpy as np
    out = np.zeros(max(int(nparts), 1), np.int64)
    _check(load_library().dgnn_disk_index_partition_counts(ctx.handle, idx.handle, int(part_rows), int(nparts),
                                                           P(out.ctypes.data)), "dgnn_disk_index_partition_counts")
    return out[:int(nparts)]


def dgnn_pack_partition(ctx: Ctx, idx: DiskIndex, part, p0: int, p1: int, row_bytes: int, chunk_off: torch.Tensor,
                        group_buf):
    _check(load_library().dgnn_pack_partition(ctx.handle, idx.handle, _ptr(part), int(p0), int(p1), int(row_bytes),
                                              _ptr(chunk_off), _ptr(group_buf)), "dgnn_pack_partition")


def dgnn_pack_tails(ctx: Ctx, idx: DiskIndex, row_bytes: int, chunk_off: torch.Tensor, group_buf):
    _check(load_library().dgnn_pack_tails(ctx.handle, idx.handle, int(row_bytes), _ptr(chunk_off), _ptr(group_buf)),
           "dgnn_pack_tails")


# ------------------------------------------------ one-sided peer-memory tier ----
IPC_HANDLE_BYTES = 64


def dgnn_assemble_group_peer(ctx: Ctx, addr: torch.Tensor, node_off: torch.Tensor, n: int, peers: torch.Tensor,
                             k_gpu: int, world: int, host_tier, k_host: int, chunk_base, chunk_off: torch.Tensor,
                             chunk_rows: torch.Tensor, row_bytes: int, out, host_map=None):
    """peers: device int64 [world] of shard base addresses (dgnn_device_alloc / dgnn_ipc_open)."""
    _check(load_library().dgnn_assemble_group_peer(
        ctx.handle, _ptr(addr), _ptr(node_off), node_off.numel() - 1, int(n), _ptr(peers), int(k_gpu), int(world),
        _ptr(host_tier), int(k_host), _ptr(host_map), _ptr(chunk_base), _ptr(chunk_off), _ptr(chunk_rows),
        int(row_bytes), _ptr(out)), "dgnn_assemble_group_peer")


class DeviceBuffer:
    """A plain cudaMalloc allocation (dgnn_device_alloc) that CUDA IPC can export."""

    def __init__(self, device: int, nbytes: int):
        L = load_library()
        p = P()
        _check(L.dgnn_device_alloc(int(device), int(nbytes), ctypes.byref(p)), "dgnn_device_alloc")
        self.ptr, self.nbytes, self.device = int(p.value or 0), int(nbytes), int(device)
        self._fin = weakref.finalize(self, L.dgnn_device_free, P(self.ptr))

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(load_library().dgnn_ipc_handle(P(self.ptr), buf), "dgnn_ipc_handle")
        return buf.raw

    def view(self, shape, dtype=torch.uint8) -> torch.Tensor:
        n = 1
        for d in shape:
            n *= int(d)
        return _view(self.ptr, n * torch.empty(0, dtype=dtype).element_size(), torch.uint8, self,
                     torch.device("cuda", self.device)).view(dtype).view(*shape)


class IpcMapping:
    """Another process's DeviceBuffer mapped into this one (dgnn_ipc_open)."""

    def __init__(self, device: int, handle: bytes):
        L = load_library()
        p = P()
        _check(L.dgnn_ipc_open(int(device), ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES),
                               ctypes.byref(p)), "dgnn_ipc_open")
        self.ptr = int(p.value or 0)
        self._fin = weakref.finalize(self, L.dgnn_ipc_close, P(self.ptr))


def dgnn_stage_file_read_pages(ctx: Ctx, f: DiskFile, base_off: int, pages, dev_dst, bounce, bounce_bytes: int,
                               threads: int = 4) -> int:
    """Read 4 KiB pages (host int32 page indices) of the file's cache region into dev_dst."""
    import numpy as np
    pg = np.ascontiguousarray(pages, dtype=np.int32)
    t = i64()
    _check(load_library().dgnn_stage_file_read_pages(ctx.handle, f.handle, int(base_off),
                                                     P(pg.ctypes.data) if pg.size else P(0), int(pg.size),
                                                     _ptr(dev_dst), _ptr(bounce), int(bounce_bytes), int(threads),
                                                     ctypes.byref(t)), "dgnn_stage_file_read_pages")
    return int(t.value)


def dgnn_host_window_runs(ctx: Ctx, stamp: torch.Tensor, k_host: int, window_id: int, smap: torch.Tensor,
                          runs: torch.Tensor, run_count: torch.Tensor):
    _check(load_library().dgnn_host_window_runs(ctx.handle, _ptr(stamp), int(k_host), int(window_id), _ptr(smap),
                                                _ptr(runs), _ptr(run_count)), "dgnn_host_window_runs")


def dgnn_gather_runs_dev(ctx: Ctx, src, row_bytes: int, lst: torch.Tensor, count: torch.Tensor, runs: torch.Tensor,
                         run_count: torch.Tensor, max_runs: int, out):
    _check(load_library().dgnn_gather_runs_dev(ctx.handle, _ptr(src), int(row_bytes), _ptr(lst), _ptr(count),
                                               _ptr(runs), _ptr(run_count), int(max_runs), _ptr(out)),
           "dgnn_gather_runs_dev")
