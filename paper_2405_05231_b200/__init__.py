"""B200-native DiskGNN offline hot path (arXiv 2405.05231).

The compute lives in ``libdgnn.so`` (hand-written CUDA for sm_100a behind the C
ABI in ``include/dgnn.h``); this package is its thin Python binding
(``_abi``) and the offline-layout driver (``layout``).  Importing the package
loads the shared library and fails loudly if it is missing.
"""
from . import _abi
from ._abi import (Ctx, Samples, CachePlan, DgnnError, dgnn_sample, dgnn_build_cache, dgnn_classify,
                   dgnn_chunk_layout, dgnn_pack, dgnn_gather_rows, dgnn_stage_copy, dgnn_stage_wait,
                   dgnn_stage_sync, dgnn_assemble, load_library, TIER_GPU, TIER_HOST, TIER_DISK, TIER_SHIFT,
                   SLOT_MASK, DiskIndex, DiskPlan, dgnn_disk_space, dgnn_disk_search, dgnn_disk_plan_build,
                   dgnn_disk_cache_fill, dgnn_disk_partial, dgnn_train_stub, dgnn_chunk_layout_graph,
                   dgnn_pack_graph, dgnn_samples_load)
from .layout import HostBuffer, Layout, Workspace, offline_layout, batch_range

load_library()

__all__ = ["Ctx", "Samples", "CachePlan", "DgnnError", "dgnn_sample", "dgnn_build_cache", "dgnn_classify",
           "dgnn_chunk_layout", "dgnn_pack", "dgnn_gather_rows", "dgnn_stage_copy", "dgnn_stage_wait",
           "dgnn_stage_sync", "dgnn_assemble", "load_library", "HostBuffer", "Layout", "Workspace", "offline_layout",
           "batch_range", "TIER_GPU", "TIER_HOST", "TIER_DISK", "TIER_SHIFT", "SLOT_MASK", "DiskIndex", "DiskPlan",
           "dgnn_disk_space", "dgnn_disk_search", "dgnn_disk_plan_build", "dgnn_disk_cache_fill", "dgnn_disk_partial",
           "dgnn_train_stub", "dgnn_chunk_layout_graph", "dgnn_pack_graph", "dgnn_samples_load"]
