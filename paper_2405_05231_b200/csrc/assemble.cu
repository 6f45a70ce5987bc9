// assemble.cu -- a9: feature assembly of one mini-batch.
// P:303-305 (Sec. 4, Fig. 3): "the GPU reads the GPU cache, CPU cache, and
// partial input to obtain all the required features"; P:488 (Sec. 6): UVA
// fetches of CPU-resident features.  out[j] = row(addr[j]) with addr from
// dgnn_classify (reading c18).
//
// One warp-per-row gather over three sources: GPU-tier rows from HBM, host-tier
// rows from pinned host memory read directly over PCIe through UVA (no staging
// copy), disk-tier rows from the batch's staged chunk (HBM after the side-stream
// H2D of a8, or pinned host).  An address whose slot is beyond its tier writes
// a zero row and raises DGNN_ERANGE at the next dgnn_ctx_sync.
#include "rowcopy.cuh"

namespace dgnn {
namespace {

constexpr int kAsmU = 4;

struct AsmRow {
    const uint32_t* addr;
    const uint8_t* gpu;
    int64_t kg;
    const uint8_t* host;
    int64_t kh;
    const uint8_t* chunk;
    int64_t cr;
    int64_t row_bytes;
    uint8_t* out;
    int* err;
    __device__ __forceinline__ bool operator()(int64_t j, const uint8_t*& s, uint8_t*& d) const {
        const uint32_t a = addr[j];
        const uint32_t tier = a >> DGNN_TIER_SHIFT;
        const int64_t slot = a & DGNN_SLOT_MASK;
        d = out + j * row_bytes;
        if (tier == DGNN_TIER_GPU && slot < kg) s = gpu + slot * row_bytes;
        else if (tier == DGNN_TIER_HOST && slot < kh) s = host + slot * row_bytes;
        else if (tier == DGNN_TIER_DISK && slot < cr) s = chunk + slot * row_bytes;
        else {
            atomicOr(err, DEVERR_ADDR_RANGE);
            s = nullptr;
            return false;
        }
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256, 6) k_assemble(AsmRow fn, int64_t n) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(n, fn.row_bytes, fn, warp, nwarps);
}

// A run of consecutive batches in one launch: row j belongs to batch b =
// segment(node_off, j); its DISK slot indexes that batch's chunk at
// chunk_base + chunk_off[b] (chunks of consecutive batches are contiguous in
// the disk tier, so one staging copy brings the whole run).
constexpr int kMaxSeg = 1024;

struct AsmGroupRow {
    const uint32_t* addr;
    const int64_t* node_off;   // [nb+1] relative to addr (smem copy)
    const int64_t* chunk_off;  // [nb+1] byte offsets relative to chunk_base
    const int64_t* chunk_rows; // [nb+1] exclusive prefix of packed rows
    int nb;
    const uint8_t* gpu;
    int64_t kg;
    const uint8_t* host;
    int64_t kh;
    const int32_t* host_map;   // NULL: host = the host tier; else host = staged rows, row host_map[slot]
    const uint8_t* chunk_base;
    int64_t row_bytes;
    uint8_t* out;
    int* err;
    int gpu_world;             // > 1: the GPU tier is sharded, slot s lives on rank s % world at s / world
    int gpu_rank;
    const uint8_t* const* peers;  // non-NULL: every shard's base (peer memory), read one-sided
    __device__ __forceinline__ bool operator()(int64_t j, const uint8_t*& s, uint8_t*& d) const {
        const uint32_t a = addr[j];
        const uint32_t tier = a >> DGNN_TIER_SHIFT;
        const int64_t slot = a & DGNN_SLOT_MASK;
        d = out + j * row_bytes;
        if (tier == DGNN_TIER_GPU && slot < kg) {
            if (peers) {  // one-sided: the owner's shard is mapped into this GPU's address space
                s = peers[slot % gpu_world] + (slot / gpu_world) * row_bytes;
            } else if (gpu_world > 1) {
                if (slot % gpu_world != gpu_rank) {  // remote row: delivered by dgnn_scatter_rows
                    d = nullptr;
                    s = nullptr;
                    return true;
                }
                s = gpu + (slot / gpu_world) * row_bytes;
            } else {
                s = gpu + slot * row_bytes;
            }
        } else if (tier == DGNN_TIER_HOST && slot < kh) {
            s = host + (host_map ? (int64_t)host_map[slot] : slot) * row_bytes;
        } else if (tier == DGNN_TIER_DISK) {
            const int b = segment_of(node_off, nb + 1, j);
            if (slot >= chunk_rows[b + 1] - chunk_rows[b]) {
                atomicOr(err, DEVERR_ADDR_RANGE);
                s = nullptr;
                return false;
            }
            s = chunk_base + chunk_off[b] + slot * row_bytes;
        } else {
            atomicOr(err, DEVERR_ADDR_RANGE);
            s = nullptr;
            return false;
        }
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256, 6) k_assemble_group(AsmGroupRow fn, int64_t n) {
    __shared__ int64_t s_no[kMaxSeg + 1], s_co[kMaxSeg + 1], s_cr[kMaxSeg + 1];
    if (fn.nb <= kMaxSeg) {
        for (int i = threadIdx.x; i <= fn.nb; i += blockDim.x) {
            s_no[i] = fn.node_off[i];
            s_co[i] = fn.chunk_off[i];
            s_cr[i] = fn.chunk_rows[i];
        }
        __syncthreads();
        fn.node_off = s_no;
        fn.chunk_off = s_co;
        fn.chunk_rows = s_cr;
    }
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(n, fn.row_bytes, fn, warp, nwarps);
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// Host-row merging over a window of batches: every host-tier slot the window reads
// gets the window's stamp (plain stores: all writers store the same value); a scan
// over the stamps then lists the slots once each, in ascending order.
__global__ void __launch_bounds__(256) k_host_mark(const uint32_t* __restrict__ addr, int64_t n, int32_t wid,
                                                   int32_t* __restrict__ stamp, int64_t kh) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = addr[i];
        const int64_t slot = a & DGNN_SLOT_MASK;
        if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_HOST && slot < kh) stamp[slot] = wid;
    }
}

struct Row {
    const uint8_t* src;
    int64_t rb;
    const int32_t* ids;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t r, const uint8_t*& s, uint8_t*& d) const {
        s = src + (int64_t)ids[r] * rb;
        d = dst + r * rb;
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256, 6) k_gather_dev(const uint8_t* __restrict__ src, int64_t row_bytes,
                                                    const int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                                    int64_t n_max, uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(min(*n_dev, n_max), row_bytes, Row{src, row_bytes, ids, dst}, warp, nwarps);
}

// Staging gather of a window's host rows (PCIe-bound): each warp owns a chunk of
// kGatherCH consecutive list positions, and every lane keeps kGatherV 16-byte loads
// in flight across the chunk's rows (vector q of the chunk is row q / vpr, offset
// q % vpr), i.e. up to 4 KiB per warp before the stores.  Rows of consecutive host
// slots (runs) come out as contiguous requests without any run bookkeeping, and a
// dense window (every slot, as on Friendster-shaped bounded epochs) is split evenly
// over the warps.
__global__ void k_check_count(const int64_t* count, int64_t capacity, int* err) {
    if (*count > capacity) atomicOr(err, DEVERR_OVERFLOW);
}

constexpr int kGatherCH = 8;
constexpr int kGatherV = 8;
__global__ void __launch_bounds__(256) k_gather_chunks(const uint8_t* __restrict__ src, int64_t row_bytes,
                                                       const int32_t* __restrict__ ids,
                                                       const int64_t* __restrict__ n_dev, int64_t n_max,
                                                       uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t n = min(*n_dev, n_max);  // never past the caller's list / output capacity
    const int vpr = (int)(row_bytes >> 4);
    for (int64_t p0 = warp * kGatherCH; p0 < n; p0 += nwarps * kGatherCH) {
        const int rows = (int)(n - p0 < kGatherCH ? n - p0 : kGatherCH);
        const int64_t my_id = lane < rows ? (int64_t)ids[p0 + lane] : 0;
        const int total = rows * vpr;
        const uint4* d0 = reinterpret_cast<const uint4*>(dst + p0 * row_bytes);
        for (int q0 = 0; q0 < total; q0 += 32 * kGatherV) {
            uint4 v[kGatherV];
            int qq[kGatherV];
#pragma unroll
            for (int i = 0; i < kGatherV; ++i) {
                const int q = q0 + i * 32 + lane;
                const int u = q / vpr;  // row of the chunk (warp-uniform per 32 consecutive q when vpr % 32 == 0)
                const int64_t id = __shfl_sync(0xffffffffu, my_id, u < rows ? u : 0);
                qq[i] = q;
                if (q < total) v[i] = __ldg(reinterpret_cast<const uint4*>(src + id * row_bytes) + (q - u * vpr));
            }
#pragma unroll
            for (int i = 0; i < kGatherV; ++i)
                if (qq[i] < total) __stcs(const_cast<uint4*>(d0) + qq[i], v[i]);
        }
    }
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_assemble(dgnn_ctx* c, const uint32_t* addr, int64_t n, const void* gpu_tier, int64_t k_gpu,
                                     const void* host_tier, int64_t k_host, const void* chunk, int64_t chunk_rows,
                                     int64_t row_bytes, void* out) {
    DGNN_REQUIRE(c && (n == 0 || (addr && out)), "dgnn_assemble: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0 && k_gpu >= 0 && k_host >= 0 && chunk_rows >= 0,
                 "dgnn_assemble: bad sizes");
    DGNN_REQUIRE((k_gpu == 0 || gpu_tier) && (k_host == 0 || host_tier) && (chunk_rows == 0 || chunk),
                 "dgnn_assemble: a non-empty source is NULL");
    if (n == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(gpu_tier) && al16(host_tier) && al16(chunk) && al16(out);
    AsmRow fn{addr,        (const uint8_t*)gpu_tier, k_gpu,     (const uint8_t*)host_tier, k_host, (const uint8_t*)chunk,
              chunk_rows,  row_bytes,                (uint8_t*)out, c->dev_err};
    const int grid = v16 ? grid_resident(c, k_assemble<uint4>, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm)
                         : grid_resident(c, k_assemble<uint32_t>, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_host_window(dgnn_ctx* c, const uint32_t* addr, int64_t n, int32_t window_id,
                                        int32_t* stamp, int64_t k_host, int32_t* list, int64_t capacity,
                                        int32_t* smap, int64_t* count) {
    DGNN_REQUIRE(c && stamp && list && smap && count && (n == 0 || addr), "dgnn_host_window: NULL argument");
    DGNN_REQUIRE(n >= 0 && k_host >= 0 && capacity >= 0 && window_id >= 0, "dgnn_host_window: bad sizes");
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_TRY(memset_async(c, count, 0, sizeof(int64_t)));
    if (n == 0 || k_host == 0) return DGNN_OK;
    // mark the window's host slots, then list them in ascending slot order with one scan
    // over the host tier: the staging gather then walks host memory in address order
    launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] {
        k_host_mark<<<grid_for(c, n, 256, 8), 256, 0, c->stream>>>(addr, n, window_id, stamp, k_host);
    });
    DGNN_CK_LAUNCH();
    const int32_t* st = stamp;
    const int32_t wid = window_id;
    auto in = [=] __device__(int64_t s) -> int32_t { return st[s] == wid ? 1 : 0; };
    auto outf = [=] __device__(int64_t s, int64_t excl, int64_t val) {
        if (val && excl < capacity) {
            list[excl] = (int32_t)s;
            smap[s] = (int32_t)excl;
        }
    };
    DGNN_TRY(scan::run(c, k_host, nullptr, in, outf, count));
    // a window with more distinct host rows than the list holds: only `capacity` were listed
    // (the gathers clamp to their n_max); reported as DGNN_ECUDA "capacity overflow" at the next sync
    launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] { k_check_count<<<1, 1, 0, c->stream>>>(count, capacity, c->dev_err); });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

namespace dgnn {
namespace {
// Runs of consecutive host slots in a window's (ascending) list: one contiguous copy per run.
// A run of k rows is k*row_bytes contiguous bytes in the host tier and in the staging buffer;
// lanes move 16-byte vectors, four 512-byte strides in flight per warp.
__global__ void __launch_bounds__(256) k_gather_runs(const uint8_t* __restrict__ src, int64_t row_bytes,
                                                     const int32_t* __restrict__ list,
                                                     const int64_t* __restrict__ count,
                                                     const int32_t* __restrict__ runs,
                                                     const int64_t* __restrict__ run_count,
                                                     uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t nr = *run_count, n = *count;
    for (int64_t r = warp; r < nr; r += nwarps) {
        const int64_t p0 = runs[r], p1 = r + 1 < nr ? runs[r + 1] : n;
        const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)list[p0] * row_bytes);
        uint4* d = reinterpret_cast<uint4*>(dst + p0 * row_bytes);
        const int64_t nv = (p1 - p0) * row_bytes / 16;
        for (int64_t q = lane; q < nv; q += 4 * 32) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (q + u * 32 < nv) v[u] = __ldg(s + q + u * 32);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (q + u * 32 < nv) __stcs(d + q + u * 32, v[u]);
        }
    }
}
}  // namespace
}  // namespace dgnn

extern "C" dgnn_status dgnn_host_window_runs(dgnn_ctx* c, const int32_t* stamp, int64_t k_host, int32_t window_id,
                                             const int32_t* smap, int32_t* runs, int64_t* run_count) {
    DGNN_REQUIRE(c && stamp && smap && runs && run_count && k_host >= 0 && window_id >= 0,
                 "dgnn_host_window_runs: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_TRY(memset_async(c, run_count, 0, sizeof(int64_t)));
    if (k_host == 0) return DGNN_OK;
    const int32_t wid = window_id;
    auto in = [=] __device__(int64_t s) -> int32_t {
        return (stamp[s] == wid && (s == 0 || stamp[s - 1] != wid)) ? 1 : 0;
    };
    auto outf = [=] __device__(int64_t s, int64_t excl, int64_t val) {
        if (val) runs[excl] = smap[s];
    };
    DGNN_TRY(scan::run(c, k_host, nullptr, in, outf, run_count));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_gather_runs_dev(dgnn_ctx* c, const void* src, int64_t row_bytes, const int32_t* list,
                                            const int64_t* count, const int32_t* runs, const int64_t* run_count,
                                            int64_t max_runs, void* out) {
    DGNN_REQUIRE(c && count && run_count && (max_runs == 0 || (src && list && runs && out)),
                 "dgnn_gather_runs_dev: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && al16(src) && al16(out) && max_runs >= 0,
                 "dgnn_gather_runs_dev: rows and buffers must be 16-byte aligned");
    if (max_runs == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const int grid = grid_resident(c, k_gather_runs, max_runs * 32, 256, c->assemble_blocks_per_sm);
    launch(c, DGNN_K_HOST_GATHER, 0.0, [&] {
        k_gather_runs<<<grid, 256, 0, c->stream>>>((const uint8_t*)src, row_bytes, list, count, runs, run_count,
                                                   (uint8_t*)out);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_gather_rows_dev(dgnn_ctx* c, const void* features, int64_t num_rows, int64_t row_bytes,
                                            const int32_t* ids, const int64_t* n_dev, int64_t n_max, void* out) {
    DGNN_REQUIRE(c && n_dev && (n_max == 0 || (features && ids && out)), "dgnn_gather_rows_dev: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n_max >= 0, "dgnn_gather_rows_dev: bad sizes");
    if (n_max == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(features) && al16(out);
    const int grid = v16 ? grid_resident(c, k_gather_chunks, ceil_div(n_max, (int64_t)kGatherCH) * 32, 256,
                                         c->assemble_blocks_per_sm)
                         : grid_resident(c, k_gather_dev<uint32_t>, n_max * 32 / kAsmU, 256,
                                         c->assemble_blocks_per_sm);
    launch(c, DGNN_K_HOST_GATHER, 0.0, [&] {
        if (v16)
            k_gather_chunks<<<grid, 256, 0, c->stream>>>((const uint8_t*)features, row_bytes, ids, n_dev, n_max,
                                                         (uint8_t*)out);
        else
            k_gather_dev<uint32_t><<<grid, 256, 0, c->stream>>>((const uint8_t*)features, row_bytes, ids, n_dev,
                                                                n_max, (uint8_t*)out);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_assemble_group(dgnn_ctx* c, const uint32_t* addr, const int64_t* node_off, int64_t nb,
                                           int64_t n, const void* gpu_tier, int64_t k_gpu, const void* host_tier,
                                           int64_t k_host, const int32_t* host_map, const void* chunk_base,
                                           const int64_t* chunk_off, const int64_t* chunk_rows, int64_t row_bytes,
                                           void* out) {
    return dgnn_assemble_group_sharded(c, addr, node_off, nb, n, gpu_tier, k_gpu, 0, 1, host_tier, k_host, host_map,
                                       chunk_base, chunk_off, chunk_rows, row_bytes, out);
}

// ------------------------------------------------------- sharded GPU tier (C2)
namespace dgnn {
namespace {

__global__ void k_shard_fill_ids(const int32_t* __restrict__ gpu_ids, int64_t k_gpu, int rank, int world,
                                 int32_t* __restrict__ ids, int64_t n_local) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n_local; l += (int64_t)gridDim.x * blockDim.x)
        ids[l] = gpu_ids[l * world + rank];
}

constexpr int kMaxWorld = 256;

__global__ void k_owner_count(const uint32_t* __restrict__ addr, int64_t n, int64_t k_gpu, int rank, int world,
                              unsigned long long* __restrict__ counts) {
    __shared__ unsigned int sh[kMaxWorld];
    for (int i = threadIdx.x; i < world; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = addr[j];
        const int64_t slot = a & DGNN_SLOT_MASK;
        if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_GPU && slot < k_gpu && slot % world != rank)
            atomicAdd(&sh[slot % world], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < world; i += blockDim.x)
        if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

__global__ void k_owner_scatter(const uint32_t* __restrict__ addr, int64_t n, int64_t k_gpu, int rank, int world,
                                unsigned long long* __restrict__ cursor, int32_t* __restrict__ req_slot,
                                int32_t* __restrict__ req_pos) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = addr[j];
        const int64_t slot = a & DGNN_SLOT_MASK;
        if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_GPU && slot < k_gpu && slot % world != rank) {
            const unsigned long long p = atomicAdd(&cursor[slot % world], 1ull);
            req_slot[p] = (int32_t)(slot / world);  // the owner's local row
            req_pos[p] = (int32_t)j;
        }
    }
}

struct ScatterRow {
    const uint8_t* src;
    const int32_t* pos;
    int64_t rb;
    uint8_t* out;
    __device__ __forceinline__ bool operator()(int64_t r, const uint8_t*& s, uint8_t*& d) const {
        s = src + r * rb;
        d = out + (int64_t)pos[r] * rb;
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256, 6) k_scatter_rows(ScatterRow fn, int64_t n) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(n, fn.rb, fn, warp, nwarps);
}

}  // namespace
}  // namespace dgnn

extern "C" dgnn_status dgnn_tier_shard_ids(dgnn_ctx* c, const int32_t* gpu_ids, int64_t k_gpu, int32_t rank,
                                           int32_t world, int32_t* ids, int64_t* n_local) {
    DGNN_REQUIRE(c && n_local && world >= 1 && world <= kMaxWorld && rank >= 0 && rank < world && k_gpu >= 0,
                 "dgnn_tier_shard_ids: bad argument");
    const int64_t nl = k_gpu > rank ? (k_gpu - rank + world - 1) / world : 0;
    *n_local = nl;
    if (nl == 0) return DGNN_OK;
    DGNN_REQUIRE(gpu_ids && ids, "dgnn_tier_shard_ids: NULL array");
    DGNN_CK(cudaSetDevice(c->device));
    launch(c, DGNN_K_GATHER, 0.0, [&] {
        k_shard_fill_ids<<<grid_for(c, nl, 256), 256, 0, c->stream>>>(gpu_ids, k_gpu, rank, world, ids, nl);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_shard_requests(dgnn_ctx* c, const uint32_t* addr, int64_t n, int64_t k_gpu, int32_t rank,
                                           int32_t world, int64_t* req_off_host, int32_t* req_slot,
                                           int32_t* req_pos) {
    DGNN_REQUIRE(c && req_off_host && world >= 1 && world <= kMaxWorld && rank >= 0 && rank < world && n >= 0,
                 "dgnn_shard_requests: bad argument");
    DGNN_REQUIRE(n == 0 || (addr && req_slot && req_pos), "dgnn_shard_requests: NULL array");
    DGNN_CK(cudaSetDevice(c->device));
    DevBuf<unsigned long long> cnt;
    DGNN_TRY(cnt.alloc(c, (size_t)world));
    DGNN_TRY(memset_async(c, cnt.p, 0, sizeof(unsigned long long) * world));
    if (n > 0) {
        launch(c, DGNN_K_ASSEMBLE, 0.0, [&] {
            k_owner_count<<<grid_for(c, n, 256, 4), 256, 0, c->stream>>>(addr, n, k_gpu, rank, world, cnt.p);
        });
        DGNN_CK_LAUNCH();
    }
    // the per-owner counts are the host's (the exchange sizes its all-to-all with them): the one
    // synchronization of the call; the cursors go back in kernel parameters (no second wait)
    std::vector<unsigned long long> h(world);
    DGNN_TRY(read_small(c, h.data(), cnt.p, sizeof(unsigned long long) * world));
    req_off_host[0] = 0;
    for (int o = 0; o < world; ++o) req_off_host[o + 1] = req_off_host[o] + (int64_t)h[o];
    if (req_off_host[world] == 0) return DGNN_OK;
    std::vector<unsigned long long> cur(world);
    for (int o = 0; o < world; ++o) cur[o] = (unsigned long long)req_off_host[o];
    DGNN_TRY(upload_small(c, cnt.p, cur.data(), sizeof(unsigned long long) * world));
    launch(c, DGNN_K_ASSEMBLE, 0.0, [&] {
        k_owner_scatter<<<grid_for(c, n, 256, 4), 256, 0, c->stream>>>(addr, n, k_gpu, rank, world, cnt.p, req_slot,
                                                                        req_pos);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_scatter_rows(dgnn_ctx* c, const void* rows, int64_t n, int64_t row_bytes,
                                         const int32_t* pos, void* out) {
    DGNN_REQUIRE(c && (n == 0 || (rows && pos && out)), "dgnn_scatter_rows: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0, "dgnn_scatter_rows: bad sizes");
    if (n == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(rows) && al16(out);
    ScatterRow fn{(const uint8_t*)rows, pos, row_bytes, (uint8_t*)out};
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16)
            k_scatter_rows<uint4><<<grid_resident(c, k_scatter_rows<uint4>, n * 32 / kAsmU, 256, 8), 256, 0,
                                    c->stream>>>(fn, n);
        else
            k_scatter_rows<uint32_t><<<grid_resident(c, k_scatter_rows<uint32_t>, n * 32 / kAsmU, 256, 8), 256, 0,
                                       c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_assemble_group_sharded(dgnn_ctx* c, const uint32_t* addr, const int64_t* node_off,
                                                   int64_t nb, int64_t n, const void* gpu_tier, int64_t k_gpu,
                                                   int32_t gpu_rank, int32_t gpu_world, const void* host_tier,
                                                   int64_t k_host, const int32_t* host_map, const void* chunk_base,
                                                   const int64_t* chunk_off, const int64_t* chunk_rows,
                                                   int64_t row_bytes, void* out) {
    DGNN_REQUIRE(gpu_world >= 1 && gpu_rank >= 0 && gpu_rank < gpu_world, "dgnn_assemble_group: bad shard");
    DGNN_REQUIRE(c && (n == 0 || (addr && out && node_off && chunk_off && chunk_rows)),
                 "dgnn_assemble_group: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0 && nb >= 0 && nb < (1 << 30) && k_gpu >= 0 &&
                     k_host >= 0, "dgnn_assemble_group: bad sizes");
    DGNN_REQUIRE((k_gpu == 0 || gpu_tier) && (k_host == 0 || host_tier), "dgnn_assemble_group: NULL tier");
    if (n == 0 || nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(gpu_tier) && al16(host_tier) && al16(chunk_base) && al16(out);
    AsmGroupRow fn{addr,     node_off, chunk_off, chunk_rows, (int)nb,   (const uint8_t*)gpu_tier, k_gpu,
                   (const uint8_t*)host_tier, k_host, host_map, (const uint8_t*)chunk_base, row_bytes,
                   (uint8_t*)out, c->dev_err, gpu_world, gpu_rank, nullptr};
    const int grid = v16 ? grid_resident(c, k_assemble_group<uint4>, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm)
                         : grid_resident(c, k_assemble_group<uint32_t>, n * 32 / kAsmU, 256,
                                         c->assemble_blocks_per_sm);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble_group<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble_group<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

// --------------------------------------------- one-sided peer-memory tier (NEXT #3)
extern "C" dgnn_status dgnn_assemble_group_peer(dgnn_ctx* c, const uint32_t* addr, const int64_t* node_off, int64_t nb,
                                                int64_t n, const void* const* peers, int64_t k_gpu, int32_t world,
                                                const void* host_tier, int64_t k_host, const int32_t* host_map,
                                                const void* chunk_base, const int64_t* chunk_off,
                                                const int64_t* chunk_rows, int64_t row_bytes, void* out) {
    DGNN_REQUIRE(world >= 1 && (k_gpu == 0 || peers), "dgnn_assemble_group_peer: bad shard table");
    DGNN_REQUIRE(c && (n == 0 || (addr && out && node_off && chunk_off && chunk_rows)),
                 "dgnn_assemble_group_peer: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && n >= 0 && nb >= 0 && nb < (1 << 30) && k_gpu >= 0 &&
                     k_host >= 0, "dgnn_assemble_group_peer: bad sizes (row_bytes must be a multiple of 16)");
    DGNN_REQUIRE(k_host == 0 || host_tier, "dgnn_assemble_group_peer: NULL host tier");
    if (n == 0 || nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = al16(host_tier) && al16(chunk_base) && al16(out);
    AsmGroupRow fn{addr,     node_off, chunk_off, chunk_rows, (int)nb,   nullptr, k_gpu,
                   (const uint8_t*)host_tier, k_host, host_map, (const uint8_t*)chunk_base, row_bytes,
                   (uint8_t*)out, c->dev_err, world, 0, (const uint8_t* const*)peers};
    const int grid = v16 ? grid_resident(c, k_assemble_group<uint4>, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm)
                         : grid_resident(c, k_assemble_group<uint32_t>, n * 32 / kAsmU, 256,
                                         c->assemble_blocks_per_sm);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble_group<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble_group<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_device_alloc(int32_t device, int64_t bytes, void** out) {
    DGNN_REQUIRE(out && bytes >= 0, "dgnn_device_alloc: bad argument");
    *out = nullptr;
    DGNN_CK(cudaSetDevice(device));
    DGNN_CK(cudaMalloc(out, (size_t)(bytes > 0 ? bytes : 16)));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_device_free(void* p) {
    if (p) DGNN_CK(cudaFree(p));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_ipc_handle(const void* dev_ptr, void* handle) {
    DGNN_REQUIRE(dev_ptr && handle, "dgnn_ipc_handle: NULL argument");
    cudaIpcMemHandle_t h;
    DGNN_CK(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    static_assert(sizeof(h) == DGNN_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_ipc_open(int32_t device, const void* handle, void** dev_ptr) {
    DGNN_REQUIRE(handle && dev_ptr, "dgnn_ipc_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    DGNN_CK(cudaSetDevice(device));
    DGNN_CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_ipc_close(void* dev_ptr) {
    if (dev_ptr) DGNN_CK(cudaIpcCloseMemHandle(dev_ptr));
    return DGNN_OK;
}
