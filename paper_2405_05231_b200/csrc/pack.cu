// pack.cu -- a6 address tables and a7 batched feature packing.
// a6: P:488 (Sec. 6) "we prepare interpreted address tables during
//     pre-processing".  Readings c18, c21.
// a7: P:228-230 (Sec. 3) "collect all node features it requires and store them
//     contiguously"; P:437-443 (Sec. 5.2) batched packing, and the GPU / CPU
//     caches filled "by treating them as special mini-batches".  Chunk layout:
//     reading c20 (dense rows, 4 KiB-aligned chunk starts, zero tail).
//
// On B200 the whole feature table of the single-GPU configurations is HBM
// resident, so "batched packing" (one sequential pass over a feature partition
// shared by many batches) becomes one gather launch per packing group: every
// packed row of every batch in the group is an independent 16-byte-vectorized
// row copy, HBM-bandwidth bound.
#include <algorithm>

#include "rowcopy.cuh"

namespace dgnn {
namespace {

constexpr int kPackU = 4;
constexpr int kPackBlocksPerSM = 4;  // 32 warps per SM: measured best for 512-byte rows (tools/pack_sweep.py)
constexpr int kMaxSmemSeg = 2048;

// Row sources: one table (HBM, or pinned host through UVA), or a table partitioned by node range
// over several devices' memory (shard r holds rows [r * shard_rows, (r + 1) * shard_rows), read
// through peer mappings: SURVEY 8(e)(4), the IGB-shaped table that no single GPU holds)
struct FlatSrc {
    const uint8_t* base;
    int64_t row_bytes;
    __device__ __forceinline__ const uint8_t* operator()(int32_t id) const { return base + (int64_t)id * row_bytes; }
};
struct ShardSrc {
    const uint8_t* const* peers;
    int64_t shard_rows;
    int64_t row_bytes;
    __device__ __forceinline__ const uint8_t* operator()(int32_t id) const {
        const int64_t r = id / shard_rows;
        return peers[r] + (id - r * shard_rows) * row_bytes;
    }
};

template <class Src>
struct PackRow {
    Src src;
    int64_t row_bytes;
    const int32_t* ids;
    const int64_t* seg;  // packed_off (smem or global), nb+1
    const int64_t* chunk_off;
    int nb;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t r, const uint8_t*& s, uint8_t*& d) const {
        const int b = segment_of(seg, nb + 1, r);
        s = src(ids[r]);
        d = dst + chunk_off[b] + (r - seg[b]) * row_bytes;
        return true;
    }
};

template <class V, int U = kPackU, class Src = FlatSrc>
__global__ void __launch_bounds__(256) k_pack(Src src, int64_t row_bytes,
                                              const int32_t* __restrict__ ids, const int64_t* __restrict__ packed_off,
                                              const int64_t* __restrict__ chunk_off, int nb, int64_t R,
                                              uint8_t* __restrict__ dst) {
    __shared__ int64_t s_seg[kMaxSmemSeg + 1];
    const bool in_smem = nb <= kMaxSmemSeg;
    if (in_smem)
        for (int i = threadIdx.x; i <= nb; i += blockDim.x) s_seg[i] = packed_off[i];
    __syncthreads();
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    // zero tail of each chunk (reading c20): warp b handles batch b
    for (int64_t b = warp; b < nb; b += nwarps) {
        const int64_t rows = packed_off[b + 1] - packed_off[b];
        uint32_t* z = reinterpret_cast<uint32_t*>(dst + chunk_off[b] + rows * row_bytes);
        const int64_t nz = (chunk_off[b + 1] - chunk_off[b] - rows * row_bytes) >> 2;
        for (int64_t i = threadIdx.x & 31; i < nz; i += 32) z[i] = 0u;
    }
    PackRow<Src> fn{src, row_bytes, ids, in_smem ? s_seg : packed_off, chunk_off, nb, dst};
    copy_rows_warp<U, V>(R, row_bytes, fn, warp, nwarps);
}

template <class Src>
struct GatherRow {
    Src src;
    int64_t row_bytes;
    const int32_t* ids;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t r, const uint8_t*& s, uint8_t*& d) const {
        s = src(ids[r]);
        d = dst + r * row_bytes;
        return true;
    }
};

template <class V, class Src = FlatSrc>
__global__ void __launch_bounds__(256) k_gather(Src src, int64_t row_bytes, const int32_t* __restrict__ ids, int64_t R,
                                                uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kPackU, V>(R, row_bytes, GatherRow<Src>{src, row_bytes, ids, dst}, warp, nwarps);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// a6's second pass, one CTA per batch (grid-stride over batches): the batch's first DISK node
// holds its smallest packed index (DISK slots are the scan's running count, ascending in node
// order), so packed_off[b] = the minimum DISK slot of the batch (block-wide min; batches without
// DISK nodes keep the memset's sentinel for k_classify_fill), then the batch's DISK addresses are
// made relative to it.  Two coalesced passes over the batch's addresses, no per-node batch search
// and no atomics across batches.
__global__ void k_classify_batches(uint32_t* __restrict__ addr, const int64_t* __restrict__ seg, int nseg,
                                   int64_t n0, int64_t* __restrict__ packed_off) {
    __shared__ unsigned long long s_min;
    for (int b = blockIdx.x; b < nseg; b += gridDim.x) {
        if (threadIdx.x == 0) s_min = ~0ull;
        __syncthreads();
        const int64_t lo = seg[b] - n0, hi = seg[b + 1] - n0;
        unsigned long long m = ~0ull;
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const uint32_t a = addr[i];
            if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_DISK) m = min(m, (unsigned long long)(a & DGNN_SLOT_MASK));
        }
        for (int d = 16; d; d >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, d));
        if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(&s_min, m);
        __syncthreads();
        const unsigned long long first = s_min;
        if (first != ~0ull) {
            if (threadIdx.x == 0) packed_off[b] = (int64_t)first;
            const uint32_t f = (uint32_t)first;
            for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const uint32_t a = addr[i];
                if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_DISK) addr[i] = a - f;
            }
        }
        __syncthreads();
    }
}

// per-batch row counts of each tier (block per batch): sizing metadata for the assembler
__global__ void k_tier_counts(const uint32_t* __restrict__ addr, const int64_t* __restrict__ node_off, int64_t n0,
                              int nb, int64_t* __restrict__ out) {
    __shared__ unsigned long long s[3];
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        if (threadIdx.x < 3) s[threadIdx.x] = 0;
        __syncthreads();
        unsigned long long c[3] = {0, 0, 0};
        for (int64_t i = node_off[b] - n0 + threadIdx.x; i < node_off[b + 1] - n0; i += blockDim.x) {
            const uint32_t t = addr[i] >> DGNN_TIER_SHIFT;
            if (t < 3) c[t] += 1;
        }
        for (int t = 0; t < 3; ++t) {
            unsigned long long v = c[t];
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s[t], v);
        }
        __syncthreads();
        if (threadIdx.x < 3) out[(int64_t)b * 3 + threadIdx.x] = (int64_t)s[threadIdx.x];
        __syncthreads();
    }
}

// batches without DISK nodes: packed_off[b] = packed_off[b+1] (packed_off[nseg] = total)
__global__ void k_classify_fill(int64_t* packed_off, int nseg) {
    if (threadIdx.x != 0) return;
    for (int b = nseg - 1; b >= 0; --b)
        if (packed_off[b] > packed_off[b + 1]) packed_off[b] = packed_off[b + 1];
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_classify(dgnn_ctx* c, const dgnn_cache_plan* plan, const dgnn_samples* S, int64_t b_lo,
                                     int64_t b_hi, uint32_t* addr, int32_t* packed_ids, int64_t* packed_off,
                                     int64_t* packed_off_host) {
    DGNN_REQUIRE(c && plan && S && addr && packed_ids && packed_off, "dgnn_classify: NULL argument");
    DGNN_REQUIRE(0 <= b_lo && b_lo <= b_hi && b_hi <= S->nb, "dgnn_classify: batch range [%lld, %lld) outside [0, %lld)",
                 (long long)b_lo, (long long)b_hi, (long long)S->nb);
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t nbg = b_hi - b_lo;
    const int64_t n0 = S->node_off_h[b_lo];
    const int64_t n = S->node_off_h[b_hi] - n0;
    DGNN_TRY(memset_async(c, packed_off, 0, sizeof(int64_t)));
    if (n > 0) {
        const int32_t* nodes = S->nodes + n0;
        const int64_t* seg = S->node_off + b_lo;  // absolute offsets of batches b_lo..b_hi
        const uint32_t* tm = plan->tier_map;
        const int nseg = (int)nbg;
        // pass 1: one gather of tier_map per node (parked in addr by the scan input), the
        // compaction of the DISK nodes (P_b concatenated) and their global packed index
        auto in = [=] __device__(int64_t i) -> int32_t {
            const uint32_t t = tm[nodes[i]];
            addr[i] = t;
            return (int32_t)((t >> DGNN_TIER_SHIFT) == DGNN_TIER_DISK);
        };
        auto outf = [=] __device__(int64_t i, int64_t excl, int64_t val) {
            if (val) {
                packed_ids[excl] = nodes[i];
                addr[i] = (DGNN_TIER_DISK << DGNN_TIER_SHIFT) | (uint32_t)excl;
            }
        };
        DGNN_TRY(scan::run(c, n, nullptr, in, outf, packed_off + nbg));
        // pass 2: packed_off[b] = the smallest global packed index of batch b (batches
        // without DISK nodes take their successor's), then DISK slots relative to the batch
        DGNN_TRY(memset_async(c, packed_off, 0x7F, sizeof(int64_t) * nbg));
        launch(c, DGNN_K_CLASSIFY, 12.0 * n, [&] {
            k_classify_batches<<<(int)std::min<int64_t>(nbg, (int64_t)c->num_sms * 8), 256, 0, c->stream>>>(
                addr, seg, nseg, n0, packed_off);
            k_classify_fill<<<1, 32, 0, c->stream>>>(packed_off, nseg);
        });
        DGNN_CK_LAUNCH();
    } else {
        DGNN_TRY(memset_async(c, packed_off, 0, sizeof(int64_t) * (nbg + 1)));
    }
    if (packed_off_host) {
        DGNN_TRY(read_small(c, packed_off_host, packed_off, sizeof(int64_t) * (nbg + 1)));
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_batch_tier_counts(dgnn_ctx* c, const dgnn_samples* S, int64_t b_lo, int64_t b_hi,
                                              const uint32_t* addr, int64_t* counts_host) {
    DGNN_REQUIRE(c && S && counts_host && (addr || b_hi == b_lo), "dgnn_batch_tier_counts: NULL argument");
    DGNN_REQUIRE(0 <= b_lo && b_lo <= b_hi && b_hi <= S->nb, "dgnn_batch_tier_counts: bad batch range");
    const int64_t nbg = b_hi - b_lo;
    if (nbg == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    DevBuf<int64_t> d;
    DGNN_TRY(d.alloc(c, (size_t)(3 * nbg)));
    launch(c, DGNN_K_CLASSIFY, 0.0, [&] {
        k_tier_counts<<<(int)std::min<int64_t>(nbg, (int64_t)c->num_sms * 8), 256, 0, c->stream>>>(
            addr, S->node_off + b_lo, S->node_off_h[b_lo], (int)nbg, d.p);
    });
    DGNN_CK_LAUNCH();
    DGNN_TRY(read_small(c, counts_host, d.p, sizeof(int64_t) * 3 * nbg));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_packing_groups(const int64_t* po, int64_t nb, int64_t row_bytes, int64_t group_size,
                                           int64_t group_budget, int64_t* group_lo, int64_t* n_groups) {
    DGNN_REQUIRE(po && group_lo && n_groups && nb >= 0 && row_bytes > 0, "dgnn_packing_groups: bad argument");
    int64_t n = 0, g0 = 0;
    while (g0 < nb) {
        int64_t g1 = g0 + 1;
        while (g1 < nb && (group_size <= 0 || g1 - g0 < group_size) &&
               (po[g1 + 1] - po[g0]) * row_bytes + 4096 * (g1 + 1 - g0) <= group_budget)
            ++g1;
        group_lo[n++] = g0;
        g0 = g1;
    }
    group_lo[n] = nb;
    *n_groups = n;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_assembly_runs(const int64_t* no, int64_t nb, int64_t max_rows, int64_t max_batches,
                                          int64_t* run_lo, int64_t* n_runs) {
    DGNN_REQUIRE(no && run_lo && n_runs && nb >= 0 && max_rows >= 1 && max_batches >= 1,
                 "dgnn_assembly_runs: bad argument");
    int64_t n = 0, b0 = 0;
    while (b0 < nb) {
        // the last b1 with no[b1] - no[b0] <= max_rows (upper bound in the non-decreasing offsets),
        // then at least one batch, at most max_batches
        const int64_t* it = std::upper_bound(no, no + nb + 1, no[b0] + max_rows);
        int64_t b1 = (int64_t)(it - no) - 1;
        b1 = std::min(std::max(b1, b0 + 1), std::min(b0 + max_batches, nb));
        run_lo[n++] = b0;
        b0 = b1;
    }
    run_lo[n] = nb;
    *n_runs = n;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_assembly_tables(const int64_t* no, const int64_t* cst, const int64_t* crows,
                                            const int64_t* drows, const int64_t* sec, int64_t nb, int64_t chunk_bytes,
                                            int64_t row_bytes, const int64_t* run_lo, int64_t n_runs, int64_t* tab,
                                            int64_t tab_cap, int64_t* tab_off, int64_t* spans) {
    DGNN_REQUIRE(no && cst && crows && run_lo && tab_off && spans && nb >= 0 && n_runs >= 0 && row_bytes > 0 &&
                     (tab || tab_cap == 0),
                 "dgnn_assembly_tables: bad argument");
    int64_t o = 0;
    auto put = [&](int64_t v) -> bool {
        if (o >= tab_cap) return false;
        tab[o++] = v;
        return true;
    };
    for (int64_t r = 0; r < n_runs; ++r) {
        const int64_t b0 = run_lo[r], b1 = run_lo[r + 1];
        DGNN_REQUIRE(0 <= b0 && b0 < b1 && b1 <= nb, "dgnn_assembly_tables: bad run [%lld, %lld)", (long long)b0,
                     (long long)b1);
        const int64_t c_lo = cst[b0], c_hi = b1 < nb ? cst[b1] : chunk_bytes;
        tab_off[r] = o;
        bool ok = true;
        for (int64_t b = b0; b <= b1; ++b) ok = ok && put(no[b] - no[b0]);
        if (!drows) {
            for (int64_t b = b0; b < b1; ++b) ok = ok && put(cst[b] - c_lo);
            ok = ok && put(c_hi - c_lo);
            int64_t acc = 0;
            ok = ok && put(0);
            for (int64_t b = b0; b < b1; ++b) ok = ok && put(acc += crows[b]);
            if (sec)
                for (int64_t b = b0; b < b1; ++b) ok = ok && put(sec[b] - c_lo);
        } else {
            int64_t acc = 0;
            ok = ok && put(0);
            for (int64_t b = b0; b < b1; ++b) ok = ok && put((acc += drows[b]) * row_bytes);
            acc = 0;
            ok = ok && put(0);
            for (int64_t b = b0; b < b1; ++b) ok = ok && put(acc += drows[b]);
            for (int64_t b = b0; b < b1; ++b) ok = ok && put(cst[b] - c_lo);
            ok = ok && put(c_hi - c_lo);
        }
        DGNN_REQUIRE(ok, "dgnn_assembly_tables: tab_cap %lld too small", (long long)tab_cap);
        spans[4 * r] = no[b0];
        spans[4 * r + 1] = no[b1];
        spans[4 * r + 2] = c_lo;
        spans[4 * r + 3] = c_hi;
    }
    tab_off[n_runs] = o;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_chunk_layout(const int64_t* packed_off_host, int64_t nb, int64_t row_bytes,
                                         int64_t* chunk_off_host) {
    DGNN_REQUIRE(packed_off_host && chunk_off_host && nb >= 0 && row_bytes > 0, "dgnn_chunk_layout: bad argument");
    chunk_off_host[0] = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t rows = packed_off_host[i + 1] - packed_off_host[i];
        DGNN_REQUIRE(rows >= 0, "dgnn_chunk_layout: packed_off must be non-decreasing");
        const int64_t end = chunk_off_host[i] + rows * row_bytes;
        chunk_off_host[i + 1] = (end + 4095) / 4096 * 4096;
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_pack(dgnn_ctx* c, const void* features, int64_t num_rows, int64_t row_bytes,
                                 const int32_t* packed_ids, const int64_t* packed_off, const int64_t* chunk_off,
                                 int64_t nb, int64_t total_rows, int64_t group_bytes, void* group_buf) {
    DGNN_REQUIRE(c && (features || num_rows == 0) && packed_off && chunk_off && (group_buf || group_bytes == 0),
                 "dgnn_pack: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0, "dgnn_pack: row_bytes must be a positive multiple of 4");
    DGNN_REQUIRE(nb >= 0 && nb < (1 << 30) && total_rows >= 0 && (packed_ids || total_rows == 0),
                 "dgnn_pack: bad sizes");
    DGNN_REQUIRE(total_rows * row_bytes <= group_bytes, "dgnn_pack: group_bytes too small for the packed rows");
    if (nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && aligned16(features) && aligned16(group_buf);
    const int pu = getenv("DGNN_PACK_U") ? atoi(getenv("DGNN_PACK_U")) : kPackU;  // tuning experiment
    const int pbs = getenv("DGNN_PACK_BPS") ? atoi(getenv("DGNN_PACK_BPS")) : kPackBlocksPerSM;
    using PackK = void (*)(FlatSrc, int64_t, const int32_t*, const int64_t*, const int64_t*, int, int64_t, uint8_t*);
    const PackK kern = !v16 ? (PackK)k_pack<uint32_t> : pu == 8 ? (PackK)k_pack<uint4, 8>
                                                      : pu == 2 ? (PackK)k_pack<uint4, 2> : (PackK)k_pack<uint4>;
    const int64_t work = std::max<int64_t>(total_rows * 32 / pu, nb * 32);
    const int grid = grid_resident(c, kern, work, 256, pbs);
    const double bytes = (double)total_rows * (2.0 * row_bytes + 4.0);
    launch(c, DGNN_K_PACK, bytes, [&] {
        kern<<<grid, 256, 0, c->stream>>>(FlatSrc{(const uint8_t*)features, row_bytes}, row_bytes, packed_ids,
                                          packed_off, chunk_off, (int)nb, total_rows, (uint8_t*)group_buf);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_gather_rows(dgnn_ctx* c, const void* features, int64_t num_rows, int64_t row_bytes,
                                        const int32_t* ids, int64_t n, void* out) {
    DGNN_REQUIRE(c && (n == 0 || (features && ids && out)), "dgnn_gather_rows: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0, "dgnn_gather_rows: bad sizes");
    if (n == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && aligned16(features) && aligned16(out);
    const int grid = v16 ? grid_resident(c, k_gather<uint4>, n * 32 / kPackU, 256, 8)
                         : grid_resident(c, k_gather<uint32_t>, n * 32 / kPackU, 256, 8);
    // a gather that reads or writes pinned host memory crosses PCIe: its own kernel family
    // (bytes = the rows that cross the link), so the HBM-bound GPU-tier fill is reported alone
    auto on_host = [](const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    const bool pcie = on_host(features) || on_host(out);
    launch(c, pcie ? DGNN_K_GATHER_PCIE : DGNN_K_GATHER, pcie ? (double)n * row_bytes : (double)n * (2.0 * row_bytes + 4.0), [&] {
        const FlatSrc src{(const uint8_t*)features, row_bytes};
        if (v16)
            k_gather<uint4><<<grid, 256, 0, c->stream>>>(src, row_bytes, ids, n, (uint8_t*)out);
        else
            k_gather<uint32_t><<<grid, 256, 0, c->stream>>>(src, row_bytes, ids, n, (uint8_t*)out);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

// ------------------------------------------- a7 from a table partitioned by node range
extern "C" dgnn_status dgnn_pack_sharded(dgnn_ctx* c, const void* const* peers_dev, int64_t shard_rows,
                                         int32_t nshards, int64_t row_bytes, const int32_t* packed_ids,
                                         const int64_t* packed_off, const int64_t* chunk_off, int64_t nb,
                                         int64_t total_rows, int64_t group_bytes, void* group_buf) {
    DGNN_REQUIRE(c && peers_dev && packed_off && chunk_off && (group_buf || group_bytes == 0),
                 "dgnn_pack_sharded: NULL argument");
    DGNN_REQUIRE(shard_rows > 0 && nshards >= 1 && row_bytes > 0 && row_bytes % 16 == 0,
                 "dgnn_pack_sharded: shard_rows > 0, nshards >= 1, row_bytes a positive multiple of 16");
    DGNN_REQUIRE(nb >= 0 && nb < (1 << 30) && total_rows >= 0 && (packed_ids || total_rows == 0) &&
                     total_rows * row_bytes <= group_bytes,
                 "dgnn_pack_sharded: bad sizes");
    if (nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_REQUIRE(aligned16(group_buf), "dgnn_pack_sharded: group_buf must be 16-byte aligned");
    auto kern = k_pack<uint4, kPackU, ShardSrc>;
    const int grid = grid_resident(c, kern, std::max<int64_t>(total_rows * 32 / kPackU, nb * 32), 256,
                                   kPackBlocksPerSM);
    launch(c, DGNN_K_PACK, (double)total_rows * (2.0 * row_bytes + 4.0), [&] {
        kern<<<grid, 256, 0, c->stream>>>(ShardSrc{(const uint8_t* const*)peers_dev, shard_rows, row_bytes}, row_bytes,
                                          packed_ids, packed_off, chunk_off, (int)nb, total_rows, (uint8_t*)group_buf);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_gather_rows_sharded(dgnn_ctx* c, const void* const* peers_dev, int64_t shard_rows,
                                                int32_t nshards, int64_t row_bytes, const int32_t* ids, int64_t n,
                                                void* out) {
    DGNN_REQUIRE(c && peers_dev && (n == 0 || (ids && out)), "dgnn_gather_rows_sharded: NULL argument");
    DGNN_REQUIRE(shard_rows > 0 && nshards >= 1 && row_bytes > 0 && row_bytes % 16 == 0 && n >= 0,
                 "dgnn_gather_rows_sharded: bad sizes");
    if (n == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_REQUIRE(aligned16(out), "dgnn_gather_rows_sharded: out must be 16-byte aligned");
    auto kern = k_gather<uint4, ShardSrc>;
    const int grid = grid_resident(c, kern, n * 32 / kPackU, 256, 8);
    launch(c, DGNN_K_GATHER, (double)n * (2.0 * row_bytes + 4.0), [&] {
        kern<<<grid, 256, 0, c->stream>>>(ShardSrc{(const uint8_t* const*)peers_dev, shard_rows, row_bytes}, row_bytes,
                                          ids, n, (uint8_t*)out);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}
