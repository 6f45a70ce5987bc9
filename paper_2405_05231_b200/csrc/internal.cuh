// internal.cuh -- shared plumbing of libdgnn.so (context, allocation, launch
// accounting, errors) plus two device building blocks used by several steps:
// the Philox4x32-10 draw and a single-pass decoupled look-back prefix scan.
// Nothing here is shared with oracle/ (see DESIGN.md "Oracle independence").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dgnn.h"

// ------------------------------------------------------------------ context
struct dgnn_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;
    bool own_stream = false;
    dgnn_allocator alloc{};
    bool has_alloc = false;
    int* dev_err = nullptr;  // device word: OR of DEVERR_* bits
    int64_t launches = 0;
    int32_t sample_group = 0;
    int32_t sample_mode = DGNN_SAMPLE_NODEWISE;
    int64_t sample_n_hint = 0;  // largest batch (nodes) of the last dgnn_sample on this ctx
    int assemble_blocks_per_sm = 8;  // grid cap for a9 (lower it to leave SMs to a concurrent pass)
    int grid_cap = 0;                // > 0: no launch of this ctx uses more CTAs (dgnn_ctx_set_grid_cap)
    // per-launch CUDA-event timing
    bool timing = false;
    uint64_t timing_mask = ~0ull;  // kernel families timed when timing is on (dgnn_ctx_set_timing_mask)
    struct Pending {
        cudaEvent_t a, b;
        int kid;
        double bytes;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double stat_ms[DGNN_K_NUM] = {};
    double stat_bytes[DGNN_K_NUM] = {};
    int64_t stat_n[DGNN_K_NUM] = {};
    // staging tickets (a8)
    static constexpr int kStageRing = 8192;
    cudaEvent_t stage_ev[kStageRing] = {};
    int64_t stage_next = 0;
    cudaEvent_t order_ev = nullptr;
    // pinned host scratch for the small size read-backs / uploads (grow-only): pageable
    // copies would stage through the driver and serialize with other streams' copies
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    int* pinned_err = nullptr;  // check_dev_err's read-back word
    // small device -> host read-backs (sizes, flags) land here from SM stores over PCIe
    // (readback_enqueue): a cudaMemcpy D2H would queue on a copy engine behind the gigabytes of
    // stage-out / tier-fill copies another stream has in flight
    void* rb = nullptr;
    size_t rb_bytes = 0;
    // recycled device buffers (keep_take / keep_put): the sample arenas and the sampler's group
    // scratch of one call are handed to the next call on the same ctx instead of going back to
    // the allocator, so a steady stream of offline passes reaches a fixed HBM footprint
    struct Kept {
        void* p;
        size_t bytes;
    };
    std::vector<Kept> kept;
    size_t kept_bytes = 0;
    size_t kept_limit = (size_t)24 << 30;      // dgnn_ctx_set_keep_limit
    // grow-only scan scratch (status words + tile counter), plain cudaMalloc: the scans of a ctx run
    // in its stream order, so one buffer serves them all, and no allocator callback (Python, the
    // GIL) sits on the sampler's hot path
    void* scan_buf = nullptr;
    size_t scan_bytes = 0;
    size_t sample_budget = (size_t)3 << 30;    // sampler group scratch budget (dgnn_ctx_set_sample_budget)
};

namespace dgnn {

enum DevErr : int {
    DEVERR_SEED_RANGE = 1,
    DEVERR_SEED_DUP = 2,
    DEVERR_ADDR_RANGE = 4,
    DEVERR_OVERFLOW = 8,
    DEVERR_TABLE = 16,
    DEVERR_PART = 32,  // a (batch, ID range) bucket of the partitioned dedup overflowed its table
};

void set_error(const char* fmt, ...);
dgnn_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define DGNN_CK(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) return dgnn::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

#define DGNN_CK_LAUNCH() DGNN_CK(cudaGetLastError())

#define DGNN_REQUIRE(cond, ...)          \
    do {                                 \
        if (!(cond)) {                   \
            dgnn::set_error(__VA_ARGS__); \
            return DGNN_EINVAL;          \
        }                                \
    } while (0)

#define DGNN_TRY(expr)                   \
    do {                                 \
        dgnn_status s_ = (expr);         \
        if (s_ != DGNN_OK) return s_;    \
    } while (0)

// ------------------------------------------------------------- allocation
void* dev_alloc(dgnn_ctx* c, size_t bytes);
void dev_free(dgnn_ctx* c, void* p, size_t bytes);
// The smallest kept buffer of >= need bytes (and not more than 2 x need + 256 MiB), else a fresh
// allocation of exactly need bytes; *got = the buffer's size.  NULL on allocation failure.
void* keep_take(dgnn_ctx* c, size_t need, size_t* got);
// Hand a buffer back to the ctx for reuse (stream-ordered on the ctx stream like dev_free);
// beyond the ctx's kept-bytes limit the oldest kept buffers are freed.
void keep_put(dgnn_ctx* c, void* p, size_t bytes);
void keep_trim(dgnn_ctx* c, size_t limit);

// RAII device buffer, freed stream-ordered on the ctx stream.
template <class T>
struct DevBuf {
    dgnn_ctx* c = nullptr;
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    size_t kept_bytes = 0;  // > 0: the buffer came from keep_take and goes back with keep_put
    dgnn_status alloc(dgnn_ctx* ctx, size_t count) {
        reset();
        c = ctx;
        n = count;
        p = static_cast<T*>(dev_alloc(ctx, (count ? count : 1) * sizeof(T)));
        if (!p) {
            set_error("device allocation of %zu bytes failed", count * sizeof(T));
            return DGNN_ENOMEM;
        }
        return DGNN_OK;
    }
    // same, recycled through the ctx's kept buffers (for scratch every call needs again)
    dgnn_status alloc_kept(dgnn_ctx* ctx, size_t count) {
        reset();
        c = ctx;
        n = count;
        p = static_cast<T*>(keep_take(ctx, (count ? count : 1) * sizeof(T), &kept_bytes));
        if (!p) {
            set_error("device allocation of %zu bytes failed", count * sizeof(T));
            return DGNN_ENOMEM;
        }
        return DGNN_OK;
    }
    void reset() {
        if (p && kept_bytes) keep_put(c, p, kept_bytes);
        else if (p) dev_free(c, p, (n ? n : 1) * sizeof(T));
        p = nullptr;
        n = 0;
        kept_bytes = 0;
    }
    T* release() {
        T* q = p;
        p = nullptr;
        n = 0;
        kept_bytes = 0;
        return q;
    }
};

// ------------------------------------------------------- launch accounting
cudaEvent_t take_event(dgnn_ctx* c);
void fold_pending(dgnn_ctx* c, bool sync);

// Wrap a kernel launch on the ctx stream: counts it and, with timing on,
// brackets it with CUDA events on that same stream.
template <class F>
inline void launch(dgnn_ctx* c, int kid, double bytes, F&& f) {
    dgnn_ctx::Pending p{};
    const bool timed = c->timing && ((c->timing_mask >> kid) & 1ull);
    if (timed) {
        p.a = take_event(c);
        p.b = take_event(c);
        cudaEventRecord(p.a, c->stream);
    }
    f();
    c->launches++;
    if (timed) {
        cudaEventRecord(p.b, c->stream);
        p.kid = kid;
        p.bytes = bytes;
        c->pending.push_back(p);
        if (c->pending.size() > 8192) fold_pending(c, true);
    }
}

dgnn_status memset_async(dgnn_ctx* c, void* p, int value, size_t bytes);
void* pinned_scratch(dgnn_ctx* c, size_t bytes);  // NULL on failure; valid until the next call
dgnn_status check_dev_err(dgnn_ctx* c);  // synchronizes
dgnn_status read_dev_err(dgnn_ctx* c, int* flags);  // synchronizes; clears the device word
// Small device -> host read-backs by SM stores into the ctx's pinned read-back buffer (no copy
// engine): readback_reserve(c, bytes) first (grow-only; nothing may be in flight), then any number
// of readback_enqueue(c, off, src, n) on the ctx stream (off, n multiples of 4, src 4-byte
// aligned), then cudaStreamSynchronize; the bytes are at readback_host(c) + off.
// DGNN_SMALL_D2H=copy uses cudaMemcpyAsync into the same buffer instead (A/B measurement).
dgnn_status readback_reserve(dgnn_ctx* c, size_t bytes);
dgnn_status readback_enqueue(dgnn_ctx* c, size_t off, const void* src_dev, size_t n);
inline uint8_t* readback_host(dgnn_ctx* c) { return static_cast<uint8_t*>(c->rb); }
// the three together: n bytes of device memory into any host memory (synchronizes)
dgnn_status read_small(dgnn_ctx* c, void* dst_host, const void* src_dev, size_t n);
// Small host -> device uploads carried in kernel parameters (copied at launch: no copy engine, and
// the host source may be reused as soon as the call returns); above kUploadMax bytes, or with
// DGNN_SMALL_D2H=copy, an ordinary cudaMemcpyAsync on the ctx stream.
constexpr size_t kUploadMax = (size_t)256 << 10;
dgnn_status upload_small(dgnn_ctx* c, void* dst_dev, const void* src_host, size_t n);
dgnn_status dev_err_status(int flags);               // DEVERR_* bits -> status + message

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int grid_for(dgnn_ctx* c, int64_t work_items, int per_block, int blocks_per_sm = 8) {
    int64_t need = ceil_div(work_items > 0 ? work_items : 1, per_block);
    int64_t cap = (int64_t)c->num_sms * blocks_per_sm;
    if (c->grid_cap > 0 && cap > c->grid_cap) cap = c->grid_cap;
    return (int)(need < cap ? need : cap);
}

// Persistent grid-stride kernels: never launch more CTAs than fit on the GPU at once.  A
// second, partial wave of CTAs that each own an equal share of the rows finishes a whole
// share late (the a7 pack at 8 CTAs/SM with 5 resident ran 1.35 ms, at 4 resident 1.26 ms).
template <class K>
inline int grid_resident(dgnn_ctx* c, K kernel, int64_t work_items, int per_block, int blocks_per_sm,
                         size_t smem = 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, per_block, smem) != cudaSuccess || occ < 1)
        occ = 1;
    return grid_for(c, work_items, per_block, blocks_per_sm < occ ? blocks_per_sm : occ);
}

// ------------------------------------------------------------------- philox
// Philox4x32-10 (Salmon et al., SC'11) with the counter packing of DESIGN.md
// reading c5: ctr = {v, lo32(bid), h<<16 | s, hi32(bid)}, key = {lo32(seed), hi32(seed)}.
__device__ __forceinline__ uint64_t draw64(uint64_t seed, uint32_t v, uint64_t bid, uint32_t h, uint32_t s) {
    uint32_t c0 = v, c1 = (uint32_t)bid, c2 = (h << 16) | (s & 0xFFFFu), c3 = (uint32_t)(bid >> 32);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return ((uint64_t)c1 << 32) | c0;
}

// ------------------------------------------------------- relaxed atomics
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// upper_bound over a short sorted array (in shared or global memory): the
// largest s in [0, n-1) with a[s] <= x, i.e. the segment containing x.
template <class T, class U>
__device__ __forceinline__ int segment_of(const T* a, int n_plus_1, U x) {
    int lo = 0, hi = n_plus_1 - 1;  // answer in [lo, hi)
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if ((int64_t)a[mid] <= (int64_t)x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ------------------------------------------------ decoupled look-back scan
// Exclusive prefix sum of int64 values produced by `in(i)` for i < n, handed to
// `out(i, exclusive_prefix, value)`.  One pass: tiles are taken in order from an
// atomic counter; each tile publishes its aggregate, then its inclusive prefix,
// in a single 64-bit status word (2 flag bits + 62 value bits), so a relaxed
// 64-bit load sees flag and value together.  n may live on the device (n_dev)
// so that data-dependent sizes need no host round trip.
namespace scan {
constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;
constexpr unsigned long long kFlagA = 1ull << 62;
constexpr unsigned long long kFlagP = 2ull << 62;
constexpr unsigned long long kMask = (1ull << 62) - 1;

template <class In, class Out>
__global__ void __launch_bounds__(kThreads) scan_kernel(const int64_t* n_dev, int64_t n_host, In in, Out out,
                                                        unsigned long long* status, unsigned int* tile_counter,
                                                        int64_t* total) {
    const int64_t n = n_dev ? *n_dev : n_host;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    __shared__ int64_t s_warp[kThreads / 32];
    __shared__ int64_t s_prefix;
    __shared__ int64_t s_tile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && total) *total = 0;
        return;
    }
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        const int64_t base = tile * kTile + (int64_t)warp * (32 * kItems);
        // V = the input's value type: int32 inputs keep the per-warp arrays in 32-bit
        // registers (the warp covers 256 items, so int32 sums cannot overflow for them)
        using V = decltype(in(int64_t(0)));
        V val[kItems], incl[kItems];
        V run = 0;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int64_t idx = base + i * 32 + lane;
            const V x = idx < n ? in(idx) : V(0);
            V s = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const V y = __shfl_up_sync(0xffffffffu, s, d);
                if (lane >= d) s += y;
            }
            val[i] = x;
            incl[i] = run + s;
            run += __shfl_sync(0xffffffffu, s, 31);
        }
        if (lane == 0) s_warp[warp] = (int64_t)run;
        __syncthreads();
        int64_t warp_excl = 0, block_total = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            const int64_t t = s_warp[w];
            warp_excl += (w < warp) ? t : 0;
            block_total += t;
        }
        if (warp == 0) {
            // warp-parallel look-back: lane l inspects predecessor tile-1-l of the window
            int64_t prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_relaxed(&status[0], kFlagP | (unsigned long long)block_total);
            } else {
                if (lane == 0) st_relaxed(&status[tile], kFlagA | (unsigned long long)block_total);
                int64_t t = tile - 1;
                for (;;) {
                    const int64_t idx = t - lane;
                    const unsigned long long s = idx >= 0 ? ld_relaxed(&status[idx]) : kFlagP;
                    const unsigned long long flag = s & ~kMask;
                    const unsigned pmask = __ballot_sync(0xffffffffu, flag == kFlagP);
                    const unsigned xmask = __ballot_sync(0xffffffffu, flag == 0);
                    const int first_p = pmask ? __ffs(pmask) - 1 : 31;
                    const unsigned need = (first_p == 31) ? 0xffffffffu : ((2u << first_p) - 1u);
                    if (xmask & need) continue;  // a needed predecessor has not published yet
                    int64_t v = (lane <= first_p) ? (int64_t)(s & kMask) : 0;
#pragma unroll
                    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                    prefix += v;
                    if (pmask) break;
                    t -= 32;
                }
                if (lane == 0) st_relaxed(&status[tile], kFlagP | (unsigned long long)(prefix + block_total));
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (tile == ntiles - 1 && total) *total = prefix + block_total;
            }
        }
        __syncthreads();
        const int64_t pre = s_prefix + warp_excl;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int64_t idx = base + i * 32 + lane;
            if (idx < n) out(idx, pre + (int64_t)(incl[i] - val[i]), (int64_t)val[i]);
        }
        __syncthreads();
    }
}

dgnn_status scratch(dgnn_ctx* c, size_t bytes, unsigned long long** status);  // ctx.cu

template <class In, class Out>
dgnn_status run(dgnn_ctx* c, int64_t max_n, const int64_t* n_dev, In in, Out out, int64_t* total_dev) {
    if (max_n < 0) max_n = 0;
    const int64_t tiles = (max_n + kTile - 1) / kTile;
    const size_t nst = (size_t)(tiles > 0 ? tiles : 1);
    unsigned long long* status = nullptr;
    DGNN_TRY(scratch(c, sizeof(unsigned long long) * (nst + 1), &status));
    unsigned int* counter = reinterpret_cast<unsigned int*>(status + nst);
    DGNN_TRY(memset_async(c, status, 0, sizeof(unsigned long long) * (nst + 1)));
    int blocks = (int)(tiles < (int64_t)c->num_sms * 4 ? tiles : (int64_t)c->num_sms * 4);
    if (blocks < 1) blocks = 1;
    launch(c, DGNN_K_SCAN, 0.0, [&] {
        scan_kernel<In, Out><<<blocks, kThreads, 0, c->stream>>>(n_dev, max_n, in, out, status, counter, total_dev);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}
}  // namespace scan

// ------------------------------------------------------------ radix sort
// Stable LSD radix sort of (uint32 key, uint32 value) pairs by key bits
// [0, end_bit) (sort.cu).  On entry (*keys, *vals) hold the input and
// (*keys_alt, *vals_alt) are scratch of the same size; the pointers are swapped
// pass by pass, so on return (*keys, *vals) point at the sorted pairs.
namespace radix {
dgnn_status sort_pairs(dgnn_ctx* c, int64_t n, int end_bit, uint32_t** keys, uint32_t** vals, uint32_t** keys_alt,
                       uint32_t** vals_alt);
}  // namespace radix

}  // namespace dgnn

// Library-owned result objects.
struct dgnn_samples {
    dgnn_ctx* ctx = nullptr;
    int64_t nb = 0;
    int32_t H = 0;
    int32_t mode = DGNN_SAMPLE_NODEWISE;
    int64_t batch_id_base = 0;
    int64_t total_nodes = 0, total_edges = 0, total_eptr = 0;
    int64_t cap_nodes = 0, cap_edges = 0, cap_eptr = 0;
    int64_t* node_off = nullptr;
    int32_t* nodes = nullptr;
    int32_t* hop_off = nullptr;
    int64_t* eptr_off = nullptr;
    int32_t* eptr = nullptr;
    int64_t* edge_off = nullptr;
    int32_t* src_local = nullptr;
    std::vector<int64_t> node_off_h, edge_off_h, eptr_off_h;
    std::vector<int32_t> hop_off_h;
};

struct dgnn_cache_plan {
    dgnn_ctx* ctx = nullptr;
    int64_t N = 0, k_gpu = 0, k_host = 0;
    uint32_t* tier_map = nullptr;
    int32_t* gpu_ids = nullptr;
    int32_t* host_ids = nullptr;
    uint32_t gpu_min = 0, host_min = 0;
};
