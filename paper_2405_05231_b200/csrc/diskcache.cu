// diskcache.cu -- the segmented disk cache (Sec. 5.1).
//
// Readings d1-d8 are stated in include/dgnn.h and DESIGN.md.  GPU design:
//  * index: an epoch's packed rows (the DISK occurrences, batch-major) are radix
//    sorted once by node ID (stable, so each node's run lists its batches in
//    ascending order).  For any s, the rows of node v inside segment g are then
//    one contiguous run, so the local frequency of (v, g) is a run length.
//  * space(s, m) (Eq. 2) is one streaming pass over the sorted rows per s; many s
//    are evaluated by one launch (blockIdx.y), which makes the heuristic's
//    linear search for the minimum feasible s a handful of launches.
//  * plan: runs longer than m become cache entries; Algorithm 1's signatures
//    are per-run minima of a (batch, hash) table of permutation ranks; "Sort(S)"
//    is k+1 stable LSD radix passes over (segment, S_0..S_{k-1}, node), entries
//    starting in node order; merged page requests come from per-batch bitmaps
//    over the segment's pages (ascending by construction).
#include <memory>
#include <type_traits>

#include "rowcopy.cuh"

struct dgnn_disk_index {
    dgnn_ctx* ctx = nullptr;
    int64_t nb = 0, R = 0, N = 0;
    int32_t* packed_ids = nullptr;  // [R]
    int64_t* packed_off = nullptr;  // [nb+1]
    std::vector<int64_t> packed_off_h;
    uint32_t* rv = nullptr;  // node of sorted row j
    int32_t* rb = nullptr;   // batch of sorted row j
    uint32_t* rr = nullptr;  // input row index of sorted row j
};

struct dgnn_disk_plan {
    dgnn_ctx* ctx = nullptr;
    int64_t nb = 0, R = 0, nseg = 0, s = 0, m = 0, fpp = 0, row_bytes = 0;
    int64_t n_cache = 0, n_pk = 0, n_req = 0;
    int64_t totals[4] = {};
    int64_t* packed_off = nullptr;
    int64_t* seg_off = nullptr;
    int32_t* cache_ids = nullptr;
    int64_t* seg_page_off = nullptr;
    int32_t* pk_ids = nullptr;
    int64_t* pk_off = nullptr;
    int32_t* req_pages = nullptr;
    int64_t* req_off = nullptr;
    uint32_t* dc_addr = nullptr;
    std::vector<int64_t> packed_off_h, pk_off_h, req_off_h, seg_off_h, seg_page_off_h;
};

namespace dgnn {
namespace {

constexpr int64_t kPage = 4096;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kSmemBatches = 2048;
constexpr int kSpaceChunk = 32;  // s values per launch of the search

int bits_for(int64_t max_value) {
    int b = 0;
    while (b < 32 && (max_value >> b) > 0) ++b;
    return b;
}

__global__ void k_iota_keys(const int32_t* __restrict__ ids, int64_t R, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        keys[r] = (uint32_t)ids[r];
        vals[r] = (uint32_t)r;
    }
}

__global__ void k_batch_of(const uint32_t* __restrict__ rr, int64_t R, const int64_t* __restrict__ packed_off, int nb,
                           int32_t* __restrict__ rb) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R; j += (int64_t)gridDim.x * blockDim.x)
        rb[j] = segment_of(packed_off, nb + 1, (int64_t)rr[j]);
}

// run of node rv[j] inside segment g starting at j: its length (0 if j does not start a run)
__device__ __forceinline__ int run_length(const uint32_t* rv, const int32_t* rb, int64_t R, int64_t j, int s) {
    const uint32_t v = rv[j];
    const int g = rb[j] / s;
    if (j > 0 && rv[j - 1] == v && rb[j - 1] / s == g) return 0;
    int len = 1;
    while (j + len < R && rv[j + len] == v && rb[j + len] / s == g) ++len;
    return len;
}

// Eq. 2 space counts for several s at once: per s (blockIdx.y) the cached entries per
// segment and the rows that stay packed per batch.
__global__ void __launch_bounds__(256) k_space_counts(const uint32_t* __restrict__ rv, const int32_t* __restrict__ rb,
                                                      int64_t R, const int64_t* __restrict__ s_list, int64_t m, int nb,
                                                      uint32_t* __restrict__ seg_cnt, uint32_t* __restrict__ pk_cnt) {
    __shared__ uint32_t s_seg[kSmemBatches], s_pk[kSmemBatches];
    const int si = blockIdx.y;
    const int s = (int)s_list[si];
    const bool sm = nb <= kSmemBatches;
    uint32_t* gseg = seg_cnt + (int64_t)si * nb;
    uint32_t* gpk = pk_cnt + (int64_t)si * nb;
    if (sm) {
        for (int i = threadIdx.x; i < nb; i += blockDim.x) s_seg[i] = s_pk[i] = 0;
        __syncthreads();
    }
    uint32_t* cs = sm ? s_seg : gseg;
    uint32_t* cp = sm ? s_pk : gpk;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R; j += (int64_t)gridDim.x * blockDim.x) {
        const int len = run_length(rv, rb, R, j, s);
        if (len == 0) continue;
        if (len > m) atomicAdd(&cs[rb[j] / s], 1u);
        else
            for (int q = 0; q < len; ++q) atomicAdd(&cp[rb[j + q]], 1u);
    }
    if (sm) {
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            if (s_seg[i]) atomicAdd(&gseg[i], s_seg[i]);
            if (s_pk[i]) atomicAdd(&gpk[i], s_pk[i]);
        }
    }
}

__device__ __forceinline__ int64_t block_sum(int64_t v) {
    __shared__ int64_t s_part[32];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
    __syncthreads();
    return t;  // valid in thread 0
}

__global__ void k_space_reduce(const uint32_t* __restrict__ seg_cnt, const uint32_t* __restrict__ pk_cnt,
                               const int64_t* __restrict__ s_list, int nb, int64_t fpp, int64_t row_bytes,
                               int64_t* __restrict__ pages) {
    const int si = blockIdx.x;
    const int64_t s = s_list[si];
    const int nseg = (int)((nb + s - 1) / s);
    int64_t acc = 0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        if (i < nseg) acc += ((int64_t)seg_cnt[(int64_t)si * nb + i] + fpp - 1) / fpp;
        acc += ((int64_t)pk_cnt[(int64_t)si * nb + i] * row_bytes + kPage - 1) / kPage;
    }
    const int64_t t = block_sum(acc);
    if (threadIdx.x == 0) pages[si] = t;
}

// ---- plan kernels
__global__ void k_runs(const uint32_t* __restrict__ rv, const int32_t* __restrict__ rb, int64_t R, int s,
                       uint32_t* __restrict__ glen) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R; j += (int64_t)gridDim.x * blockDim.x)
        glen[j] = (uint32_t)run_length(rv, rb, R, j, s);
}

// d5: Philox key of (local index i, segment g, hash t)
__global__ void k_perm_x(int nb, int s, int k, uint64_t seed, unsigned long long* __restrict__ X) {
    const int64_t n = (int64_t)nb * k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / k), t = (int)(q % k);
        const int g = b / s;
        X[q] = draw64(seed, (uint32_t)(b - g * s), (0x4D48ull << 32) | (uint32_t)g, 0u, (uint32_t)t);
    }
}

// H[b*k+t] = rank of b's local index among its segment's indices ordered by (X, index)
__global__ void k_perm_rank(int nb, int s, int k, const unsigned long long* __restrict__ X, uint32_t* __restrict__ H) {
    const int64_t n = (int64_t)nb * k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / k), t = (int)(q % k);
        const int g0 = (b / s) * s, g1 = min(g0 + s, nb);
        const unsigned long long x = X[q];
        uint32_t rank = 0;
        for (int c = g0; c < g1; ++c) {
            const unsigned long long y = X[(int64_t)c * k + t];
            rank += (y < x || (y == x && c < b)) ? 1u : 0u;
        }
        H[q] = rank;
    }
}

// Algorithm 1 lines 4-8 per cache entry (reading d6): S_t = min over the run's batches
__global__ void k_signatures(const uint32_t* __restrict__ ent_j, int64_t ne, const uint32_t* __restrict__ glen,
                             const int32_t* __restrict__ rb, int s, int k, const uint32_t* __restrict__ H,
                             uint32_t* __restrict__ sig, uint32_t* __restrict__ ent_seg) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j0 = ent_j[e];
        const uint32_t len = glen[j0];
        ent_seg[e] = (uint32_t)(rb[j0] / s);
        for (int t = 0; t < k; ++t) {
            uint32_t mn = kNone;
            for (uint32_t q = 0; q < len; ++q) mn = min(mn, H[(int64_t)rb[j0 + q] * k + t]);
            sig[(int64_t)t * ne + e] = mn;
        }
    }
}

// reading d6 vs Algorithm 1 line 8 as printed (reorder = 2): S(v) = min over t of S_t(v)
__global__ void k_sig_min(uint32_t* __restrict__ sig, int64_t ne, int k) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t mn = sig[e];
        for (int t = 1; t < k; ++t) mn = min(mn, sig[(int64_t)t * ne + e]);
        sig[e] = mn;
    }
}

__global__ void k_iota(uint32_t* __restrict__ a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

__global__ void k_gather_key(const uint32_t* __restrict__ src, const uint32_t* __restrict__ ord, int64_t n,
                             uint32_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = src[ord[i]];
}

__global__ void k_seg_count(const uint32_t* __restrict__ ent_seg, int64_t ne, uint32_t* __restrict__ cnt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[ent_seg[e]], 1u);
}

// V_r: position p of the sorted order holds entry ord[p]
__global__ void k_place(const uint32_t* __restrict__ ord, int64_t ne, const uint32_t* __restrict__ ent_j,
                        const uint32_t* __restrict__ rv, int32_t* __restrict__ cache_ids, uint32_t* __restrict__ ent_pos) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < ne; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = ord[p];
        cache_ids[p] = (int32_t)rv[ent_j[e]];
        ent_pos[e] = (uint32_t)p;
    }
}

// cache position of every input row that belongs to a cached run
__global__ void k_mark(const uint32_t* __restrict__ ent_j, int64_t ne, const uint32_t* __restrict__ glen,
                       const uint32_t* __restrict__ ent_pos, const uint32_t* __restrict__ rr, uint32_t* __restrict__ cpos) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j0 = ent_j[e], len = glen[j0], p = ent_pos[e];
        for (uint32_t q = 0; q < len; ++q) cpos[rr[j0 + q]] = p;
    }
}

__global__ void k_pk_off(const int64_t* __restrict__ packed_off, int nb, int64_t R, const uint32_t* __restrict__ pkx,
                         const int64_t* __restrict__ n_pk, int64_t* __restrict__ pk_off) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        const int64_t r = packed_off[b];
        pk_off[b] = r < R ? (int64_t)pkx[r] : *n_pk;
    }
}

__global__ void k_set_bits(const uint32_t* __restrict__ cpos, int64_t R, const int64_t* __restrict__ packed_off, int nb,
                           int s, const int64_t* __restrict__ seg_off, int64_t fpp, const int64_t* __restrict__ bm_off,
                           uint32_t* __restrict__ bm) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = cpos[r];
        if (p == kNone) continue;
        const int b = segment_of(packed_off, nb + 1, r);
        const int64_t lp = ((int64_t)p - seg_off[b / s]) / fpp;
        atomicOr(&bm[bm_off[b] + (lp >> 5)], 1u << (lp & 31));
    }
}

__global__ void k_req_off(const int64_t* __restrict__ bm_off, int nb, int64_t W, const uint32_t* __restrict__ wpos,
                          const int64_t* __restrict__ n_req, int64_t* __restrict__ req_off) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x)
        req_off[b] = bm_off[b] < W ? (int64_t)wpos[bm_off[b]] : *n_req;
}

__global__ void k_emit_pages(const uint32_t* __restrict__ bm, int64_t W, const int64_t* __restrict__ bm_off, int nb,
                             int s, const int64_t* __restrict__ seg_page_off, const uint32_t* __restrict__ wpos,
                             int32_t* __restrict__ req_pages) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t word = bm[w];
        if (!word) continue;
        const int b = segment_of(bm_off, nb + 1, w);
        const int64_t first = seg_page_off[b / s] + (w - bm_off[b]) * 32;
        uint32_t o = wpos[w];
        while (word) {
            const int bit = __ffs(word) - 1;
            req_pages[o++] = (int32_t)(first + bit);
            word &= word - 1;
        }
    }
}

// reading d8
__global__ void k_addr(const uint32_t* __restrict__ cpos, const uint32_t* __restrict__ pkx, int64_t R,
                       const int64_t* __restrict__ packed_off, int nb, int s, const int64_t* __restrict__ pk_off,
                       const int64_t* __restrict__ seg_off, int64_t fpp, const int64_t* __restrict__ bm_off,
                       const uint32_t* __restrict__ bm, const uint32_t* __restrict__ wpos,
                       const int64_t* __restrict__ req_off, uint32_t* __restrict__ dc_addr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const int b = segment_of(packed_off, nb + 1, r);
        const uint32_t p = cpos[r];
        if (p == kNone) {
            dc_addr[r] = (uint32_t)((int64_t)pkx[r] - pk_off[b]);
            continue;
        }
        const int64_t in_seg = (int64_t)p - seg_off[b / s];
        const int64_t lp = in_seg / fpp;
        const int64_t w = bm_off[b] + (lp >> 5);
        const int64_t q = (int64_t)wpos[w] - req_off[b] + __popc(bm[w] & ((1u << (lp & 31)) - 1u));
        dc_addr[r] = 0x80000000u | (uint32_t)(q * fpp + in_seg % fpp);
    }
}

__global__ void k_totals(const int64_t* __restrict__ pk_off, const int64_t* __restrict__ req_off, int nb,
                         int64_t row_bytes, unsigned long long* __restrict__ out) {
    int64_t chunk = 0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x)
        chunk += ((pk_off[b + 1] - pk_off[b]) * row_bytes + kPage - 1) / kPage;
    const int64_t t = block_sum(chunk);
    if (threadIdx.x == 0 && t) atomicAdd(out, (unsigned long long)t);
}

// ---- materialization
struct CacheRow {
    const uint8_t* src;
    int64_t row_bytes, fpp;
    const int32_t* ids;
    const int64_t* seg_off;
    const int64_t* seg_page_off;
    int nseg;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t p, const uint8_t*& s, uint8_t*& d) const {
        const int g = segment_of(seg_off, nseg + 1, p);
        const int64_t lp = p - seg_off[g];
        s = src + (int64_t)ids[p] * row_bytes;
        d = dst + (seg_page_off[g] + lp / fpp) * kPage + (lp % fpp) * row_bytes;
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256) k_cache_fill(CacheRow fn, int64_t n) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<4, V>(n, fn.row_bytes, fn, warp, nwarps);
}

// zero every byte of a cache page past its rows (warp per page)
__global__ void k_cache_zero(const int64_t* __restrict__ seg_off, const int64_t* __restrict__ seg_page_off, int nseg,
                             int64_t pages, int64_t fpp, int64_t row_bytes, uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (int64_t P = warp; P < pages; P += nwarps) {
        const int g = segment_of(seg_page_off, nseg + 1, P);
        const int64_t rows = min(fpp, seg_off[g + 1] - seg_off[g] - (P - seg_page_off[g]) * fpp);
        uint4* z = reinterpret_cast<uint4*>(dst + P * kPage + rows * row_bytes);
        const int64_t nz = (kPage - rows * row_bytes) / 16;
        for (int64_t i = lane; i < nz; i += 32) __stcs(z + i, make_uint4(0, 0, 0, 0));
    }
}

struct PartialRow {
    const uint8_t* pages;
    const uint8_t* chunks;
    const int64_t* chunk_off;
    const int64_t* packed_off;  // input packed lists, global
    const int64_t* req_off;
    const uint32_t* dc_addr;
    const int64_t* out_off;
    int64_t row_bytes, fpp;
    int b_lo, nbr;
    int64_t r0;
    uint8_t* out;
    __device__ __forceinline__ bool operator()(int64_t i, const uint8_t*& s, uint8_t*& d) const {
        const int64_t r = r0 + i;
        const int bl = segment_of(packed_off + b_lo, nbr + 1, r);
        const int b = b_lo + bl;
        const uint32_t a = dc_addr[r];
        if (a & 0x80000000u) {
            const int64_t x = a & 0x7FFFFFFFu;
            s = pages + (req_off[b] - req_off[b_lo] + x / fpp) * kPage + (x % fpp) * row_bytes;
        } else {
            s = chunks + chunk_off[bl] + (int64_t)a * row_bytes;
        }
        d = out + out_off[bl] + (r - packed_off[b]) * row_bytes;
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256) k_partial(PartialRow fn, int64_t n) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<4, V>(n, fn.row_bytes, fn, warp, nwarps);
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <class T>
dgnn_status d2h(dgnn_ctx* c, T* host, const T* dev, size_t n) {
    if (n) DGNN_CK(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    DGNN_CK(cudaStreamSynchronize(c->stream));
    return DGNN_OK;
}

int grid1(dgnn_ctx* c, int64_t n) { return grid_for(c, n, 256); }

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_disk_index_build(dgnn_ctx* c, const int32_t* packed_ids, const int64_t* packed_off,
                                             const int64_t* packed_off_host, int64_t nb, int64_t num_nodes,
                                             dgnn_disk_index** out) {
    DGNN_REQUIRE(c && out && packed_off && packed_off_host && nb >= 0, "dgnn_disk_index_build: NULL argument");
    *out = nullptr;
    const int64_t R = packed_off_host[nb];
    DGNN_REQUIRE(R >= 0 && R < (int64_t(1) << 31) && num_nodes >= 0 && num_nodes <= (int64_t(1) << 31) &&
                     nb < (int64_t(1) << 31) && (R == 0 || packed_ids),
                 "dgnn_disk_index_build: sizes out of range (R=%lld, N=%lld)", (long long)R, (long long)num_nodes);
    DGNN_CK(cudaSetDevice(c->device));
    auto* x = new dgnn_disk_index();
    std::unique_ptr<dgnn_disk_index, void (*)(dgnn_disk_index*)> guard(x, dgnn_disk_index_free);
    x->ctx = c;
    x->nb = nb;
    x->R = R;
    x->N = num_nodes;
    x->packed_off_h.assign(packed_off_host, packed_off_host + nb + 1);
    DevBuf<int32_t> ids, rb;
    DevBuf<int64_t> off;
    DevBuf<uint32_t> k0, v0, k1, v1;
    DGNN_TRY(ids.alloc(c, (size_t)R));
    DGNN_TRY(off.alloc(c, (size_t)nb + 1));
    DGNN_TRY(rb.alloc(c, (size_t)R));
    DGNN_TRY(k0.alloc(c, (size_t)R));
    DGNN_TRY(v0.alloc(c, (size_t)R));
    DGNN_TRY(k1.alloc(c, (size_t)R));
    DGNN_TRY(v1.alloc(c, (size_t)R));
    if (R) DGNN_CK(cudaMemcpyAsync(ids.p, packed_ids, R * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
    DGNN_CK(cudaMemcpyAsync(off.p, packed_off, (nb + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
    uint32_t *kk = k0.p, *vv = v0.p, *ka = k1.p, *va = v1.p;
    if (R) {
        launch(c, DGNN_K_SORT, 12.0 * R, [&] { k_iota_keys<<<grid1(c, R), 256, 0, c->stream>>>(ids.p, R, kk, vv); });
        DGNN_CK_LAUNCH();
        DGNN_TRY(radix::sort_pairs(c, R, bits_for(num_nodes > 0 ? num_nodes - 1 : 0), &kk, &vv, &ka, &va));
        launch(c, DGNN_K_SORT, 8.0 * R,
               [&] { k_batch_of<<<grid1(c, R), 256, 0, c->stream>>>(vv, R, off.p, (int)nb, rb.p); });
        DGNN_CK_LAUNCH();
    }
    // keep the sorted pair, the scratch pair is freed with its DevBufs
    x->rv = kk;
    x->rr = vv;
    if (kk == k0.p) k0.release(); else k1.release();
    if (vv == v0.p) v0.release(); else v1.release();
    x->packed_ids = ids.release();
    x->packed_off = off.release();
    x->rb = rb.release();
    DGNN_TRY(check_dev_err(c));
    *out = guard.release();
    return DGNN_OK;
}

extern "C" void dgnn_disk_index_free(dgnn_disk_index* x) {
    if (!x) return;
    dgnn_ctx* c = x->ctx;
    cudaSetDevice(c->device);
    dev_free(c, x->packed_ids, (size_t)(x->R ? x->R : 1) * sizeof(int32_t));
    dev_free(c, x->packed_off, (size_t)(x->nb + 1) * sizeof(int64_t));
    dev_free(c, x->rv, (size_t)(x->R ? x->R : 1) * sizeof(uint32_t));
    dev_free(c, x->rr, (size_t)(x->R ? x->R : 1) * sizeof(uint32_t));
    dev_free(c, x->rb, (size_t)(x->R ? x->R : 1) * sizeof(int32_t));
    delete x;
}

namespace dgnn {
namespace {
dgnn_status space_many(dgnn_ctx* c, const dgnn_disk_index* x, int64_t row_bytes, const int64_t* s_host, int64_t n_s,
                       int64_t m, int64_t* pages_host) {
    const int nb = (int)x->nb;
    if (nb == 0) {
        for (int64_t i = 0; i < n_s; ++i) pages_host[i] = 0;
        return DGNN_OK;
    }
    const int64_t fpp = kPage / row_bytes;
    DevBuf<int64_t> sl, pg;
    DevBuf<uint32_t> sc, pc;
    DGNN_TRY(sl.alloc(c, (size_t)n_s));
    DGNN_TRY(pg.alloc(c, (size_t)n_s));
    DGNN_TRY(sc.alloc(c, (size_t)(n_s * nb)));
    DGNN_TRY(pc.alloc(c, (size_t)(n_s * nb)));
    DGNN_CK(cudaMemcpyAsync(sl.p, s_host, n_s * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    DGNN_TRY(memset_async(c, sc.p, 0, (size_t)(n_s * nb) * sizeof(uint32_t)));
    DGNN_TRY(memset_async(c, pc.p, 0, (size_t)(n_s * nb) * sizeof(uint32_t)));
    if (x->R) {
        int bx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(x->R, 256), (int64_t)c->num_sms * 8 / n_s));
        dim3 grid(bx, (unsigned)n_s);
        launch(c, DGNN_K_DISK_PLAN, 8.0 * x->R * n_s, [&] {
            k_space_counts<<<grid, 256, 0, c->stream>>>(x->rv, x->rb, x->R, sl.p, m, nb, sc.p, pc.p);
        });
        DGNN_CK_LAUNCH();
    }
    launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
        k_space_reduce<<<(unsigned)n_s, 256, 0, c->stream>>>(sc.p, pc.p, sl.p, nb, fpp, row_bytes, pg.p);
    });
    DGNN_CK_LAUNCH();
    return d2h(c, pages_host, pg.p, (size_t)n_s);
}
}  // namespace
}  // namespace dgnn

extern "C" dgnn_status dgnn_disk_space(dgnn_ctx* c, const dgnn_disk_index* x, int64_t row_bytes,
                                       const int64_t* s_list_host, int64_t n_s, int64_t m, int64_t* pages_host) {
    DGNN_REQUIRE(c && x && (n_s == 0 || (s_list_host && pages_host)) && n_s >= 0, "dgnn_disk_space: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes <= kPage && m >= 0, "dgnn_disk_space: bad row_bytes or m");
    for (int64_t i = 0; i < n_s; ++i) DGNN_REQUIRE(s_list_host[i] >= 1, "dgnn_disk_space: s must be >= 1");
    DGNN_CK(cudaSetDevice(c->device));
    for (int64_t i0 = 0; i0 < n_s; i0 += kSpaceChunk) {
        const int64_t n = std::min<int64_t>(kSpaceChunk, n_s - i0);
        DGNN_TRY(space_many(c, x, row_bytes, s_list_host + i0, n, m, pages_host + i0));
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_disk_search(dgnn_ctx* c, const dgnn_disk_index* x, int64_t row_bytes, int64_t m,
                                        int64_t budget_pages, int64_t* s_out, int64_t* pages_out) {
    DGNN_REQUIRE(c && x && s_out && pages_out, "dgnn_disk_search: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes <= kPage && m >= 0, "dgnn_disk_search: bad row_bytes or m");
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t s_max = x->nb > 0 ? x->nb : 1;
    int64_t sl[kSpaceChunk], pg[kSpaceChunk];
    int64_t last = 0;
    for (int64_t s0 = 1; s0 <= s_max; s0 += kSpaceChunk) {
        const int64_t n = std::min<int64_t>(kSpaceChunk, s_max - s0 + 1);
        for (int64_t i = 0; i < n; ++i) sl[i] = s0 + i;
        DGNN_TRY(space_many(c, x, row_bytes, sl, n, m, pg));
        for (int64_t i = 0; i < n; ++i)
            if (pg[i] <= budget_pages) {
                *s_out = sl[i];
                *pages_out = pg[i];
                return DGNN_OK;
            }
        last = pg[n - 1];
    }
    *s_out = 0;
    *pages_out = last;
    return DGNN_OK;
}

extern "C" void dgnn_disk_plan_free(dgnn_disk_plan* p) {
    if (!p) return;
    dgnn_ctx* c = p->ctx;
    cudaSetDevice(c->device);
    auto fr = [&](void* q, int64_t n, size_t el) { dev_free(c, q, (size_t)(n > 0 ? n : 1) * el); };
    fr(p->packed_off, p->nb + 1, 8);
    fr(p->seg_off, p->nseg + 1, 8);
    fr(p->cache_ids, p->n_cache, 4);
    fr(p->seg_page_off, p->nseg + 1, 8);
    fr(p->pk_ids, p->n_pk, 4);
    fr(p->pk_off, p->nb + 1, 8);
    fr(p->req_pages, p->n_req, 4);
    fr(p->req_off, p->nb + 1, 8);
    fr(p->dc_addr, p->R, 4);
    delete p;
}

extern "C" dgnn_status dgnn_disk_plan_build(dgnn_ctx* c, const dgnn_disk_index* x, int64_t row_bytes, int64_t s,
                                            int64_t m, int32_t k, uint64_t seed, int32_t reorder, dgnn_disk_plan** out) {
    DGNN_REQUIRE(c && x && out, "dgnn_disk_plan_build: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes <= kPage && s >= 1 && m >= 0 && k >= 1 && k <= 16,
                 "dgnn_disk_plan_build: bad row_bytes/s/m/k");
    *out = nullptr;
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t nb = x->nb, R = x->R;
    const int si = (int)std::min<int64_t>(s, nb > 0 ? nb : 1);  // s > nb behaves as s = nb
    const int64_t nseg = nb > 0 ? ceil_div(nb, si) : 0;
    const int64_t fpp = kPage / row_bytes;
    auto* p = new dgnn_disk_plan();
    p->ctx = c;
    p->nb = nb;
    p->R = R;
    p->nseg = nseg;
    p->s = s;
    p->m = m;
    p->fpp = fpp;
    p->row_bytes = row_bytes;
    p->packed_off_h = x->packed_off_h;
    std::unique_ptr<dgnn_disk_plan, void (*)(dgnn_disk_plan*)> guard(p, dgnn_disk_plan_free);
    auto alloc = [&](auto** ptr, int64_t n) -> dgnn_status {
        using T = std::remove_pointer_t<std::remove_reference_t<decltype(*ptr)>>;
        *ptr = static_cast<T*>(dev_alloc(c, (size_t)(n > 0 ? n : 1) * sizeof(T)));
        if (!*ptr) {
            set_error("device allocation failed");
            return DGNN_ENOMEM;
        }
        return DGNN_OK;
    };
    DGNN_TRY(alloc(&p->packed_off, nb + 1));
    DGNN_CK(cudaMemcpyAsync(p->packed_off, x->packed_off, (nb + 1) * 8, cudaMemcpyDeviceToDevice, c->stream));
    DGNN_TRY(alloc(&p->seg_off, nseg + 1));
    DGNN_TRY(alloc(&p->seg_page_off, nseg + 1));
    DGNN_TRY(alloc(&p->pk_off, nb + 1));
    DGNN_TRY(alloc(&p->req_off, nb + 1));
    DGNN_TRY(alloc(&p->dc_addr, R));
    DevBuf<int64_t> tot;  // device scalars: [0] n_ent, [1] n_pk, [2] n_req, [3] W, [4] chunk pages
    DGNN_TRY(tot.alloc(c, 5));
    DGNN_TRY(memset_async(c, tot.p, 0, 5 * sizeof(int64_t)));
    int64_t h[5] = {};

    // 1. runs and cache entries (d2)
    DevBuf<uint32_t> glen, ent_j;
    DGNN_TRY(glen.alloc(c, (size_t)R));
    DGNN_TRY(ent_j.alloc(c, (size_t)R));
    if (R) {
        launch(c, DGNN_K_DISK_PLAN, 8.0 * R,
               [&] { k_runs<<<grid1(c, R), 256, 0, c->stream>>>(x->rv, x->rb, R, si, glen.p); });
        DGNN_CK_LAUNCH();
        const uint32_t* gl = glen.p;
        uint32_t* ej = ent_j.p;
        DGNN_TRY(scan::run(
            c, R, nullptr, [gl, m] __device__(int64_t j) -> int32_t { return gl[j] > (uint32_t)m ? 1 : 0; },
            [ej] __device__(int64_t j, int64_t excl, int64_t v) {
                if (v) ej[excl] = (uint32_t)j;
            },
            tot.p + 0));
    }
    DGNN_TRY(d2h(c, h, tot.p, 1));
    const int64_t ne = h[0];
    p->n_cache = ne;

    // 2. permutations and signatures (d5, d6); 3. Line 9 sort
    DevBuf<uint32_t> ent_seg, ord, ord_alt, keys, keys_alt;
    DGNN_TRY(ent_seg.alloc(c, (size_t)ne));
    DGNN_TRY(ord.alloc(c, (size_t)ne));
    DGNN_TRY(ord_alt.alloc(c, (size_t)ne));
    DGNN_TRY(keys.alloc(c, (size_t)ne));
    DGNN_TRY(keys_alt.alloc(c, (size_t)ne));
    {
        DevBuf<unsigned long long> X;
        DevBuf<uint32_t> H, sig;
        const int kk = reorder ? k : 1;
        DGNN_TRY(X.alloc(c, (size_t)(nb * kk)));
        DGNN_TRY(H.alloc(c, (size_t)(nb * kk)));
        DGNN_TRY(sig.alloc(c, (size_t)(ne * kk)));
        if (nb) {
            launch(c, DGNN_K_DISK_PLAN, 0.0,
                   [&] { k_perm_x<<<grid1(c, nb * kk), 256, 0, c->stream>>>((int)nb, si, kk, seed, X.p); });
            DGNN_CK_LAUNCH();
            launch(c, DGNN_K_DISK_PLAN, 0.0,
                   [&] { k_perm_rank<<<grid1(c, nb * kk), 256, 0, c->stream>>>((int)nb, si, kk, X.p, H.p); });
            DGNN_CK_LAUNCH();
        }
        if (ne) {
            launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
                k_signatures<<<grid1(c, ne), 256, 0, c->stream>>>(ent_j.p, ne, glen.p, x->rb, si, kk, H.p, sig.p,
                                                                  ent_seg.p);
            });
            DGNN_CK_LAUNCH();
            launch(c, DGNN_K_DISK_PLAN, 0.0, [&] { k_iota<<<grid1(c, ne), 256, 0, c->stream>>>(ord.p, ne); });
            DGNN_CK_LAUNCH();
            uint32_t *o = ord.p, *oa = ord_alt.p, *ky = keys.p, *ka = keys_alt.p;
            auto pass = [&](const uint32_t* src, int bits) -> dgnn_status {
                launch(c, DGNN_K_SORT, 12.0 * ne,
                       [&] { k_gather_key<<<grid1(c, ne), 256, 0, c->stream>>>(src, o, ne, ky); });
                DGNN_CK_LAUNCH();
                return radix::sort_pairs(c, ne, bits, &ky, &o, &ka, &oa);
            };
            if (reorder == 2) {  // Algorithm 1 line 8 verbatim: one scalar min over the k functions
                launch(c, DGNN_K_DISK_PLAN, 0.0,
                       [&] { k_sig_min<<<grid1(c, ne), 256, 0, c->stream>>>(sig.p, ne, kk); });
                DGNN_CK_LAUNCH();
                DGNN_TRY(pass(sig.p, bits_for(si - 1)));
            } else if (reorder) {
                for (int t = k - 1; t >= 0; --t) DGNN_TRY(pass(sig.p + (int64_t)t * ne, bits_for(si - 1)));
            }
            DGNN_TRY(pass(ent_seg.p, bits_for(nseg - 1)));
            if (o != ord.p) std::swap(ord.p, ord_alt.p);  // the sorted order lives in ord.p
        }
    }

    // 4. segment offsets (cache rows, pages), V_r, cache position of every row
    DevBuf<uint32_t> seg_cnt, ent_pos, cpos, pkx;
    DGNN_TRY(seg_cnt.alloc(c, (size_t)nseg));
    DGNN_TRY(memset_async(c, seg_cnt.p, 0, (size_t)(nseg > 0 ? nseg : 1) * 4));
    if (ne) {
        launch(c, DGNN_K_DISK_PLAN, 0.0,
               [&] { k_seg_count<<<grid1(c, ne), 256, 0, c->stream>>>(ent_seg.p, ne, seg_cnt.p); });
        DGNN_CK_LAUNCH();
    }
    {
        const uint32_t* sc = seg_cnt.p;
        int64_t* so = p->seg_off;
        int64_t* spo = p->seg_page_off;
        DGNN_TRY(scan::run(
            c, nseg + 1, nullptr, [sc, nseg] __device__(int64_t g) -> int64_t { return g < nseg ? (int64_t)sc[g] : 0; },
            [so] __device__(int64_t g, int64_t excl, int64_t) { so[g] = excl; }, nullptr));
        DGNN_TRY(scan::run(
            c, nseg + 1, nullptr,
            [sc, nseg, fpp] __device__(int64_t g) -> int64_t {
                return g < nseg ? ((int64_t)sc[g] + fpp - 1) / fpp : 0;
            },
            [spo] __device__(int64_t g, int64_t excl, int64_t) { spo[g] = excl; }, nullptr));
    }
    DGNN_TRY(alloc(&p->cache_ids, ne));
    DGNN_TRY(ent_pos.alloc(c, (size_t)ne));
    DGNN_TRY(cpos.alloc(c, (size_t)R));
    DGNN_TRY(memset_async(c, cpos.p, 0xFF, (size_t)(R > 0 ? R : 1) * 4));
    if (ne) {
        launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
            k_place<<<grid1(c, ne), 256, 0, c->stream>>>(ord.p, ne, ent_j.p, x->rv, p->cache_ids, ent_pos.p);
        });
        DGNN_CK_LAUNCH();
        launch(c, DGNN_K_DISK_PLAN, 0.0,
               [&] { k_mark<<<grid1(c, ne), 256, 0, c->stream>>>(ent_j.p, ne, glen.p, ent_pos.p, x->rr, cpos.p); });
        DGNN_CK_LAUNCH();
    }

    // 5. reduced packed lists P_b'
    DGNN_TRY(pkx.alloc(c, (size_t)R));
    DGNN_TRY(alloc(&p->pk_ids, R));  // capacity R; n_pk <= R
    if (R) {
        const uint32_t* cp = cpos.p;
        uint32_t* px = pkx.p;
        int32_t* pid = p->pk_ids;
        const int32_t* ids = x->packed_ids;
        DGNN_TRY(scan::run(
            c, R, nullptr, [cp] __device__(int64_t r) -> int32_t { return cp[r] == kNone ? 1 : 0; },
            [px, pid, ids] __device__(int64_t r, int64_t excl, int64_t v) {
                px[r] = (uint32_t)excl;
                if (v) pid[excl] = ids[r];
            },
            tot.p + 1));
    }
    launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
        k_pk_off<<<grid1(c, nb + 1), 256, 0, c->stream>>>(p->packed_off, (int)nb, R, pkx.p, tot.p + 1, p->pk_off);
    });
    DGNN_CK_LAUNCH();

    // 6. merged page requests: per-batch bitmaps over the segment's pages (d7)
    DevBuf<int64_t> bm_off;
    DGNN_TRY(bm_off.alloc(c, (size_t)nb + 1));
    {
        const int64_t* spo = p->seg_page_off;
        int64_t* bo = bm_off.p;
        DGNN_TRY(scan::run(
            c, nb + 1, nullptr,
            [spo, nb, si] __device__(int64_t b) -> int64_t {
                if (b >= nb) return 0;
                const int64_t g = b / si;
                return (spo[g + 1] - spo[g] + 31) / 32;
            },
            [bo] __device__(int64_t b, int64_t excl, int64_t) { bo[b] = excl; }, tot.p + 3));
    }
    DGNN_TRY(d2h(c, h, tot.p, 5));
    p->n_pk = h[1];
    const int64_t W = h[3];
    DevBuf<uint32_t> bm, wpos;
    DGNN_TRY(bm.alloc(c, (size_t)W));
    DGNN_TRY(wpos.alloc(c, (size_t)W));
    DGNN_TRY(memset_async(c, bm.p, 0, (size_t)(W > 0 ? W : 1) * 4));
    if (R && ne) {
        launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
            k_set_bits<<<grid1(c, R), 256, 0, c->stream>>>(cpos.p, R, p->packed_off, (int)nb, si, p->seg_off, fpp,
                                                           bm_off.p, bm.p);
        });
        DGNN_CK_LAUNCH();
    }
    if (W) {
        const uint32_t* bmp = bm.p;
        uint32_t* wp = wpos.p;
        DGNN_TRY(scan::run(
            c, W, nullptr, [bmp] __device__(int64_t w) -> int32_t { return __popc(bmp[w]); },
            [wp] __device__(int64_t w, int64_t excl, int64_t) { wp[w] = (uint32_t)excl; }, tot.p + 2));
    }
    launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
        k_req_off<<<grid1(c, nb + 1), 256, 0, c->stream>>>(bm_off.p, (int)nb, W, wpos.p, tot.p + 2, p->req_off);
    });
    DGNN_CK_LAUNCH();
    DGNN_TRY(d2h(c, h, tot.p, 5));
    p->n_req = h[2];
    DGNN_TRY(alloc(&p->req_pages, p->n_req));
    if (W) {
        launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
            k_emit_pages<<<grid1(c, W), 256, 0, c->stream>>>(bm.p, W, bm_off.p, (int)nb, si, p->seg_page_off, wpos.p,
                                                             p->req_pages);
        });
        DGNN_CK_LAUNCH();
    }
    // 7. disk addresses (d8) and totals
    if (R) {
        launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
            k_addr<<<grid1(c, R), 256, 0, c->stream>>>(cpos.p, pkx.p, R, p->packed_off, (int)nb, si, p->pk_off,
                                                       p->seg_off, fpp, bm_off.p, bm.p, wpos.p, p->req_off, p->dc_addr);
        });
        DGNN_CK_LAUNCH();
    }
    if (nb) {
        launch(c, DGNN_K_DISK_PLAN, 0.0, [&] {
            k_totals<<<std::min<int64_t>(ceil_div(nb, 256), 64), 256, 0, c->stream>>>(
                p->pk_off, p->req_off, (int)nb, row_bytes, (unsigned long long*)(tot.p + 4));
        });
        DGNN_CK_LAUNCH();
    }
    DGNN_TRY(d2h(c, h, tot.p, 5));
    p->pk_off_h.resize(nb + 1);
    p->req_off_h.resize(nb + 1);
    p->seg_off_h.resize(nseg + 1);
    p->seg_page_off_h.resize(nseg + 1);
    DGNN_TRY(d2h(c, p->pk_off_h.data(), p->pk_off, nb + 1));
    DGNN_TRY(d2h(c, p->req_off_h.data(), p->req_off, nb + 1));
    DGNN_TRY(d2h(c, p->seg_off_h.data(), p->seg_off, nseg + 1));
    DGNN_TRY(d2h(c, p->seg_page_off_h.data(), p->seg_page_off, nseg + 1));
    const int64_t chunk_pages = h[4], cache_pages = p->seg_page_off_h[nseg];
    p->totals[0] = cache_pages + chunk_pages;
    p->totals[1] = chunk_pages + p->n_req;
    p->totals[2] = cache_pages;
    p->totals[3] = chunk_pages;
    DGNN_TRY(check_dev_err(c));
    *out = guard.release();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_disk_plan_get_info(const dgnn_disk_plan* p, dgnn_disk_plan_info* info) {
    DGNN_REQUIRE(p && info, "dgnn_disk_plan_get_info: NULL argument");
    info->nb = p->nb;
    info->nseg = p->nseg;
    info->s = p->s;
    info->m = p->m;
    info->fpp = p->fpp;
    info->row_bytes = p->row_bytes;
    info->n_cache = p->n_cache;
    info->n_packed = p->n_pk;
    info->n_req = p->n_req;
    info->space_pages = p->totals[0];
    info->io_pages = p->totals[1];
    info->cache_pages = p->totals[2];
    info->chunk_pages = p->totals[3];
    info->seg_off = p->seg_off;
    info->cache_ids = p->cache_ids;
    info->seg_page_off = p->seg_page_off;
    info->pk_ids = p->pk_ids;
    info->pk_off = p->pk_off;
    info->req_pages = p->req_pages;
    info->req_off = p->req_off;
    info->dc_addr = p->dc_addr;
    info->pk_off_host = p->pk_off_h.data();
    info->req_off_host = p->req_off_h.data();
    info->seg_off_host = p->seg_off_h.data();
    info->seg_page_off_host = p->seg_page_off_h.data();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_disk_cache_fill(dgnn_ctx* c, const dgnn_disk_plan* p, const void* features,
                                           int64_t num_rows, void* out) {
    DGNN_REQUIRE(c && p && (p->totals[2] == 0 || (features && out)), "dgnn_disk_cache_fill: NULL argument");
    DGNN_REQUIRE(p->row_bytes % 16 == 0 && al16(out) && (features == nullptr || al16(features)),
                 "dgnn_disk_cache_fill: rows and buffers must be 16-byte aligned");
    (void)num_rows;
    const int64_t pages = p->totals[2];
    if (pages == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    CacheRow fn{(const uint8_t*)features, p->row_bytes, p->fpp, p->cache_ids, p->seg_off, p->seg_page_off,
                (int)p->nseg, (uint8_t*)out};
    const double bytes = 2.0 * p->n_cache * p->row_bytes;
    launch(c, DGNN_K_DISK_GATHER, bytes, [&] {
        k_cache_fill<uint4><<<grid_for(c, p->n_cache * 32 / 4, 256, 6), 256, 0, c->stream>>>(fn, p->n_cache);
    });
    DGNN_CK_LAUNCH();
    launch(c, DGNN_K_DISK_GATHER, 0.0, [&] {
        k_cache_zero<<<grid_for(c, pages * 32, 256, 6), 256, 0, c->stream>>>(
            p->seg_off, p->seg_page_off, (int)p->nseg, pages, p->fpp, p->row_bytes, (uint8_t*)out);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_disk_partial(dgnn_ctx* c, const dgnn_disk_plan* p, int64_t b_lo, int64_t b_hi,
                                         const void* pages, const void* chunks, const int64_t* chunk_off, void* out,
                                         const int64_t* out_off) {
    DGNN_REQUIRE(c && p && 0 <= b_lo && b_lo <= b_hi && b_hi <= p->nb, "dgnn_disk_partial: bad batch range");
    const int64_t r0 = p->packed_off_h[b_lo], n = p->packed_off_h[b_hi] - r0;
    if (n == 0) return DGNN_OK;
    DGNN_REQUIRE(out && out_off && chunk_off, "dgnn_disk_partial: NULL argument");
    DGNN_CK(cudaSetDevice(c->device));
    PartialRow fn{(const uint8_t*)pages, (const uint8_t*)chunks, chunk_off, p->packed_off, p->req_off, p->dc_addr,
                  out_off, p->row_bytes, p->fpp, (int)b_lo, (int)(b_hi - b_lo), r0, (uint8_t*)out};
    const bool v16 = p->row_bytes % 16 == 0 && al16(out) && (!pages || al16(pages)) && (!chunks || al16(chunks));
    const int grid = grid_for(c, n * 32 / 4, 256, 6);
    launch(c, DGNN_K_DISK_GATHER, 2.0 * n * p->row_bytes, [&] {
        if (v16) k_partial<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_partial<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

// ----------------------------------------- batched packing from partitions (NEXT #3)
namespace dgnn {
namespace {

__global__ void k_part_counts(const uint32_t* __restrict__ rv, int64_t R, int64_t part_rows, int64_t nparts,
                              unsigned long long* __restrict__ cnt) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = rv[j] / part_rows;
        // rows are sorted by node: only the first row of each partition's run adds the run length
        if (j > 0 && rv[j - 1] / part_rows == p) continue;
        int64_t lo = j, hi = R;  // first row of the next partition
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(rv[mid] / part_rows) <= p) lo = mid + 1;
            else hi = mid;
        }
        if (p < nparts) cnt[p] = (unsigned long long)(lo - j);
    }
}

// [j0, j1) = rows of the sorted index with node in [p0, p1)
__global__ void k_part_bounds(const uint32_t* __restrict__ rv, int64_t R, int64_t p0, int64_t p1,
                              int64_t* __restrict__ bounds) {
    const int64_t key = threadIdx.x == 0 ? p0 : p1;
    if (threadIdx.x > 1) return;
    int64_t lo = 0, hi = R;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)rv[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    bounds[threadIdx.x] = lo;
}

struct PartRow {
    const uint8_t* part;
    int64_t p0, row_bytes, j0;
    const uint32_t* rv;
    const uint32_t* rr;
    const int32_t* rb;
    const int64_t* packed_off;
    const int64_t* chunk_off;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t i, const uint8_t*& s, uint8_t*& d) const {
        const int64_t j = j0 + i;
        const int b = rb[j];
        s = part + ((int64_t)rv[j] - p0) * row_bytes;
        d = dst + chunk_off[b] + ((int64_t)rr[j] - packed_off[b]) * row_bytes;
        return true;
    }
};

__global__ void __launch_bounds__(256) k_pack_part(PartRow fn, const int64_t* __restrict__ bounds) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    PartRow f = fn;
    f.j0 = bounds[0];
    copy_rows_warp<4, uint4>(bounds[1] - bounds[0], f.row_bytes, f, warp, nwarps);
}

__global__ void k_pack_tails(const int64_t* __restrict__ packed_off, const int64_t* __restrict__ chunk_off, int nb,
                             int64_t row_bytes, uint8_t* __restrict__ dst) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (int64_t b = warp; b < nb; b += nwarps) {
        const int64_t start = chunk_off[b] + (packed_off[b + 1] - packed_off[b]) * row_bytes;
        const int64_t nz = (chunk_off[b + 1] - start) / 16;  // row_bytes % 16 == 0: 16-byte aligned
        uint4* z = reinterpret_cast<uint4*>(dst + start);
        for (int64_t i = lane; i < nz; i += 32) __stcs(z + i, make_uint4(0, 0, 0, 0));
    }
}

}  // namespace
}  // namespace dgnn

extern "C" dgnn_status dgnn_disk_index_partition_counts(dgnn_ctx* c, const dgnn_disk_index* x, int64_t part_rows,
                                                        int64_t nparts, int64_t* counts_host) {
    DGNN_REQUIRE(c && x && part_rows > 0 && nparts >= 0 && (nparts == 0 || counts_host),
                 "dgnn_disk_index_partition_counts: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    DevBuf<unsigned long long> cnt;
    DGNN_TRY(cnt.alloc(c, (size_t)nparts));
    DGNN_TRY(memset_async(c, cnt.p, 0, (size_t)(nparts > 0 ? nparts : 1) * 8));
    if (x->R) {
        launch(c, DGNN_K_PACK, 0.0, [&] {
            k_part_counts<<<grid1(c, x->R), 256, 0, c->stream>>>(x->rv, x->R, part_rows, nparts, cnt.p);
        });
        DGNN_CK_LAUNCH();
    }
    return d2h(c, reinterpret_cast<unsigned long long*>(counts_host), cnt.p, (size_t)nparts);
}

extern "C" dgnn_status dgnn_pack_partition(dgnn_ctx* c, const dgnn_disk_index* x, const void* part, int64_t p0,
                                           int64_t p1, int64_t row_bytes, const int64_t* chunk_off, void* group_buf) {
    DGNN_REQUIRE(c && x && chunk_off && 0 <= p0 && p0 <= p1, "dgnn_pack_partition: bad argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && al16(part) && al16(group_buf),
                 "dgnn_pack_partition: rows and buffers must be 16-byte aligned");
    if (x->R == 0 || p0 == p1) return DGNN_OK;
    DGNN_REQUIRE(part && group_buf, "dgnn_pack_partition: NULL buffer");
    DGNN_CK(cudaSetDevice(c->device));
    DevBuf<int64_t> bounds;
    DGNN_TRY(bounds.alloc(c, 2));
    launch(c, DGNN_K_PACK, 0.0, [&] { k_part_bounds<<<1, 32, 0, c->stream>>>(x->rv, x->R, p0, p1, bounds.p); });
    DGNN_CK_LAUNCH();
    PartRow fn{(const uint8_t*)part, p0, row_bytes, 0, x->rv, x->rr, x->rb, x->packed_off, chunk_off, (uint8_t*)group_buf};
    const int grid = grid_for(c, std::min<int64_t>(x->R, p1 - p0) * 32 / 4, 256, 5);
    launch(c, DGNN_K_PACK, 0.0, [&] { k_pack_part<<<grid, 256, 0, c->stream>>>(fn, bounds.p); });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_pack_tails(dgnn_ctx* c, const dgnn_disk_index* x, int64_t row_bytes,
                                       const int64_t* chunk_off, void* group_buf) {
    DGNN_REQUIRE(c && x && chunk_off && row_bytes > 0 && row_bytes % 16 == 0, "dgnn_pack_tails: bad argument");
    if (x->nb == 0) return DGNN_OK;
    DGNN_REQUIRE(group_buf && al16(group_buf), "dgnn_pack_tails: bad buffer");
    DGNN_CK(cudaSetDevice(c->device));
    launch(c, DGNN_K_PACK, 0.0, [&] {
        k_pack_tails<<<grid_for(c, x->nb * 32, 256), 256, 0, c->stream>>>(x->packed_off, chunk_off, (int)x->nb,
                                                                        row_bytes, (uint8_t*)group_buf);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}
