// sort.cu -- stable LSD radix sort of (uint32 key, uint32 value) pairs.
//
// Used by the segmented disk cache (diskcache.cu): once to order an epoch's
// packed rows by (node, batch), and k+1 times per plan for Algorithm 1's
// "Sort(S)" over (segment, S_0..S_{k-1}, node).  Each pass handles 8
// key bits in three launches: a per-tile digit histogram, one decoupled
// look-back scan over the digit-major (digit, tile) matrix, and a scatter that
// ranks each tile's items stably with warp match_any + per-warp digit counters.
#include "internal.cuh"

namespace dgnn {
namespace radix {
namespace {

constexpr int kThreads = 256;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // items per tile
constexpr int kBins = 256;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) k_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                   int64_t ntiles, uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_cnt[kBins];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        s_cnt[threadIdx.x] = 0;
        __syncthreads();
        const int64_t base = tile * kTile;
        for (int r = 0; r < kRounds; ++r) {
            const int64_t i = base + r * kThreads + threadIdx.x;
            if (i < n) atomicAdd(&s_cnt[(keys[i] >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        hist[(int64_t)threadIdx.x * ntiles + tile] = s_cnt[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_scatter(const uint32_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ vals, int64_t n, int shift,
                                                      int64_t ntiles, const uint32_t* __restrict__ base_off,
                                                      uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t s_run[kBins];
    __shared__ uint32_t s_base[kBins];
    __shared__ uint32_t s_wcnt[kWarps][kBins];
    const int warp = threadIdx.x >> 5;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        s_run[threadIdx.x] = 0;
        s_base[threadIdx.x] = base_off[(int64_t)threadIdx.x * ntiles + tile];
        for (int w = 0; w < kWarps; ++w) s_wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t base = tile * kTile;
        for (int r = 0; r < kRounds; ++r) {
            // items in index order across the block: stability within the tile
            const int64_t i = base + r * kThreads + threadIdx.x;
            const bool ok = i < n;
            const uint32_t k = ok ? keys[i] : 0u;
            const uint32_t v = ok ? vals[i] : 0u;
            const uint32_t d = ok ? ((k >> shift) & 0xFFu) : kBins;  // kBins: no digit
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const uint32_t rank = __popc(peers & lanemask_lt());
            if (ok && rank == 0) s_wcnt[warp][d] = __popc(peers);
            __syncthreads();
            if (ok) {
                uint32_t off = s_base[d] + s_run[d] + rank;
                for (int w = 0; w < warp; ++w) off += s_wcnt[w][d];
                keys_out[off] = k;
                vals_out[off] = v;
            }
            __syncthreads();
            uint32_t tot = 0;
            for (int w = 0; w < kWarps; ++w) {
                tot += s_wcnt[w][threadIdx.x];
                s_wcnt[w][threadIdx.x] = 0;
            }
            s_run[threadIdx.x] += tot;
            __syncthreads();
        }
    }
}

}  // namespace

dgnn_status sort_pairs(dgnn_ctx* c, int64_t n, int end_bit, uint32_t** keys, uint32_t** vals, uint32_t** keys_alt,
                       uint32_t** vals_alt) {
    DGNN_REQUIRE(n >= 0 && n < (int64_t(1) << 32) && end_bit >= 0 && end_bit <= 32, "radix sort: bad size");
    if (n <= 1 || end_bit == 0) return DGNN_OK;
    const int64_t ntiles = ceil_div(n, kTile);
    DevBuf<uint32_t> hist;
    DGNN_TRY(hist.alloc(c, (size_t)(ntiles * kBins)));
    const int blocks = (int)(ntiles < (int64_t)c->num_sms * 8 ? ntiles : (int64_t)c->num_sms * 8);
    for (int shift = 0; shift < end_bit; shift += 8) {
        const uint32_t* kin = *keys;
        const uint32_t* vin = *vals;
        uint32_t* h = hist.p;
        launch(c, DGNN_K_SORT, 4.0 * n, [&] {
            k_hist<<<blocks, kThreads, 0, c->stream>>>(kin, n, shift, ntiles, h);
        });
        DGNN_CK_LAUNCH();
        DGNN_TRY(scan::run(
            c, ntiles * kBins, nullptr, [h] __device__(int64_t i) -> int32_t { return (int32_t)h[i]; },
            [h] __device__(int64_t i, int64_t excl, int64_t) { h[i] = (uint32_t)excl; }, nullptr));
        uint32_t* ko = *keys_alt;
        uint32_t* vo = *vals_alt;
        launch(c, DGNN_K_SORT, 16.0 * n, [&] {
            k_scatter<<<blocks, kThreads, 0, c->stream>>>(kin, vin, n, shift, ntiles, h, ko, vo);
        });
        DGNN_CK_LAUNCH();
        std::swap(*keys, *keys_alt);
        std::swap(*vals, *vals_alt);
    }
    return DGNN_OK;
}

}  // namespace radix
}  // namespace dgnn
