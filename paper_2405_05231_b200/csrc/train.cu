// train.cu -- the trainer stub: the surrogate of Eq. 1
// fixed by SPEC S:409-413, h^k_v = h^{k-1}_v + mean{h^{k-1}_u : u in N(v)},
// run over a run of assembled batches in place (reading t1: layer k = 1..H handles
// sampling hop h = H - k, deepest first; nodes outside hop h, and hop-h nodes
// without edges, keep their value).
//
// Per layer: one warp per frontier node of hop h (across the run's batches)
// sums its neighbours' rows in edge order with 16-byte loads (lane q owns
// elements 4q..4q+3, so every element is summed in edge order exactly as the
// oracle does), divides once by the edge count, adds the node's own row, and
// writes the result to a scratch row; a second launch copies the scratch rows
// back.  The scratch keeps every read of the layer on h^{k-1}: a hop-h node can be
// another hop-h node's neighbour.  fp32 adds and the IEEE division (no fast-math)
// give results bit-identical to the oracle.
#include "internal.cuh"

namespace dgnn {
namespace {

struct RunView {
    const int64_t* node_off;  // samples (global)
    const int32_t* hop_off;   // [nb*(H+2)]
    const int64_t* eptr_off;
    const int32_t* eptr;
    const int64_t* edge_off;
    const int32_t* src_local;
    int H;
    int b_lo, nbr;
    int blocks;  // DGNN_SAMPLE_BLOCKS: hop h's destinations are local [0, hop_off[h+1]), eptr per hop
};

// first destination of hop h and the start of hop h's eptr array (relative to the batch's eptr)
__device__ __forceinline__ void hop_geometry(const RunView& v, const int32_t* ho, int h, int64_t& first,
                                             int64_t& eptr_base) {
    if (!v.blocks) {
        first = ho[h];
        eptr_base = 0;
        return;
    }
    first = 0;
    eptr_base = 0;
    for (int i = 0; i < h; ++i) eptr_base += ho[i + 1] + 1;
}

// fr_off[bl] = exclusive prefix over the run's batches of |hop h| (single block)
__global__ void k_frontier_off(RunView v, int h, int64_t* __restrict__ fr_off) {
    __shared__ int64_t s_carry;
    __shared__ int64_t s_warp[32];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base <= v.nbr; base += blockDim.x) {
        const int bl = base + threadIdx.x;
        int64_t x = 0;
        if (bl < v.nbr) {
            const int32_t* ho = v.hop_off + (int64_t)(v.b_lo + bl) * (v.H + 2);
            x = v.blocks ? ho[h + 1] : ho[h + 1] - ho[h];
        }
        int64_t s = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += y;
        }
        if (lane == 31) s_warp[warp] = s;
        __syncthreads();
        int64_t wpre = 0, tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            wpre += (w < warp) ? s_warp[w] : 0;
            tot += s_warp[w];
        }
        if (bl <= v.nbr) fr_off[bl] = s_carry + wpre + s - x;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
}

template <class V>
__device__ __forceinline__ void acc(V& s, const V& x);
template <>
__device__ __forceinline__ void acc<float4>(float4& s, const float4& x) {
    s.x += x.x;
    s.y += x.y;
    s.z += x.z;
    s.w += x.w;
}
template <>
__device__ __forceinline__ void acc<float>(float& s, const float& x) {
    s += x;
}
__device__ __forceinline__ float4 upd(const float4& self, const float4& s, float c) {
    return make_float4(self.x + s.x / c, self.y + s.y / c, self.z + s.z / c, self.w + s.w / c);
}
__device__ __forceinline__ float upd(const float& self, const float& s, float c) { return self + s / c; }
template <class V>
__device__ __forceinline__ V vzero();
template <>
__device__ __forceinline__ float4 vzero<float4>() {
    return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <>
__device__ __forceinline__ float vzero<float>() {
    return 0.f;
}

// warp per frontier node f of hop h: scratch[f] = x[j] + (sum_e x[src_e]) / cnt
template <class V>
__global__ void __launch_bounds__(256) k_layer(RunView v, int h, const int64_t* __restrict__ fr_off, int64_t F,
                                               const float* __restrict__ x, int64_t dim, float* __restrict__ scratch) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    constexpr int W = sizeof(V) / sizeof(float);
    const int64_t nvec = dim / W;
    const int64_t x0 = v.node_off[v.b_lo];
    for (int64_t f = warp; f < F; f += nwarps) {
        const int bl = segment_of(fr_off, v.nbr + 1, f);
        const int b = v.b_lo + bl;
        const int32_t* ho = v.hop_off + (int64_t)b * (v.H + 2);
        int64_t first, ebase;
        hop_geometry(v, ho, h, first, ebase);
        const int64_t j = first + (f - fr_off[bl]);
        const int32_t* ep = v.eptr + v.eptr_off[b] + ebase;
        const int32_t e0 = ep[j], e1 = ep[j + 1];
        const int64_t rb = v.node_off[b] - x0;  // the batch's first row in x
        const V* self = reinterpret_cast<const V*>(x + (rb + j) * dim);
        V* dst = reinterpret_cast<V*>(scratch + f * dim);
        const int32_t* src = v.src_local + v.edge_off[b];
        const float cnt = (float)(e1 - e0);
        for (int64_t q0 = 0; q0 < nvec; q0 += 32) {
            const int64_t q = q0 + lane;
            const bool in = q < nvec;
            if (e1 == e0) {
                if (in) dst[q] = self[q];
                continue;
            }
            V s = vzero<V>();
            // neighbour ids of 32 edges at a time, one per lane, broadcast with shuffles; four
            // row loads in flight per lane, accumulated strictly in edge order
            for (int32_t eb = e0; eb < e1; eb += 32) {
                const int ne = min(32, e1 - eb);
                const int32_t my = lane < ne ? src[eb + lane] : 0;
                int t = 0;
                for (; t + 4 <= ne; t += 4) {
                    const int32_t u0 = __shfl_sync(0xffffffffu, my, t);
                    const int32_t u1 = __shfl_sync(0xffffffffu, my, t + 1);
                    const int32_t u2 = __shfl_sync(0xffffffffu, my, t + 2);
                    const int32_t u3 = __shfl_sync(0xffffffffu, my, t + 3);
                    if (in) {
                        const V r0 = reinterpret_cast<const V*>(x + (rb + u0) * dim)[q];
                        const V r1 = reinterpret_cast<const V*>(x + (rb + u1) * dim)[q];
                        const V r2 = reinterpret_cast<const V*>(x + (rb + u2) * dim)[q];
                        const V r3 = reinterpret_cast<const V*>(x + (rb + u3) * dim)[q];
                        acc<V>(s, r0);
                        acc<V>(s, r1);
                        acc<V>(s, r2);
                        acc<V>(s, r3);
                    }
                }
                for (; t < ne; ++t) {
                    const int32_t u = __shfl_sync(0xffffffffu, my, t);
                    if (in) acc<V>(s, reinterpret_cast<const V*>(x + (rb + u) * dim)[q]);
                }
            }
            if (in) dst[q] = upd(self[q], s, cnt);
        }
    }
}

template <class V>
__global__ void __launch_bounds__(256) k_copyback(RunView v, int h, const int64_t* __restrict__ fr_off, int64_t F,
                                                  float* __restrict__ x, int64_t dim, const float* __restrict__ scratch) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    constexpr int W = sizeof(V) / sizeof(float);
    const int64_t nvec = dim / W;
    const int64_t x0 = v.node_off[v.b_lo];
    for (int64_t f = warp; f < F; f += nwarps) {
        const int bl = segment_of(fr_off, v.nbr + 1, f);
        const int b = v.b_lo + bl;
        const int64_t j = (v.blocks ? 0 : v.hop_off[(int64_t)b * (v.H + 2) + h]) + (f - fr_off[bl]);
        V* d = reinterpret_cast<V*>(x + (v.node_off[b] - x0 + j) * dim);
        const V* s = reinterpret_cast<const V*>(scratch + f * dim);
        for (int64_t q = lane; q < nvec; q += 32) d[q] = s[q];
    }
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_train_stub(dgnn_ctx* c, const dgnn_samples* s, int64_t b_lo, int64_t b_hi, float* x,
                                       int64_t dim) {
    DGNN_REQUIRE(c && s && 0 <= b_lo && b_lo <= b_hi && b_hi <= s->nb && dim > 0, "dgnn_train_stub: bad argument");
    if (b_lo == b_hi) return DGNN_OK;
    DGNN_REQUIRE(x, "dgnn_train_stub: NULL features");
    DGNN_CK(cudaSetDevice(c->device));
    const int H = s->H;
    const int nbr = (int)(b_hi - b_lo);
    // host-side sizes from the host mirror of hop_off: no device round trip
    int64_t F_max = 0;
    std::vector<int64_t> F(H, 0);
    for (int h = 0; h < H; ++h) {
        for (int64_t b = b_lo; b < b_hi; ++b)
            F[h] += s->hop_off_h[b * (H + 2) + h + 1] -
                    (s->mode == DGNN_SAMPLE_BLOCKS ? 0 : s->hop_off_h[b * (H + 2) + h]);
        F_max = std::max(F_max, F[h]);
    }
    if (F_max == 0) return DGNN_OK;
    DevBuf<float> scratch;
    DevBuf<int64_t> fr;
    DGNN_TRY(scratch.alloc(c, (size_t)(F_max * dim)));
    DGNN_TRY(fr.alloc(c, (size_t)nbr + 1));
    RunView v{s->node_off, s->hop_off, s->eptr_off, s->eptr, s->edge_off, s->src_local, H, (int)b_lo, nbr,
              s->mode == DGNN_SAMPLE_BLOCKS ? 1 : 0};
    const bool v4 = dim % 4 == 0 && ((uintptr_t)x & 15) == 0;
    for (int h = H - 1; h >= 0; --h) {
        if (F[h] == 0) continue;
        launch(c, DGNN_K_TRAIN, 0.0, [&] { k_frontier_off<<<1, 1024, 0, c->stream>>>(v, h, fr.p); });
        DGNN_CK_LAUNCH();
        const int grid = grid_for(c, F[h] * 32, 256, 8);
        launch(c, DGNN_K_TRAIN, 0.0, [&] {
            if (v4) k_layer<float4><<<grid, 256, 0, c->stream>>>(v, h, fr.p, F[h], x, dim, scratch.p);
            else k_layer<float><<<grid, 256, 0, c->stream>>>(v, h, fr.p, F[h], x, dim, scratch.p);
        });
        DGNN_CK_LAUNCH();
        launch(c, DGNN_K_TRAIN, 0.0, [&] {
            if (v4) k_copyback<float4><<<grid, 256, 0, c->stream>>>(v, h, fr.p, F[h], x, dim, scratch.p);
            else k_copyback<float><<<grid, 256, 0, c->stream>>>(v, h, fr.p, F[h], x, dim, scratch.p);
        });
        DGNN_CK_LAUNCH();
    }
    return DGNN_OK;
}
