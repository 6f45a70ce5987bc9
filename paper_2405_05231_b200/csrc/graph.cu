// graph.cu -- the graph sample kept in the chunk (Sec. 4: "the graph sample of
// the mini-batch is also kept in the chunk") and the graph-loader stage that reads it back at
// training time (Sec. 5.3: "the graph loader ... loads the graph samples").
// Byte layout: reading c22b in DESIGN.md / include/dgnn.h.
//
//   dgnn_chunk_layout_graph  host: chunk offsets with a graph section after each batch's rows
//   dgnn_pack_graph          a7 + P:283: every batch's sample serialized into its chunk
//   dgnn_samples_load        the loader: a run's staged chunks -> a samples object (device)
//   dgnn_samples_drop_device the offline samples' device arrays freed once they are in chunks
#include <algorithm>

#include "internal.cuh"

namespace dgnn {
namespace {

constexpr int64_t kSecAlign = 16;

struct SampleSrc {
    const int64_t* node_off;
    const int32_t* nodes;
    const int32_t* hop_off;
    const int64_t* eptr_off;
    const int32_t* eptr;
    const int64_t* edge_off;
    const int32_t* src_local;
    int H;
};

// word w of batch b's section: header {H, n, m, e}, hop_off[H+2], nodes[n], eptr[m], src_local[e]
__device__ __forceinline__ int32_t section_word(const SampleSrc& s, int64_t b, int64_t w) {
    const int64_t n0 = s.node_off[b], n = s.node_off[b + 1] - n0;
    const int64_t m0 = s.eptr_off[b], m = s.eptr_off[b + 1] - m0;
    const int64_t e0 = s.edge_off[b], e = s.edge_off[b + 1] - e0;
    const int64_t hw = 4 + s.H + 2;
    if (w < 4) return (int32_t)(w == 0 ? s.H : w == 1 ? n : w == 2 ? m : e);
    if (w < hw) return s.hop_off[b * (s.H + 2) + (w - 4)];
    w -= hw;
    if (w < n) return s.nodes[n0 + w];
    w -= n;
    if (w < m) return s.eptr[m0 + w];
    return s.src_local[e0 + (w - m)];
}

__global__ void k_pack_graph(SampleSrc s, int64_t b_lo, int64_t nb, const int64_t* __restrict__ sec_off,
                             uint8_t* __restrict__ buf) {
    for (int64_t i = blockIdx.y; i < nb; i += gridDim.y) {
        const int64_t b = b_lo + i;
        const int64_t words = 4 + s.H + 2 + (s.node_off[b + 1] - s.node_off[b]) + (s.eptr_off[b + 1] - s.eptr_off[b]) +
                              (s.edge_off[b + 1] - s.edge_off[b]);
        int32_t* out = reinterpret_cast<int32_t*>(buf + sec_off[i]);
        for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
            out[w] = section_word(s, b, w);
    }
}

struct LoadDst {
    int64_t* node_off;  // [nb+2]: offsets, then node_off[nb+1] = 1 if the headers are inconsistent
    int32_t* nodes;
    int32_t* hop_off;
    int64_t* eptr_off;
    int32_t* eptr;
    int64_t* edge_off;
    int32_t* src_local;
    int H;
};

// the loader: section i -> batch i of the run's samples object (offsets from k_load_offsets)
__global__ void k_load_graph(LoadDst d, int64_t nb, const uint8_t* __restrict__ base,
                             const int64_t* __restrict__ sec_off, int*) {
    if (d.node_off[nb + 1]) return;  // inconsistent headers (k_load_offsets): write nothing
    for (int64_t i = blockIdx.y; i < nb; i += gridDim.y) {
        const int32_t* in = reinterpret_cast<const int32_t*>(base + sec_off[i]);
        const int64_t n = d.node_off[i + 1] - d.node_off[i], m = d.eptr_off[i + 1] - d.eptr_off[i],
                      e = d.edge_off[i + 1] - d.edge_off[i];
        const int64_t hw = 4 + d.H + 2, words = hw + n + m + e;
        for (int64_t w = 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
             w += (int64_t)gridDim.x * blockDim.x) {
            const int32_t v = in[w];
            int64_t x = w - hw;
            if (x < 0) d.hop_off[i * (d.H + 2) + (w - 4)] = v;
            else if (x < n) d.nodes[d.node_off[i] + x] = v;
            else if ((x -= n) < m) d.eptr[d.eptr_off[i] + x] = v;
            else d.src_local[d.edge_off[i] + (x - m)] = v;
        }
    }
}

// the loader's offsets, from the section headers alone (one block; a running block-wide scan
// over the run's batches); the totals must equal the layout's (else DEVERR_OVERFLOW)
__global__ void __launch_bounds__(1024) k_load_offsets(LoadDst d, int64_t nb, const uint8_t* __restrict__ base,
                                                      const int64_t* __restrict__ sec_off, int64_t n_tot,
                                                      int64_t m_tot, int64_t e_tot, int* err) {
    __shared__ int64_t s_w[3][32];
    __shared__ int64_t s_run[3];
    __shared__ int s_bad;
    if (threadIdx.x < 3) s_run[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t i0 = 0; i0 < nb; i0 += blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        int64_t v[3] = {0, 0, 0};
        if (i < nb) {
            const int32_t* in = reinterpret_cast<const int32_t*>(base + sec_off[i]);
            if (in[0] != d.H || in[1] < 0 || in[2] < 0 || in[3] < 0) s_bad = 1;
            v[0] = in[1];
            v[1] = in[2];
            v[2] = in[3];
        }
        int64_t incl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int64_t x = v[k];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            incl[k] = x;
            if (lane == 31) s_w[k][warp] = x;
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int nw = (int)(blockDim.x >> 5);
                int64_t x = lane < nw ? s_w[k][lane] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (lane < nw) s_w[k][lane] = x;  // inclusive over warps
            }
        }
        __syncthreads();
        int64_t* outs[3] = {d.node_off, d.eptr_off, d.edge_off};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int64_t excl = s_run[k] + (warp ? s_w[k][warp - 1] : 0) + incl[k] - v[k];
            if (i < nb) outs[k][i] = excl;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k = 0; k < 3; ++k) s_run[k] += s_w[k][(int)(blockDim.x >> 5) - 1];
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        d.node_off[nb] = s_run[0];
        d.eptr_off[nb] = s_run[1];
        d.edge_off[nb] = s_run[2];
        const int bad = s_bad || s_run[0] != n_tot || s_run[1] != m_tot || s_run[2] != e_tot;
        d.node_off[nb + 1] = bad;
        if (bad) atomicOr(err, DEVERR_OVERFLOW);
    }
}

int64_t section_words(const dgnn_samples* s, int64_t b) {
    return 4 + s->H + 2 + (s->node_off_h[b + 1] - s->node_off_h[b]) + (s->eptr_off_h[b + 1] - s->eptr_off_h[b]) +
           (s->edge_off_h[b + 1] - s->edge_off_h[b]);
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_chunk_layout_graph(const dgnn_samples* s, int64_t b_lo, const int64_t* packed_off_host,
                                               int64_t nb, int64_t row_bytes, int64_t* chunk_off_host,
                                               int64_t* sec_off_host) {
    DGNN_REQUIRE(s && packed_off_host && chunk_off_host && sec_off_host && nb >= 0 && row_bytes > 0 && b_lo >= 0 &&
                     b_lo + nb <= s->nb,
                 "dgnn_chunk_layout_graph: bad argument");
    chunk_off_host[0] = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t rows = packed_off_host[i + 1] - packed_off_host[i];
        DGNN_REQUIRE(rows >= 0, "dgnn_chunk_layout_graph: packed_off must be non-decreasing");
        const int64_t sec = (chunk_off_host[i] + rows * row_bytes + kSecAlign - 1) / kSecAlign * kSecAlign;
        sec_off_host[i] = sec;
        const int64_t end = sec + 4 * section_words(s, b_lo + i);
        chunk_off_host[i + 1] = (end + 4095) / 4096 * 4096;
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_pack_graph(dgnn_ctx* c, const dgnn_samples* s, int64_t b_lo, int64_t nb,
                                       const int64_t* sec_off_dev, void* group_buf) {
    DGNN_REQUIRE(c && s && nb >= 0 && b_lo >= 0 && b_lo + nb <= s->nb && (nb == 0 || (sec_off_dev && group_buf)),
                 "dgnn_pack_graph: bad argument");
    DGNN_REQUIRE(nb == 0 || (s->nodes && s->src_local && s->eptr),
                 "dgnn_pack_graph: the samples' device arrays were dropped");
    if (nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    SampleSrc src{s->node_off, s->nodes, s->hop_off, s->eptr_off, s->eptr, s->edge_off, s->src_local, s->H};
    int64_t max_words = 0;
    for (int64_t i = 0; i < nb; ++i) max_words = std::max(max_words, section_words(s, b_lo + i));
    const dim3 grid((unsigned)std::min<int64_t>(ceil_div(max_words, 256), 64), (unsigned)std::min<int64_t>(nb, 65535));
    int64_t bytes = 0;
    for (int64_t i = 0; i < nb; ++i) bytes += 8 * section_words(s, b_lo + i);
    launch(c, DGNN_K_PACK_GRAPH, (double)bytes,
           [&] { k_pack_graph<<<grid, 256, 0, c->stream>>>(src, b_lo, nb, sec_off_dev, (uint8_t*)group_buf); });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_samples_load(dgnn_ctx* c, const dgnn_samples* meta, int64_t b_lo, int64_t b_hi,
                                         const void* base_dev, const int64_t* sec_off_dev, dgnn_samples** out) {
    DGNN_REQUIRE(c && meta && out && 0 <= b_lo && b_lo <= b_hi && b_hi <= meta->nb &&
                     (b_lo == b_hi || (base_dev && sec_off_dev)),
                 "dgnn_samples_load: bad argument");
    *out = nullptr;
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t nb = b_hi - b_lo;
    const int H = meta->H;
    auto* S = new dgnn_samples();
    struct Guard {
        dgnn_samples* s;
        ~Guard() { if (s) dgnn_samples_free(s); }
    } guard{S};
    S->ctx = c;
    S->nb = nb;
    S->H = H;
    S->mode = meta->mode;
    S->batch_id_base = meta->batch_id_base + b_lo;
    S->node_off_h.assign(nb + 1, 0);
    S->edge_off_h.assign(nb + 1, 0);
    S->eptr_off_h.assign(nb + 1, 0);
    S->hop_off_h.assign((size_t)nb * (H + 2), 0);
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t b = b_lo + i;
        S->node_off_h[i + 1] = S->node_off_h[i] + meta->node_off_h[b + 1] - meta->node_off_h[b];
        S->edge_off_h[i + 1] = S->edge_off_h[i] + meta->edge_off_h[b + 1] - meta->edge_off_h[b];
        S->eptr_off_h[i + 1] = S->eptr_off_h[i] + meta->eptr_off_h[b + 1] - meta->eptr_off_h[b];
        for (int x = 0; x < H + 2; ++x) S->hop_off_h[i * (H + 2) + x] = meta->hop_off_h[b * (H + 2) + x];
    }
    S->total_nodes = S->node_off_h[nb];
    S->total_edges = S->edge_off_h[nb];
    S->total_eptr = S->eptr_off_h[nb];
    S->cap_nodes = std::max<int64_t>(S->total_nodes, 1);
    S->cap_edges = std::max<int64_t>(S->total_edges, 1);
    S->cap_eptr = std::max<int64_t>(S->total_eptr, 1);
    S->nodes = (int32_t*)dev_alloc(c, 4 * (size_t)S->cap_nodes);
    S->src_local = (int32_t*)dev_alloc(c, 4 * (size_t)S->cap_edges);
    S->eptr = (int32_t*)dev_alloc(c, 4 * (size_t)S->cap_eptr);
    S->node_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 2));  // + the loader's consistency flag
    S->edge_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 1));
    S->eptr_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 1));
    S->hop_off = (int32_t*)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(1, nb * (H + 2)));
    if (!S->nodes || !S->src_local || !S->eptr || !S->node_off || !S->edge_off || !S->eptr_off || !S->hop_off) {
        set_error("dgnn_samples_load: device allocation failed");
        return DGNN_ENOMEM;
    }
    // every device array, offsets included, comes from the chunks' sections; the host mirrors
    // are the layout's metadata (no host round trip, no device sync)
    LoadDst d{S->node_off, S->nodes, S->hop_off, S->eptr_off, S->eptr, S->edge_off, S->src_local, H};
    launch(c, DGNN_K_PACK_GRAPH, 0.0, [&] {
        k_load_offsets<<<1, 1024, 0, c->stream>>>(d, nb, (const uint8_t*)base_dev, sec_off_dev, S->total_nodes,
                                                  S->total_eptr, S->total_edges, c->dev_err);
    });
    DGNN_CK_LAUNCH();
    if (nb) {
        int64_t max_words = 0;
        for (int64_t i = 0; i < nb; ++i) max_words = std::max(max_words, section_words(S, i));
        const dim3 grid((unsigned)std::min<int64_t>(ceil_div(max_words, 256), 64),
                        (unsigned)std::min<int64_t>(nb, 65535));
        launch(c, DGNN_K_PACK_GRAPH, 0.0, [&] {
            k_load_graph<<<grid, 256, 0, c->stream>>>(d, nb, (const uint8_t*)base_dev, sec_off_dev, c->dev_err);
        });
        DGNN_CK_LAUNCH();
    }
    *out = S;
    guard.s = nullptr;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_samples_drop_device(dgnn_samples* s) {
    DGNN_REQUIRE(s, "dgnn_samples_drop_device: NULL samples");
    dgnn_ctx* c = s->ctx;
    if (c) {
        DGNN_CK(cudaSetDevice(c->device));
        keep_put(c, s->nodes, (size_t)s->cap_nodes * 4);
        keep_put(c, s->src_local, (size_t)s->cap_edges * 4);
        keep_put(c, s->eptr, (size_t)s->cap_eptr * 4);
    }
    s->nodes = s->src_local = s->eptr = nullptr;
    s->cap_nodes = s->cap_edges = s->cap_eptr = 0;
    return DGNN_OK;
}
