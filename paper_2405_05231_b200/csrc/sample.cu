// sample.cu -- a1-a3: offline K-hop node-wise neighbour sampling of many
// mini-batches (Sec. 2 "node-wise sampling ... uses a fan-out
// vector"; Sec. 3 "sample many mini-batches before running their
// model computation"), with the per-node access counter of P:271 fused into
// the dedup step.  Semantics: DESIGN.md readings c1-c14, c24, c26.
//
// Design (B200): batches are processed in sampling groups of G slots; every
// step of a hop runs over the flattened frontier / candidate / new-node sets of
// all G batches at once, sized on the device (no host round trip inside a
// group):
//   hop_begin   frontier prefix over slots                        (1 block)
//   scan        cand offsets = exclusive scan of min(k, deg(v))   (decoupled look-back)
//   sample_hop  warp per frontier node: Philox draws (lane s = slot s), Floyd
//               resolution with warp ballots, rank-sort of the k positions,
//               gather of indices[], per-batch hash-set insert (CAS); first
//               insert -> counts[u] += 1 and warp-aggregated append
//   order       bucket sort of each batch's new IDs: histogram on (slot,
//               id >> shift), scan, scatter, per-bucket insertion sort, and
//               local-ID assignment into the hash set
//   remap       cand[i] = local(cand[i])
//   hop_end     frontier <- the new nodes                          (1 block)
// then one host sync per group sizes the batch-major compaction into the
// output arena.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <string>

#include "internal.cuh"

namespace dgnn {
namespace {

constexpr int kMaxGroup = 256;
constexpr int kMaxHops = 30;  // hops of the partitioned dedup path (slices of nodes-so-far)
constexpr int32_t kEmpty = -1;
constexpr unsigned kFull = 0xffffffffu;

struct Grp {
    int G;
    int blocks;  // DGNN_SAMPLE_BLOCKS: every node so far is in the next frontier (reading c27)
    int tlog;
    uint32_t tmask;
    uint32_t max_probes;  // k_insert gives up (DEVERR_TABLE -> redo at the bound) after this many probes
    int H;
    int64_t cap_n;
    int32_t* nodes;      // [G*cap_n]
    int32_t* table;      // [G << tlog] keys (kEmpty = free); the insert CASes only these
    int32_t* local;      // [G << tlog] local ID of the key in the same slot (written after the insert)
    int32_t* n;          // [G] nodes so far
    int32_t* fr_lo;      // [G]
    int32_t* fr_hi;      // [G]
    int32_t* new_cnt;    // [G]
    int64_t* fr_off;     // [G+1]
    int64_t* cand_base;  // [G+1]
    int64_t* new_off;    // [G+1]
    int64_t* cand_total; // [1]
    int32_t* hop_bound;  // [G*(H+2)]
    int64_t* hop_fr_off; // [H*(kMaxGroup+1)]
    int64_t* hop_cbase;  // [H*(kMaxGroup+1)]
    int32_t* fv;         // [frontier] node id
    int64_t* fst;        // [frontier] indptr[v]
    int32_t* fdg;        // [frontier] degree
};

__device__ __forceinline__ uint32_t slot_hash(int32_t key, int tlog) {
    return ((uint32_t)key * 2654435761u) >> (32 - tlog);
}

// 1 = inserted, 0 = already present, -1 = table full
__device__ __forceinline__ int table_insert(int32_t* tab, int32_t* loc, int tlog, uint32_t mask, int32_t key,
                                            int32_t value) {
    uint32_t p = slot_hash(key, tlog);
    for (uint32_t probes = 0; probes <= mask; ++probes) {
        const int prev = atomicCAS(&tab[p], kEmpty, key);
        if (prev == kEmpty) {
            if (value >= 0) loc[p] = value;
            return 1;
        }
        if (prev == key) return 0;
        p = (p + 1) & mask;
    }
    return -1;
}

// ----------------------------------------------------------------- seeds
__global__ void k_seed_init(Grp g, const int32_t* __restrict__ seeds, int64_t num_seeds, int32_t B, int64_t t0,
                            int64_t N, uint32_t* counts, int* err, int use_table) {
    const int s = blockIdx.x;
    const int64_t a = (t0 + s) * (int64_t)B;
    const int64_t ns = min((int64_t)B, num_seeds - a);
    if (threadIdx.x == 0) {
        g.n[s] = (int32_t)ns;
        g.fr_lo[s] = 0;
        g.fr_hi[s] = (int32_t)ns;
        g.new_cnt[s] = 0;
        g.hop_bound[s * (g.H + 2) + 0] = 0;
        g.hop_bound[s * (g.H + 2) + 1] = (int32_t)ns;
    }
    int32_t* tab = g.table + ((int64_t)s << g.tlog);
    int32_t* loc = g.local + ((int64_t)s << g.tlog);
    for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const int32_t u = seeds[a + i];
        if (u < 0 || (int64_t)u >= N) {
            atomicOr(err, DEVERR_SEED_RANGE);
            g.nodes[(int64_t)s * g.cap_n + i] = 0;
            continue;
        }
        g.nodes[(int64_t)s * g.cap_n + i] = u;
        if (!use_table) continue;  // partitioned path: k_seed_sort checks duplicates
        const int r = table_insert(tab, loc, g.tlog, g.tmask, u, (int32_t)i);
        if (r == 0) atomicOr(err, DEVERR_SEED_DUP);
        else if (r < 0) atomicOr(err, DEVERR_TABLE);
        else if (counts) atomicAdd(&counts[u], 1u);
    }
}

// access counter over a group's compacted node lists (batch nodes are distinct): counts[v] += 1
__global__ void k_count_nodes(const int32_t* __restrict__ nodes, int64_t n, uint32_t* __restrict__ counts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[nodes[i]], 1u);
}

__global__ void k_seed_range(const int32_t* __restrict__ seeds, int64_t n, int64_t N, int* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = seeds[i];
        if (u < 0 || (int64_t)u >= N) atomicOr(err, DEVERR_SEED_RANGE);
    }
}

// ------------------------------------------------------ per-hop bookkeeping
// frontier offsets of the group's slots: an exclusive scan over G <= kMaxGroup frontier sizes, one
// thread per slot and one for the total (launched with kSlotThreads threads)
constexpr int kSlotThreads = kMaxGroup + 32;
__global__ void k_hop_begin(Grp g, int h) {
    static_assert(kSlotThreads <= 1024 && kMaxGroup % 32 == 0, "one thread per slot");
    __shared__ int64_t s_warp[kSlotThreads / 32];
    const int s = threadIdx.x, lane = s & 31, w = s >> 5;
    const int64_t len = s < g.G ? (int64_t)(g.fr_hi[s] - g.fr_lo[s]) : 0;
    int64_t x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    int64_t pre = x - len;
    for (int k = 0; k < w; ++k) pre += s_warp[k];
    if (s <= g.G) {  // s == G: the total (len 0 there)
        g.fr_off[s] = pre;
        g.hop_fr_off[h * (kMaxGroup + 1) + s] = pre;
    }
}

// candidate bases of the group's slots (one thread per slot and one for the total, kSlotThreads)
__global__ void k_hop_cands(Grp g, int h, int64_t* cptr) {
    const int s = threadIdx.x;
    const int64_t F = g.fr_off[g.G];
    if (s > g.G) return;
    // (slots whose frontier offset is F -- the total, and empty trailing slots -- take the total)
    const int64_t o = g.fr_off[s];
    const int64_t c = o == F ? *g.cand_total : cptr[o];
    if (s == g.G) cptr[F] = c;
    g.cand_base[s] = c;
    g.hop_cbase[h * (kMaxGroup + 1) + s] = c;
}

// new_off[s] = start of slot s's new nodes in the flattened bucket order
__global__ void k_new_setup(Grp g, const int64_t* __restrict__ bstart, int64_t NB, const int64_t* __restrict__ total) {
    for (int s = threadIdx.x; s <= g.G; s += blockDim.x) g.new_off[s] = s < g.G ? bstart[(int64_t)s * NB] : *total;
}

__global__ void k_hop_end(Grp g, int h) {
    for (int s = threadIdx.x; s < g.G; s += blockDim.x) {
        const int32_t n0 = g.n[s], c = (int32_t)(g.new_off[s + 1] - g.new_off[s]);
        g.hop_bound[s * (g.H + 2) + h + 2] = n0 + c;
        g.fr_lo[s] = g.blocks ? 0 : n0;
        g.fr_hi[s] = n0 + c;
        g.n[s] = n0 + c;
    }
}

// ------------------------------------------------ a2: the sampling kernels
// Scan input: frontier node t -> min(k, deg); records (v, indptr[v], deg) so the
// sampling kernel reads them coalesced instead of chasing pointers.
struct DegIn {
    Grp g;
    const int64_t* indptr;
    int k;
    int* err;
    __device__ __forceinline__ int32_t operator()(int64_t t) const {
        const int s = segment_of(g.fr_off, g.G + 1, t);
        const int64_t j = g.fr_lo[s] + (t - g.fr_off[s]);
        const int32_t v = g.nodes[(int64_t)s * g.cap_n + j];
        const int64_t start = indptr[v];
        const int64_t d = indptr[v + 1] - start;
        g.fv[t] = v;
        g.fst[t] = start;
        if (d >= (int64_t)INT32_MAX) atomicOr(err, DEVERR_OVERFLOW);
        g.fdg[t] = (int32_t)d;
        return (int32_t)(d < k ? d : k);
    }
};

struct StoreExcl {
    int64_t* out;
    __device__ __forceinline__ void operator()(int64_t i, int64_t excl, int64_t) const { out[i] = excl; }
};

// W lanes per frontier node (W = next power of two >= k, k <= 32): lane s of a
// sub-warp draws slot s (Philox keyed (seed, v, bid, h, s)), Floyd's resolution
// runs in slot order with sub-warp ballots, the k positions are ranked (they are
// distinct) and the neighbour IDs gathered into cand[cptr[t] + rank].
template <int W>
__global__ void __launch_bounds__(256) k_sample_hop(Grp g, const int32_t* __restrict__ indices, int k, uint64_t seed,
                                                    int64_t bid0, int h, const int64_t* __restrict__ cptr,
                                                    int32_t* __restrict__ cand) {
    __shared__ int64_t s_fr[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_fr[i] = g.fr_off[i];
    __syncthreads();
    constexpr int NPW = 32 / W;  // frontier nodes per warp
    const int64_t F = s_fr[g.G];
    const int lane = threadIdx.x & 31, sub = lane / W, sl = lane % W;
    const unsigned gmask = (W == 32) ? kFull : (((1u << W) - 1u) << (sub * W));
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NPW; t0 < F;
         t0 += nwarps * NPW) {
        const int64_t t = t0 + sub;
        const bool live = t < F;
        int32_t v = 0, d = 0;
        int64_t start = 0, base = 0;
        int s = 0;
        if (live) {
            v = g.fv[t];
            start = g.fst[t];
            d = g.fdg[t];
            base = cptr[t];
            s = segment_of(s_fr, g.G + 1, t);
        }
        const bool floyd = live && d > k;
        if (live && !floyd) {
            // reading c3: take every position, in CSR order
            for (int p = sl; p < d; p += W) cand[base + p] = indices[start + p];
        }
        if (__ballot_sync(kFull, floyd)) {
            // Floyd (readings c6, c7): draw t_s in [0, d-k+s]; slot s takes i_s if t_s was taken
            const int64_t i = (int64_t)d - k + sl;
            int64_t tdraw = 0;
            if (floyd && sl < k)
                tdraw = (int64_t)__umul64hi(draw64(seed, (uint32_t)v, (uint64_t)(bid0 + s), (uint32_t)h, (uint32_t)sl),
                                            (uint64_t)(i + 1));
            int64_t S = -1;
            for (int r = 0; r < k; ++r) {
                const int64_t tr = __shfl_sync(kFull, tdraw, r, W);
                const unsigned hit = __ballot_sync(kFull, sl < r && S == tr) & gmask;
                if (sl == r) S = hit ? i : tr;
            }
            int rank = 0;
            for (int q = 0; q < k; ++q) {
                const int64_t Sq = __shfl_sync(kFull, S, q, W);
                rank += (Sq < S) ? 1 : 0;
            }
            if (floyd && sl < k) cand[base + rank] = indices[start + S];
        }
    }
}

// Thread per frontier node (k <= KMAX <= 32): the node's k Philox draws, Floyd's resolution and
// the ranking of the k positions all stay in registers (unrolled to KMAX, predicated on k), so a
// draw costs its Philox rounds plus a few compares -- no shuffles or ballots, no idle lanes.
template <int KMAX>
__global__ void __launch_bounds__(256) k_sample_hop_t(Grp g, const int32_t* __restrict__ indices, int k,
                                                      uint64_t seed, int64_t bid0, int h,
                                                      const int64_t* __restrict__ cptr, int32_t* __restrict__ cand) {
    __shared__ int64_t s_fr[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_fr[i] = g.fr_off[i];
    __syncthreads();
    const int64_t F = s_fr[g.G];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < F; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = g.fv[t];
        const int64_t start = g.fst[t];
        const int32_t d = g.fdg[t];
        const int64_t base = cptr[t];
        if (d <= k) {  // reading c3: every position, in CSR order
            for (int p = 0; p < d; ++p) cand[base + p] = indices[start + p];
            continue;
        }
        const int s = segment_of(s_fr, g.G + 1, t);
        const uint64_t bid = (uint64_t)(bid0 + s);
        int32_t S[KMAX];
        // Floyd (readings c6, c7): slot q draws t_q in [0, i_q], i_q = d - k + q; takes i_q if
        // t_q was already taken
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            if (q < k) {
                const int32_t i = d - k + q;
                const int32_t tq =
                    (int32_t)__umul64hi(draw64(seed, (uint32_t)v, bid, (uint32_t)h, (uint32_t)q), (uint64_t)i + 1);
                bool hit = false;
#pragma unroll
                for (int r = 0; r < q; ++r) hit |= S[r] == tq;
                S[q] = hit ? i : tq;
            }
        }
        // positions ascending: slot q's rank among the k distinct positions
#pragma unroll
        for (int q = 0; q < KMAX; ++q) {
            if (q < k) {
                int rank = 0;
#pragma unroll
                for (int r = 0; r < KMAX; ++r) rank += (r < k && S[r] < S[q]) ? 1 : 0;
                cand[base + rank] = indices[start + S[q]];
            }
        }
    }
}

// k > 32: one lane per frontier node runs Floyd sequentially, using the node's
// candidate slots as scratch for the positions, then the warp gathers.
__global__ void __launch_bounds__(256) k_sample_hop_wide(Grp g, const int32_t* __restrict__ indices, int k,
                                                         uint64_t seed, int64_t bid0, int h,
                                                         const int64_t* __restrict__ cptr, int32_t* __restrict__ cand) {
    __shared__ int64_t s_fr[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_fr[i] = g.fr_off[i];
    __syncthreads();
    const int64_t F = s_fr[g.G];
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < F; t += nwarps) {
        const int s = segment_of(s_fr, g.G + 1, t);
        const int32_t v = g.fv[t];
        const int64_t start = g.fst[t];
        const int32_t d = g.fdg[t];
        const int64_t base = cptr[t];
        if (d <= k) {
            for (int p = lane; p < d; p += 32) cand[base + p] = indices[start + p];
            continue;
        }
        if (lane == 0) {
            for (int s2 = 0; s2 < k; ++s2) {
                const int64_t i = (int64_t)d - k + s2;
                const int64_t tt = (int64_t)__umul64hi(
                    draw64(seed, (uint32_t)v, (uint64_t)(bid0 + s), (uint32_t)h, (uint32_t)s2), (uint64_t)(i + 1));
                bool present = false;
                for (int r = 0; r < s2; ++r)
                    if ((int64_t)cand[base + r] == tt) {
                        present = true;
                        break;
                    }
                cand[base + s2] = (int32_t)(present ? i : tt);
            }
            for (int a = 1; a < k; ++a) {
                const int32_t x = cand[base + a];
                int b = a - 1;
                while (b >= 0 && cand[base + b] > x) {
                    cand[base + b + 1] = cand[base + b];
                    --b;
                }
                cand[base + b + 1] = x;
            }
        }
        __syncwarp();
        for (int p = lane; p < k; p += 32) cand[base + p] = indices[start + cand[base + p]];
        __syncwarp();
    }
}

// ------------------------- a3: dedup insert + access counter + bucket histogram
// Thread per candidate: insert into the batch's hash set; the first insert of u
// in a batch is the node's discovery: counts[u] += 1 and a slot in the
// (batch, u >> shift) bucket; the table index is kept so the local ID can be
// written back without probing.
__global__ void __launch_bounds__(256) k_insert(Grp g, const int32_t* __restrict__ cand, int64_t NB, int shift,
                                                int32_t* __restrict__ hist, int32_t* __restrict__ npos,
                                                int32_t* __restrict__ ntab, uint32_t* counts, int* err) {
    __shared__ int64_t s_cb[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_cb[i] = g.cand_base[i];
    __syncthreads();
    const int64_t C = s_cb[g.G];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int s = segment_of(s_cb, g.G + 1, i);
        const int32_t u = cand[i];
        int32_t* tab = g.table + ((int64_t)s << g.tlog);
        uint32_t p = slot_hash(u, g.tlog);
        int pos = -1;
        for (uint32_t probes = 0;; ++probes) {
            if (probes >= g.max_probes) {
                atomicOr(err, DEVERR_TABLE);
                break;
            }
            const int prev = atomicCAS(&tab[p], kEmpty, u);
            if (prev == kEmpty) {
                if (counts) atomicAdd(&counts[u], 1u);
                pos = atomicAdd(&hist[(int64_t)s * NB + (u >> shift)], 1);
                break;
            }
            if (prev == u) break;
            p = (p + 1) & g.tmask;
        }
        npos[i] = pos;
        ntab[i] = (int32_t)p;
    }
}

__global__ void k_bucket_scatter(Grp g, const int32_t* __restrict__ cand, int64_t NB, int shift,
                                 const int64_t* __restrict__ bstart, const int32_t* __restrict__ npos,
                                 const int32_t* __restrict__ ntab, unsigned long long* __restrict__ sorted) {
    __shared__ int64_t s_cb[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_cb[i] = g.cand_base[i];
    __syncthreads();
    const int64_t C = s_cb[g.G];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t pos = npos[i];
        if (pos < 0) continue;
        const int s = segment_of(s_cb, g.G + 1, i);
        const int32_t u = cand[i];
        sorted[bstart[(int64_t)s * NB + (u >> shift)] + pos] =
            ((unsigned long long)(uint32_t)u << 32) | (uint32_t)ntab[i];
    }
}

// thread per bucket: insertion sort of its (few) (id, table index) pairs by id,
// then the ascending-ID local numbering (reading c10) into nodes[] and the hash set
__global__ void k_bucket_sort_assign(Grp g, int64_t NB, const int64_t* __restrict__ bstart,
                                     const int32_t* __restrict__ hist, unsigned long long* __restrict__ sorted) {
    const int64_t nbk = (int64_t)g.G * NB;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbk; b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = hist[b];
        if (c == 0) continue;
        const int64_t lo = bstart[b];
        unsigned long long* a = sorted + lo;
        for (int x = 1; x < c; ++x) {
            const unsigned long long key = a[x];
            int y = x - 1;
            while (y >= 0 && a[y] > key) {
                a[y + 1] = a[y];
                --y;
            }
            a[y + 1] = key;
        }
        const int s = (int)(b / NB);
        const int64_t off = g.new_off[s];
        const int32_t n0 = g.n[s];
        int32_t* loc = g.local + ((int64_t)s << g.tlog);
        int32_t* nodes = g.nodes + (int64_t)s * g.cap_n;
        for (int x = 0; x < c; ++x) {
            const unsigned long long e = a[x];
            const int32_t local = n0 + (int32_t)(lo + x - off);
            nodes[local] = (int32_t)(e >> 32);
            loc[(uint32_t)e] = local;
        }
    }
}

// Edge remap: the insert kept each candidate's table slot (ntab), so the local ID is one
// load from the slot k_bucket_sort_assign filled -- no second probe sequence.
__global__ void k_remap(Grp g, int32_t* __restrict__ cand, const int32_t* __restrict__ ntab) {
    __shared__ int64_t s_cb[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_cb[i] = g.cand_base[i];
    __syncthreads();
    const int64_t C = s_cb[g.G];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C; i += (int64_t)gridDim.x * blockDim.x) {
        const int s = segment_of(s_cb, g.G + 1, i);
        cand[i] = g.local[((int64_t)s << g.tlog) + (uint32_t)ntab[i]];
    }
}

// ------------------------- a3, partitioned path: shared-memory dedup per (batch, ID range)
// The per-batch global hash sets above cost one random CAS into a 4-8 MB table per candidate,
// 64 batches at once (0.5 GB of tables against a 126 MB L2).  This path instead splits each
// batch's candidates by ID range (partition p = u >> pshift, P = 2^pbits ranges) and dedups
// each (batch, range) bucket inside one CTA's shared memory:
//   k_seed_sort    per batch: the seeds sorted by ID with their local IDs (the one unsorted
//                  slice of nodes-so-far; every hop's new nodes are already ID-ascending)
//   k_part_bounds  per (batch, slice) and range: where the range starts in the sorted slice
//   k_part_count   candidates per bucket (shared-memory histogram per tile)
//   scan           bucket starts
//   k_part_scatter (u, candidate index) pairs into their buckets
//   k_part_dedup   one CTA per bucket, taken in (batch, range) order: the bucket's old nodes
//                  and candidates go into a shared-memory hash set; the new IDs are sorted in
//                  shared memory; the bucket's first local ID is the batch's node count plus
//                  the new nodes of the lower ranges (decoupled look-back over the batch's
//                  buckets); nodes[] is written and every candidate remapped to its local ID.
// A bucket whose distinct IDs would load its table past 3/4 raises DEVERR_PART and the group
// is redone on the hash-set path (adversarial ID distributions only).  Results are identical
// by construction: the dedup is a set operation, new nodes are ordered by ID (reading c10), and
// the remap is per candidate.
// (the DGNN_PART_* macros exist for A/B builds, tools/build_variant.sh)
#ifndef DGNN_PART_THREADS
#define DGNN_PART_THREADS 512
#endif
#ifndef DGNN_PART_TABLE_LOG
#define DGNN_PART_TABLE_LOG 12
#endif
#ifndef DGNN_PART_TARGET
#define DGNN_PART_TARGET 1024  // distinct IDs a bucket is sized to expect
#endif
constexpr int kPartThreads = DGNN_PART_THREADS;
constexpr int kPartTableLog = DGNN_PART_TABLE_LOG;      // 4096 slots: keys + locals + sort keys = 64 KB
constexpr int kPartTable = 1 << kPartTableLog;
constexpr size_t kPartSmem = (size_t)kPartTable * 16;  // dynamic shared memory of k_part_dedup
constexpr int kRankBits = kPartTableLog - 2;  // sub-ranges of a bucket's ID range in the counting order
constexpr int kRankMax = kPartTable / 2;      // new IDs a bucket ranks by counting (above: bitonic sort)
constexpr int kPartTarget = DGNN_PART_TARGET;
static_assert((kPartTable - kRankMax) * 2 >= (1 << kRankBits) + 1 + kRankMax, "rank scratch in s_new");

constexpr int kSeedSortMax = 4096;                      // batch_size limit of the partitioned path
constexpr int kPartTile = 8192;                         // candidates per tile in count / scatter
constexpr int kPartTileThreads = 512;
constexpr int kPartBins = 2048;                         // shared-memory bins per tile

struct Part {
    int pbits;   // P = 1 << pbits ranges per batch
    int pshift;  // range of u = u >> pshift
    int nslices; // slices of nodes-so-far: sorted seeds + one per finished hop
    int rank_max;  // buckets with at most this many new IDs order them by counting, others sort
    int32_t* sid;     // [G * B] seeds sorted by ID
    int32_t* sloc;    // [G * B] their local IDs
    int32_t* bnd;     // [G * (H+1) * (P+1)] start of range p in slice x, relative to the slice
    int64_t* bstart;  // [G * P + 1] bucket starts (exclusive scan of the counts), total at the end
    int64_t* bcur;    // [G * P] scatter cursors
    int32_t* bcnt;    // [G * P] candidates per bucket
    int2* pui;        // [C] bucketed (candidate ID, candidate index) pairs: one 8-byte store per
                      // candidate in the scatter, so a bin's run of pairs fills whole sectors
    unsigned long long* status;  // [G * P] look-back words of k_part_dedup
    unsigned int* ticket;        // bucket ticket counter
    int32_t B;        // batch size (seed slice stride)
};

template <class T>
__device__ __forceinline__ void bitonic_sort_smem(T* a, int n2) {
    // ascending bitonic sort of a[0, n2) (n2 a power of two), all threads of the block, one
    // compare-exchange pair per thread and stage.  Thread t's pairs q = t + m*blockDim touch
    // elements [64*(q/32), 64*(q/32) + 64) while j <= 32, so those stages need only the warp's
    // own barrier; a stage with j >= 64, and the stage after it, synchronize the block.
    const int half = n2 >> 1;
    int prev_j = 1 << 30;  // the caller synchronized before the call
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 64 || prev_j >= 64) __syncthreads();
            else __syncwarp();
            prev_j = j;
            for (int q = threadIdx.x; q < half; q += blockDim.x) {
                const int i = 2 * q - (q & (j - 1));
                const int l = i + j;
                const T x = a[i], y = a[l];
                if ((x > y) == ((i & k) == 0)) {
                    a[i] = y;
                    a[l] = x;
                }
            }
        }
    }
    __syncthreads();
}

// in-place exclusive prefix sum of a[0, n) in shared memory, all threads of the block (each
// thread sums a contiguous piece, warp scan of the piece totals, block combine)
__device__ __forceinline__ void block_excl_scan_smem(int32_t* a, int n, int32_t* warp_tmp) {
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
    int32_t sum = 0;
    for (int i = lo; i < hi; ++i) sum += a[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[warp] = x;
    __syncthreads();
    int32_t pre = x - sum;
    for (int w = 0; w < warp; ++w) pre += warp_tmp[w];
    for (int i = lo; i < hi; ++i) {
        const int32_t v = a[i];
        a[i] = pre;
        pre += v;
    }
    __syncthreads();
}

// one CTA per batch slot: seeds sorted by ID (local ID = input position); duplicates are the
// EINVAL of reading c12
__global__ void __launch_bounds__(kPartThreads) k_seed_sort(Grp g, Part pt, int* err) {
    __shared__ unsigned long long s_k[kSeedSortMax];
    const int s = blockIdx.x;
    const int ns = g.hop_bound[s * (g.H + 2) + 1];
    int n2 = 1;
    while (n2 < ns) n2 <<= 1;
    const int32_t* nodes = g.nodes + (int64_t)s * g.cap_n;
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        s_k[i] = i < ns ? ((unsigned long long)(uint32_t)nodes[i] << 32) | (uint32_t)i : ~0ull;
    __syncthreads();
    bitonic_sort_smem(s_k, n2);
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        const unsigned long long e = s_k[i];
        pt.sid[(int64_t)s * pt.B + i] = (int32_t)(e >> 32);
        pt.sloc[(int64_t)s * pt.B + i] = (int32_t)(uint32_t)e;
        if (i > 0 && (s_k[i - 1] >> 32) == (e >> 32)) atomicOr(err, DEVERR_SEED_DUP);
    }
}

// Range starts inside each sorted slice of nodes-so-far: slice 0 = the sorted seeds, slice x >= 1
// = the new nodes of hop x-1 (local [hb[x], hb[x+1]), ID-ascending).  The element that opens a
// range writes its start for every (empty) range in between, so bnd[.][p] for p in [0, P] is
// written exactly once per non-empty slice (empty slices keep the memset's zeros).
__global__ void k_part_bounds(Grp g, Part pt) {
    const int s = blockIdx.y;
    const int32_t* hb = g.hop_bound + s * (g.H + 2);
    const int P = 1 << pt.pbits;
    const int32_t n = hb[pt.nslices];  // nodes so far
    const int32_t* nodes = g.nodes + (int64_t)s * g.cap_n;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int x = 0;
        while (j >= hb[x + 1]) ++x;
        const int32_t a = hb[x], e = hb[x + 1];
        const int32_t id = x == 0 ? pt.sid[(int64_t)s * pt.B + j] : nodes[j];
        const int q = id >> pt.pshift;
        int qprev = -1;
        if (j > a) qprev = (x == 0 ? pt.sid[(int64_t)s * pt.B + j - 1] : nodes[j - 1]) >> pt.pshift;
        int32_t* bnd = pt.bnd + ((int64_t)s * (g.H + 1) + x) * (P + 1);
        for (int r = qprev + 1; r <= q; ++r) bnd[r] = j - a;
        if (j == e - 1)
            for (int r = q + 1; r <= P; ++r) bnd[r] = e - a;
    }
}

// Shared-memory histogram of a tile's candidates over (batch, range) bins; the tile's batches
// span [s0, s1].  mode 0: add the counts to bcnt; mode 1: reserve the bins' runs at the cursors
// and write the (u, index) pairs.
template <int MODE>
__global__ void __launch_bounds__(kPartTileThreads) k_part_tile(Grp g, Part pt, const int32_t* __restrict__ cand) {
    constexpr int kIt = kPartTile / kPartTileThreads;
    __shared__ int64_t s_cb[kMaxGroup + 1];
    __shared__ int32_t s_h[kPartBins];
    __shared__ int64_t s_base[MODE ? kPartBins : 1];
    for (int i = threadIdx.x; i <= g.G; i += blockDim.x) s_cb[i] = g.cand_base[i];
    __syncthreads();
    const int64_t C = s_cb[g.G];
    const int P = 1 << pt.pbits;
    for (int64_t t0 = (int64_t)blockIdx.x * kPartTile; t0 < C; t0 += (int64_t)gridDim.x * kPartTile) {
        const int64_t t1 = min(C, t0 + kPartTile);
        const int s0 = segment_of(s_cb, g.G + 1, t0), s1 = segment_of(s_cb, g.G + 1, t1 - 1);
        const bool local = (int64_t)(s1 - s0 + 1) * P <= kPartBins;
        if (local) {
            for (int i = threadIdx.x; i < (s1 - s0 + 1) * P; i += blockDim.x) s_h[i] = 0;
            __syncthreads();
        }
        int32_t bin[kIt], rk[kIt], u[kIt];
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int64_t i = t0 + it * kPartTileThreads + threadIdx.x;
            bin[it] = -1;
            if (i < t1) {
                const int s = s0 == s1 ? s0 : segment_of(s_cb, g.G + 1, i);
                u[it] = cand[i];
                const int b = s * P + (u[it] >> pt.pshift);
                if (local) {
                    bin[it] = b - s0 * P;
                    rk[it] = atomicAdd(&s_h[bin[it]], 1);
                } else if (MODE == 0) {
                    atomicAdd(&pt.bcnt[b], 1);
                } else {
                    const int64_t pos = atomicAdd((unsigned long long*)&pt.bcur[b], 1ull);
                    pt.pui[pos] = make_int2(u[it], (int32_t)i);
                }
            }
        }
        if (local) {
            __syncthreads();
            for (int i = threadIdx.x; i < (s1 - s0 + 1) * P; i += blockDim.x) {
                const int c = s_h[i];
                if (MODE == 0) {
                    if (c) atomicAdd(&pt.bcnt[s0 * P + i], c);
                } else if (c) {
                    s_base[i] = (int64_t)atomicAdd((unsigned long long*)&pt.bcur[s0 * P + i], (unsigned long long)c);
                }
            }
            __syncthreads();
            if (MODE == 1) {
#pragma unroll
                for (int it = 0; it < kIt; ++it) {
                    if (bin[it] < 0) continue;
                    const int64_t pos = s_base[bin[it]] + rk[it];
                    pt.pui[pos] = make_int2(u[it], (int32_t)(t0 + it * kPartTileThreads + threadIdx.x));
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t part_hash(int32_t key, int tlog) {
    return ((uint32_t)key * 2654435761u) >> (32 - tlog);
}

__global__ void __launch_bounds__(kPartThreads) k_part_dedup(Grp g, Part pt, int32_t* __restrict__ cand, int* err) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    unsigned long long* s_new = reinterpret_cast<unsigned long long*>(s_dyn);
    int32_t* s_key = reinterpret_cast<int32_t*>(s_new + kPartTable);
    int32_t* s_loc = s_key + kPartTable;
    __shared__ int32_t s_scan_tmp[kPartThreads / 32];
    __shared__ int s_nnew;
    __shared__ volatile int s_over;
    __shared__ unsigned s_ticket;
    __shared__ int64_t s_prefix;
    __shared__ int32_t s_lo[kMaxHops + 1], s_hi[kMaxHops + 1], s_hb[kMaxHops + 2];
    __shared__ int64_t s_c0, s_c1;
    const int P = 1 << pt.pbits;
    const unsigned nbk = (unsigned)g.G * P;
    const int lane = threadIdx.x & 31;
    const int X = pt.nslices;
    for (;;) {
        if (threadIdx.x == 0) {
            s_ticket = atomicAdd(pt.ticket, 1u);
            s_nnew = 0;
            s_over = 0;
        }
        __syncthreads();
        const unsigned b = s_ticket;
        if (b >= nbk) break;
        const int s = (int)(b >> pt.pbits), p = (int)(b & (P - 1));
        // the bucket's extents, loaded in parallel: its old nodes (one run per slice of
        // nodes-so-far) and its candidates
        {
            const int t = threadIdx.x;
            if (t < X) {
                s_lo[t] = pt.bnd[((int64_t)s * (g.H + 1) + t) * (P + 1) + p];
            } else if (t >= 32 && t < 32 + X) {
                s_hi[t - 32] = pt.bnd[((int64_t)s * (g.H + 1) + (t - 32)) * (P + 1) + p + 1];
            } else if (t >= 64 && t < 64 + X + 1) {
                s_hb[t - 64] = g.hop_bound[s * (g.H + 2) + (t - 64)];
            } else if (t == 96) {
                s_c0 = pt.bstart[b];
            } else if (t == 97) {
                s_c1 = pt.bstart[b + 1];
            }
        }
        __syncthreads();
        int nold = 0;
        for (int x = 0; x < X; ++x) nold += s_hi[x] - s_lo[x];
        const int64_t c0 = s_c0, c1 = s_c1;
        // table size: twice the bucket's distinct-ID bound, at most kPartTable
        const int64_t bound = (int64_t)nold + (c1 - c0);
        int tlog = 6;
        while (tlog < kPartTableLog && ((int64_t)1 << tlog) < 2 * bound) ++tlog;
        const int tsize = 1 << tlog;
        const uint32_t tmask = (uint32_t)tsize - 1;
        const int limit = tsize - tsize / 4;  // distinct IDs before DEVERR_PART
        for (int i = threadIdx.x; i < tsize; i += blockDim.x) s_key[i] = kEmpty;
        if (nold > limit && threadIdx.x == 0) s_over = 1;
        __syncthreads();
        if (!s_over) {
            // old nodes: (id, local) into the table; IDs are distinct
            for (int r = threadIdx.x; r < nold; r += blockDim.x) {
                int x = 0, rr = r;
                while (rr >= s_hi[x] - s_lo[x]) {
                    rr -= s_hi[x] - s_lo[x];
                    ++x;
                }
                const int32_t j = s_lo[x] + rr;
                int32_t id, loc;
                if (x == 0) {
                    id = pt.sid[(int64_t)s * pt.B + j];
                    loc = pt.sloc[(int64_t)s * pt.B + j];
                } else {
                    loc = s_hb[x] + j;
                    id = g.nodes[(int64_t)s * g.cap_n + loc];
                }
                uint32_t q = part_hash(id, tlog);
                while (atomicCAS(&s_key[q], kEmpty, id) != kEmpty) q = (q + 1) & tmask;
                s_loc[q] = loc;
            }
            __syncthreads();
            // candidates: the first insert of an ID is a new node
            for (int64_t j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
                const int32_t u = pt.pui[j].x;
                uint32_t q = part_hash(u, tlog);
                for (int probes = 0;; ++probes) {
                    if (probes >= tsize) {  // unreachable below the limit; never spin
                        s_over = 1;
                        break;
                    }
                    const int32_t prev = atomicCAS(&s_key[q], kEmpty, u);
                    if (prev == kEmpty) {
                        const int r = atomicAdd(&s_nnew, 1);
                        if (r + nold >= limit) s_over = 1;  // the bucket is abandoned
                        else s_new[r] = ((unsigned long long)(uint32_t)u << 32) | q;
                        break;
                    }
                    if (prev == u) break;
                    q = (q + 1) & tmask;
                }
                if (s_over) break;
            }
        }
        __syncthreads();
        const bool over = s_over != 0;
        const int nnew = over ? 0 : s_nnew;
        if (over && threadIdx.x == 0) atomicOr(err, DEVERR_PART);
        // publish this bucket's new-node count first (its successors in the batch look back at
        // it), sort, and only then look back: the predecessors publish while this CTA sorts
        if (threadIdx.x == 0)
            st_relaxed(&pt.status[b], (p == 0 ? scan::kFlagP : scan::kFlagA) | (unsigned long long)nnew);
        // ranked: s_new[r] = (rank << 32 | slot) instead of sorted (u << 32 | slot)
        const bool ranked = !over && nnew > 1 && nnew <= pt.rank_max;
        if (ranked) {
            // order (reading c10) by counting: the bucket's ID range in 2^kRankBits sub-ranges
            // (counts and the grouped list live in s_new past its kRankMax used entries); an ID's
            // rank = the new IDs of lower sub-ranges + those of its own sub-range below it
            int32_t* s_cnt = reinterpret_cast<int32_t*>(s_new + kRankMax);  // [nsub + 1]
            int32_t* s_grp = s_cnt + (1 << kRankBits) + 1;                  // [nnew]
            const int rs = pt.pshift > kRankBits ? pt.pshift - kRankBits : 0;
            const int nsub = 1 << (pt.pshift < kRankBits ? pt.pshift : kRankBits);
            const int32_t base_id = p << pt.pshift;
            for (int i = threadIdx.x; i <= nsub; i += blockDim.x) s_cnt[i] = 0;
            __syncthreads();
            for (int r = threadIdx.x; r < nnew; r += blockDim.x)
                atomicAdd(&s_cnt[((int32_t)(s_new[r] >> 32) - base_id) >> rs], 1);
            __syncthreads();
            block_excl_scan_smem(s_cnt, nsub, s_scan_tmp);  // s_cnt[sub] = start of sub
            for (int r = threadIdx.x; r < nnew; r += blockDim.x)
                s_grp[atomicAdd(&s_cnt[((int32_t)(s_new[r] >> 32) - base_id) >> rs], 1)] = r;
            __syncthreads();  // now s_cnt[sub] = end of sub = start of sub + 1
            int rk[kRankMax / kPartThreads];
#pragma unroll
            for (int k = 0; k < kRankMax / kPartThreads; ++k) {
                const int r = threadIdx.x + k * kPartThreads;
                if (r >= nnew) break;
                const int32_t u = (int32_t)(s_new[r] >> 32);
                const int sub = (u - base_id) >> rs;
                const int lo = sub ? s_cnt[sub - 1] : 0, hi = s_cnt[sub];
                int rank = lo;
                for (int q = lo; q < hi; ++q) rank += ((int32_t)(s_new[s_grp[q]] >> 32) < u) ? 1 : 0;
                rk[k] = rank;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kRankMax / kPartThreads; ++k) {
                const int r = threadIdx.x + k * kPartThreads;
                if (r >= nnew) break;
                s_new[r] = ((unsigned long long)(uint32_t)rk[k] << 32) | (uint32_t)s_new[r];
            }
        } else if (!over) {
            int n2 = 1;
            while (n2 < nnew) n2 <<= 1;
            for (int i = nnew + threadIdx.x; i < n2; i += blockDim.x) s_new[i] = ~0ull;
            __syncthreads();
            if (nnew > 1) bitonic_sort_smem(s_new, n2);
        }
        // decoupled look-back over the batch's lower ranges (never past range 0 of batch s)
        if (threadIdx.x < 32) {
            int64_t prefix = 0;
            if (p > 0) {
                int t = p - 1;  // range index inside the batch
                for (;;) {
                    const int idx = t - lane;
                    const unsigned long long w =
                        idx >= 0 ? ld_relaxed(&pt.status[(unsigned)s * P + idx]) : scan::kFlagP;
                    const unsigned long long flag = w & ~scan::kMask;
                    const unsigned pmask = __ballot_sync(kFull, flag == scan::kFlagP);
                    const unsigned xmask = __ballot_sync(kFull, flag == 0);
                    const int first_p = pmask ? __ffs(pmask) - 1 : 31;
                    const unsigned need = (first_p == 31) ? kFull : ((2u << first_p) - 1u);
                    if (xmask & need) continue;
                    int64_t v = (lane <= first_p && idx >= 0) ? (int64_t)(w & scan::kMask) : 0;
#pragma unroll
                    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
                    prefix += v;
                    if (pmask) break;
                    t -= 32;
                }
                if (lane == 0) st_relaxed(&pt.status[b], scan::kFlagP | (unsigned long long)(prefix + nnew));
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (p == P - 1) g.new_cnt[s] = (int32_t)(prefix + nnew);
            }
        }
        __syncthreads();
        if (!over) {
            const int32_t base = s_hb[X] + (int32_t)s_prefix;  // nodes so far + lower ranges' new nodes
            int32_t* onodes = g.nodes + (int64_t)s * g.cap_n;
            for (int r = threadIdx.x; r < nnew; r += blockDim.x) {
                const unsigned long long e = s_new[r];
                const int32_t local = ranked ? base + (int32_t)(e >> 32) : base + r;  // (rank | slot) or sorted
                onodes[local] = ranked ? s_key[(uint32_t)e] : (int32_t)(e >> 32);
                s_loc[(uint32_t)e] = local;
            }
            __syncthreads();
            // remap: every candidate of the bucket to its local ID
            for (int64_t j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
                const int2 ui = pt.pui[j];
                uint32_t q = part_hash(ui.x, tlog);
                while (s_key[q] != ui.x) q = (q + 1) & tmask;
                cand[ui.y] = s_loc[q];
            }
        }
        __syncthreads();
    }
}

__global__ void k_hop_end_part(Grp g, int h) {
    for (int s = threadIdx.x; s < g.G; s += blockDim.x) {
        const int32_t n0 = g.n[s], c = g.new_cnt[s];
        g.hop_bound[s * (g.H + 2) + h + 2] = n0 + c;
        g.fr_lo[s] = g.blocks ? 0 : n0;
        g.fr_hi[s] = n0 + c;
        g.n[s] = n0 + c;
    }
}

// ------------------------------- a4: the access counter, range-major over the epoch
// counts[v] += the number of batches whose node list holds v.  One random RED per
// (batch, node) spreads ~0.5 G read-modify-writes over the whole 444 MB array (papers); instead,
// once every batch is sampled, each CTA owns one range of 2^kCntBits IDs, accumulates that range's
// counts over every batch in shared memory and adds them to counts[] with plain coalesced
// read-modify-writes (it is the range's only writer).  Every hop slice of a batch's node list is
// ID-ascending (reading c10), so a range is one contiguous run per slice: k_cnt_bounds finds the
// runs, k_cnt_ranges consumes them.  Seeds (input order) take one RED each.
constexpr int kCntBits = 14;                   // 16384 IDs = 64 KB of shared counters per CTA
constexpr int kCntThreads = 512;
constexpr int kCntChunk = 2048;                // slices per block-scan chunk in k_cnt_ranges

struct CntPlan {
    const int64_t* node_off;  // [nb+1]
    const int32_t* hop_off;   // [nb*(H+2)]
    const int32_t* nodes;
    int H;
    int64_t nb;
    int64_t P;                // ranges
    int32_t* bnd;             // [(P+1) * nb*H]: row p = start of range p in every slice; row P = lengths
};

// blockIdx.y = batch: the run boundaries of its hop slices (x = 1..H), plus one RED per seed
__global__ void k_cnt_bounds(CntPlan c, uint32_t* __restrict__ counts) {
    const int64_t NS = c.nb * c.H;
    for (int64_t b = blockIdx.y; b < c.nb; b += gridDim.y) {
        const int32_t* hb = c.hop_off + b * (c.H + 2);
        const int32_t* nodes = c.nodes + c.node_off[b];
        const int32_t n = hb[c.H + 1];
        for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
            const int32_t id = nodes[j];
            if (j < hb[1]) {  // a seed
                atomicAdd(&counts[id], 1u);
                continue;
            }
            int x = 1;
            while (j >= hb[x + 1]) ++x;
            const int32_t a = hb[x], e = hb[x + 1];
            const int64_t col = b * c.H + (x - 1);
            const int64_t q = id >> kCntBits;
            const int64_t qprev = j > a ? (int64_t)(nodes[j - 1] >> kCntBits) : -1;
            for (int64_t r = qprev + 1; r <= q; ++r) c.bnd[r * NS + col] = j - a;
            if (j == e - 1)
                for (int64_t r = q + 1; r <= c.P; ++r) c.bnd[r * NS + col] = e - a;
        }
    }
}

// CTA per range p (grid-stride): shared counters over every slice's run of the range
__global__ void __launch_bounds__(kCntThreads) k_cnt_ranges(CntPlan c, uint32_t* __restrict__ counts,
                                                            int64_t N) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_dyn);
    __shared__ int64_t s_pre[kCntChunk + 1];
    __shared__ int64_t s_base[kCntChunk];  // per slice of the chunk: node position of its run's entry 0 minus s_pre
    __shared__ int64_t s_wsum[kCntThreads / 32];
    const int64_t NS = c.nb * c.H;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t p = blockIdx.x; p < c.P; p += gridDim.x) {
        for (int i = threadIdx.x; i < (1 << kCntBits); i += blockDim.x) s_cnt[i] = 0;
        const int32_t* lo_row = c.bnd + p * NS;
        const int32_t* hi_row = c.bnd + (p + 1) * NS;
        for (int64_t s0 = 0; s0 < NS; s0 += kCntChunk) {
            const int ns = (int)min((int64_t)kCntChunk, NS - s0);
            // run lengths of this chunk of slices -> inclusive block scan into s_pre[1..ns]
            __syncthreads();
            constexpr int kPer = kCntChunk / kCntThreads;
            int64_t len[kPer], run = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int i = threadIdx.x * kPer + k;
                len[k] = i < ns ? (int64_t)(hi_row[s0 + i] - lo_row[s0 + i]) : 0;
                run += len[k];
            }
            int64_t incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            int64_t wpre = 0;
            for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
            int64_t acc = wpre + incl - run;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int i = threadIdx.x * kPer + k;
                if (i < ns) {
                    s_pre[i] = acc;
                    const int64_t sl = s0 + i;
                    const int64_t b = sl / c.H;
                    const int x = (int)(sl - b * c.H) + 1;
                    s_base[i] = c.node_off[b] + c.hop_off[b * (c.H + 2) + x] + lo_row[sl] - acc;
                }
                acc += len[k];
            }
            if (threadIdx.x == kCntThreads - 1) s_pre[ns] = acc;  // chunk total
            __syncthreads();
            const int64_t total = s_pre[ns];
            // flattened over the chunk's runs: entry t is in slice i with s_pre[i] <= t < s_pre[i+1]
            for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
                int lo = 0, hi = ns;  // s_pre[lo] <= t < s_pre[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_pre[mid] <= t) lo = mid;
                    else hi = mid;
                }
                atomicAdd(&s_cnt[c.nodes[s_base[lo] + t] - (p << kCntBits)], 1u);
            }
        }
        __syncthreads();
        const int64_t v0 = p << kCntBits;
        for (int i = threadIdx.x; i < (1 << kCntBits) && v0 + i < N; i += blockDim.x)
            if (s_cnt[i]) counts[v0 + i] += s_cnt[i];
        __syncthreads();
    }
}

// ------------------------------------------------ batch-major compaction
struct CompactPlan {
    int G;
    int H;
    int64_t cap_n;
    const int64_t* node_pre;     // [G+1] group-relative node prefix
    const int64_t* edge_pre;     // [G+1]
    const int64_t* eptr_pre;     // [G+1]
    const int64_t* edges_before; // [H*G]
    const int64_t* hop_fr_off;   // [H*(kMaxGroup+1)]
    const int64_t* hop_cbase;    // [H*(kMaxGroup+1)]
    const int32_t* hop_bound;    // [G*(H+2)]
    int64_t* const* cptr;        // [H] device pointers
    int blocks;
};

// blockIdx.y = batch slot s: its nodes are one contiguous run in the slot's scratch and one in the
// arena, so each CTA row copies its slot's run (no per-element search for the slot)
__global__ void k_compact_nodes(CompactPlan p, const int32_t* __restrict__ gnodes, int32_t* __restrict__ out) {
    const int s = blockIdx.y;
    const int64_t pre = p.node_pre[s], n = p.node_pre[s + 1] - pre;
    const int32_t* src = gnodes + (int64_t)s * p.cap_n;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        out[pre + j] = src[j];
}

// blockIdx.y = batch slot s: hop h's candidates of slot s are one contiguous run of cand
__global__ void k_compact_edges(CompactPlan p, int h, const int32_t* __restrict__ cand, int32_t* __restrict__ out) {
    const int s = blockIdx.y;
    const int64_t* cb = p.hop_cbase + h * (kMaxGroup + 1);
    const int64_t c0 = cb[s], n = cb[s + 1] - c0;
    int32_t* dst = out + p.edge_pre[s] + p.edges_before[h * p.G + s];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        dst[j] = cand[c0 + j];
}

__global__ void k_compact_eptr(CompactPlan p, int32_t* __restrict__ out) {
    __shared__ int64_t s_pre[kMaxGroup + 1];
    for (int i = threadIdx.x; i <= p.G; i += blockDim.x) s_pre[i] = p.eptr_pre[i];
    __syncthreads();
    const int64_t T = s_pre[p.G];
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < T; q += (int64_t)gridDim.x * blockDim.x) {
        const int s = segment_of(s_pre, p.G + 1, q);
        int64_t j = q - s_pre[s];
        const int32_t* hb = p.hop_bound + s * (p.H + 2);
        int64_t val;
        if (!p.blocks) {
            if (j == hb[p.H]) {
                val = p.edge_pre[s + 1] - p.edge_pre[s];
            } else {
                int h = 0;
                while (!(j < hb[h + 1])) ++h;  // frontier of hop h: local [hb[h], hb[h+1])
                const int64_t t = p.hop_fr_off[h * (kMaxGroup + 1) + s] + (j - hb[h]);
                val = p.cptr[h][t] - p.hop_cbase[h * (kMaxGroup + 1) + s] + p.edges_before[h * p.G + s];
            }
        } else {
            // blocks: hop h's array has hb[h+1] + 1 entries (its frontier is local [0, hb[h+1]))
            int h = 0;
            while (j > hb[h + 1]) {
                j -= hb[h + 1] + 1;
                ++h;
            }
            if (j == hb[h + 1]) {
                val = h + 1 < p.H ? p.edges_before[(h + 1) * p.G + s] : p.edge_pre[s + 1] - p.edge_pre[s];
            } else {
                const int64_t t = p.hop_fr_off[h * (kMaxGroup + 1) + s] + j;
                val = p.cptr[h][t] - p.hop_cbase[h * (kMaxGroup + 1) + s] + p.edges_before[h * p.G + s];
            }
        }
        out[q] = (int32_t)val;
    }
}

// ------------------------------------------------------------ host side
int ceil_log2(int64_t x) {
    int b = 0;
    while (((int64_t)1 << b) < x) ++b;
    return b;
}

int64_t sat_mul(int64_t a, int64_t b, int64_t cap) {
    if (a == 0 || b == 0) return 0;
    if (a > cap / b) return cap;
    return std::min(a * b, cap);
}

// sub-buffers carved from one allocation (sizing pass with base = NULL, then the real pass)
struct Slab {
    uint8_t* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T* q = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += std::max<size_t>(count, 1) * sizeof(T);
        return q;
    }
};

struct Arena {
    // an output array of dgnn_sample; its buffer comes from (and, on an error path, goes back
    // to) the ctx's kept buffers, so an epoch resampled on the same ctx reuses the previous
    // epoch's arena at its final size instead of growing a fresh one by copies
    dgnn_ctx* c;
    int32_t* p = nullptr;
    int64_t cap = 0;
    ~Arena() {
        if (p) keep_put(c, p, (size_t)cap * 4);
    }
    int32_t* release() {
        int32_t* q = p;
        p = nullptr;
        return q;
    }
    dgnn_status reserve(int64_t need, int64_t used) {
        if (need <= cap) return DGNN_OK;
        // a fresh arena gets 1/8 headroom: the next epoch's estimate (made after its first group)
        // then still fits the kept buffer
        const int64_t want = p ? std::max<int64_t>(need, cap + cap / 2) : need + need / 8;
        size_t got = 0;
        int32_t* q = (int32_t*)keep_take(c, (size_t)want * 4, &got);
        if (!q) {
            set_error("sample arena allocation of %lld bytes failed", (long long)want * 4);
            return DGNN_ENOMEM;
        }
        if (p) {
            if (used) DGNN_CK(cudaMemcpyAsync(q, p, (size_t)used * 4, cudaMemcpyDeviceToDevice, c->stream));
            dev_free(c, p, (size_t)cap * 4);
        }
        p = q;
        cap = (int64_t)(got / 4);
        return DGNN_OK;
    }
};

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_sample(dgnn_ctx* c, const dgnn_csr* csr, const int32_t* seeds, int64_t num_seeds,
                                   int32_t batch_size, int64_t batch_id_base, const int32_t* fanout,
                                   int32_t num_hops, uint64_t rng_seed, uint32_t* counts, dgnn_samples** out) {
    DGNN_REQUIRE(c && csr && out, "dgnn_sample: NULL argument");
    *out = nullptr;
    DGNN_REQUIRE(csr->num_nodes > 0 && csr->num_nodes < ((int64_t)1 << DGNN_TIER_SHIFT),
                 "dgnn_sample: num_nodes must be in [1, 2^30)");
    DGNN_REQUIRE(csr->indptr && (csr->indices || csr->num_edges == 0), "dgnn_sample: CSR arrays are NULL");
    DGNN_REQUIRE(batch_size > 0, "dgnn_sample: batch_size must be positive");
    DGNN_REQUIRE(num_seeds >= 0 && (seeds || num_seeds == 0), "dgnn_sample: bad seeds");
    DGNN_REQUIRE(batch_id_base >= 0, "dgnn_sample: batch_id_base must be >= 0");
    DGNN_REQUIRE(num_hops >= 1 && num_hops <= 65535 && fanout, "dgnn_sample: num_hops must be in [1, 65535]");
    for (int h = 0; h < num_hops; ++h)
        DGNN_REQUIRE(fanout[h] >= 0 && fanout[h] <= 65535, "dgnn_sample: fanout[%d]=%d outside [0, 65535]", h,
                     fanout[h]);
    DGNN_CK(cudaSetDevice(c->device));
    const auto t_entry = std::chrono::steady_clock::now();  // (DGNN_TRACE_SAMPLE only)
    auto t_synced = t_entry;
    const int64_t N = csr->num_nodes;
    const int H = num_hops;
    const int64_t B = batch_size;
    const int64_t nb = (num_seeds + B - 1) / B;

    auto* S = new dgnn_samples();
    S->ctx = c;
    S->nb = nb;
    S->H = H;
    S->batch_id_base = batch_id_base;
    S->mode = c->sample_mode;
    struct Guard {
        dgnn_samples* s;
        ~Guard() { if (s) dgnn_samples_free(s); }
    } guard{S};
    S->node_off_h.assign(nb + 1, 0);
    S->edge_off_h.assign(nb + 1, 0);
    S->eptr_off_h.assign(nb + 1, 0);
    S->hop_off_h.assign(nb * (H + 2), 0);
    // a4 counter: range-major over the finished epoch (default) or per group (DGNN_SAMPLE_COUNT=group)
    const char* cm = std::getenv("DGNN_SAMPLE_COUNT");
    const bool range_count = !(cm && std::string(cm) == "group");

    if (nb > 0) {
        // all seeds in range before any counting
        launch(c, DGNN_K_SAMPLE_SEED, 0.0, [&] {
            k_seed_range<<<grid_for(c, num_seeds, 256), 256, 0, c->stream>>>(seeds, num_seeds, N, c->dev_err);
        });
        DGNN_CK_LAUNCH();
        DGNN_TRY(check_dev_err(c));
        t_synced = std::chrono::steady_clock::now();

        // ---- capacities (exact upper bounds; reading c26 for k = 0) ----
        const int64_t kCap = (int64_t)1 << 40;
        std::vector<int64_t> fr_bound(H), cand_bound(H), new_bound(H);
        const bool blocks = c->sample_mode == DGNN_SAMPLE_BLOCKS;
        int64_t prod = B, nodes_bound = B;
        for (int h = 0; h < H; ++h) {
            fr_bound[h] = blocks ? nodes_bound : prod;  // blocks: every node so far expands
            prod = sat_mul(fr_bound[h], fanout[h], kCap);
            new_bound[h] = prod;
            nodes_bound = std::min(kCap, nodes_bound + prod);
        }
        const int64_t cap_n = std::min(nodes_bound, N);  // a batch's nodes are distinct IDs
        for (int h = 0; h < H; ++h) {
            fr_bound[h] = std::min(fr_bound[h], cap_n);
            new_bound[h] = std::min(new_bound[h], cap_n);
            cand_bound[h] = sat_mul(fr_bound[h], fanout[h], kCap);
        }
        const int tlog = std::max(4, ceil_log2(2 * cap_n));
        std::vector<int> bb(H), shift(H);
        const int idbits = std::max(1, ceil_log2(N));
        int64_t hist_per_slot = 1;
        for (int h = 0; h < H; ++h) {
            int b = ceil_log2(std::max<int64_t>(1, new_bound[h] / 4));
            b = std::min(b, idbits);
            bb[h] = b;
            shift[h] = idbits - b;
            hist_per_slot = std::max<int64_t>(hist_per_slot, (int64_t)1 << b);
        }
        int64_t max_fr = 1, max_cand = 1;
        for (int h = 0; h < H; ++h) {
            max_fr = std::max(max_fr, fr_bound[h]);
            max_cand = std::max(max_cand, cand_bound[h]);
        }
        // Hash-set size: the first group uses the exact bound (2 x the node bound) unless the ctx
        // carries the largest batch of its previous call (an epoch resamples the same workload);
        // later groups use 2 x the largest node count seen so far (a table that stays closer to
        // L2), and a group that overflows is redone at the bound.  The access counter is
        // therefore applied after a group succeeds, over its compacted nodes.
        const int tlog_safe = tlog;
        const bool adaptive = !(std::getenv("DGNN_SAMPLE_TABLE") && std::string(std::getenv("DGNN_SAMPLE_TABLE")) == "bound");
        int tlog_cur = (adaptive && c->sample_n_hint > 0)
                           ? std::min(tlog_safe, std::max(4, ceil_log2(2 * c->sample_n_hint)))
                           : tlog_safe;
        // group size from the scratch budget (the table counted at its expected size)
        int64_t per_slot = cap_n * (4 + 8) + ((int64_t)8 << tlog_cur) + hist_per_slot * 12 + max_fr * 16 + max_cand * 8;
        for (int h = 0; h < H; ++h) per_slot += (fr_bound[h] + 1) * 8 + cand_bound[h] * 4;
        int64_t G = c->sample_group;
        if (G <= 0) {
            const int64_t budget = (int64_t)c->sample_budget;
            G = std::max<int64_t>(1, std::min<int64_t>(64, budget / std::max<int64_t>(per_slot, 1)));
        }
        G = std::min<int64_t>(std::min<int64_t>(G, kMaxGroup), nb);

        // ---- dedup path: partitioned shared-memory buckets unless the batch is too large for the
        // seed sort or DGNN_SAMPLE_DEDUP=table; per hop, P ranges so that a bucket expects ~1024
        // distinct IDs (from the node bound after the hop, capped by the ctx's hint) ----
        const char* dd = std::getenv("DGNN_SAMPLE_DEDUP");
        bool part = batch_size <= kSeedSortMax && H <= kMaxHops && !(dd && std::string(dd) == "table");
        const char* so = std::getenv("DGNN_SAMPLE_ORDER");  // "sort": bitonic order for every bucket
        const int rank_max = (so && std::string(so) == "sort") ? 0 : kRankMax;
        const int pbits_max = std::min(idbits, 12);
        std::vector<int64_t> after_bound(H), after_seen(H, 0);
        {
            int64_t acc = B;
            for (int h = 0; h < H; ++h) {
                acc = std::min<int64_t>(cap_n, acc + new_bound[h]);
                after_bound[h] = acc;
            }
        }
        auto pbits_for = [&](int h) {
            int64_t est = after_bound[h];
            if (after_seen[h] > 0) est = std::min(est, after_seen[h] + after_seen[h] / 4);
            else if (c->sample_n_hint > 0) est = std::min(est, c->sample_n_hint + c->sample_n_hint / 4);
            return std::min(pbits_max, std::max(0, ceil_log2((est + kPartTarget - 1) / kPartTarget)));
        };
        const int64_t Pmax = (int64_t)1 << pbits_max;

        // ---- group scratch: one slab recycled through the ctx (keep_take / keep_put) ----
        int32_t *d_nodes = nullptr, *d_small32 = nullptr, *d_hist = nullptr, *d_npos = nullptr, *d_ntab = nullptr,
                *d_fv = nullptr, *d_fdg = nullptr;
        unsigned long long* d_sorted = nullptr;
        int64_t *d_small64 = nullptr, *d_bstart = nullptr, *d_plan = nullptr, *d_fst = nullptr;
        std::vector<int32_t*> d_cand(H);
        std::vector<int64_t*> d_cptr(H);
        int64_t** d_cptr_list = nullptr;
        Part pt{};
        pt.B = batch_size;
        const size_t plan_max = 3 * (size_t)(G + 1) + (size_t)H * G;
        auto carve = [&](Slab& sl) {
            d_nodes = sl.take<int32_t>((size_t)(G * cap_n));
            d_small32 = sl.take<int32_t>((size_t)(4 * G + G * (H + 2)));
            d_small64 = sl.take<int64_t>((size_t)(3 * (G + 1) + 2 + 2 * H * (kMaxGroup + 1)));
            d_npos = sl.take<int32_t>((size_t)(G * max_cand));
            d_ntab = sl.take<int32_t>((size_t)(G * max_cand));
            d_fv = sl.take<int32_t>((size_t)(G * max_fr));
            d_fdg = sl.take<int32_t>((size_t)(G * max_fr));
            d_fst = sl.take<int64_t>((size_t)(G * max_fr));
            for (int h = 0; h < H; ++h) {
                d_cand[h] = sl.take<int32_t>((size_t)std::max<int64_t>(1, G * cand_bound[h]));
                d_cptr[h] = sl.take<int64_t>((size_t)(G * fr_bound[h] + 1));
            }
            d_cptr_list = sl.take<int64_t*>((size_t)H);
            d_plan = sl.take<int64_t>(plan_max);
            if (part) {
                pt.sid = sl.take<int32_t>((size_t)G * batch_size);
                pt.sloc = sl.take<int32_t>((size_t)G * batch_size);
                pt.bnd = sl.take<int32_t>((size_t)G * (H + 1) * (Pmax + 1));
                pt.bstart = sl.take<int64_t>((size_t)(G * Pmax + 1));
                pt.bcur = sl.take<int64_t>((size_t)(G * Pmax));
                pt.bcnt = sl.take<int32_t>((size_t)(G * Pmax));
                pt.status = sl.take<unsigned long long>((size_t)(G * Pmax));
                pt.ticket = sl.take<unsigned int>(1);
            }
        };
        Slab sizing;
        carve(sizing);
        DevBuf<uint8_t> d_slab;
        DGNN_TRY(d_slab.alloc_kept(c, sizing.off));
        {
            Slab sl;
            sl.base = d_slab.p;
            carve(sl);
        }
        pt.pui = reinterpret_cast<int2*>(d_npos);  // spans d_npos and d_ntab (the hash-set path's pair)
        // hash-set path scratch (bucket sort arrays + the hash sets), taken when that path runs
        DevBuf<uint8_t> d_legacy;
        DevBuf<int32_t> d_tabs;
        int tlog_alloc = 0;
        auto take_legacy = [&]() -> dgnn_status {
            if (!d_legacy.p) {
                auto carve_l = [&](Slab& sl) {
                    d_hist = sl.take<int32_t>((size_t)(G * hist_per_slot));
                    d_bstart = sl.take<int64_t>((size_t)(G * hist_per_slot));
                    d_sorted = sl.take<unsigned long long>((size_t)(G * cap_n));
                };
                Slab sz;
                carve_l(sz);
                DGNN_TRY(d_legacy.alloc_kept(c, sz.off));
                Slab sl;
                sl.base = d_legacy.p;
                carve_l(sl);
            }
            return DGNN_OK;
        };
        {
            std::vector<int64_t*> ptrs(H);
            for (int h = 0; h < H; ++h) ptrs[h] = d_cptr[h];
            DGNN_TRY(upload_small(c, d_cptr_list, ptrs.data(), sizeof(int64_t*) * H));
        }
        if (part) DGNN_CK(cudaFuncSetAttribute(k_part_dedup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPartSmem));
        const int part_grid = part ? grid_resident(c, k_part_dedup, (int64_t)1 << 40, kPartThreads, 8, kPartSmem) : 0;
        Grp g{};
        g.blocks = blocks ? 1 : 0;
        g.tlog = tlog;
        g.tmask = (uint32_t)((1ull << tlog) - 1);
        g.max_probes = g.tmask + 1;
        g.H = H;
        g.cap_n = cap_n;
        g.nodes = d_nodes;
        g.n = d_small32;
        g.fr_lo = g.n + G;
        g.fr_hi = g.fr_lo + G;
        g.new_cnt = g.fr_hi + G;
        g.hop_bound = g.new_cnt + G;
        g.fr_off = d_small64;
        g.cand_base = g.fr_off + (G + 1);
        g.new_off = g.cand_base + (G + 1);
        g.cand_total = g.new_off + (G + 1);
        int64_t* new_total = g.cand_total + 1;
        g.hop_fr_off = new_total + 1;
        g.hop_cbase = g.hop_fr_off + H * (kMaxGroup + 1);
        g.fv = d_fv;
        g.fst = d_fst;
        g.fdg = d_fdg;

        Arena a_nodes{c}, a_edges{c}, a_eptr{c};
        int64_t used_nodes = 0, used_edges = 0, used_eptr = 0;
        // host views of the per-group sizes and the compaction plan, in pinned memory
        const size_t n_frs = (size_t)H * (kMaxGroup + 1);
        const size_t plan_cap = 3 * (size_t)(G + 1) + (size_t)H * G;
        const size_t pin_bytes = sizeof(int64_t) * plan_cap;
        auto* pin = static_cast<uint8_t*>(pinned_scratch(c, pin_bytes));
        if (!pin) {
            set_error("pinned host allocation of %zu bytes failed", pin_bytes);
            return DGNN_ENOMEM;
        }
        int64_t* h_plan = reinterpret_cast<int64_t*>(pin);  // (upload source)
        // the group-end sizes come back through the read-back buffer (SM stores, no copy engine);
        // its first 64 bytes are read_dev_err's
        const size_t rb_frs = 64, rb_cbs = rb_frs + sizeof(int64_t) * n_frs, rb_n = rb_cbs + sizeof(int64_t) * n_frs,
                     rb_hb = rb_n + sizeof(int32_t) * G, rb_end = rb_hb + sizeof(int32_t) * G * (H + 2);
        DGNN_TRY(readback_reserve(c, rb_end));
        int64_t* h_frs = reinterpret_cast<int64_t*>(readback_host(c) + rb_frs);
        int64_t* h_cbs = reinterpret_cast<int64_t*>(readback_host(c) + rb_cbs);
        int32_t* h_n = reinterpret_cast<int32_t*>(readback_host(c) + rb_n);
        int32_t* h_hb = reinterpret_cast<int32_t*>(readback_host(c) + rb_hb);

        // DGNN_TRACE_SAMPLE=1: host-side split of the call (enqueue vs waiting in the group syncs)
        const bool trace = std::getenv("DGNN_TRACE_SAMPLE") != nullptr;
        using clk = std::chrono::steady_clock;
        double t_wait = 0.0, t_enq = 0.0, t_post = 0.0;
        const auto t_start = clk::now();
        int64_t max_n_seen = 0;
        int64_t redone = 0;
        for (int64_t t0 = 0; t0 < nb;) {
            const auto tg0 = clk::now();
            const int Gc = (int)std::min<int64_t>(G, nb - t0);
            g.G = Gc;
            if (!part) {
                DGNN_TRY(take_legacy());
                if (!d_tabs.p || tlog_cur > tlog_alloc) {  // a bigger table than the one taken
                    tlog_alloc = tlog_cur;
                    DGNN_TRY(d_tabs.alloc_kept(c, (size_t)(2 * G) << tlog_alloc));
                }
                g.table = d_tabs.p;
                g.local = d_tabs.p + ((size_t)G << tlog_alloc);
                g.tlog = tlog_cur;
                g.tmask = (uint32_t)((1ull << tlog_cur) - 1);
                // inserts into a table below the bound give up after a bounded probe run (the group
                // is then redone at the bound); at the bound the load is <= 1/2 and every insert
                // succeeds
                g.max_probes = tlog_cur < tlog_safe ? 128u : g.tmask + 1;
                DGNN_TRY(memset_async(c, g.table, 0xFF, sizeof(int32_t) * ((size_t)Gc << tlog_cur)));
            }
            launch(c, DGNN_K_SAMPLE_SEED, 0.0, [&] {
                k_seed_init<<<Gc, 256, 0, c->stream>>>(g, seeds, num_seeds, batch_size, t0, N, nullptr, c->dev_err,
                                                       part ? 0 : 1);
            });
            DGNN_CK_LAUNCH();
            if (part) {
                launch(c, DGNN_K_SAMPLE_SEED, 0.0,
                       [&] { k_seed_sort<<<Gc, kPartThreads, 0, c->stream>>>(g, pt, c->dev_err); });
                DGNN_CK_LAUNCH();
            }
            for (int h = 0; h < H; ++h) {
                const int k = fanout[h];
                const int64_t fmax = Gc * fr_bound[h], cmax = Gc * cand_bound[h];
                launch(c, DGNN_K_SAMPLE_SETUP, 0.0, [&] { k_hop_begin<<<1, kSlotThreads, 0, c->stream>>>(g, h); });
                DGNN_CK_LAUNCH();
                // a2: candidate offsets (and the frontier's (v, start, deg) records)
                DGNN_TRY(scan::run(c, fmax, g.fr_off + Gc, DegIn{g, csr->indptr, k, c->dev_err},
                                   StoreExcl{d_cptr[h]}, g.cand_total));
                launch(c, DGNN_K_SAMPLE_SETUP, 0.0,
                       [&] { k_hop_cands<<<1, kSlotThreads, 0, c->stream>>>(g, h, d_cptr[h]); });
                DGNN_CK_LAUNCH();
                // a2: draws + gather
                if (k > 0) {
                    const int64_t cb = batch_id_base + t0;
                    const int64_t* cp = d_cptr[h];
                    int32_t* cd = d_cand[h];
                    const bool warp_hop = std::getenv("DGNN_SAMPLE_HOP") &&
                                          std::string(std::getenv("DGNN_SAMPLE_HOP")) == "warp";
                    launch(c, DGNN_K_SAMPLE_HOP, 0.0, [&] {
                        const int tg = grid_for(c, fmax, 256);
                        if (!warp_hop && k <= 4)
                            k_sample_hop_t<4><<<tg, 256, 0, c->stream>>>(g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (!warp_hop && k <= 8)
                            k_sample_hop_t<8><<<tg, 256, 0, c->stream>>>(g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (!warp_hop && k <= 16)
                            k_sample_hop_t<16><<<tg, 256, 0, c->stream>>>(g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (!warp_hop && k <= 32)
                            k_sample_hop_t<32><<<tg, 256, 0, c->stream>>>(g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (k <= 4)
                            k_sample_hop<4><<<grid_for(c, fmax * 4, 256), 256, 0, c->stream>>>(
                                g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (k <= 8)
                            k_sample_hop<8><<<grid_for(c, fmax * 8, 256), 256, 0, c->stream>>>(
                                g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (k <= 16)
                            k_sample_hop<16><<<grid_for(c, fmax * 16, 256), 256, 0, c->stream>>>(
                                g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else if (k <= 32)
                            k_sample_hop<32><<<grid_for(c, fmax * 32, 256), 256, 0, c->stream>>>(
                                g, csr->indices, k, rng_seed, cb, h, cp, cd);
                        else
                            k_sample_hop_wide<<<grid_for(c, fmax * 32, 256), 256, 0, c->stream>>>(
                                g, csr->indices, k, rng_seed, cb, h, cp, cd);
                    });
                    DGNN_CK_LAUNCH();
                }
                if (part) {
                    // a3, partitioned: bucket the candidates by (batch, ID range), dedup + order +
                    // remap each bucket in shared memory
                    pt.pbits = pbits_for(h);
                    pt.pshift = idbits - pt.pbits;
                    pt.nslices = h + 1;
                    pt.rank_max = rank_max;
                    const int64_t P = (int64_t)1 << pt.pbits, nbk = Gc * P;
                    DGNN_TRY(memset_async(c, pt.bnd, 0, sizeof(int32_t) * (size_t)Gc * (H + 1) * (P + 1)));
                    DGNN_TRY(memset_async(c, pt.bcnt, 0, sizeof(int32_t) * (size_t)nbk));
                    launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                        k_part_bounds<<<dim3(8, Gc), 256, 0, c->stream>>>(g, pt);
                    });
                    DGNN_CK_LAUNCH();
                    const int tgrid = grid_for(c, cmax, kPartTile);
                    launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                        k_part_tile<0><<<tgrid, kPartTileThreads, 0, c->stream>>>(g, pt, d_cand[h]);
                    });
                    DGNN_CK_LAUNCH();
                    {
                        const int32_t* cnt = pt.bcnt;
                        int64_t* bst = pt.bstart;
                        int64_t* bcu = pt.bcur;
                        DGNN_TRY(scan::run(
                            c, nbk, nullptr, [=] __device__(int64_t i) -> int32_t { return cnt[i]; },
                            [=] __device__(int64_t i, int64_t e, int64_t) {
                                bst[i] = e;
                                bcu[i] = e;
                            },
                            pt.bstart + nbk));
                    }
                    launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                        k_part_tile<1><<<tgrid, kPartTileThreads, 0, c->stream>>>(g, pt, d_cand[h]);
                    });
                    DGNN_CK_LAUNCH();
                    DGNN_TRY(memset_async(c, pt.status, 0, sizeof(unsigned long long) * (size_t)nbk));
                    DGNN_TRY(memset_async(c, pt.ticket, 0, sizeof(unsigned int)));
                    launch(c, DGNN_K_SAMPLE_DEDUP, 0.0, [&] {
                        k_part_dedup<<<(int)std::min<int64_t>(part_grid, nbk), kPartThreads, kPartSmem, c->stream>>>(
                            g, pt, d_cand[h], c->dev_err);
                    });
                    DGNN_CK_LAUNCH();
                    launch(c, DGNN_K_SAMPLE_SETUP, 0.0, [&] { k_hop_end_part<<<1, 256, 0, c->stream>>>(g, h); });
                    DGNN_CK_LAUNCH();
                    continue;
                }
                // a3: dedup insert + count + bucket histogram of (slot, id >> shift)
                const int64_t NB = (int64_t)1 << bb[h];
                const int64_t nbk = Gc * NB;
                DGNN_TRY(memset_async(c, d_hist, 0, sizeof(int32_t) * (size_t)nbk));
                launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                    k_insert<<<grid_for(c, cmax, 256), 256, 0, c->stream>>>(g, d_cand[h], NB, shift[h], d_hist,
                                                                            d_npos, d_ntab, nullptr, c->dev_err);
                });
                DGNN_CK_LAUNCH();
                {
                    const int32_t* hist = d_hist;
                    int64_t* bst = d_bstart;
                    DGNN_TRY(scan::run(
                        c, nbk, nullptr, [=] __device__(int64_t i) -> int32_t { return hist[i]; },
                        [=] __device__(int64_t i, int64_t e, int64_t) { bst[i] = e; }, new_total));
                }
                launch(c, DGNN_K_SAMPLE_SETUP, 0.0,
                       [&] { k_new_setup<<<1, 256, 0, c->stream>>>(g, d_bstart, NB, new_total); });
                DGNN_CK_LAUNCH();
                launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                    k_bucket_scatter<<<grid_for(c, cmax, 256), 256, 0, c->stream>>>(
                        g, d_cand[h], NB, shift[h], d_bstart, d_npos, d_ntab, d_sorted);
                });
                DGNN_CK_LAUNCH();
                launch(c, DGNN_K_SAMPLE_ORDER, 0.0, [&] {
                    k_bucket_sort_assign<<<grid_for(c, nbk, 256), 256, 0, c->stream>>>(g, NB, d_bstart, d_hist,
                                                                                         d_sorted);
                });
                DGNN_CK_LAUNCH();
                launch(c, DGNN_K_SAMPLE_REMAP, 0.0, [&] {
                    k_remap<<<grid_for(c, cmax, 256), 256, 0, c->stream>>>(g, d_cand[h], d_ntab);
                });
                DGNN_CK_LAUNCH();
                launch(c, DGNN_K_SAMPLE_SETUP, 0.0, [&] { k_hop_end<<<1, 256, 0, c->stream>>>(g, h); });
                DGNN_CK_LAUNCH();
            }
            // ---- group end: read sizes, then compact into the batch-major arena ----
            DGNN_TRY(readback_enqueue(c, rb_n, g.n, sizeof(int32_t) * Gc));
            DGNN_TRY(readback_enqueue(c, rb_hb, g.hop_bound, sizeof(int32_t) * Gc * (H + 2)));
            DGNN_TRY(readback_enqueue(c, rb_frs, g.hop_fr_off, sizeof(int64_t) * n_frs));
            DGNN_TRY(readback_enqueue(c, rb_cbs, g.hop_cbase, sizeof(int64_t) * n_frs));
            const auto tg1 = clk::now();
            int flags = 0;
            DGNN_TRY(read_dev_err(c, &flags));  // synchronizes
            const auto tg2 = clk::now();
            if (trace) {
                t_enq += std::chrono::duration<double, std::milli>(tg1 - tg0).count();
                t_wait += std::chrono::duration<double, std::milli>(tg2 - tg1).count();
            }
            if ((flags & DEVERR_PART) && part && !(flags & (DEVERR_SEED_RANGE | DEVERR_SEED_DUP))) {
                // a bucket of the partitioned dedup overflowed: this group and the rest of the call
                // run on the hash-set path
                part = false;
                ++redone;
                continue;
            }
            if ((flags & DEVERR_TABLE) && !part && tlog_cur < tlog_safe) {  // the smaller table overflowed: redo
                tlog_cur = tlog_safe;
                ++redone;
                continue;
            }
            DGNN_TRY(dev_err_status(flags));
            for (int s = 0; s < Gc; ++s) max_n_seen = std::max<int64_t>(max_n_seen, h_n[s]);
            for (int s = 0; s < Gc; ++s)
                for (int h = 0; h < H; ++h)
                    after_seen[h] = std::max<int64_t>(after_seen[h], h_hb[s * (H + 2) + h + 2]);
            if (adaptive) tlog_cur = std::min(tlog_safe, std::max(4, ceil_log2(2 * max_n_seen)));
            // plan: node_pre[G+1], edge_pre[G+1], eptr_pre[G+1], edges_before[H*G]
            const size_t plan_n = 3 * (size_t)(Gc + 1) + (size_t)H * Gc;
            std::fill(h_plan, h_plan + plan_n, int64_t(0));
            int64_t* node_pre = h_plan;
            int64_t* edge_pre = node_pre + (Gc + 1);
            int64_t* eptr_pre = edge_pre + (Gc + 1);
            int64_t* ebef = eptr_pre + (Gc + 1);
            for (int s = 0; s < Gc; ++s) {
                int64_t e = 0;
                for (int h = 0; h < H; ++h) {
                    ebef[h * Gc + s] = e;
                    e += h_cbs[h * (kMaxGroup + 1) + s + 1] - h_cbs[h * (kMaxGroup + 1) + s];
                }
                node_pre[s + 1] = node_pre[s] + h_n[s];
                edge_pre[s + 1] = edge_pre[s] + e;
                int64_t ne = h_hb[s * (H + 2) + H] + 1;
                if (blocks) {
                    ne = 0;
                    for (int h = 0; h < H; ++h) ne += h_hb[s * (H + 2) + h + 1] + 1;
                }
                eptr_pre[s + 1] = eptr_pre[s] + ne;
                const int64_t b = t0 + s;
                S->node_off_h[b + 1] = S->node_off_h[b] + h_n[s];
                S->edge_off_h[b + 1] = S->edge_off_h[b] + e;
                S->eptr_off_h[b + 1] = S->eptr_off_h[b] + ne;
                for (int x = 0; x < H + 2; ++x) S->hop_off_h[b * (H + 2) + x] = h_hb[s * (H + 2) + x];
            }
            // grow the arena (estimate the whole run from the groups seen so far)
            const double frac = (double)nb / (double)(t0 + Gc);
            auto est = [&](int64_t used, int64_t add) {
                return (int64_t)((double)(used + add) * frac * 1.02) + 1024;
            };
            DGNN_TRY(a_nodes.reserve(used_nodes + node_pre[Gc] > a_nodes.cap ? est(used_nodes, node_pre[Gc]) : 0,
                                     used_nodes));
            DGNN_TRY(a_edges.reserve(used_edges + edge_pre[Gc] > a_edges.cap ? est(used_edges, edge_pre[Gc]) : 0,
                                     used_edges));
            DGNN_TRY(a_eptr.reserve(used_eptr + eptr_pre[Gc] > a_eptr.cap ? est(used_eptr, eptr_pre[Gc]) : 0,
                                    used_eptr));
            DGNN_TRY(upload_small(c, d_plan, h_plan, sizeof(int64_t) * plan_n));
            CompactPlan p{};
            p.G = Gc;
            p.H = H;
            p.cap_n = cap_n;
            p.node_pre = d_plan;
            p.edge_pre = p.node_pre + (Gc + 1);
            p.eptr_pre = p.edge_pre + (Gc + 1);
            p.edges_before = p.eptr_pre + (Gc + 1);
            p.hop_fr_off = g.hop_fr_off;
            p.hop_cbase = g.hop_cbase;
            p.hop_bound = g.hop_bound;
            p.cptr = d_cptr_list;
            p.blocks = g.blocks;
            launch(c, DGNN_K_SAMPLE_COMPACT, 8.0 * node_pre[Gc], [&] {
                const int gx = std::max(1, grid_for(c, node_pre[Gc], 256) / Gc);
                k_compact_nodes<<<dim3(gx, Gc), 256, 0, c->stream>>>(p, g.nodes, a_nodes.p + used_nodes);
            });
            DGNN_CK_LAUNCH();
            if (counts && node_pre[Gc] && !range_count) {  // one count per batch containing the node
                launch(c, DGNN_K_SAMPLE_COUNT, 0.0, [&] {
                    k_count_nodes<<<grid_for(c, node_pre[Gc], 256), 256, 0, c->stream>>>(
                        a_nodes.p + used_nodes, node_pre[Gc], counts);
                });
                DGNN_CK_LAUNCH();
            }
            for (int h = 0; h < H; ++h) {
                const int64_t Ch = h_cbs[h * (kMaxGroup + 1) + Gc];
                if (Ch == 0) continue;
                launch(c, DGNN_K_SAMPLE_COMPACT, 8.0 * Ch, [&] {
                    const int gx = std::max(1, grid_for(c, Ch, 256) / Gc);
                    k_compact_edges<<<dim3(gx, Gc), 256, 0, c->stream>>>(p, h, d_cand[h], a_edges.p + used_edges);
                });
                DGNN_CK_LAUNCH();
            }
            launch(c, DGNN_K_SAMPLE_COMPACT, 0.0, [&] {
                k_compact_eptr<<<grid_for(c, eptr_pre[Gc], 256), 256, 0, c->stream>>>(p, a_eptr.p + used_eptr);
            });
            DGNN_CK_LAUNCH();
            used_nodes += node_pre[Gc];
            used_edges += edge_pre[Gc];
            used_eptr += eptr_pre[Gc];
            t0 += Gc;
        }
        if (max_n_seen > 0) c->sample_n_hint = max_n_seen;
        if (trace) {
            const double tot = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
            t_post = tot - t_enq - t_wait;
            const double ms_sync0 = std::chrono::duration<double, std::milli>(t_synced - t_entry).count();
            const double ms_setup = std::chrono::duration<double, std::milli>(t_start - t_synced).count();
            fprintf(stderr, "[dgnn_sample] groups=%lld G=%lld first sync %.1f ms, setup %.1f ms, then total %.1f ms: "
                    "enqueue %.1f, sync-wait %.1f, post-sync host+compaction enqueue %.1f; table 2^%d (bound 2^%d), "
                    "%lld groups redone\n",
                    (long long)((nb + G - 1) / G), (long long)G, ms_sync0, ms_setup, tot, t_enq, t_wait, t_post,
                    tlog_cur, tlog_safe, (long long)redone);
        }
        S->cap_nodes = a_nodes.cap;
        S->nodes = a_nodes.release();
        S->cap_edges = a_edges.cap;
        S->src_local = a_edges.release();
        S->cap_eptr = a_eptr.cap;
        S->eptr = a_eptr.release();
        S->total_nodes = used_nodes;
        S->total_edges = used_edges;
        S->total_eptr = used_eptr;
    }
    // offset arrays (device copies of the host mirrors)
    S->node_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 1));
    S->edge_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 1));
    S->eptr_off = (int64_t*)dev_alloc(c, sizeof(int64_t) * (nb + 1));
    S->hop_off = (int32_t*)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(1, nb * (H + 2)));
    if (!S->node_off || !S->edge_off || !S->eptr_off || !S->hop_off) {
        set_error("dgnn_sample: offset allocation failed");
        return DGNN_ENOMEM;
    }
    DGNN_TRY(upload_small(c, S->node_off, S->node_off_h.data(), sizeof(int64_t) * (nb + 1)));
    DGNN_TRY(upload_small(c, S->edge_off, S->edge_off_h.data(), sizeof(int64_t) * (nb + 1)));
    DGNN_TRY(upload_small(c, S->eptr_off, S->eptr_off_h.data(), sizeof(int64_t) * (nb + 1)));
    if (nb) DGNN_TRY(upload_small(c, S->hop_off, S->hop_off_h.data(), sizeof(int32_t) * nb * (H + 2)));
    if (counts && nb && S->total_nodes && range_count) {
        // a4, range-major over the epoch (see k_cnt_ranges); DGNN_SAMPLE_COUNT=group counted per group
        const int64_t P = (N + (1 << kCntBits) - 1) >> kCntBits;
        const int64_t NS = nb * H;
        DevBuf<int32_t> bnd;
        DGNN_TRY(bnd.alloc_kept(c, (size_t)((P + 1) * NS)));
        DGNN_TRY(memset_async(c, bnd.p, 0, sizeof(int32_t) * (size_t)((P + 1) * NS)));
        CntPlan cp{S->node_off, S->hop_off, S->nodes, H, nb, P, bnd.p};
        launch(c, DGNN_K_SAMPLE_COUNT, 0.0, [&] {
            k_cnt_bounds<<<dim3(16, (unsigned)std::min<int64_t>(nb, 65535)), 256, 0, c->stream>>>(cp, counts);
        });
        DGNN_CK_LAUNCH();
        const size_t smem = sizeof(uint32_t) << kCntBits;
        DGNN_CK(cudaFuncSetAttribute(k_cnt_ranges, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = grid_resident(c, k_cnt_ranges, P, 1, 8, smem);
        launch(c, DGNN_K_SAMPLE_COUNT, 4.0 * S->total_nodes, [&] {
            k_cnt_ranges<<<grid, kCntThreads, smem, c->stream>>>(cp, counts, N);
        });
        DGNN_CK_LAUNCH();
    }
    DGNN_CK(cudaStreamSynchronize(c->stream));  // host mirrors are the copy sources
    *out = S;
    guard.s = nullptr;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_samples_get_info(const dgnn_samples* s, dgnn_samples_info* i) {
    DGNN_REQUIRE(s && i, "dgnn_samples_get_info: NULL argument");
    i->num_batches = s->nb;
    i->num_hops = s->H;
    i->batch_id_base = s->batch_id_base;
    i->total_nodes = s->total_nodes;
    i->total_edges = s->total_edges;
    i->total_eptr = s->total_eptr;
    i->node_off = s->node_off;
    i->nodes = s->nodes;
    i->hop_off = s->hop_off;
    i->eptr_off = s->eptr_off;
    i->eptr = s->eptr;
    i->edge_off = s->edge_off;
    i->src_local = s->src_local;
    i->node_off_host = s->node_off_h.data();
    i->edge_off_host = s->edge_off_h.data();
    i->eptr_off_host = s->eptr_off_h.data();
    i->hop_off_host = s->hop_off_h.data();
    i->mode = s->mode;
    return DGNN_OK;
}

extern "C" void dgnn_samples_free(dgnn_samples* s) {
    if (!s) return;
    dgnn_ctx* c = s->ctx;
    if (c) {
        cudaSetDevice(c->device);
        // the arenas go back to the ctx for the next dgnn_sample call (keep_put)
        keep_put(c, s->nodes, (size_t)s->cap_nodes * 4);
        keep_put(c, s->src_local, (size_t)s->cap_edges * 4);
        keep_put(c, s->eptr, (size_t)s->cap_eptr * 4);
        dev_free(c, s->node_off, sizeof(int64_t) * (s->nb + 1));
        dev_free(c, s->edge_off, sizeof(int64_t) * (s->nb + 1));
        dev_free(c, s->eptr_off, sizeof(int64_t) * (s->nb + 1));
        dev_free(c, s->hop_off, sizeof(int32_t) * std::max<int64_t>(1, s->nb * (s->H + 2)));
    }
    delete s;
}
