/*
 * dgnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the DiskGNN offline
 * hot path (arXiv 2405.05231), written from the paper and from the
 * readings fixed in DESIGN.md ("Readings of the paper").  It is the parity
 * oracle for the CUDA path in paper_2405_05231_b200/csrc and shares NO code,
 * header, table or helper with it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *
 * Every step is written in the order the method states it; library
 * primitives used: qsort (sorting), bsearch (set membership), memcpy (row copy).
 *
 * Pinning (tests/test_oracle_*.py): Philox against Random123 known-answer
 * vectors and against curand_Philox4x32_10 compiled on the host; Floyd by
 * exhaustive enumeration of draw tuples; the sampler by the paper's Fig. 1
 * worked example, full-fanout == BFS ball, star graph
 * (S:58), fanout [0]; counts by S:128/S:129; tier selection by Fig. 3
 * and by the tie-break-free optimality statement of P:226; pack and
 * assemble by row identity with the closed-form feature generator.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ERANGE 2
#define OR_ENOMEM 3

#define TIER_GPU 0u
#define TIER_HOST 1u
#define TIER_DISK 2u
#define TIER_SHIFT 30
#define SLOT_MASK ((1u << TIER_SHIFT) - 1u)

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  DESIGN.md reading c5. */
/* ------------------------------------------------------------------------ */
static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* One 64-bit draw keyed by (rng_seed, node v, batch bid, hop h, slot s).
 * Counter packing = DESIGN.md reading c5/c8: ctr = {v, lo32(bid), h<<16|s, hi32(bid)},
 * key = {lo32(seed), hi32(seed)}, result = out.y << 32 | out.x. */
uint64_t oracle_draw64(uint64_t rng_seed, uint32_t v, uint64_t bid, uint32_t h, uint32_t s)
{
    uint32_t ctr[4] = {v, (uint32_t)bid, (h << 16) | (s & 0xFFFFu), (uint32_t)(bid >> 32)};
    uint32_t key[2] = {(uint32_t)rng_seed, (uint32_t)(rng_seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return ((uint64_t)out[1] << 32) | (uint64_t)out[0];
}

/* Uniform integer in [0, n) from a 64-bit draw: floor(x * n / 2^64) (reading c6). */
static uint64_t mulhi64(uint64_t x, uint64_t n)
{
    return (uint64_t)(((unsigned __int128)x * (unsigned __int128)n) >> 64);
}

static int cmp_i64(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

static int cmp_i32(const void* a, const void* b)
{
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* Floyd's algorithm (Bentley & Floyd, CACM 30(9) 1987): a uniform k-subset of
 * [0, d) from exactly k draws, then sorted ascending (readings c2, c7).
 *   for s = 0..k-1: i = d-k+s; t = draw_s in [0, i]; S += (t in S) ? i : t
 * oracle_floyd_core takes the k draws t[s] (each already in [0, d-k+s]). */
void oracle_floyd_core(int64_t d, int32_t k, const int64_t* t, int64_t* out)
{
    for (int32_t s = 0; s < k; ++s) {
        int64_t i = d - k + s;
        int present = 0;
        for (int32_t r = 0; r < s; ++r)
            if (out[r] == t[s]) { present = 1; break; }
        out[s] = present ? i : t[s];
    }
    qsort(out, (size_t)k, sizeof(int64_t), cmp_i64);
}

void oracle_floyd(int64_t d, int32_t k, uint64_t rng_seed, uint32_t v, uint64_t bid,
                  uint32_t h, int64_t* out)
{
    int64_t* t = (int64_t*)malloc((size_t)(k > 0 ? k : 1) * sizeof(int64_t));
    for (int32_t s = 0; s < k; ++s) {
        int64_t i = d - k + s;
        t[s] = (int64_t)mulhi64(oracle_draw64(rng_seed, v, bid, h, (uint32_t)s), (uint64_t)(i + 1));
    }
    oracle_floyd_core(d, k, t, out);
    free(t);
}

/* ------------------------------------------------------------------------ */
/* One graph sample (P:205 node-wise sampling).           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t status;
    int32_t num_hops;
    int64_t num_nodes;   /* n_i                                             */
    int32_t* nodes;      /* [n_i] global IDs: seeds, then per hop new ascending (c10) */
    int32_t* hop_off;    /* [H+2] local boundaries: 0, |seeds|, ..., n_i      */
    int64_t num_edges;
    int32_t* eptr;       /* [hop_off[H]+1] edges of frontier node j: eptr[j]..eptr[j+1] */
    int32_t* src_local;  /* [num_edges] local index of the sampled neighbour (c11) */
} oracle_batch;

typedef struct { int32_t id; int32_t local; } id_local;

static int cmp_id_local(const void* a, const void* b)
{
    int32_t x = ((const id_local*)a)->id, y = ((const id_local*)b)->id;
    return (x > y) - (x < y);
}

static int cmp_id_only(const void* key, const void* elem)
{
    int32_t x = *(const int32_t*)key, y = ((const id_local*)elem)->id;
    return (x > y) - (x < y);
}

void oracle_batch_free(oracle_batch* b)
{
    if (!b) return;
    free(b->nodes); free(b->hop_off); free(b->eptr); free(b->src_local);
    free(b);
}

/* Sample batch `bid` with seeds seeds[0..ns).  Oracle algorithm steps 2-3
 * of DESIGN.md: the frontier at hop h is the set of nodes first discovered
 * at hop h-1 (reading c4, following Fig. 1 P:205 where v0 does not resample).
 * blocks != 0: the DGL-block variant ("the
 * multi-layer GNN computation ... the neighbors of each node", reading c27):
 * the frontier at hop h is EVERY node of the sample so far (local [0,
 * hop_off[h+1])), so every destination node of a layer resamples; eptr then
 * holds one array of hop_off[h+1] + 1 entries per hop, concatenated. */
oracle_batch* oracle_sample_batch(const int64_t* indptr, const int32_t* indices, int64_t num_nodes,
                                  const int32_t* seeds, int64_t ns, const int32_t* fanout,
                                  int32_t num_hops, uint64_t rng_seed, uint64_t bid, int32_t blocks)
{
    oracle_batch* B = (oracle_batch*)calloc(1, sizeof(oracle_batch));
    if (!B) return NULL;
    B->num_hops = num_hops;
    B->hop_off = (int32_t*)calloc((size_t)num_hops + 2, sizeof(int32_t));

    /* capacity for nodes: grows as needed */
    int64_t cap_nodes = ns > 0 ? ns : 1;
    B->nodes = (int32_t*)malloc((size_t)cap_nodes * sizeof(int32_t));
    int64_t cap_edges = 16;
    B->src_local = (int32_t*)malloc((size_t)cap_edges * sizeof(int32_t));
    if (!B->hop_off || !B->nodes || !B->src_local) { B->status = OR_ENOMEM; return B; }

    /* step 2: nodes = seeds (in input order); seeds must be valid and distinct (c12) */
    for (int64_t i = 0; i < ns; ++i) {
        if (seeds[i] < 0 || (int64_t)seeds[i] >= num_nodes) { B->status = OR_EINVAL; return B; }
        B->nodes[i] = seeds[i];
    }
    {
        int32_t* tmp = (int32_t*)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int32_t));
        memcpy(tmp, seeds, (size_t)ns * sizeof(int32_t));
        qsort(tmp, (size_t)ns, sizeof(int32_t), cmp_i32);
        for (int64_t i = 1; i < ns; ++i)
            if (tmp[i] == tmp[i - 1]) { free(tmp); B->status = OR_EINVAL; return B; }
        free(tmp);
    }
    int64_t n = ns;
    B->hop_off[0] = 0;
    B->hop_off[1] = (int32_t)ns;

    /* node-wise: eptr is indexed by frontier local index; every node with local
     * index < hop_off[H] is a frontier node of exactly one hop.
     * blocks: hop h's array starts at eptr_base = sum over i < h of (hop_off[i+1] + 1). */
    int64_t cap_eptr = ns + 1;
    B->eptr = (int32_t*)malloc((size_t)cap_eptr * sizeof(int32_t));
    B->eptr[0] = 0;
    int64_t ne = 0;
    int64_t eptr_base = 0;

    int64_t lo = 0, hi = ns; /* frontier = local [lo, hi) */
    for (int32_t h = 0; h < num_hops; ++h) {
        int32_t k = fanout[h];
        /* eptr must cover frontier nodes lo..hi-1 */
        int64_t need = blocks ? eptr_base + hi + 1 : hi + 1;
        if (need > cap_eptr) {
            cap_eptr = need;
            B->eptr = (int32_t*)realloc(B->eptr, (size_t)cap_eptr * sizeof(int32_t));
        }
        int32_t* ep = blocks ? B->eptr + eptr_base : B->eptr;  /* ep[j] .. ep[j+1]: node j's edges */
        if (blocks) ep[0] = (int32_t)ne;
        int64_t cand_begin = ne;
        /* step 3: per frontier node, ascending local j */
        for (int64_t j = lo; j < hi; ++j) {
            int32_t v = B->nodes[j];
            int64_t start = indptr[v];
            int64_t d = indptr[(int64_t)v + 1] - start;
            int64_t take = (k >= d) ? d : k;
            if (ne + take > cap_edges) {
                while (ne + take > cap_edges) cap_edges *= 2;
                B->src_local = (int32_t*)realloc(B->src_local, (size_t)cap_edges * sizeof(int32_t));
            }
            if (k >= d) {
                for (int64_t p = 0; p < d; ++p) B->src_local[ne++] = indices[start + p]; /* c3: all positions */
            } else {
                int64_t* P = (int64_t*)malloc((size_t)k * sizeof(int64_t));
                oracle_floyd(d, k, rng_seed, (uint32_t)v, bid, (uint32_t)h, P);
                for (int32_t s = 0; s < k; ++s) B->src_local[ne++] = indices[start + P[s]];
                free(P);
            }
            ep[j + 1] = (int32_t)ne;
        }
        if (blocks) eptr_base += hi + 1;
        /* new = sorted(set(candidates) - set(nodes)) ascending global ID (c10) */
        int64_t nc = ne - cand_begin;
        int32_t* cs = (int32_t*)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(int32_t));
        memcpy(cs, B->src_local + cand_begin, (size_t)nc * sizeof(int32_t));
        qsort(cs, (size_t)nc, sizeof(int32_t), cmp_i32);
        id_local* known = (id_local*)malloc((size_t)(n > 0 ? n : 1) * sizeof(id_local));
        for (int64_t i = 0; i < n; ++i) { known[i].id = B->nodes[i]; known[i].local = (int32_t)i; }
        qsort(known, (size_t)n, sizeof(id_local), cmp_id_local);
        int64_t nnew = 0;
        for (int64_t i = 0; i < nc; ++i) {
            if (i > 0 && cs[i] == cs[i - 1]) continue;
            if (bsearch(&cs[i], known, (size_t)n, sizeof(id_local), cmp_id_only)) continue;
            cs[nnew++] = cs[i]; /* compaction in place keeps ascending order */
        }
        free(known);
        if (n + nnew > cap_nodes) {
            cap_nodes = n + nnew;
            B->nodes = (int32_t*)realloc(B->nodes, (size_t)cap_nodes * sizeof(int32_t));
        }
        memcpy(B->nodes + n, cs, (size_t)nnew * sizeof(int32_t));
        free(cs);
        int64_t n_before = n;
        n += nnew;
        B->hop_off[h + 2] = (int32_t)n;

        /* remap this hop's candidates to local indices: local[u] = index in nodes */
        id_local* all = (id_local*)malloc((size_t)(n > 0 ? n : 1) * sizeof(id_local));
        for (int64_t i = 0; i < n; ++i) { all[i].id = B->nodes[i]; all[i].local = (int32_t)i; }
        qsort(all, (size_t)n, sizeof(id_local), cmp_id_local);
        for (int64_t e = cand_begin; e < ne; ++e) {
            id_local* hit = (id_local*)bsearch(&B->src_local[e], all, (size_t)n, sizeof(id_local), cmp_id_only);
            if (!hit) { free(all); B->status = OR_ERANGE; return B; }
            B->src_local[e] = hit->local;
        }
        free(all);
        lo = blocks ? 0 : n_before;
        hi = n;
    }
    B->num_nodes = n;
    B->num_edges = ne;
    return B;
}

/* Partition seeds in order into ceil(S/B) batches (reading c24) and
 * sample batches t in [t_lo, t_hi); out[t - t_lo] receives each sample. */
int oracle_sample_range(const int64_t* indptr, const int32_t* indices, int64_t num_nodes,
                        const int32_t* seeds, int64_t num_seeds, int32_t batch_size,
                        int64_t batch_id_base, const int32_t* fanout, int32_t num_hops,
                        uint64_t rng_seed, int64_t t_lo, int64_t t_hi, int32_t threads,
                        oracle_batch** out, int32_t blocks)
{
    if (batch_size <= 0 || num_hops < 1) return OR_EINVAL;
    (void)threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int64_t t = t_lo; t < t_hi; ++t) {
        int64_t a = t * batch_size;
        int64_t b = a + batch_size < num_seeds ? a + batch_size : num_seeds;
        out[t - t_lo] = oracle_sample_batch(indptr, indices, num_nodes, seeds + a, b - a, fanout,
                                            num_hops, rng_seed, (uint64_t)(batch_id_base + t), blocks);
    }
    for (int64_t t = t_lo; t < t_hi; ++t) {
        if (!out[t - t_lo]) return OR_ENOMEM;
        if (out[t - t_lo]->status) return out[t - t_lo]->status;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Access frequency: counts[v] = #batches whose node set contains v          */
/* ("keeps a counter for each node and streams the graph samples";    */
/*  S:125; reading c14).                                                     */
/* ------------------------------------------------------------------------ */
void oracle_count_add(const int32_t* nodes, int64_t n, uint32_t* counts)
{
    for (int64_t i = 0; i < n; ++i) counts[nodes[i]] += 1u;
}

/* ------------------------------------------------------------------------ */
/* Tier selection ("rank the nodes by their access frequencies and     */
/* cache more popular nodes in faster memory"; P:275-277 GPU cache = most    */
/* popular, CPU cache = second most popular; readings c15-c17).             */
/* ------------------------------------------------------------------------ */
typedef struct { uint32_t count; int32_t id; } count_id;

static int cmp_rank(const void* a, const void* b)
{
    const count_id* x = (const count_id*)a;
    const count_id* y = (const count_id*)b;
    if (x->count != y->count) return x->count > y->count ? -1 : 1; /* count descending */
    return (x->id > y->id) - (x->id < y->id);                      /* then ID ascending */
}

int oracle_select_tiers(const uint32_t* counts, int64_t num_nodes, int64_t gpu_rows, int64_t host_rows,
                        uint32_t* tier_map, int32_t* gpu_ids, int32_t* host_ids,
                        int64_t* k_gpu, int64_t* k_host)
{
    if (num_nodes >= ((int64_t)1 << TIER_SHIFT) || gpu_rows < 0 || host_rows < 0) return OR_EINVAL;
    int64_t nnz = 0;
    for (int64_t v = 0; v < num_nodes; ++v) nnz += counts[v] > 0;
    count_id* order = (count_id*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(count_id));
    if (!order) return OR_ENOMEM;
    int64_t m = 0;
    for (int64_t v = 0; v < num_nodes; ++v)
        if (counts[v] > 0) { order[m].count = counts[v]; order[m].id = (int32_t)v; ++m; }
    qsort(order, (size_t)nnz, sizeof(count_id), cmp_rank);
    int64_t kg = gpu_rows < nnz ? gpu_rows : nnz;
    int64_t kh = host_rows < nnz - kg ? host_rows : nnz - kg;
    for (int64_t i = 0; i < kg; ++i) gpu_ids[i] = order[i].id;
    for (int64_t i = 0; i < kh; ++i) host_ids[i] = order[kg + i].id;
    free(order);
    /* slots: position in the tier's ascending-ID list (c17) */
    qsort(gpu_ids, (size_t)kg, sizeof(int32_t), cmp_i32);
    qsort(host_ids, (size_t)kh, sizeof(int32_t), cmp_i32);
    for (int64_t v = 0; v < num_nodes; ++v) tier_map[v] = TIER_DISK << TIER_SHIFT;
    for (int64_t s = 0; s < kg; ++s) tier_map[gpu_ids[s]] = (TIER_GPU << TIER_SHIFT) | (uint32_t)s;
    for (int64_t s = 0; s < kh; ++s) tier_map[host_ids[s]] = (TIER_HOST << TIER_SHIFT) | (uint32_t)s;
    *k_gpu = kg;
    *k_host = kh;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Address table of one batch ("interpreted address tables"):  */
/* addr[j] = tier<<30 | slot; DISK slot = rank among the batch's DISK nodes  */
/* in local order; P = the DISK nodes in local order (reading c21).          */
/* Returns |P|.                                                              */
/* ------------------------------------------------------------------------ */
int64_t oracle_classify(const int32_t* nodes, int64_t n, const uint32_t* tier_map,
                        uint32_t* addr, int32_t* packed)
{
    int64_t p = 0;
    for (int64_t j = 0; j < n; ++j) {
        uint32_t t = tier_map[nodes[j]];
        if ((t >> TIER_SHIFT) == TIER_DISK) {
            addr[j] = (TIER_DISK << TIER_SHIFT) | (uint32_t)p;
            packed[p++] = nodes[j];
        } else {
            addr[j] = t;
        }
    }
    return p;
}

/* ------------------------------------------------------------------------ */
/* Batched packing of one packing group ("collect all node features   */
/* it requires and store them contiguously"): chunk i starts at   */
/* chunk_off[i], chunk_off[i+1] = roundup(chunk_off[i] + |P_i|*row_bytes,    */
/* 4096) (reading c20); padding bytes are zero.                             */
/* ------------------------------------------------------------------------ */
void oracle_chunk_offsets(const int64_t* packed_rows, int64_t nb, int64_t row_bytes, int64_t* chunk_off)
{
    chunk_off[0] = 0;
    for (int64_t i = 0; i < nb; ++i) {
        int64_t end = chunk_off[i] + packed_rows[i] * row_bytes;
        chunk_off[i + 1] = (end + 4095) / 4096 * 4096;
    }
}

void oracle_pack(const uint8_t* features, int64_t row_bytes, const int32_t* packed_concat,
                 const int64_t* packed_rows, int64_t nb, const int64_t* chunk_off, uint8_t* group_buf)
{
    memset(group_buf, 0, (size_t)chunk_off[nb]);
    int64_t r0 = 0;
    for (int64_t i = 0; i < nb; ++i) {
        for (int64_t r = 0; r < packed_rows[i]; ++r)
            memcpy(group_buf + chunk_off[i] + r * row_bytes,
                   features + (int64_t)packed_concat[r0 + r] * row_bytes, (size_t)row_bytes);
        r0 += packed_rows[i];
    }
}

/* out[s] = features[ids[s]] (tier buffers as "special mini-batches", P:443;
 * direct-gather assembly out[j] = features[nodes[j]]). */
void oracle_gather_rows(const uint8_t* features, int64_t row_bytes, const int32_t* ids, int64_t n,
                        uint8_t* out)
{
    for (int64_t s = 0; s < n; ++s)
        memcpy(out + s * row_bytes, features + (int64_t)ids[s] * row_bytes, (size_t)row_bytes);
}

/* Three-source reconstruction (Fig. 3): the GPU reads the GPU
 * cache, the CPU cache and the partial input (this batch's chunk). */
int oracle_assemble_tiers(const uint32_t* addr, int64_t n, const uint8_t* gpu_buf, int64_t k_gpu,
                          const uint8_t* host_buf, int64_t k_host, const uint8_t* chunk, int64_t chunk_rows,
                          int64_t row_bytes, uint8_t* out)
{
    for (int64_t j = 0; j < n; ++j) {
        uint32_t t = addr[j] >> TIER_SHIFT, s = addr[j] & SLOT_MASK;
        const uint8_t* src;
        if (t == TIER_GPU && s < k_gpu) src = gpu_buf + (int64_t)s * row_bytes;
        else if (t == TIER_HOST && s < k_host) src = host_buf + (int64_t)s * row_bytes;
        else if (t == TIER_DISK && s < chunk_rows) src = chunk + (int64_t)s * row_bytes;
        else return OR_ERANGE; /* unresolvable address */
        memcpy(out + j * row_bytes, src, (size_t)row_bytes);
    }
    return OR_OK;
}

/* ======================================================================== */
/* Segmented disk cache (Sec. 5.1).          */
/*                                                                          */
/* Input: the packed lists P_b of an epoch (the DISK-tier nodes of each      */
/* batch in local order, as oracle_classify returns them, concatenated with  */
/* offsets packed_off[nb+1]).  Readings (DESIGN.md d1-d8):                   */
/*  d1 segments = consecutive batches [g*s, min((g+1)*s, nb)).   */
/*  d2 local frequency of v in segment g = number of the segment's batches   */
/*     whose P_b holds v; > m -> disk cache V_d of g, <= m -> stays packed    */
/*     in every P_b that holds it.  m = 0 is allowed (pure cache).    */
/*  d3 space (Eq. 2) in 4096-byte pages: per segment              */
/*     ceil(|V_d| / fpp) with fpp = floor(4096 / row_bytes) rows per page    */
/*     (a cached row never straddles a page), per batch ceil(|P_b'| *        */
/*     row_bytes / 4096) (the chunk of reading c20).  Constraint: <= budget.  */
/*  d4 heuristic: m = 1 (caller's choice), s = the minimum s in   */
/*     1..nb with space <= budget, by linear scan.                           */
/*  d5 Permute (Alg. 1 line 3): H_t(i) for local batch index i of segment g   */
/*     = rank of i when the segment's indices are ordered by (x_t(i), i),     */
/*     x_t(i) = Philox4x32-10(ctr = {i, g, t, 0x4D48}, key = seed) as         */
/*     out.y << 32 | out.x.                                                  */
/*  d6 signature (Alg. 1 lines 4-8) read per hash function: S_t(v) =          */
/*     min over the segment's batches i holding v of H_t(i) (the MinHash      */
/*     signature of HashOrder); V_r = V_d sorted by (S_0..S_{k-1}, v)         */
/*     lexicographically (line 9).  For k = 1 this is Algorithm 1 verbatim.  */
/*     reorder = 0 gives the identity order (ascending v) for comparison;    */
/*     reorder = 2 is line 8 verbatim for any k: the scalar S(v) = min over   */
/*     t of S_t(v), V_r sorted by (S(v), v).                          */
/*  d7 I/O (Eq. 2 objective): per batch ceil(|P_b'| * row_bytes / 4096)      */
/*     chunk pages + the number of distinct cache pages holding D_b          */
/*     (requests to one page merged).                                 */
/*  d8 disk address of the r-th packed row of batch b (local DISK order):     */
/*     cached -> 1 << 31 | (q * fpp + slot), q = index of its page in the     */
/*     batch's ascending request list, slot = position inside the page;      */
/*     packed -> rank of the row in P_b'.                                    */
/* ======================================================================== */
#define DC_PAGE 4096

static int64_t dc_chunk_pages(int64_t rows, int64_t row_bytes)
{
    return (rows * row_bytes + DC_PAGE - 1) / DC_PAGE;
}

/* Eq. 2 space of configuration (s, m), in pages (d1-d3). */
int oracle_disk_space(const int32_t* packed_ids, const int64_t* packed_off, int64_t nb, int64_t num_nodes,
                      int64_t row_bytes, int64_t s, int64_t m, int64_t* pages_out)
{
    if (s < 1 || m < 0 || row_bytes < 1 || row_bytes > DC_PAGE) return OR_EINVAL;
    int64_t fpp = DC_PAGE / row_bytes;
    uint32_t* cnt = (uint32_t*)calloc((size_t)(num_nodes > 0 ? num_nodes : 1), sizeof(uint32_t));
    if (!cnt) return OR_ENOMEM;
    int64_t total = 0;
    for (int64_t g0 = 0; g0 < nb; g0 += s) {
        int64_t g1 = g0 + s < nb ? g0 + s : nb;
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) cnt[packed_ids[r]] += 1;
        for (int64_t b = g0; b < g1; ++b) {
            int64_t kept = 0;
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r)
                if (cnt[packed_ids[r]] <= (uint64_t)m) kept += 1;
            total += dc_chunk_pages(kept, row_bytes);
        }
        int64_t cached = 0;
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r)
                if (cnt[packed_ids[r]] > (uint64_t)m) { cached += 1; cnt[packed_ids[r]] = 0; }
        total += (cached + fpp - 1) / fpp;
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) cnt[packed_ids[r]] = 0;
    }
    free(cnt);
    *pages_out = total;
    return OR_OK;
}

/* Heuristic search (d4): s_out = minimum feasible s, or 0 when even s = nb
 * exceeds the budget; pages_out = the space of s_out (of s = nb if infeasible). */
int oracle_disk_search(const int32_t* packed_ids, const int64_t* packed_off, int64_t nb, int64_t num_nodes,
                       int64_t row_bytes, int64_t m, int64_t budget_pages, int64_t* s_out, int64_t* pages_out)
{
    int64_t sp = 0;
    int64_t s_max = nb > 0 ? nb : 1;
    for (int64_t s = 1; s <= s_max; ++s) {
        int rc = oracle_disk_space(packed_ids, packed_off, nb, num_nodes, row_bytes, s, m, &sp);
        if (rc) return rc;
        if (sp <= budget_pages) { *s_out = s; *pages_out = sp; return OR_OK; }
    }
    *s_out = 0;
    *pages_out = sp;
    return OR_OK;
}

/* d5: one permutation H of the n local batch indices of segment g. */
typedef struct { uint64_t x; int64_t i; } dc_key;

static int cmp_dc_key(const void* a, const void* b)
{
    const dc_key* p = (const dc_key*)a;
    const dc_key* q = (const dc_key*)b;
    if (p->x != q->x) return p->x < q->x ? -1 : 1;
    return (p->i > q->i) - (p->i < q->i);
}

int oracle_disk_perm(uint64_t seed, int64_t g, int64_t t, int64_t n, int64_t* H)
{
    dc_key* keys = (dc_key*)malloc((size_t)(n > 0 ? n : 1) * sizeof(dc_key));
    if (!keys) return OR_ENOMEM;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t i = 0; i < n; ++i) {
        uint32_t ctr[4] = {(uint32_t)i, (uint32_t)g, (uint32_t)t, 0x4D48u};
        uint32_t out[4];
        oracle_philox4x32_10(ctr, key, out);
        keys[i].x = ((uint64_t)out[1] << 32) | out[0];
        keys[i].i = i;
    }
    qsort(keys, (size_t)n, sizeof(dc_key), cmp_dc_key);
    for (int64_t p = 0; p < n; ++p) H[keys[p].i] = p;
    free(keys);
    return OR_OK;
}

/* cache entry of one segment for the Line-9 sort */
typedef struct { int32_t v; int32_t k; const int64_t* sig; } dc_entry;

static int cmp_dc_entry(const void* a, const void* b)
{
    const dc_entry* p = (const dc_entry*)a;
    const dc_entry* q = (const dc_entry*)b;
    for (int32_t t = 0; t < p->k; ++t)
        if (p->sig[t] != q->sig[t]) return p->sig[t] < q->sig[t] ? -1 : 1;
    return (p->v > q->v) - (p->v < q->v);
}

static int cmp_i64_asc(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Full plan for (s, m) (d1-d8).  Output capacities: R = packed_off[nb] rows.
 *   seg_off[nseg+1]       prefix of |V_d| per segment; cache_ids[R]: V_r of every
 *                         segment, concatenated (segment g at seg_off[g]).
 *   seg_page_off[nseg+1]  prefix of cache pages per segment.
 *   pk_ids[R], pk_off[nb+1]       the reduced packed lists P_b'.
 *   req_pages[R], req_off[nb+1]   per batch, the ascending distinct global cache
 *                                 pages (seg_page_off[g] + page in segment).
 *   dc_addr[R]                     d8, one per packed row of the input.
 *   totals[4] = {space pages, io pages, cache pages, chunk pages}. */
int oracle_disk_plan(const int32_t* packed_ids, const int64_t* packed_off, int64_t nb, int64_t num_nodes,
                     int64_t row_bytes, int64_t s, int64_t m, int32_t k, uint64_t seed, int32_t reorder,
                     int64_t* seg_off, int32_t* cache_ids, int64_t* seg_page_off, int32_t* pk_ids, int64_t* pk_off,
                     int64_t* req_pages, int64_t* req_off, uint32_t* dc_addr, int64_t* totals)
{
    if (s < 1 || m < 0 || k < 1 || row_bytes < 1 || row_bytes > DC_PAGE) return OR_EINVAL;
    int64_t fpp = DC_PAGE / row_bytes;
    int64_t N = num_nodes > 0 ? num_nodes : 1;
    uint32_t* cnt = (uint32_t*)calloc((size_t)N, sizeof(uint32_t));
    int64_t* ent = (int64_t*)malloc((size_t)N * sizeof(int64_t));  /* v -> entry index, -1 if none */
    int64_t R = packed_off[nb];
    int64_t cap = R > 0 ? R : 1;
    dc_entry* es = (dc_entry*)malloc((size_t)cap * sizeof(dc_entry));
    int64_t* sig = (int64_t*)malloc((size_t)cap * (size_t)k * sizeof(int64_t));
    int64_t* rank = (int64_t*)malloc((size_t)cap * sizeof(int64_t));  /* entry (by v) -> position in V_r */
    int64_t* H = (int64_t*)malloc((size_t)(s > 0 ? s : 1) * (size_t)k * sizeof(int64_t));
    int64_t* pages = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    if (!cnt || !ent || !es || !sig || !rank || !H || !pages) {
        free(cnt); free(ent); free(es); free(sig); free(rank); free(H); free(pages);
        return OR_ENOMEM;
    }
    for (int64_t v = 0; v < N; ++v) ent[v] = -1;
    int64_t nseg = (nb + s - 1) / s;
    int64_t n_cache = 0, n_pk = 0, n_req = 0, cache_pages = 0, chunk_pages = 0, io = 0;
    seg_off[0] = 0;
    seg_page_off[0] = 0;
    pk_off[0] = 0;
    req_off[0] = 0;
    for (int64_t g = 0; g < nseg; ++g) {
        int64_t g0 = g * s, g1 = g0 + s < nb ? g0 + s : nb, sg = g1 - g0;
        /* d2: local frequencies */
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) cnt[packed_ids[r]] += 1;
        /* V_d of the segment, first-seen order (re-sorted below) */
        int64_t e0 = n_cache, ne = 0;
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
                int32_t v = packed_ids[r];
                if (cnt[v] > (uint64_t)m && ent[v] < 0) {
                    ent[v] = ne;
                    es[ne].v = v;
                    es[ne].k = k;
                    es[ne].sig = sig + ne * k;
                    for (int32_t t = 0; t < k; ++t) sig[ne * k + t] = INT64_MAX;  /* Alg. 1 line 1: inf */
                    ne += 1;
                }
            }
        /* Alg. 1 lines 2-3: k permutations of the local batch indices (d5) */
        for (int32_t t = 0; t < k; ++t) {
            int rc = oracle_disk_perm(seed, g, t, sg, H + (int64_t)t * sg);
            if (rc) { free(cnt); free(ent); free(es); free(sig); free(rank); free(H); free(pages); return rc; }
        }
        /* Alg. 1 lines 4-8 (d6) */
        for (int64_t i = 0; i < sg; ++i) {
            int64_t b = g0 + i;
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
                int64_t e = ent[packed_ids[r]];
                if (e < 0) continue;  /* line 5: V_i intersect V_d */
                for (int32_t t = 0; t < k; ++t)
                    if (H[(int64_t)t * sg + i] < sig[e * k + t]) sig[e * k + t] = H[(int64_t)t * sg + i];
            }
        }
        /* line 8 read literally (reorder = 2, P:368 / P:377: "the MinHash value is the minimum
           over the outputs of the k hash functions"): one scalar S(v) = min_t S_t(v) */
        if (reorder == 2)
            for (int64_t e = 0; e < ne; ++e) {
                int64_t mn = INT64_MAX;
                for (int32_t t = 0; t < k; ++t) mn = es[e].sig[t] < mn ? es[e].sig[t] : mn;
                sig[e * k] = mn;  /* es[e].sig == sig + e * k before the sort */
                es[e].k = 1;
            }
        /* line 9: V_r = V_d[Sort(S)] */
        if (reorder) {
            qsort(es, (size_t)ne, sizeof(dc_entry), cmp_dc_entry);
        } else {
            for (int64_t e = 0; e < ne; ++e) es[e].k = 0;  /* compare by v only */
            qsort(es, (size_t)ne, sizeof(dc_entry), cmp_dc_entry);
        }
        for (int64_t p = 0; p < ne; ++p) {
            cache_ids[e0 + p] = es[p].v;
            rank[ent[es[p].v]] = p;
        }
        n_cache += ne;
        seg_off[g + 1] = n_cache;
        int64_t segp = (ne + fpp - 1) / fpp;
        seg_page_off[g + 1] = seg_page_off[g] + segp;
        cache_pages += segp;
        /* per batch: P_b', merged page requests, disk addresses (d7, d8) */
        for (int64_t b = g0; b < g1; ++b) {
            int64_t kept = 0, np = 0;
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
                int32_t v = packed_ids[r];
                if (ent[v] >= 0) pages[np++] = seg_page_off[g] + rank[ent[v]] / fpp;
                else { pk_ids[n_pk + kept] = v; dc_addr[r] = (uint32_t)kept; kept += 1; }
            }
            qsort(pages, (size_t)np, sizeof(int64_t), cmp_i64_asc);
            int64_t nu = 0;
            for (int64_t q = 0; q < np; ++q)
                if (nu == 0 || pages[q] != req_pages[n_req + nu - 1]) { req_pages[n_req + nu] = pages[q]; nu += 1; }
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
                int32_t v = packed_ids[r];
                if (ent[v] < 0) continue;
                int64_t pos = rank[ent[v]];
                int64_t pg = seg_page_off[g] + pos / fpp;
                int64_t q = 0;
                while (req_pages[n_req + q] != pg) q += 1;
                dc_addr[r] = 0x80000000u | (uint32_t)(q * fpp + pos % fpp);
            }
            n_pk += kept;
            pk_off[b + 1] = n_pk;
            n_req += nu;
            req_off[b + 1] = n_req;
            chunk_pages += dc_chunk_pages(kept, row_bytes);
            io += dc_chunk_pages(kept, row_bytes) + nu;
        }
        for (int64_t b = g0; b < g1; ++b)
            for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
                cnt[packed_ids[r]] = 0;
                ent[packed_ids[r]] = -1;
            }
    }
    totals[0] = cache_pages + chunk_pages;
    totals[1] = io;
    totals[2] = cache_pages;
    totals[3] = chunk_pages;
    free(cnt); free(ent); free(es); free(sig); free(rank); free(H); free(pages);
    return OR_OK;
}

/* Materialized segment caches ("laid out on disk by reordering"): the rows of
 * V_r of segment g fill pages seg_page_off[g].. in order, fpp rows per page at
 * slot * row_bytes; the rest of every page is zero. */
void oracle_disk_cache_fill(const uint8_t* features, int64_t row_bytes, const int32_t* cache_ids,
                            const int64_t* seg_off, const int64_t* seg_page_off, int64_t nseg, uint8_t* out)
{
    int64_t fpp = DC_PAGE / row_bytes;
    memset(out, 0, (size_t)(seg_page_off[nseg] * DC_PAGE));
    for (int64_t g = 0; g < nseg; ++g)
        for (int64_t p = 0; p < seg_off[g + 1] - seg_off[g]; ++p)
            memcpy(out + (seg_page_off[g] + p / fpp) * DC_PAGE + (p % fpp) * row_bytes,
                   features + (int64_t)cache_ids[seg_off[g] + p] * row_bytes, (size_t)row_bytes);
}

/* ======================================================================== */
/* Trainer stub: the surrogate of Eq. 1  */
/* that SPEC S:409-413 fixes -- h^k_v = h^{k-1}_v + mean{h^{k-1}_u : u in   */
/* N(v)}, no W^k, no sigma.  Reading t1: layer k = 1..H runs    */
/* over sampling hop h = H - k (deepest first); N(v) = v's sampled          */
/* neighbours at the hop v expanded in; a node of hop h without edges, and  */
/* every node outside hop h, keeps h^{k-1}.  fp32 throughout: the sum starts */
/* at 0 and adds the neighbours in edge order, then one division by the     */
/* edge count and one addition.  x: the batch's assembled rows [n][dim],    */
/* updated in place; the seeds' embeddings are rows [0, hop_off[1]).         */
/* ======================================================================== */
int oracle_train_stub(float* x, int64_t n, int64_t dim, const int32_t* hop_off, int32_t H, const int32_t* eptr,
                      const int32_t* src_local, int32_t blocks)
{
    float* prev = (float*)malloc((size_t)(n > 0 ? n : 1) * (size_t)dim * sizeof(float));
    if (!prev) return OR_ENOMEM;
    for (int32_t k = 1; k <= H; ++k) {
        int32_t h = H - k;
        memcpy(prev, x, (size_t)n * (size_t)dim * sizeof(float));  /* h^{k-1} */
        /* layer k's destination nodes: hop h's frontier (node-wise: the nodes discovered at
         * hop h-1; blocks: every node of the sample so far) and where their edges start */
        int64_t lo = blocks ? 0 : hop_off[h];
        const int32_t* ep = eptr;
        if (blocks) {
            int64_t base = 0;
            for (int32_t i = 0; i < h; ++i) base += hop_off[i + 1] + 1;
            ep = eptr + base;
        }
        for (int64_t j = lo; j < hop_off[h + 1]; ++j) {
            int32_t e0 = ep[j], e1 = ep[j + 1];
            if (e1 == e0) continue;
            for (int64_t d = 0; d < dim; ++d) {
                float s = 0.0f;
                for (int32_t e = e0; e < e1; ++e) s += prev[(int64_t)src_local[e] * dim + d];
                x[j * dim + d] = prev[j * dim + d] + s / (float)(e1 - e0);
            }
        }
    }
    free(prev);
    return OR_OK;
}

/* ======================================================================== */
/* Sec. 5.2 source-page accounting (Fig. 6). */
/* The feature file holds row v at byte v * row_bytes, read in 4096-byte    */
/* pages.  Individual packing fetches every needed row on its own, batch by */
/* batch: the pages the row spans, re-read for every batch that needs it.   */
/* Batched packing reads each partition of part_rows consecutive rows that  */
/* holds at least one needed row exactly once, whole (part_rows * row_bytes */
/* is a multiple of 4096: partitions never split a page).                  */
/* ======================================================================== */
int oracle_pack_pages(const int32_t* packed_ids, const int64_t* packed_off, int64_t nb, int64_t num_nodes,
                      int64_t row_bytes, int64_t part_rows, int64_t* individual, int64_t* batched)
{
    if (row_bytes < 1 || part_rows < 1 || (part_rows * row_bytes) % DC_PAGE) return OR_EINVAL;
    int64_t ind = 0;
    int64_t nparts = (num_nodes + part_rows - 1) / part_rows;
    uint8_t* touched = (uint8_t*)calloc((size_t)(nparts > 0 ? nparts : 1), 1);
    if (!touched) return OR_ENOMEM;
    for (int64_t b = 0; b < nb; ++b)
        for (int64_t r = packed_off[b]; r < packed_off[b + 1]; ++r) {
            int64_t v = packed_ids[r];
            int64_t first = v * row_bytes / DC_PAGE, last = ((v + 1) * row_bytes - 1) / DC_PAGE;
            ind += last - first + 1;
            touched[v / part_rows] = 1;
        }
    int64_t bat = 0;
    int64_t file_pages = (num_nodes * row_bytes + DC_PAGE - 1) / DC_PAGE;
    for (int64_t p = 0; p < nparts; ++p) {
        if (!touched[p]) continue;
        int64_t p0 = p * part_rows * row_bytes / DC_PAGE;
        int64_t p1 = (p + 1) * part_rows * row_bytes / DC_PAGE;
        if (p1 > file_pages) p1 = file_pages;
        bat += p1 - p0;
    }
    free(touched);
    *individual = ind;
    *batched = bat;
    return OR_OK;
}
