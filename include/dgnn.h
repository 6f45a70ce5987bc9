/*
 * dgnn.h -- C ABI of the B200-native DiskGNN offline hot path (libdgnn.so).
 *
 * The path (DiskGNN, arXiv 2405.05231; PAPER.md cited as P:n, SPEC.md as S:n):
 *   a1-a3  dgnn_sample       offline K-hop node-wise neighbour sampling of many
 *                             mini-batches (Sec. 2; Sec. 3) with the
 *                             per-node access counter fused in (Sec. 4).
 *   a4-a5  dgnn_build_cache  popularity ranking: most popular nodes -> GPU cache, next
 *                             most popular -> CPU (host) cache.
 *   a6     dgnn_classify     per-batch "interpreted address tables" (Sec. 6) and
 *                             the list of each batch's disk-resident features.
 *   a7     dgnn_pack         batched feature packing into per-batch contiguous chunks,
 *                             and the tier buffers as "special mini-batches" (P:228-230,
 *                             P:437-443 Sec. 5.2).
 *   a8     dgnn_stage_*      moving chunks to/from the disk tier (pinned host memory or a
 *                             file) on a side stream.
 *   a9     dgnn_assemble     feature assembly from GPU cache, CPU cache (UVA) and the
 *                             staged partial input (Sec. 4, Fig. 3).
 * The exact semantics (RNG keying, node order, tie-breaks, chunk layout) are the
 * readings c1-c26 listed in DESIGN.md; the CPU oracle in oracle/ implements them
 * independently and the GPU results are required to be byte-identical to it.
 *
 * Conventions
 *  - Every call returns dgnn_status; nothing throws across the boundary.  On a non-OK
 *    status, dgnn_last_error() returns a thread-local message.
 *  - "device" pointers are CUDA device pointers of the ctx's device; "host" pointers are
 *    ordinary CPU memory; "UVA" pointers may be either device memory or pinned host
 *    memory mapped into the device address space (cudaHostAlloc / cudaHostRegister).
 *  - All work is enqueued on the ctx stream (see dgnn_ctx_create) unless stated;
 *    inputs are borrowed and must stay valid until that stream has passed the call.
 *  - Variable-size outputs (dgnn_samples, dgnn_cache_plan) are library-owned, allocated
 *    with the ctx allocator and released by *_free; they must not outlive their ctx.
 *    Fixed-size outputs are caller-allocated.
 *  - Node IDs are int32, N < 2^30 (the address encoding keeps 30 slot bits).
 *  - Feature rows are opaque bytes: row_bytes > 0 and a multiple of 4; rows are copied,
 *    never combined, so every result is bit-exact.
 */
#ifndef DGNN_H
#define DGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DGNN_OK = 0,
    DGNN_EINVAL = 1,       /* argument / precondition violation                    */
    DGNN_ERANGE = 2,       /* unresolvable node address                    */
    DGNN_ENOMEM = 3,       /* allocation failed                                           */
    DGNN_ECUDA = 4,        /* CUDA runtime error                                          */
    DGNN_ECOMM = 5,        /* collective failure (reserved for the sharded tier)          */
    DGNN_EIO = 6,          /* file staging I/O error                                      */
    DGNN_EUNSUPPORTED = 7  /* configuration outside the implemented envelope              */
} dgnn_status;

/* Address encoding (reading c18): addr = tier << 30 | slot. */
#define DGNN_TIER_GPU 0u
#define DGNN_TIER_HOST 1u
#define DGNN_TIER_DISK 2u
#define DGNN_TIER_SHIFT 30
#define DGNN_SLOT_MASK ((1u << DGNN_TIER_SHIFT) - 1u)

/* Kernel families, for dgnn_ctx_kernel_stats (per-launch CUDA-event timing). */
typedef enum {
    DGNN_K_SCAN = 0,        /* decoupled look-back prefix scan (all scans)             */
    DGNN_K_SAMPLE_SEED,     /* seed insertion / validation                             */
    DGNN_K_SAMPLE_HOP,      /* a2: Philox + Floyd draw, CSR gather, dedup insert, count */
    DGNN_K_SAMPLE_ORDER,    /* a3: bucket order of new nodes (hist, scatter, sort)      */
    DGNN_K_SAMPLE_REMAP,    /* a3: global -> local remap of sampled edges               */
    DGNN_K_SAMPLE_COMPACT,  /* a3: batch-major output compaction                        */
    DGNN_K_SAMPLE_SETUP,    /* per-hop bookkeeping (1-block kernels)                    */
    DGNN_K_CACHE_HIST,      /* a4: count histogram                                      */
    DGNN_K_CACHE_SELECT,    /* a5: tier membership + slots                              */
    DGNN_K_CLASSIFY,        /* a6: address tables + packed lists                        */
    DGNN_K_PACK,            /* a7: batched pack gather (the HBM-bound kernel)           */
    DGNN_K_GATHER,          /* a7: tier-buffer gather ("special mini-batches")          */
    DGNN_K_ASSEMBLE,        /* a9: three-source assembly                                */
    DGNN_K_MISC,            /* memsets and small helpers                                */
    DGNN_K_SORT,            /* stable LSD radix sort (disk-cache index and order)       */
    DGNN_K_DISK_PLAN,       /* segmented disk cache: groups, MinHash, pages, addresses  */
    DGNN_K_DISK_GATHER,     /* segmented disk cache: page fill, partial input           */
    DGNN_K_TRAIN,           /* trainer stub (mean aggregation per sampled hop)          */
    DGNN_K_HOST_WINDOW,     /* a9: marking a host window's distinct host-tier rows      */
    DGNN_K_HOST_GATHER,     /* a9: PCIe gather of a window's host rows into HBM staging */
    DGNN_K_GATHER_PCIE,     /* a7: tier gather from / into pinned host memory (PCIe)   */
    DGNN_K_PACK_GRAPH,      /* P:283 graph sample into / out of the chunk (pack, loader) */
    DGNN_K_SAMPLE_DEDUP,    /* a3, partitioned path: per-(batch, ID range) dedup + order */
    DGNN_K_SAMPLE_COUNT,    /* a4: access counter over a sampling group's nodes          */
    DGNN_K_NUM
} dgnn_kernel_id;

typedef struct dgnn_ctx dgnn_ctx;
typedef struct dgnn_samples dgnn_samples;
typedef struct dgnn_cache_plan dgnn_cache_plan;

/* Optional device allocator (e.g. a framework's caching allocator).  alloc must return
 * device memory usable on `stream` (a cudaStream_t) or NULL; free receives the same
 * pointer and size.  When NULL is passed to dgnn_ctx_create, cudaMallocAsync /
 * cudaFreeAsync on the ctx stream are used. */
typedef void* (*dgnn_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*dgnn_free_fn)(void* ptr, size_t bytes, void* stream, void* user);
typedef struct {
    dgnn_alloc_fn alloc;
    dgnn_free_fn free;
    void* user;
} dgnn_allocator;

/* ------------------------------------------------------------------ context ---- */
/* Create a context on CUDA device `device` enqueuing on `stream` (a cudaStream_t;
 * NULL = the legacy default stream).  A second, internal side stream carries staging
 * copies (a8).  One ctx per host thread. */
dgnn_status dgnn_ctx_create(int device, void* stream, const dgnn_allocator* allocator, dgnn_ctx** out);
void dgnn_ctx_destroy(dgnn_ctx* ctx);
dgnn_status dgnn_ctx_set_stream(dgnn_ctx* ctx, void* stream);
void* dgnn_ctx_stream(const dgnn_ctx* ctx);
void* dgnn_ctx_side_stream(const dgnn_ctx* ctx);
/* Synchronize the ctx stream and report deferred device-side errors (e.g. an
 * unresolvable address seen by dgnn_assemble -> DGNN_ERANGE). */
dgnn_status dgnn_ctx_sync(dgnn_ctx* ctx);
/* Thread-local message for the last non-OK status returned on this thread. */
const char* dgnn_last_error(void);
/* Tuning knob: batches sampled concurrently per sampling group (0 = automatic). */
dgnn_status dgnn_ctx_set_sample_group(dgnn_ctx* ctx, int32_t batches);
/* Sampling variant for later dgnn_sample calls on this ctx: DGNN_SAMPLE_NODEWISE (default;
 * reading c4: the frontier of hop h is the nodes first discovered at hop h-1) or
 * DGNN_SAMPLE_BLOCKS (the DGL-block variant, reading c27: the frontier of hop h is every node
 * of the sample so far, so each destination node of a layer resamples; eptr then holds one
 * array of hop_off[b][h+1] + 1 entries per hop h, concatenated). */
#define DGNN_SAMPLE_NODEWISE 0
#define DGNN_SAMPLE_BLOCKS 1
dgnn_status dgnn_ctx_set_sample_mode(dgnn_ctx* ctx, int32_t mode);
/* Tuning knob: resident CTAs per SM for the assemble kernels (default 8).  The assemble
 * kernel is PCIe-bound on host-tier rows; a low value leaves SMs to a concurrent offline
 * pass on another stream (epoch pipelining). */
dgnn_status dgnn_ctx_set_assemble_occupancy(dgnn_ctx* ctx, int32_t blocks_per_sm);

/* Statistics: number of kernels this ctx has launched; optional per-launch CUDA-event
 * timing on the ctx stream (enable before the region of interest). */
/* Cap every grid this ctx launches at max_blocks CTAs (0 = no cap).  For a ctx running
 * PCIe-bound UVA gathers next to latency-bound work on other streams: a few SMs' worth of
 * outstanding host reads already saturate PCIe, more only queue up in the memory system. */
dgnn_status dgnn_ctx_set_grid_cap(dgnn_ctx* ctx, int32_t max_blocks);
/* HBM footprint controls.  The ctx recycles the large buffers every dgnn_sample call needs
 * (the output arenas of a dgnn_samples released with dgnn_samples_free, and the sampler's
 * group scratch): they are kept by the ctx, up to `bytes` in total (default 24 GiB; 0 = keep
 * nothing), and handed to the next call instead of being freed and re-allocated, so repeated
 * offline passes settle on a fixed footprint.  Kept buffers are released by a lower limit, by
 * an allocation that would otherwise fail, and by dgnn_ctx_destroy.  dgnn_ctx_kept_bytes
 * reports the bytes currently kept. */
dgnn_status dgnn_ctx_set_keep_limit(dgnn_ctx* ctx, int64_t bytes);
int64_t dgnn_ctx_kept_bytes(const dgnn_ctx* ctx);
/* Budget (bytes, >= 16 MiB; default 3 GiB) of the sampler's per-group scratch: the number of
 * batches sampled concurrently (when dgnn_ctx_set_sample_group is 0) is the largest that fits
 * it, at most 64.  Results do not depend on it. */
dgnn_status dgnn_ctx_set_sample_budget(dgnn_ctx* ctx, int64_t bytes);
int64_t dgnn_ctx_launches(const dgnn_ctx* ctx);
dgnn_status dgnn_ctx_set_timing(dgnn_ctx* ctx, int enable);
/* With timing on, only the kernel families whose bit (1 << DGNN_K_*) is set in mask are bracketed
 * by events (default: all).  Two event records per launch are host API calls: a timed region that
 * should not pay them for hundreds of small launches times only the families it reports. */
dgnn_status dgnn_ctx_set_timing_mask(dgnn_ctx* ctx, uint64_t mask);
typedef struct {
    int64_t launches;  /* timed launches of this family                          */
    double ms;         /* summed CUDA-event durations (ms)                        */
    double bytes;      /* summed algorithmic bytes, 0 if n/a */
} dgnn_kernel_stat;
/* Synchronizes the ctx stream, folds pending events into the totals. */
dgnn_status dgnn_ctx_kernel_stats(dgnn_ctx* ctx, int32_t kernel_id, dgnn_kernel_stat* out);
dgnn_status dgnn_ctx_reset_stats(dgnn_ctx* ctx);
const char* dgnn_kernel_name(int32_t kernel_id);

/* ----------------------------------------------------------- a1-a3 sampling ---- */
typedef struct {
    int64_t num_nodes;       /* N (< 2^30)                                                */
    int64_t num_edges;       /* E = indptr[N]                                             */
    const int64_t* indptr;   /* device [N+1], non-decreasing, indptr[0] = 0               */
    const int32_t* indices;  /* device [E], neighbour IDs in [0, N)                       */
} dgnn_csr;

/* Sample mini-batches t = 0 .. ceil(num_seeds/batch_size)-1: batch t has
 * seeds[t*B .. min((t+1)*B, S)) and batch id bid = batch_id_base + t (reading c9).
 * Per batch, hop h = 0..H-1 with k = fanout[h] (reading c1): every node first
 * discovered at hop h-1 (the seeds at h = 0; reading c4) with out-degree d takes all d
 * CSR positions if k >= d, else the k positions chosen by Floyd's algorithm from
 * Philox4x32-10 draws keyed (rng_seed, v, bid, h, slot) (readings c2, c3, c5-c8),
 * in ascending position order.  New nodes of a hop are appended in ascending global
 * ID (c10); edges are (frontier node j -> local id of the neighbour), grouped by j,
 * then by CSR position (c11).
 *   seeds        device [num_seeds]; distinct within a batch (c12), in [0, N).
 *   fanout       HOST [num_hops], each in [0, 65535]; num_hops in [1, 65535].
 *   counts       device uint32 [N] or NULL: counts[v] += 1 for every sampled batch whose
 *                node set contains v (the access-frequency counter, c14).
 *   out          receives a library-owned dgnn_samples (free with dgnn_samples_free).
 * Blocking: returns after the samples are complete (it synchronizes the ctx stream
 * once per sampling group to size the outputs).  num_seeds == 0 returns OK with zero
 * batches.  Errors: DGNN_EINVAL for bad arguments, a seed outside [0, N) or a
 * seed repeated within one batch (in the last two cases `counts` is unspecified). */
dgnn_status dgnn_sample(dgnn_ctx* ctx, const dgnn_csr* csr, const int32_t* seeds, int64_t num_seeds,
                        int32_t batch_size, int64_t batch_id_base, const int32_t* fanout, int32_t num_hops,
                        uint64_t rng_seed, uint32_t* counts, dgnn_samples** out);

/* Concatenated, batch-major layout of all samples (device unless *_host). */
typedef struct {
    int64_t num_batches;
    int32_t num_hops;
    int64_t batch_id_base;
    int64_t total_nodes;
    int64_t total_edges;
    int64_t total_eptr;
    const int64_t* node_off;      /* [nb+1]: batch b's nodes are nodes[node_off[b] .. node_off[b+1]) */
    const int32_t* nodes;         /* [total_nodes] global IDs, seeds first, then per hop ascending   */
    const int32_t* hop_off;       /* [nb*(H+2)]: local boundaries 0, |seeds|, ..., n_b per batch      */
    const int64_t* eptr_off;      /* [nb+1]: batch b's eptr starts at eptr[eptr_off[b]]               */
    const int32_t* eptr;          /* per batch hop_off[b][H]+1 entries: edges of frontier node j are  */
                                  /* src_local[edge_off[b] + eptr[j] .. edge_off[b] + eptr[j+1])      */
                                  /* (DGNN_SAMPLE_BLOCKS: per hop h an array of hop_off[b][h+1]+1)   */
    const int64_t* edge_off;      /* [nb+1]                                                           */
    const int32_t* src_local;     /* [total_edges] local index (within the batch) of each neighbour   */
    const int64_t* node_off_host; /* host mirrors of the offset arrays                                */
    const int64_t* edge_off_host;
    const int64_t* eptr_off_host;
    const int32_t* hop_off_host;
    int32_t mode;                 /* DGNN_SAMPLE_NODEWISE or DGNN_SAMPLE_BLOCKS (eptr layout)       */
} dgnn_samples_info;
dgnn_status dgnn_samples_get_info(const dgnn_samples* s, dgnn_samples_info* info);
void dgnn_samples_free(dgnn_samples* s);

/* ------------------------------------------------------- a4-a5 cache plan ---- */
/* Rank nodes by (counts desc, ID asc), excluding zero counts (c15); the first
 * K_g = min(gpu_rows, nnz) form the GPU tier, the next K_h = min(host_rows, nnz-K_g)
 * the host tier; every other node is DISK (c18, c19).  Slots inside a tier follow
 * ascending node ID (c17); tier_map[v] = tier << 30 | slot (DISK slot 0).
 *   counts   device uint32 [num_nodes]; must already be summed over ranks when the
 *            offline pass is sharded (the Python layer all-reduces it).
 * Blocking (one small histogram read-back).  DGNN_EUNSUPPORTED if max(counts) >= 2^24. */
dgnn_status dgnn_build_cache(dgnn_ctx* ctx, const uint32_t* counts, int64_t num_nodes, int64_t gpu_rows,
                             int64_t host_rows, dgnn_cache_plan** out);
typedef struct {
    int64_t num_nodes;
    int64_t k_gpu;
    int64_t k_host;
    const uint32_t* tier_map;  /* device [num_nodes]               */
    const int32_t* gpu_ids;    /* device [k_gpu], ascending IDs     */
    const int32_t* host_ids;   /* device [k_host], ascending IDs    */
    uint32_t gpu_min_count;    /* smallest count inside the GPU tier (0 if empty)  */
    uint32_t host_min_count;   /* smallest count inside the host tier (0 if empty) */
} dgnn_plan_info;
dgnn_status dgnn_cache_plan_get_info(const dgnn_cache_plan* p, dgnn_plan_info* info);
void dgnn_cache_plan_free(dgnn_cache_plan* p);

/* --------------------------------------------------------- a6 classify ---- */
/* Address tables of batches [b_lo, b_hi) (reading c18, c21):
 * for local node j of batch b, addr = tier_map[nodes[j]] if that tier is GPU/HOST,
 * else DISK << 30 | (rank of j among the batch's DISK nodes, in local order).
 * The DISK nodes of each batch, in local order, are that batch's packed list P_b.
 *   addr        device uint32 [node_off[b_hi] - node_off[b_lo]] (caller-owned).
 *   packed_ids  device int32, same capacity: P_{b_lo} .. P_{b_hi-1} concatenated.
 *   packed_off  device int64 [b_hi-b_lo+1]: exclusive prefix of |P_b| (packed_off[0]=0).
 *   packed_off_host  host int64 [b_hi-b_lo+1] or NULL; when non-NULL the call
 *               synchronizes and copies packed_off there. */
dgnn_status dgnn_classify(dgnn_ctx* ctx, const dgnn_cache_plan* plan, const dgnn_samples* samples,
                          int64_t b_lo, int64_t b_hi, uint32_t* addr, int32_t* packed_ids, int64_t* packed_off,
                          int64_t* packed_off_host);

/* Rows of each tier per batch, from the address tables of batches [b_lo, b_hi) (as written
 * by dgnn_classify into addr): counts_host[3*(b-b_lo) + tier] (host int64; synchronizes).
 * Sizing metadata for the assembler's staging buffers. */
dgnn_status dgnn_batch_tier_counts(dgnn_ctx* ctx, const dgnn_samples* samples, int64_t b_lo, int64_t b_hi,
                                   const uint32_t* addr, int64_t* counts_host);

/* ------------------------------------------------------------- a7 pack ---- */
/* Host arithmetic of the chunk layout (reading c20): chunk_off[0] = 0,
 * chunk_off[i+1] = roundup(chunk_off[i] + (packed_off[i+1]-packed_off[i]) * row_bytes, 4096). */
dgnn_status dgnn_chunk_layout(const int64_t* packed_off_host, int64_t nb, int64_t row_bytes,
                              int64_t* chunk_off_host);

/* Host arithmetic of the packing groups (the analogue of P:439's "C - 4N" partition sizing):
 * consecutive batches, each group at most group_size batches (<= 0: unbounded) whose packed rows
 * plus one 4 KiB page of padding per batch fit group_budget bytes (a group always holds at least one
 * batch).  packed_off_host [nb+1] as from dgnn_classify; group_lo_host [nb+1] receives the first batch
 * of every group followed by nb; *n_groups their count.  Errors: DGNN_EINVAL. */
dgnn_status dgnn_packing_groups(const int64_t* packed_off_host, int64_t nb, int64_t row_bytes, int64_t group_size,
                                int64_t group_budget, int64_t* group_lo_host, int64_t* n_groups);

/* Host arithmetic of the assembler's runs (a9; one dgnn_assemble_group launch each): consecutive
 * batches whose assembled rows fit max_rows (a run holds at least one batch, at most max_batches).
 * node_off_host [nb+1] (the samples' node offsets); run_lo_host [nb+1] receives the first batch of
 * every run followed by nb; *n_runs their count.  Errors: DGNN_EINVAL. */
dgnn_status dgnn_assembly_runs(const int64_t* node_off_host, int64_t nb, int64_t max_rows, int64_t max_batches,
                               int64_t* run_lo_host, int64_t* n_runs);

/* Host arithmetic of the per-run tables the run-level assembly reads (dgnn_assemble_group*), all
 * relative to the run [b0, b1) = [run_lo[r], run_lo[r+1]), k = b1 - b0:
 *   packed-only layout (disk_rows == NULL): node offsets no[b0..b1] - no[b0] (k+1), chunk byte
 *     offsets chunk_start[b0..b1) - c_lo then c_hi - c_lo (k+1), packed-row prefix from b0 (k+1),
 *     and with sec_abs (graph samples in the chunks) sec_abs[b0..b1) - c_lo (k);
 *   segmented disk cache (disk_rows = DISK rows per batch): node offsets (k+1), dense partial-input
 *     byte offsets dpre * row_bytes (k+1), dpre (k+1), chunk byte offsets (k+1);
 * with c_lo = chunk_start[b0], c_hi = chunk_start[b1] (chunk_bytes past the last batch).  All host
 * int64: node_off [nb+1], chunk_start / chunk_rows / disk_rows / sec_abs [nb]; tab receives the tables
 * back to back (tab_off [n_runs+1] their starts; EINVAL past tab_cap); spans [4*n_runs] = (no[b0],
 * no[b1], c_lo, c_hi) per run. */
dgnn_status dgnn_assembly_tables(const int64_t* node_off, const int64_t* chunk_start, const int64_t* chunk_rows,
                                 const int64_t* disk_rows, const int64_t* sec_abs, int64_t nb, int64_t chunk_bytes,
                                 int64_t row_bytes, const int64_t* run_lo, int64_t n_runs, int64_t* tab,
                                 int64_t tab_cap, int64_t* tab_off, int64_t* spans);

/* The graph sample kept in the chunk ("the graph sample of the mini-batch is also kept in
 * the chunk"; reading c22b, opt-in).  Chunk i then holds its |P_i| packed rows at offset 0, and
 * at sec_off[i] = roundup(|P_i| * row_bytes, 16) a graph section of int32 words:
 *     H, n_i, m_i, e_i, hop_off[H+2], nodes[n_i], eptr[m_i], src_local[e_i]
 * (the batch's dgnn_samples arrays; m_i eptr entries, e_i edges), zero padding up to
 * chunk_off[i+1] = roundup(sec_off[i] + 4 * words, 4096).
 * dgnn_chunk_layout_graph: host arithmetic of chunk_off [nb+1] and sec_off [nb] for batches
 *   [b_lo, b_lo + nb) of `samples` (sizes from its host mirrors), offsets relative to the group.
 * dgnn_pack_graph: writes those sections into a group buffer already packed by dgnn_pack (which
 *   zeroes the tails the sections overwrite); sec_off_dev = the device copy of sec_off.
 *   EINVAL if the samples' device arrays were dropped.
 * dgnn_samples_load: the graph loader: a library-owned samples object (free with
 *   dgnn_samples_free) for batches [b_lo, b_hi) of `meta`, renumbered from 0, whose device arrays
 *   are read from the staged chunks -- section i at base_dev + sec_off_dev[i] (device int64 [nb]);
 *   its device offsets are a scan of the section headers.  Only the host mirrors (and the array
 *   sizes) come from `meta`, the layout's metadata; headers that disagree with them raise
 *   DGNN_ECUDA ("internal: device capacity overflow") at the next synchronizing call.  Enqueued
 *   on the ctx stream, no host synchronization; the object's arrays come from the ctx allocator
 *   (stream-ordered on the ctx stream: a consumer on another stream must finish before it is freed).
 * dgnn_samples_drop_device: frees a samples object's nodes / eptr / src_local device arrays
 *   (host mirrors and offsets stay), e.g. once they are in the chunks. */
dgnn_status dgnn_chunk_layout_graph(const dgnn_samples* samples, int64_t b_lo, const int64_t* packed_off_host,
                                    int64_t nb, int64_t row_bytes, int64_t* chunk_off_host, int64_t* sec_off_host);
dgnn_status dgnn_pack_graph(dgnn_ctx* ctx, const dgnn_samples* samples, int64_t b_lo, int64_t nb,
                            const int64_t* sec_off_dev, void* group_buf);
dgnn_status dgnn_samples_load(dgnn_ctx* ctx, const dgnn_samples* meta, int64_t b_lo, int64_t b_hi,
                              const void* base_dev, const int64_t* sec_off_dev, dgnn_samples** out);
dgnn_status dgnn_samples_drop_device(dgnn_samples* samples);

/* a7 from a feature table partitioned by node range over several devices (the
 * IGB-shaped table, 409.6 GB, exceeds one GPU): row v lives in shard r = v / shard_rows at row
 * v - r * shard_rows of peers_dev[r] (a device array of nshards pointers: this rank's own shard and
 * the CUDA IPC mappings of the others', read over NVLink).  dgnn_pack_sharded / dgnn_gather_rows_sharded
 * are dgnn_pack / dgnn_gather_rows with that source; row_bytes a multiple of 16, outputs 16-byte
 * aligned. */
dgnn_status dgnn_pack_sharded(dgnn_ctx* ctx, const void* const* peers_dev, int64_t shard_rows, int32_t nshards,
                              int64_t row_bytes, const int32_t* packed_ids, const int64_t* packed_off,
                              const int64_t* chunk_off, int64_t nb, int64_t total_rows, int64_t group_bytes,
                              void* group_buf);
dgnn_status dgnn_gather_rows_sharded(dgnn_ctx* ctx, const void* const* peers_dev, int64_t shard_rows, int32_t nshards,
                                     int64_t row_bytes, const int32_t* ids, int64_t n, void* out);

/* Batched pack of one packing group: for every batch i < nb and r <
 * |P_i|, group_buf[chunk_off[i] + r*row_bytes ..] = features[P_i[r]] (raw bytes), and
 * the tail of each chunk up to chunk_off[i+1] is zeroed.
 *   features    UVA [num_rows * row_bytes] (device HBM, or pinned host for tables that
 *               exceed HBM).
 *   packed_ids, packed_off (device, as produced by dgnn_classify), chunk_off (device
 *   int64 [nb+1]); total_rows = packed_off[nb] and group_bytes = chunk_off[nb] (host
 *   values, used for grid sizing).  group_buf: device or pinned [group_bytes]. */
dgnn_status dgnn_pack(dgnn_ctx* ctx, const void* features, int64_t num_rows, int64_t row_bytes,
                      const int32_t* packed_ids, const int64_t* packed_off, const int64_t* chunk_off, int64_t nb,
                      int64_t total_rows, int64_t group_bytes, void* group_buf);

/* Tier buffers as special mini-batches: out[s] = features[ids[s]], s < n.
 * out: device or pinned host (UVA). */
dgnn_status dgnn_gather_rows(dgnn_ctx* ctx, const void* features, int64_t num_rows, int64_t row_bytes,
                             const int32_t* ids, int64_t n, void* out);

/* ----------------------------------------------------------- a8 staging ---- */
/* Copies on the ctx side stream, ordered after all work already enqueued on the ctx
 * stream.  Each returns a ticket; dgnn_stage_wait makes the ctx stream wait for that
 * copy (and all earlier ones); dgnn_stage_sync blocks the host until it completes.
 * kind: 0 = device -> host, 1 = host -> device, 2 = device -> device. */
dgnn_status dgnn_stage_copy(dgnn_ctx* ctx, void* dst, const void* src, int64_t bytes, int32_t kind,
                            int64_t* ticket);
dgnn_status dgnn_stage_wait(dgnn_ctx* ctx, int64_t ticket);
/* Make another stream (a cudaStream_t; NULL = legacy default) wait for a staging copy, e.g.
 * the assembler's stream waiting for a packing group's stage-out. */
dgnn_status dgnn_stage_wait_stream(dgnn_ctx* ctx, int64_t ticket, void* stream);
dgnn_status dgnn_stage_sync(dgnn_ctx* ctx, int64_t ticket);
/* The disk tier as a file on local storage ("creates a disk chunk", "pread ...
 * O_Direct").  dgnn_file_open opens (create=1: creates / truncates to `size`) a file, with
 * O_DIRECT when direct=1 (offsets, sizes and the bounce buffer must then be 4096-aligned).
 * dgnn_stage_file_write / _read move bytes between device memory and the file through a
 * pinned bounce buffer (host, caller-owned, chunk_bytes): on the ctx side stream, pieces of
 * chunk_bytes / 2 alternate between the buffer's halves, each one cudaMemcpyAsync plus the file
 * engine's pwrite / pread parts, submitted and awaited in stream order (cudaLaunchHostFunc), so
 * the ticket completes when the data is on disk / in HBM.  I/O errors surface as DGNN_EIO at
 * the next dgnn_ctx_sync. */
typedef struct dgnn_file dgnn_file;
dgnn_status dgnn_file_open(const char* path, int32_t direct, int32_t create, int64_t size, dgnn_file** out);
dgnn_status dgnn_file_close(dgnn_file* f);
dgnn_status dgnn_stage_file_write(dgnn_ctx* ctx, dgnn_file* f, int64_t file_off, const void* dev_src, int64_t bytes,
                                  void* bounce, int64_t chunk_bytes, int64_t* ticket);
/* Each file owns an I/O engine (the paper's multi-queue engine): `queues` worker threads
 * with one request queue each (default 4), started at the file's first transfer; a transfer is
 * split into 4 KiB-aligned parts (>= 1 MiB) spread over the queues.  dgnn_file_set_queues sets
 * the count before the first transfer (EINVAL after it, or outside [1, 64]).  The staging calls
 * are double-buffered: the bounce buffer's two halves alternate, so the disk side of one piece
 * overlaps the PCIe copy of the next.  dgnn_file_close joins the engine: synchronize every
 * staging ticket of the file first. */
dgnn_status dgnn_file_set_queues(dgnn_file* f, int32_t queues);
/* Disk-cache page reads (P:307 merged requests; the paper's io_uring engine): the 4 KiB
 * pages pages[0..n_pages) of the cache region at file offset base_off are read (runs of
 * consecutive pages as one request each, spread over the file's I/O queues; `threads` raises the
 * queue count of an engine that has not started yet) into dev_dst back to back, through the
 * pinned bounce buffer (bounce_bytes, page-aligned; its halves alternate between fills) in stream
 * order on the side stream.  The page list is copied at the call; returns a staging ticket like
 * dgnn_stage_copy. */
dgnn_status dgnn_stage_file_read_pages(dgnn_ctx* ctx, dgnn_file* f, int64_t base_off, const int32_t* pages,
                                       int64_t n_pages, void* dev_dst, void* bounce, int64_t bounce_bytes,
                                       int32_t threads, int64_t* ticket);
dgnn_status dgnn_stage_file_read(dgnn_ctx* ctx, dgnn_file* f, int64_t file_off, void* dev_dst, int64_t bytes,
                                 void* bounce, int64_t chunk_bytes, int64_t* ticket);

/* The window-ordered host tier (the ordering idea of the paper's disk cache,
 * Sec. 5.1 / Algorithm 1, applied to the CPU-cache tier and the assembler's host-row
 * windows).  Slots and addresses are unchanged (reading c17); the tier's PHYSICAL row order is
 * (reversed mask, slot), mask = the windows that address the slot (bits reversed: window 0 most
 * significant, so window 0's rows are one contiguous range), so that every window's host rows are a
 * few contiguous ranges the copy engine moves at the link rate.
 * dgnn_host_order: addr = the address tables of all batches (device uint32, batch-major), window w =
 *   addr[win_node_off_host[w] .. win_node_off_host[w+1]), 1 <= nwin <= 32; host_ids = the plan's
 *   host tier (device int32 [k_host]).  Outputs (device, caller-owned, k_host entries):
 *   slot_mask[s] = OR of 1<<w over windows holding a HOST address of slot s; phys_of_slot[s] = its
 *   physical row (slots sorted by (bit-reversed mask, slot)); phys_ids[p] = host_ids[the slot at row p] (fill the tier with dgnn_gather_rows
 *   over phys_ids).  Host outputs: the n_groups runs of equal mask in physical order, their first
 *   row (group_start_host) and mask (group_mask_host); DGNN_ERANGE if n_groups > max_groups (the
 *   caller keeps the slot-ordered tier).  Synchronizes.
 * dgnn_host_order_ranges: host arithmetic: window w's physical ranges (merged adjacent groups) as
 *   triples (phys_lo, phys_hi, staging_lo) in ranges_host[3 * capacity]; *rows = the window's rows.
 * dgnn_host_order_schedule: host arithmetic: the staging schedule of all nwin windows in one arena
 *   of capacity_rows rows.  A group is needed by the maximal runs of consecutive windows in its
 *   mask; each (group, run) is copied once, at the prefetch of its first window, and stays in the
 *   arena until its last window is done (window w is prefetched once window w-2 is done), so rows
 *   shared by consecutive windows cross PCIe once.  Spare capacity bridges the gaps between runs of a
 *   group (shortest first, when the arena has room in every window of the gap): with capacity_rows
 *   >= the rows the windows touch, every row crosses once per pass.  Outputs per window w (CSR, copy_off / map_off
 *   [nwin+1]): the copies to issue (copy_out triples) and the map of every row w reads (map_out
 *   triples sorted by phys_lo: the input of dgnn_host_window_ranges); *rows_copied = total rows
 *   moved.  EINVAL if the capacity (>= max over w of |S_{w-1}| + |S_w| always fits) or an output
 *   capacity is exceeded.
 * dgnn_host_window_ranges: smap[s] = staging row of slot s for every slot of window w (ranges_dev =
 *   the device copy of the triples, nr <= 4096); other entries untouched.
 * dgnn_copy_ranges: one cudaMemcpyAsync (H2D, ctx stream) per triple: rows [phys_lo, phys_hi) of
 *   src_host (the pinned tier) to dst_dev rows [staging_lo, ...).
 * dgnn_remap_ids_dev: ids[i] = table[ids[i]] for i < min(*n_dev, n_max) (a window's slot list ->
 *   physical rows, for the SM gather when the windows differ from the ordering's). */
dgnn_status dgnn_host_order(dgnn_ctx* ctx, const uint32_t* addr, const int64_t* win_node_off_host, int32_t nwin,
                            const int32_t* host_ids, int64_t k_host, int32_t* phys_ids, int32_t* phys_of_slot,
                            uint32_t* slot_mask, int64_t max_groups, int64_t* group_start_host,
                            uint32_t* group_mask_host, int64_t* n_groups);
dgnn_status dgnn_host_order_ranges(const int64_t* group_start_host, const uint32_t* group_mask_host, int64_t n_groups,
                                   int64_t k_host, int32_t window, int64_t* ranges_host, int64_t capacity,
                                   int64_t* n_ranges, int64_t* rows);
dgnn_status dgnn_host_order_schedule(const int64_t* group_start_host, const uint32_t* group_mask_host,
                                     int64_t n_groups, int64_t k_host, int32_t nwin, int64_t capacity_rows,
                                     int64_t* copy_out, int64_t copy_cap, int64_t* copy_off, int64_t* map_out,
                                     int64_t map_cap, int64_t* map_off, int64_t* rows_copied);
dgnn_status dgnn_host_window_ranges(dgnn_ctx* ctx, const uint32_t* slot_mask, const int32_t* phys_of_slot,
                                    int64_t k_host, int32_t window, const int64_t* ranges_dev, int64_t nr,
                                    int32_t* smap);
/* The host tier read from the feature table itself (a host-resident table, bench.py's e2e mode):
 * instead of copying a window's physical host-tier ranges (dgnn_copy_ranges), gather, for every
 * triple t of ranges_dev (phys_lo, phys_hi, staging_lo; prefix_dev[nr+1] = rows before each
 * triple, prefix_dev[nr] = total_rows), the table rows of the nodes at physical rows [phys_lo,
 * phys_hi) -- ids = the host order's phys_ids (physical row -> node id, device) -- into dst_dev rows
 * [staging_lo, ...).  table: device or pinned host (UVA) [num_nodes, row_bytes]; row_bytes % 4 == 0.
 * The staging arena then holds exactly what dgnn_copy_ranges would have put there (the tier's
 * rows are the table's rows of its nodes).  Enqueued on the ctx stream.
 * Errors: DGNN_EINVAL. */
dgnn_status dgnn_gather_ranges(dgnn_ctx* ctx, const void* table, int64_t row_bytes, const int32_t* ids,
                               const int64_t* ranges_dev, const int64_t* prefix_dev, int64_t nr,
                               int64_t total_rows, void* dst_dev);

/* Small host -> device table upload (the per-run assembly tables, the pack's offset tables; a
 * scheduling primitive, no arithmetic of the method): `bytes` of src_host (any host memory, read
 * before the call returns) to dst_dev (device, caller-owned), enqueued on the ctx stream as kernels
 * that carry the bytes in their parameters -- not the copy engines, where a small copy queues behind
 * the gigabytes of window and stage copies in flight (and the stream's next operations with it).
 * Above 256 KiB: one cudaMemcpyAsync.  Errors: DGNN_EINVAL (NULL with bytes > 0, bytes < 0). */
dgnn_status dgnn_upload(dgnn_ctx* ctx, void* dst_dev, const void* src_host, int64_t bytes);
dgnn_status dgnn_copy_ranges(dgnn_ctx* ctx, void* dst_dev, const void* src_host, const int64_t* ranges_host,
                             int64_t nr, int64_t row_bytes);
dgnn_status dgnn_remap_ids_dev(dgnn_ctx* ctx, int32_t* ids, const int64_t* n_dev, int64_t n_max,
                               const int32_t* table);

/* Pinned, device-mapped host memory for the host tier and the disk-tier arena. */
dgnn_status dgnn_host_alloc(int64_t bytes, void** out);
dgnn_status dgnn_host_free(void* p);

/* --------------------------------------------------------- a9 assemble ---- */
/* out[j] = row(addr[j]) for j < n (Fig. 3): tier GPU -> gpu_tier[slot]
 * (device), HOST -> host_tier[slot] (pinned host, read over PCIe through UVA), DISK ->
 * chunk[slot] (the batch's staged chunk: device or pinned host).  Slots must be below
 * k_gpu / k_host / chunk_rows; an unresolvable address writes a zero row and is
 * reported as DGNN_ERANGE by the next dgnn_ctx_sync.  out: device [n * row_bytes]. */
dgnn_status dgnn_assemble(dgnn_ctx* ctx, const uint32_t* addr, int64_t n, const void* gpu_tier, int64_t k_gpu,
                          const void* host_tier, int64_t k_host, const void* chunk, int64_t chunk_rows,
                          int64_t row_bytes, void* out);

/* A run of consecutive batches in one launch (same per-row semantics as dgnn_assemble).
 *   addr        device uint32 [n]: the address tables of the batches, concatenated.
 *   node_off    device int64 [nb+1]: row offsets of the batches inside addr / out (node_off[0] = 0,
 *               node_off[nb] = n).
 *   host_tier   the host tier (pinned, UVA) when host_map is NULL; otherwise a device buffer of
 *               staged host rows and host_map (device int32 [k_host]) gives the staged row of
 *               each host slot (see dgnn_host_window).
 *   chunk_base  UVA base of the batches' staged chunks; chunk_off device int64 [nb+1] byte
 *               offsets of each chunk from chunk_base; chunk_rows device int64 [nb+1] exclusive
 *               prefix of the packed rows (a DISK slot of batch b must be < its packed rows).
 *   out         device [n * row_bytes]. */
dgnn_status dgnn_assemble_group(dgnn_ctx* ctx, const uint32_t* addr, const int64_t* node_off, int64_t nb, int64_t n,
                                const void* gpu_tier, int64_t k_gpu, const void* host_tier, int64_t k_host,
                                const int32_t* host_map, const void* chunk_base, const int64_t* chunk_off,
                                const int64_t* chunk_rows, int64_t row_bytes, void* out);

/* Host-row merging for a window of consecutive batches (the paper's request merging, P:305,
 * applied to CPU-cache rows): every host-tier slot referenced by addr[0..n) is listed once.
 *   stamp      device int32 [k_host], caller-owned, set to -1 once before the first window;
 *              window_id must differ between consecutive windows (use an increasing counter).
 *   list       device int32 [capacity]: the distinct slots (arbitrary order).
 *   smap       device int32 [k_host]: smap[slot] = position of slot in list (for listed slots).
 *   count      device int64 [1]: number of listed slots (overwritten).
 * Pair with dgnn_gather_rows_dev(host_tier, list, count -> staging) and dgnn_assemble_group
 * (host_tier = staging, host_map = smap): each host row then crosses PCIe once per window
 * instead of once per batch; outputs are unchanged. */
dgnn_status dgnn_host_window(dgnn_ctx* ctx, const uint32_t* addr, int64_t n, int32_t window_id, int32_t* stamp,
                             int64_t k_host, int32_t* list, int64_t capacity, int32_t* smap, int64_t* count);
/* Runs of consecutive slots in the window's list (after dgnn_host_window with the same stamp,
 * window_id and smap): runs[r] = list position where run r starts, *run_count = runs.  A run
 * of k slots is k*row_bytes contiguous bytes, so dgnn_gather_runs_dev moves the window's rows
 * with one contiguous copy per run (fewer, larger PCIe reads than one per row):
 * out + p*row_bytes .. = src + list[p]*row_bytes .. for every list position p < *count. */
dgnn_status dgnn_host_window_runs(dgnn_ctx* ctx, const int32_t* stamp, int64_t k_host, int32_t window_id,
                                  const int32_t* smap, int32_t* runs, int64_t* run_count);
dgnn_status dgnn_gather_runs_dev(dgnn_ctx* ctx, const void* src, int64_t row_bytes, const int32_t* list,
                                 const int64_t* count, const int32_t* runs, const int64_t* run_count,
                                 int64_t max_runs, void* out);
/* ---- sharded GPU tier (when the GPU tier does not fit replicated, slot s
 * lives on rank s % world at local row s / world; remote rows travel over NVLink with
 * all-to-all exchanges run by the caller's process group) ----
 * dgnn_tier_shard_ids: ids[l] = gpu_ids[l*world + rank] for the rank's local rows
 *   (*n_local = their count); fill the shard with dgnn_gather_rows(features, ids).
 * dgnn_shard_requests: the GPU-tier rows of addr[0..n) owned by other ranks, grouped by
 *   owner: req_off_host[world+1] (host, exclusive prefix; the call synchronizes),
 *   req_slot (device int32 [n]): owner-local row, req_pos (device int32 [n]): row in out.
 *   Order inside an owner's group is unspecified (each request carries its position).
 * dgnn_scatter_rows: out[pos[i]] = rows[i] for i < n (the received remote rows).
 * dgnn_assemble_group_sharded: dgnn_assemble_group with gpu_tier = this rank's shard;
 *   GPU-tier rows owned by other ranks are left untouched (filled by dgnn_scatter_rows). */
dgnn_status dgnn_tier_shard_ids(dgnn_ctx* ctx, const int32_t* gpu_ids, int64_t k_gpu, int32_t rank, int32_t world,
                                int32_t* ids, int64_t* n_local);
dgnn_status dgnn_shard_requests(dgnn_ctx* ctx, const uint32_t* addr, int64_t n, int64_t k_gpu, int32_t rank,
                                int32_t world, int64_t* req_off_host, int32_t* req_slot, int32_t* req_pos);
dgnn_status dgnn_scatter_rows(dgnn_ctx* ctx, const void* rows, int64_t n, int64_t row_bytes, const int32_t* pos,
                              void* out);
dgnn_status dgnn_assemble_group_sharded(dgnn_ctx* ctx, const uint32_t* addr, const int64_t* node_off, int64_t nb,
                                        int64_t n, const void* gpu_tier, int64_t k_gpu, int32_t gpu_rank,
                                        int32_t gpu_world, const void* host_tier, int64_t k_host,
                                        const int32_t* host_map, const void* chunk_base, const int64_t* chunk_off,
                                        const int64_t* chunk_rows, int64_t row_bytes, void* out);

/* ---- one-sided peer-memory GPU tier (the sharded tier without the
 * all-to-all).  Every rank's shard is a dgnn_device_alloc allocation exported with
 * dgnn_ipc_handle and mapped by the other ranks with dgnn_ipc_open (CUDA IPC; over NVLink /
 * NVSwitch the mapped loads are peer loads), so the assembly kernel reads a remote GPU-tier row
 * directly from its owner: the exchange of dgnn_shard_requests / all-to-all / dgnn_scatter_rows
 * collapses into the gather itself.  Shards must be complete (filled + a barrier across ranks)
 * before any rank assembles.
 * dgnn_assemble_group_peer: dgnn_assemble_group with GPU-tier slot s read from
 *   peers[s % world] + (s / world) * row_bytes; peers = device array [world] of shard bases
 *   (this rank's own shard included); row_bytes % 16 == 0.
 * dgnn_device_alloc / _free: plain cudaMalloc (an IPC handle names the allocation base).
 * dgnn_ipc_handle: handle (DGNN_IPC_HANDLE_BYTES bytes, host) of a dgnn_device_alloc pointer.
 * dgnn_ipc_open / _close: map / unmap another process's allocation on `device`. */
#define DGNN_IPC_HANDLE_BYTES 64
dgnn_status dgnn_assemble_group_peer(dgnn_ctx* ctx, const uint32_t* addr, const int64_t* node_off, int64_t nb,
                                     int64_t n, const void* const* peers, int64_t k_gpu, int32_t world,
                                     const void* host_tier, int64_t k_host, const int32_t* host_map,
                                     const void* chunk_base, const int64_t* chunk_off, const int64_t* chunk_rows,
                                     int64_t row_bytes, void* out);
dgnn_status dgnn_device_alloc(int32_t device, int64_t bytes, void** out);
dgnn_status dgnn_device_free(void* p);
dgnn_status dgnn_ipc_handle(const void* dev_ptr, void* handle);
dgnn_status dgnn_ipc_open(int32_t device, const void* handle, void** dev_ptr);
dgnn_status dgnn_ipc_close(void* dev_ptr);

/* dgnn_gather_rows with the row count read from device memory (*n_dev <= n_max). */
dgnn_status dgnn_gather_rows_dev(dgnn_ctx* ctx, const void* features, int64_t num_rows, int64_t row_bytes,
                                 const int32_t* ids, const int64_t* n_dev, int64_t n_max, void* out);

/* ------------------------------------------- segmented disk cache (NEXT #1) ---- */
/* Sec. 5.1: under a disk-space budget C the DISK rows of an epoch are split
 * into per-segment disk caches (shared, de-duplicated, laid out by MinHash reordering,
 * Algorithm 1) and reduced packed chunks.  Readings d1-d8 (oracle/dgnn_oracle.c):
 *  d1 segment g = batches [g*s, min((g+1)*s, nb)).
 *  d2 a node whose local frequency (batches of the segment whose packed list holds it)
 *     exceeds m joins the segment's cache V_d; otherwise it stays in each packed list.
 *  d3 space in 4096-byte pages: per segment ceil(|V_d| / fpp), fpp = floor(4096 / row_bytes),
 *     per batch ceil(|P_b'| * row_bytes / 4096); feasible when space <= budget.
 *  d4 heuristic: the minimum s in 1..nb with space <= budget (m = 1 advised).
 *  d5 H_t = ranking of the segment's local batch indices i by (x, i), x = Philox4x32-10
 *     (ctr = {i, g, t, 0x4D48}, key = seed) as out.y << 32 | out.x.
 *  d6 S_t(v) = min over the segment's batches i holding v of H_t(i); V_r = V_d sorted by
 *     (S_0, ..., S_{k-1}, v) (reorder = 1) or by v (reorder = 0).
 *  d7 I/O = sum over batches of chunk pages + distinct cache pages (merged requests).
 *  d8 dc_addr of the r-th packed row of the INPUT packed lists: cached -> 1 << 31 |
 *     (q * fpp + slot), q = index of its page in the batch's request list; packed -> its
 *     rank in P_b'.
 * Input: the packed lists of all nb batches as dgnn_classify writes them (packed_ids,
 * packed_off device int64 [nb+1], packed_off_host host int64 [nb+1]); the index copies
 * what it needs, so the inputs may be freed after dgnn_disk_index_build returns.
 * Node IDs must be < num_nodes <= 2^31; packed_off[nb] < 2^31.  All calls synchronize. */
typedef struct dgnn_disk_index dgnn_disk_index;
typedef struct dgnn_disk_plan dgnn_disk_plan;
dgnn_status dgnn_disk_index_build(dgnn_ctx* ctx, const int32_t* packed_ids, const int64_t* packed_off,
                                  const int64_t* packed_off_host, int64_t nb, int64_t num_nodes,
                                  dgnn_disk_index** out);
void dgnn_disk_index_free(dgnn_disk_index* idx);
/* Eq. 2 space (d3) of (s_list[i], m) for i < n_s: pages_host[i] (host int64). */
dgnn_status dgnn_disk_space(dgnn_ctx* ctx, const dgnn_disk_index* idx, int64_t row_bytes, const int64_t* s_list_host,
                            int64_t n_s, int64_t m, int64_t* pages_host);
/* d4: *s_out = minimum feasible s (0 if none), *pages_out = its space (of s = nb if none). */
dgnn_status dgnn_disk_search(dgnn_ctx* ctx, const dgnn_disk_index* idx, int64_t row_bytes, int64_t m,
                             int64_t budget_pages, int64_t* s_out, int64_t* pages_out);
/* The plan of (s, m) with k hash functions (d1-d8).  k in [1, 16].  reorder: 0 = identity order
 * (ascending node ID), 1 = reading d6 (sort by the per-function signatures S_0..S_{k-1}),
 * 2 = Algorithm 1 line 8 as printed (one scalar MinHash value min_t S_t(v)). */
dgnn_status dgnn_disk_plan_build(dgnn_ctx* ctx, const dgnn_disk_index* idx, int64_t row_bytes, int64_t s, int64_t m,
                                 int32_t k, uint64_t seed, int32_t reorder, dgnn_disk_plan** out);
typedef struct {
    int64_t nb, nseg, s, m, fpp, row_bytes;
    int64_t n_cache;             /* sum |V_d| over segments                              */
    int64_t n_packed;            /* sum |P_b'|                                           */
    int64_t n_req;               /* sum of merged page requests                          */
    int64_t space_pages, io_pages, cache_pages, chunk_pages;
    const int64_t* seg_off;      /* device [nseg+1]: V_r of segment g = cache_ids[seg_off[g]..) */
    const int32_t* cache_ids;    /* device [n_cache]                                     */
    const int64_t* seg_page_off; /* device [nseg+1]: first global cache page of segment g */
    const int32_t* pk_ids;       /* device [n_packed]: P_b' concatenated                 */
    const int64_t* pk_off;       /* device [nb+1]                                        */
    const int32_t* req_pages;    /* device [n_req]: per batch ascending global pages     */
    const int64_t* req_off;      /* device [nb+1]                                        */
    const uint32_t* dc_addr;     /* device [packed_off[nb]]: d8                          */
    const int64_t* pk_off_host;  /* host copies of pk_off, req_off, seg_off, seg_page_off */
    const int64_t* req_off_host;
    const int64_t* seg_off_host;
    const int64_t* seg_page_off_host;
} dgnn_disk_plan_info;
dgnn_status dgnn_disk_plan_get_info(const dgnn_disk_plan* p, dgnn_disk_plan_info* info);
void dgnn_disk_plan_free(dgnn_disk_plan* p);
/* The segment caches ("laid out on disk by reordering"): out (device or pinned,
 * [cache_pages * 4096] bytes) receives V_r of each segment, fpp rows per page at
 * slot * row_bytes, every byte past the rows zeroed.  row_bytes % 16 == 0. */
dgnn_status dgnn_disk_cache_fill(dgnn_ctx* ctx, const dgnn_disk_plan* p, const void* features, int64_t num_rows,
                                 void* out);
/* Partial input of batches [b_lo, b_hi) ("the CPU reads the features in the disk
 * cache and packed feature chunks and prepares them as partial input"; here the GPU, from
 * staged bytes): for input packed row r of batch b (local DISK rank j = r - packed_off[b]),
 *   out + out_off[b-b_lo] + j*row_bytes  <-  cached: pages + (req_off[b] - req_off[b_lo] + q)*4096
 *                                                   + slot*row_bytes
 *                                           packed: chunks + chunk_off[b-b_lo] + rank*row_bytes
 *   pages    device/pinned: the requested pages req_pages[req_off[b_lo] .. req_off[b_hi]), in order.
 *   chunks   device/pinned: the reduced chunks of the batches; chunk_off device int64 [b_hi-b_lo+1].
 *   out_off  device int64 [b_hi-b_lo+1] (e.g. the c20 layout of the input packed lists, so the
 *            result is what dgnn_pack of the input lists would have produced, minus the padding). */
dgnn_status dgnn_disk_partial(dgnn_ctx* ctx, const dgnn_disk_plan* p, int64_t b_lo, int64_t b_hi,
                              const void* pages, const void* chunks, const int64_t* chunk_off, void* out,
                              const int64_t* out_off);

/* ------------------------------- batched packing from partitions (NEXT #3) ---- */
/* Sec. 5.2 (Fig. 6): when the feature table does not fit in HBM it is read in
 * partitions of consecutive node IDs, each once and sequentially, and every packed row of every
 * batch is routed from the partition that holds it.  The packed lists come as a
 * dgnn_disk_index (its rows sorted by node, so the rows of a partition are one contiguous
 * range).  Results equal dgnn_pack's ("append these node features to pack feature
 * chunk of the mini-batch"); what differs is the source access pattern.
 * dgnn_disk_index_partition_counts: counts_host[p] = packed rows whose node lies in
 *   [p*part_rows, (p+1)*part_rows), p < nparts (host int64; synchronizes).
 * dgnn_pack_partition: for the index's rows with node v in [p0, p1):
 *   group_buf + chunk_off[b] + (r - packed_off[b]) * row_bytes  <-  part + (v - p0) * row_bytes
 *   part       device (or pinned) [(p1-p0) * row_bytes]: rows p0 .. p1-1 of the feature table.
 *   chunk_off  device int64 [nb+1]: the chunk layout (reading c20) of the index's packed lists.
 * dgnn_pack_tails: zero every chunk's bytes past its rows (reading c20).
 * Both are enqueued on the ctx stream without synchronizing; row_bytes % 16 == 0. */
dgnn_status dgnn_disk_index_partition_counts(dgnn_ctx* ctx, const dgnn_disk_index* idx, int64_t part_rows,
                                             int64_t nparts, int64_t* counts_host);
dgnn_status dgnn_pack_partition(dgnn_ctx* ctx, const dgnn_disk_index* idx, const void* part, int64_t p0, int64_t p1,
                                int64_t row_bytes, const int64_t* chunk_off, void* group_buf);
dgnn_status dgnn_pack_tails(dgnn_ctx* ctx, const dgnn_disk_index* idx, int64_t row_bytes, const int64_t* chunk_off,
                            void* group_buf);

/* ------------------------------------------------ trainer stub (NEXT #2) ---- */
/* The model-training stage of the pipeline with the surrogate of Eq. 1
 * that SPEC S:409-413 fixes: h^k_v = h^{k-1}_v + mean{h^{k-1}_u : u in N(v)}, no W, no sigma.
 * Reading t1: layer k = 1..H handles sampling hop h = H-k (deepest first); N(v) = v's sampled
 * neighbours at the hop v expanded in (src_local); a node outside hop h, or without edges,
 * keeps its value.  For DGNN_SAMPLE_BLOCKS samples, hop h's destinations are every node of
 * local index < hop_off[b][h+1] with their hop-h edges.  fp32: the sum starts at 0 and adds neighbours in edge order, then one
 * IEEE division by the edge count and one addition (bit-identical to the oracle).
 *   x    device fp32 [node_off[b_hi] - node_off[b_lo], dim]: the assembled rows of batches
 *        [b_lo, b_hi) in node order, updated IN PLACE; afterwards the rows of each batch's
 *        seeds (local [0, hop_off[b][1])) hold the seed embeddings h^H.
 * Enqueued on the ctx stream; scratch comes from the ctx allocator. */
dgnn_status dgnn_train_stub(dgnn_ctx* ctx, const dgnn_samples* samples, int64_t b_lo, int64_t b_hi, float* x,
                            int64_t dim);

#ifdef __cplusplus
}
#endif
#endif /* DGNN_H */
