// cache.cu -- a4-a5: popularity ranking and tier selection.
// P:226 (Sec. 3): "rank the nodes by their access frequencies and cache more
// popular nodes in faster memory ... optimal in that it minimizes the total
// number of node features fetched from the disk"; P:275-277 (Sec. 4): GPU
// cache = most popular, CPU cache = second most popular.  Semantics: readings
// c15-c19 (rank by (count desc, ID asc), zero counts never cached, slots in
// ascending ID).
//
// Design: a count-value histogram (shared-memory privatized) gives, on the
// host, the number of nodes ranked above every count value; only the (at most
// two) count values that straddle a tier boundary need per-node tie ranks,
// which one decoupled look-back scan provides (two 31-bit counters packed in
// one int64).  A second scan assigns ascending-ID slots and writes tier_map and
// the tier ID lists.  Traffic ~ 6 x 4N bytes; no sort.
#include <algorithm>

#include "internal.cuh"

namespace dgnn {
namespace {

constexpr int kSmemBins = 8192;
constexpr uint32_t kMaxCount = 1u << 24;
constexpr int64_t kLo31 = (1ll << 31) - 1;

__global__ void k_count_max(const uint32_t* __restrict__ counts, int64_t N, unsigned int* mx) {
    uint32_t m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, counts[i]);
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

__global__ void __launch_bounds__(512) k_count_hist(const uint32_t* __restrict__ counts, int64_t N, uint32_t nbins,
                                                    unsigned int* __restrict__ hist) {
    __shared__ unsigned int sh[kSmemBins];
    const uint32_t sbins = nbins < (uint32_t)kSmemBins ? nbins : (uint32_t)kSmemBins;
    for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = counts[i];
        if (c < sbins) atomicAdd(&sh[c], 1u);
        else atomicAdd(&hist[c], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_build_cache(dgnn_ctx* c, const uint32_t* counts, int64_t N, int64_t gpu_rows,
                                        int64_t host_rows, dgnn_cache_plan** out) {
    DGNN_REQUIRE(c && counts && out, "dgnn_build_cache: NULL argument");
    *out = nullptr;
    DGNN_REQUIRE(N > 0 && N < ((int64_t)1 << DGNN_TIER_SHIFT), "dgnn_build_cache: num_nodes must be in [1, 2^30)");
    DGNN_REQUIRE(gpu_rows >= 0 && host_rows >= 0, "dgnn_build_cache: negative capacity");
    DGNN_CK(cudaSetDevice(c->device));

    // ---- a4: max count, then the histogram of count values ----
    DevBuf<unsigned int> d_max;
    DGNN_TRY(d_max.alloc(c, 1));
    DGNN_TRY(memset_async(c, d_max.p, 0, sizeof(unsigned int)));
    launch(c, DGNN_K_CACHE_HIST, 4.0 * N, [&] {
        k_count_max<<<grid_for(c, N, 256, 8), 256, 0, c->stream>>>(counts, N, d_max.p);
    });
    DGNN_CK_LAUNCH();
    unsigned int mx = 0;
    DGNN_TRY(read_small(c, &mx, d_max.p, sizeof(mx)));
    if (mx >= kMaxCount) {
        set_error("dgnn_build_cache: max count %u >= 2^24 is outside the supported envelope", mx);
        return DGNN_EUNSUPPORTED;
    }
    const uint32_t nbins = mx + 1;
    DevBuf<unsigned int> d_hist;
    DGNN_TRY(d_hist.alloc(c, nbins));
    DGNN_TRY(memset_async(c, d_hist.p, 0, sizeof(unsigned int) * nbins));
    launch(c, DGNN_K_CACHE_HIST, 4.0 * N, [&] {
        k_count_hist<<<c->num_sms * 2, 512, 0, c->stream>>>(counts, N, nbins, d_hist.p);
    });
    DGNN_CK_LAUNCH();
    std::vector<unsigned int> hist(nbins);
    DGNN_TRY(read_small(c, hist.data(), d_hist.p, sizeof(unsigned int) * nbins));

    // ---- host: ranks above each count value, capacities and boundary values ----
    const int64_t nnz = N - (int64_t)hist[0];
    const int64_t kg = std::min(gpu_rows, nnz);
    const int64_t kh = std::min(host_rows, nnz - kg);
    std::vector<int64_t> above(nbins, 0);  // above[c] = #nodes with count > c
    {
        int64_t acc = 0;
        for (int64_t v = (int64_t)nbins - 1; v >= 0; --v) {
            above[v] = acc;
            acc += hist[v];
        }
    }
    auto value_at_rank = [&](int64_t r) -> uint32_t {  // count value of rank r (0-based) among nonzero counts
        for (int64_t v = (int64_t)nbins - 1; v >= 1; --v)
            if (above[v] <= r && r < above[v] + (int64_t)hist[v]) return (uint32_t)v;
        return 0;
    };
    const uint32_t cg = kg > 0 ? value_at_rank(kg - 1) : 0;        // boundary group of the GPU tier
    const uint32_t ch = kh > 0 ? value_at_rank(kg + kh - 1) : 0;   // boundary group of the host tier
    DevBuf<int64_t> d_above;
    DGNN_TRY(d_above.alloc(c, nbins));
    DGNN_TRY(upload_small(c, d_above.p, above.data(), sizeof(int64_t) * nbins));

    auto* P = new dgnn_cache_plan();
    P->ctx = c;
    P->N = N;
    P->k_gpu = kg;
    P->k_host = kh;
    P->gpu_min = cg;
    P->host_min = ch;
    struct Guard {
        dgnn_cache_plan* p;
        ~Guard() { if (p) dgnn_cache_plan_free(p); }
    } guard{P};
    P->tier_map = (uint32_t*)dev_alloc(c, sizeof(uint32_t) * N);
    P->gpu_ids = (int32_t*)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(kg, 1));
    P->host_ids = (int32_t*)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(kh, 1));
    if (!P->tier_map || !P->gpu_ids || !P->host_ids) {
        set_error("dgnn_build_cache: allocation failed");
        return DGNN_ENOMEM;
    }

    // ---- a5 pass 1: tier membership (tie ranks only inside the boundary groups) ----
    {
        const uint32_t* cnt = counts;
        const int64_t* ab = d_above.p;
        uint32_t* tm = P->tier_map;
        const uint32_t bg = kg > 0 ? cg : 0xFFFFFFFFu, bh = kh > 0 ? ch : 0xFFFFFFFFu;
        const int64_t KG = kg, KGH = kg + kh;
        auto in = [=] __device__(int64_t v) -> int64_t {
            const uint32_t x = cnt[v];
            return (int64_t)(x == bg) | ((int64_t)(x == bh) << 31);
        };
        auto outf = [=] __device__(int64_t v, int64_t excl, int64_t) {
            const uint32_t x = cnt[v];
            uint32_t tier = DGNN_TIER_DISK;
            if (x > 0) {
                int64_t rank = ab[x];
                if (x == bg) rank += excl & kLo31;
                else if (x == bh) rank += excl >> 31;
                tier = rank < KG ? DGNN_TIER_GPU : (rank < KGH ? DGNN_TIER_HOST : DGNN_TIER_DISK);
            }
            tm[v] = tier << DGNN_TIER_SHIFT;
        };
        DGNN_TRY(scan::run(c, N, nullptr, in, outf, nullptr));
    }
    // ---- a5 pass 2: ascending-ID slots, tier ID lists ----
    {
        uint32_t* tm = P->tier_map;
        int32_t* gid = P->gpu_ids;
        int32_t* hid = P->host_ids;
        auto in = [=] __device__(int64_t v) -> int64_t {
            const uint32_t t = tm[v] >> DGNN_TIER_SHIFT;
            return (int64_t)(t == DGNN_TIER_GPU) | ((int64_t)(t == DGNN_TIER_HOST) << 31);
        };
        auto outf = [=] __device__(int64_t v, int64_t excl, int64_t val) {
            if (val & kLo31) {
                const int64_t s = excl & kLo31;
                tm[v] = (DGNN_TIER_GPU << DGNN_TIER_SHIFT) | (uint32_t)s;
                gid[s] = (int32_t)v;
            } else if (val) {
                const int64_t s = excl >> 31;
                tm[v] = (DGNN_TIER_HOST << DGNN_TIER_SHIFT) | (uint32_t)s;
                hid[s] = (int32_t)v;
            }
        };
        DGNN_TRY(scan::run(c, N, nullptr, in, outf, nullptr));
    }
    c->launches += 0;
    DGNN_CK(cudaStreamSynchronize(c->stream));  // `above` (host) was a copy source
    *out = P;
    guard.p = nullptr;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_cache_plan_get_info(const dgnn_cache_plan* p, dgnn_plan_info* i) {
    DGNN_REQUIRE(p && i, "dgnn_cache_plan_get_info: NULL argument");
    i->num_nodes = p->N;
    i->k_gpu = p->k_gpu;
    i->k_host = p->k_host;
    i->tier_map = p->tier_map;
    i->gpu_ids = p->gpu_ids;
    i->host_ids = p->host_ids;
    i->gpu_min_count = p->gpu_min;
    i->host_min_count = p->host_min;
    return DGNN_OK;
}

extern "C" void dgnn_cache_plan_free(dgnn_cache_plan* p) {
    if (!p) return;
    if (p->ctx) {
        cudaSetDevice(p->ctx->device);
        dev_free(p->ctx, p->tier_map, sizeof(uint32_t) * p->N);
        dev_free(p->ctx, p->gpu_ids, sizeof(int32_t) * std::max<int64_t>(p->k_gpu, 1));
        dev_free(p->ctx, p->host_ids, sizeof(int32_t) * std::max<int64_t>(p->k_host, 1));
    }
    delete p;
}
