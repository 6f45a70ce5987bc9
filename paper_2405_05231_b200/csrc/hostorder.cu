// hostorder.cu -- the window-ordered host tier ("window-ordered host tier").
//
// a9 reads the host (CPU-cache) tier over PCIe once per window of W consecutive batches: each
// window needs the distinct host rows its batches address (≈ half of the tier at papers scale,
// W = 128), scattered over the tier in slot order, so an SM-driven UVA gather moves them at
// ~0.7-0.8 of the link rate.  The paper reorders its disk cache so that the rows one segment of
// batches needs share pages (Sec. 5.1, Algorithm 1); here the windows are known when the
// layout is built, so the host tier can be ordered exactly: slot s gets the window-membership mask
// m(s) (bit w = some batch of window w addresses s), and the tier is laid out physically in
// (brev(m(s)), s) order -- masks with their window bits reversed, window 0 most significant.  Rows with equal masks form one contiguous group; window w needs exactly the
// groups whose mask has bit w, i.e. a few hundred contiguous ranges, which the copy engine moves
// at the full link rate.  Slots, tier_map and every address stay as the oracle defines them
// (reading c17); only the physical row of a slot changes, and every reader goes through a map.
//
//   dgnn_host_order         masks, physical order (radix sort), phys_ids for the tier fill, groups
//   dgnn_host_order_ranges  host: window w's physical ranges and their staging offsets
//   dgnn_host_window_ranges smap[slot] = staging row of the slot in window w
//   dgnn_copy_ranges        the copy-engine copies of a window's ranges (H2D)
//   dgnn_remap_ids_dev      ids[i] = table[ids[i]] (slot -> physical row for the generic gather)
#include <algorithm>
#include <cstdlib>
#include <array>
#include <utility>
#include <vector>

#include "internal.cuh"
#include "rowcopy.cuh"

namespace dgnn {
namespace {

// (host tier read from the feature table itself) one row per staging row of a window's copies:
// row r of the copy list lies in triple t (prefix[t] <= r < prefix[t+1]); its source is the table
// row of the node at physical row lo_t + k, its destination staging row st_t + k
struct RangeRow {
    const uint8_t* table;
    int64_t row_bytes;
    const int32_t* ids;     // physical row -> node id
    const int64_t* tri;     // (phys_lo, phys_hi, staging_lo) triples
    const int64_t* prefix;  // [nr + 1] rows before each triple
    int64_t nr;
    uint8_t* dst;
    __device__ __forceinline__ bool operator()(int64_t r, const uint8_t*& s, uint8_t*& d) const {
        int64_t lo = 0, hi = nr;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (prefix[mid] <= r) lo = mid;
            else hi = mid;
        }
        const int64_t k = r - prefix[lo];
        s = table + (int64_t)ids[tri[3 * lo] + k] * row_bytes;
        d = dst + (tri[3 * lo + 2] + k) * row_bytes;
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256) k_gather_ranges(RangeRow f, int64_t R) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<8, V>(R, f.row_bytes, f, warp, nwarps);
}

__global__ void k_host_masks(const uint32_t* __restrict__ addr, int64_t n, uint32_t bit, int64_t kh,
                             uint32_t* __restrict__ mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = addr[i];
        const int64_t slot = a & DGNN_SLOT_MASK;
        if ((a >> DGNN_TIER_SHIFT) == DGNN_TIER_HOST && slot < kh && !(mask[slot] & bit)) atomicOr(&mask[slot], bit);
    }
}

// sort key of a mask: its nwin bits reversed, so window 0 is the most significant -- the rows of
// window 0 (the first one the assembler stages, and the one staged ahead of it) are one
// contiguous range at the end of the physical order
__device__ __forceinline__ uint32_t mask_key(uint32_t m, int nwin) { return __brev(m) >> (32 - nwin); }

__global__ void k_mask_keys(const uint32_t* __restrict__ mask, int64_t n, int nwin, uint32_t* __restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = mask_key(mask[i], nwin);
}

__global__ void k_iota(uint32_t* __restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

__global__ void k_phys(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sslot, int64_t kh,
                       const int32_t* __restrict__ host_ids, int32_t* __restrict__ phys_ids,
                       int32_t* __restrict__ phys_of_slot) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kh; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = sslot[i];
        phys_of_slot[s] = (int32_t)i;
        phys_ids[i] = host_ids[s];
    }
}

__global__ void k_window_smap(const uint32_t* __restrict__ mask, const int32_t* __restrict__ phys_of_slot, int64_t kh,
                              uint32_t bit, const int64_t* __restrict__ ranges, int nr, int32_t* __restrict__ smap) {
    extern __shared__ int64_t s_rg[];  // [3 * nr]: phys_lo, phys_hi, stage_lo
    for (int i = threadIdx.x; i < 3 * nr; i += blockDim.x) s_rg[i] = ranges[i];
    __syncthreads();
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < kh; s += (int64_t)gridDim.x * blockDim.x) {
        if (!(mask[s] & bit)) continue;
        const int64_t p = phys_of_slot[s];
        int lo = 0, hi = nr;  // the range with phys_lo <= p
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_rg[3 * mid] <= p) lo = mid;
            else hi = mid;
        }
        smap[s] = (int32_t)(s_rg[3 * lo + 2] + (p - s_rg[3 * lo]));
    }
}

__global__ void k_remap_ids(int32_t* __restrict__ ids, const int64_t* __restrict__ n_dev, int64_t n_max,
                            const int32_t* __restrict__ table) {
    const int64_t n = min(*n_dev, n_max);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ids[i] = table[ids[i]];
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_host_order(dgnn_ctx* c, const uint32_t* addr, const int64_t* win_node_off_host,
                                       int32_t nwin, const int32_t* host_ids, int64_t k_host, int32_t* phys_ids,
                                       int32_t* phys_of_slot, uint32_t* slot_mask, int64_t max_groups,
                                       int64_t* group_start_host, uint32_t* group_mask_host, int64_t* n_groups) {
    DGNN_REQUIRE(c && win_node_off_host && n_groups && nwin >= 1 && nwin <= 32 && k_host >= 0 && max_groups >= 1,
                 "dgnn_host_order: bad argument (1 <= nwin <= 32)");
    DGNN_REQUIRE(k_host == 0 || (host_ids && phys_ids && phys_of_slot && slot_mask && group_start_host && group_mask_host),
                 "dgnn_host_order: NULL array");
    DGNN_REQUIRE(win_node_off_host[nwin] == 0 || addr, "dgnn_host_order: NULL addr");
    *n_groups = 0;
    if (k_host == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_TRY(memset_async(c, slot_mask, 0, sizeof(uint32_t) * (size_t)k_host));
    for (int w = 0; w < nwin; ++w) {
        const int64_t a = win_node_off_host[w], n = win_node_off_host[w + 1] - a;
        DGNN_REQUIRE(n >= 0, "dgnn_host_order: window node offsets must be non-decreasing");
        if (n == 0) continue;
        launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] {
            k_host_masks<<<grid_for(c, n, 256), 256, 0, c->stream>>>(addr + a, n, 1u << w, k_host, slot_mask);
        });
        DGNN_CK_LAUNCH();
    }
    // physical order: slots sorted by (reversed mask, slot) -- a stable radix sort on nwin bits
    DevBuf<uint32_t> keys, vals, keys_alt, vals_alt;
    DGNN_TRY(keys.alloc_kept(c, (size_t)k_host));
    DGNN_TRY(vals.alloc_kept(c, (size_t)k_host));
    DGNN_TRY(keys_alt.alloc_kept(c, (size_t)k_host));
    DGNN_TRY(vals_alt.alloc_kept(c, (size_t)k_host));
    launch(c, DGNN_K_MISC, 0.0, [&] {
        k_mask_keys<<<grid_for(c, k_host, 256), 256, 0, c->stream>>>(slot_mask, k_host, nwin, keys.p);
    });
    DGNN_CK_LAUNCH();
    launch(c, DGNN_K_MISC, 0.0, [&] { k_iota<<<grid_for(c, k_host, 256), 256, 0, c->stream>>>(vals.p, k_host); });
    DGNN_CK_LAUNCH();
    uint32_t *k0 = keys.p, *v0 = vals.p, *k1 = keys_alt.p, *v1 = vals_alt.p;
    DGNN_TRY(radix::sort_pairs(c, k_host, nwin, &k0, &v0, &k1, &v1));
    launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] {
        k_phys<<<grid_for(c, k_host, 256), 256, 0, c->stream>>>(k0, v0, k_host, host_ids, phys_ids, phys_of_slot);
    });
    DGNN_CK_LAUNCH();
    // groups: maximal runs of equal mask in physical order (compacted with one scan)
    DevBuf<int64_t> gstart, total;
    DevBuf<uint32_t> gmask;
    DGNN_TRY(gstart.alloc(c, (size_t)max_groups));
    DGNN_TRY(gmask.alloc(c, (size_t)max_groups));
    DGNN_TRY(total.alloc(c, 1));
    {
        const uint32_t* sk = k0;
        int64_t* gs = gstart.p;
        uint32_t* gm = gmask.p;
        const int64_t cap = max_groups;
        const int nw = nwin;
        auto in = [=] __device__(int64_t i) -> int32_t { return (i == 0 || sk[i] != sk[i - 1]) ? 1 : 0; };
        auto out = [=] __device__(int64_t i, int64_t excl, int64_t v) {
            if (v && excl < cap) {
                gs[excl] = i;
                gm[excl] = mask_key(sk[i], nw);  // (bit reversal is its own inverse)
            }
        };
        DGNN_TRY(scan::run(c, k_host, nullptr, in, out, total.p));
    }
    int64_t ng = 0;
    DGNN_TRY(read_small(c, &ng, total.p, sizeof(int64_t)));
    *n_groups = ng;
    if (ng > max_groups) {
        set_error("dgnn_host_order: %lld mask groups exceed max_groups %lld", (long long)ng, (long long)max_groups);
        return DGNN_ERANGE;
    }
    DGNN_TRY(read_small(c, group_start_host, gstart.p, sizeof(int64_t) * (size_t)ng));
    DGNN_TRY(read_small(c, group_mask_host, gmask.p, sizeof(uint32_t) * (size_t)ng));
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_host_order_ranges(const int64_t* group_start_host, const uint32_t* group_mask_host,
                                              int64_t n_groups, int64_t k_host, int32_t window, int64_t* ranges_host,
                                              int64_t capacity, int64_t* n_ranges, int64_t* rows) {
    DGNN_REQUIRE(n_ranges && rows && n_groups >= 0 && window >= 0 && window < 32 && capacity >= 0 &&
                     (n_groups == 0 || (group_start_host && group_mask_host)) && (capacity == 0 || ranges_host),
                 "dgnn_host_order_ranges: bad argument");
    int64_t nr = 0, stage = 0;
    for (int64_t g = 0; g < n_groups; ++g) {
        if (!((group_mask_host[g] >> window) & 1u)) continue;
        const int64_t lo = group_start_host[g], hi = g + 1 < n_groups ? group_start_host[g + 1] : k_host;
        if (nr > 0 && ranges_host[3 * (nr - 1) + 1] == lo) {
            ranges_host[3 * (nr - 1) + 1] = hi;  // adjacent group: one longer range
        } else {
            DGNN_REQUIRE(nr < capacity, "dgnn_host_order_ranges: more than %lld ranges", (long long)capacity);
            ranges_host[3 * nr] = lo;
            ranges_host[3 * nr + 1] = hi;
            ranges_host[3 * nr + 2] = stage;
            ++nr;
        }
        stage += hi - lo;
    }
    *n_ranges = nr;
    *rows = stage;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_host_window_ranges(dgnn_ctx* c, const uint32_t* slot_mask, const int32_t* phys_of_slot,
                                               int64_t k_host, int32_t window, const int64_t* ranges_dev, int64_t nr,
                                               int32_t* smap) {
    DGNN_REQUIRE(c && window >= 0 && window < 32 && nr >= 0 && k_host >= 0 &&
                     (k_host == 0 || (slot_mask && phys_of_slot && smap)) && (nr == 0 || ranges_dev),
                 "dgnn_host_window_ranges: bad argument");
    DGNN_REQUIRE(nr <= 4096, "dgnn_host_window_ranges: at most 4096 ranges per window");
    if (k_host == 0 || nr == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const size_t smem = sizeof(int64_t) * 3 * (size_t)nr;
    if (smem > 48 * 1024)
        DGNN_CK(cudaFuncSetAttribute(k_window_smap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] {
        k_window_smap<<<grid_for(c, k_host, 256), 256, smem, c->stream>>>(slot_mask, phys_of_slot, k_host, 1u << window,
                                                                          ranges_dev, (int)nr, smap);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_copy_ranges(dgnn_ctx* c, void* dst_dev, const void* src_host, const int64_t* ranges_host,
                                        int64_t nr, int64_t row_bytes) {
    DGNN_REQUIRE(c && row_bytes > 0 && nr >= 0 && (nr == 0 || (dst_dev && src_host && ranges_host)),
                 "dgnn_copy_ranges: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    if (nr == 0) return DGNN_OK;
    for (int64_t r = 0; r < nr; ++r) {
        const int64_t lo = ranges_host[3 * r], hi = ranges_host[3 * r + 1], st = ranges_host[3 * r + 2];
        DGNN_REQUIRE(hi >= lo && st >= 0, "dgnn_copy_ranges: bad range");
        if (hi == lo) continue;
        DGNN_CK(cudaMemcpyAsync((uint8_t*)dst_dev + st * row_bytes, (const uint8_t*)src_host + lo * row_bytes,
                                (size_t)((hi - lo) * row_bytes), cudaMemcpyHostToDevice, c->stream));
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_gather_ranges(dgnn_ctx* c, const void* table, int64_t row_bytes, const int32_t* ids,
                                          const int64_t* ranges_dev, const int64_t* prefix_dev, int64_t nr,
                                          int64_t total_rows, void* dst_dev) {
    DGNN_REQUIRE(c && row_bytes > 0 && row_bytes % 4 == 0 && nr >= 0 && total_rows >= 0 &&
                     (total_rows == 0 || (table && ids && ranges_dev && prefix_dev && dst_dev && nr > 0)),
                 "dgnn_gather_ranges: bad argument");
    if (total_rows == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const RangeRow f{static_cast<const uint8_t*>(table), row_bytes, ids, ranges_dev, prefix_dev, nr,
                     static_cast<uint8_t*>(dst_dev)};
    const bool v16 = row_bytes % 16 == 0 && ((uintptr_t)table & 15) == 0 && ((uintptr_t)dst_dev & 15) == 0;
    const int grid = v16 ? grid_resident(c, k_gather_ranges<uint4>, total_rows * 32 / 8, 256, c->assemble_blocks_per_sm)
                         : grid_resident(c, k_gather_ranges<uint32_t>, total_rows * 32 / 8, 256,
                                         c->assemble_blocks_per_sm);
    launch(c, DGNN_K_HOST_GATHER, (double)total_rows * row_bytes, [&] {
        if (v16) k_gather_ranges<uint4><<<grid, 256, 0, c->stream>>>(f, total_rows);
        else k_gather_ranges<uint32_t><<<grid, 256, 0, c->stream>>>(f, total_rows);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_remap_ids_dev(dgnn_ctx* c, int32_t* ids, const int64_t* n_dev, int64_t n_max,
                                          const int32_t* table) {
    DGNN_REQUIRE(c && n_dev && n_max >= 0 && (n_max == 0 || (ids && table)), "dgnn_remap_ids_dev: bad argument");
    if (n_max == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    launch(c, DGNN_K_HOST_WINDOW, 0.0, [&] {
        k_remap_ids<<<grid_for(c, n_max, 256), 256, 0, c->stream>>>(ids, n_dev, n_max, table);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

// The staging schedule of the ordered windows: a row needed by consecutive windows stays in the
// HBM staging arena between them instead of crossing PCIe once per window.  A group (equal mask)
// is needed by the maximal runs [a, b] of consecutive set bits of its mask; each (group, run) is
// one "item", copied when window a is prefetched and resident until window b is done.  The
// assembler prefetches window w once window w-2's runs are done (while w-1's execute), so at that
// point the items ending at or before w-2 are freed and the items starting at w are placed in
// free staging rows (split over free fragments as needed: a copy is a range of physical rows).
// capacity_rows >= max_w |S_{w-1}| + |S_w| always suffices (both windows' rows resident).
// Spare capacity is then spent on bridging: two runs of a group separated by a gap of windows are
// merged into one item (copied once, resident through the gap) when the arena has room for it in
// every window of the gap -- shortest gaps first (a gap of one window costs no extra room at all);
// with capacity_rows >= the rows the windows touch, every row crosses PCIe exactly once per pass.
// Outputs per window (CSR over windows): the copies to issue at its prefetch, and the map of all
// its rows (every resident item whose group it needs), both as (phys_lo, phys_hi, stage_lo) triples,
// the map sorted by phys_lo.
extern "C" dgnn_status dgnn_host_order_schedule(const int64_t* group_start_host, const uint32_t* group_mask_host,
                                                int64_t n_groups, int64_t k_host, int32_t nwin, int64_t capacity_rows,
                                                int64_t* copy_out, int64_t copy_cap, int64_t* copy_off,
                                                int64_t* map_out, int64_t map_cap, int64_t* map_off,
                                                int64_t* rows_copied) {
    DGNN_REQUIRE(n_groups >= 0 && k_host >= 0 && nwin >= 1 && nwin <= 32 && capacity_rows >= 0 && copy_off &&
                     map_off && rows_copied && (n_groups == 0 || (group_start_host && group_mask_host)),
                 "dgnn_host_order_schedule: bad argument");
    struct Item {
        int64_t lo, hi;  // physical rows of the group
        int a, b;        // first and last window it stays resident for
        uint32_t m;      // the group's mask (the windows that read it)
        std::vector<std::pair<int64_t, int64_t>> frag;  // (stage_lo, rows) pieces, in phys order
    };
    // runs of consecutive set bits per group; an item occupies the arena for windows [a, b + 1]
    // (it is released when window b + 2 is prefetched)
    struct Run {
        int64_t g;
        int a, b;
    };
    std::vector<Run> runs;
    std::vector<int64_t> occ(nwin + 1, 0);
    for (int64_t g = 0; g < n_groups; ++g) {
        const uint32_t m = group_mask_host[g];
        const int64_t rows = (g + 1 < n_groups ? group_start_host[g + 1] : k_host) - group_start_host[g];
        for (int w = 0; w < nwin;) {
            if (!((m >> w) & 1u)) {
                ++w;
                continue;
            }
            int e = w;
            while (e + 1 < nwin && ((m >> (e + 1)) & 1u)) ++e;
            runs.push_back(Run{g, w, e});
            for (int x = w; x <= std::min(e + 1, nwin - 1); ++x) occ[x] += rows;
            w = e + 1;
        }
    }
    // bridging: gap k lies between runs k and k + 1 of the same group; bridged[k] merges them
    std::vector<char> bridged(runs.size(), 0);
    const char* nb_env = std::getenv("DGNN_HOST_BRIDGE");  // "0": no bridging (A/B measurement)
    if (!(nb_env && nb_env[0] == '0')) {
        std::vector<size_t> gaps;
        for (size_t k = 0; k + 1 < runs.size(); ++k)
            if (runs[k].g == runs[k + 1].g) gaps.push_back(k);
        std::stable_sort(gaps.begin(), gaps.end(), [&](size_t x, size_t y) {
            return runs[x + 1].a - runs[x].b < runs[y + 1].a - runs[y].b;
        });
        for (size_t k : gaps) {
            const int64_t g = runs[k].g;
            const int64_t rows = (g + 1 < n_groups ? group_start_host[g + 1] : k_host) - group_start_host[g];
            const int w0 = runs[k].b + 2, w1 = runs[k + 1].a - 1;  // windows neither run occupies
            bool fits = true;
            for (int x = w0; x <= w1 && fits; ++x) fits = occ[x] + rows <= capacity_rows;
            if (!fits) continue;
            for (int x = w0; x <= w1; ++x) occ[x] += rows;
            bridged[k] = 1;
        }
    }
    std::vector<Item> items;
    for (size_t k = 0; k < runs.size();) {
        size_t e = k;
        while (bridged[e]) ++e;  // (a bridged gap always has a next run of the same group)
        const int64_t g = runs[k].g;
        const int64_t lo = group_start_host[g], hi = g + 1 < n_groups ? group_start_host[g + 1] : k_host;
        items.push_back(Item{lo, hi, runs[k].a, runs[e].b, group_mask_host[g], {}});
        k = e + 1;
    }
    std::vector<std::pair<int64_t, int64_t>> freel{{0, capacity_rows}};  // [start, end) free staging rows
    int64_t nc = 0, nm = 0, copied = 0;
    auto release = [&](const Item& it) {
        for (auto& f : it.frag) freel.push_back({f.first, f.first + f.second});
        std::sort(freel.begin(), freel.end());
        std::vector<std::pair<int64_t, int64_t>> merged;
        for (auto& f : freel) {
            if (!merged.empty() && merged.back().second == f.first) merged.back().second = f.second;
            else merged.push_back(f);
        }
        freel.swap(merged);
    };
    for (int w = 0; w < nwin; ++w) {
        copy_off[w] = nc;
        for (auto& it : items)
            if (it.b == w - 2) release(it);
        for (auto& it : items) {
            if (it.a != w) continue;
            int64_t need = it.hi - it.lo, p = it.lo;
            while (need > 0) {
                DGNN_REQUIRE(!freel.empty(), "dgnn_host_order_schedule: staging capacity of %lld rows exceeded",
                             (long long)capacity_rows);
                auto& f = freel.front();
                const int64_t take = std::min(need, f.second - f.first);
                it.frag.push_back({f.first, take});
                DGNN_REQUIRE(nc < copy_cap, "dgnn_host_order_schedule: copy_cap too small");
                copy_out[3 * nc] = p;
                copy_out[3 * nc + 1] = p + take;
                copy_out[3 * nc + 2] = f.first;
                ++nc;
                f.first += take;
                if (f.first == f.second) freel.erase(freel.begin());
                p += take;
                need -= take;
                copied += take;
            }
        }
        // the map of window w: every piece of every item covering w, by physical row
        map_off[w] = nm;
        std::vector<std::array<int64_t, 3>> mp;
        for (auto& it : items) {
            if (it.a > w || it.b < w || !((it.m >> w) & 1u)) continue;
            int64_t p = it.lo;
            for (auto& f : it.frag) {
                mp.push_back({p, p + f.second, f.first});
                p += f.second;
            }
        }
        std::sort(mp.begin(), mp.end());
        for (auto& t : mp) {
            DGNN_REQUIRE(nm < map_cap, "dgnn_host_order_schedule: map_cap too small");
            map_out[3 * nm] = t[0];
            map_out[3 * nm + 1] = t[1];
            map_out[3 * nm + 2] = t[2];
            ++nm;
        }
    }
    copy_off[nwin] = nc;
    map_off[nwin] = nm;
    *rows_copied = copied;
    return DGNN_OK;
}
