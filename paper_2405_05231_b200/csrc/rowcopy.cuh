// rowcopy.cuh -- the warp-per-row gather engine shared by a7 (pack, tier
// gather) and a9 (assemble).  Rows are opaque byte strings; each warp moves U
// rows per iteration: lanes < U resolve (src, dst) for one row each, then all
// lanes issue U coalesced 16-byte loads (one row = row_bytes/16 vectors spread
// over the lanes) before the U stores, so every warp keeps U*row_bytes in
// flight.  Loads go through the read-only path (rows shared by several batches
// stay L2-resident); stores are streaming (st.global.cs) because a packed
// chunk is written once and not re-read by this kernel.
#pragma once

#include "internal.cuh"

namespace dgnn {

template <class V>
__device__ __forceinline__ V ld_row(const void* p) {
    return __ldg(reinterpret_cast<const V*>(p));
}
template <>
__device__ __forceinline__ uint4 ld_row<uint4>(const void* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st_row(void* p, uint4 v) { __stcs(reinterpret_cast<uint4*>(p), v); }
__device__ __forceinline__ void st_row(void* p, uint32_t v) { __stcs(reinterpret_cast<unsigned int*>(p), v); }
__device__ __forceinline__ uint4 zero_of(uint4) { return make_uint4(0, 0, 0, 0); }
__device__ __forceinline__ uint32_t zero_of(uint32_t) { return 0u; }

// RowFn: __device__ bool operator()(int64_t r, const uint8_t*& src, uint8_t*& dst) const
// returns false to write a zero row (unresolvable address) -- dst must still be set;
// dst == nullptr skips the row (written by someone else, e.g. a remote GPU-tier row).
template <int U, class V, class RowFn>
__device__ __forceinline__ void copy_rows_warp(int64_t R, int64_t row_bytes, const RowFn& fn, int64_t warp_id,
                                               int64_t nwarps) {
    const int lane = threadIdx.x & 31;
    const int nvec = (int)(row_bytes / (int64_t)sizeof(V));
    for (int64_t r0 = warp_id * U; r0 < R; r0 += nwarps * U) {
        const uint8_t* my_src = nullptr;
        uint8_t* my_dst = nullptr;
        bool my_ok = false;
        if (lane < U && r0 + lane < R) my_ok = fn(r0 + lane, my_src, my_dst);
        const uint8_t* src[U];
        uint8_t* dst[U];
        bool ok[U], live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            src[u] = (const uint8_t*)__shfl_sync(0xffffffffu, (unsigned long long)my_src, u);
            dst[u] = (uint8_t*)__shfl_sync(0xffffffffu, (unsigned long long)my_dst, u);
            ok[u] = __shfl_sync(0xffffffffu, my_ok, u);
            live[u] = r0 + u < R && dst[u] != nullptr;
        }
        for (int q0 = 0; q0 < nvec; q0 += 32) {
            const int q = q0 + lane;
            const bool in = q < nvec;
            V v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = (in && live[u] && ok[u]) ? ld_row<V>(src[u] + (int64_t)q * sizeof(V)) : zero_of(V{});
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (in && live[u]) st_row(dst[u] + (int64_t)q * sizeof(V), v[u]);
        }
    }
}

}  // namespace dgnn
