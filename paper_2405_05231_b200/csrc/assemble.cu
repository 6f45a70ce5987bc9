// assemble.cu -- a9: feature assembly of one mini-batch.
// P:303-305 (Sec. 4, Fig. 3): "the GPU reads the GPU cache, CPU cache, and
// partial input to obtain all the required features"; P:488 (Sec. 6): UVA
// fetches of CPU-resident features.  out[j] = row(addr[j]) with addr from
// dgnn_classify (reading c18).
//
// One warp-per-row gather over three sources: GPU-tier rows from HBM, host-tier
// rows from pinned host memory read directly over PCIe through UVA (no staging
// copy), disk-tier rows from the batch's staged chunk (HBM after the side-stream
// H2D of a8, or pinned host).  An address whose slot is beyond its tier writes
// a zero row and raises DGNN_ERANGE at the next dgnn_ctx_sync.
#include "rowcopy.cuh"

namespace dgnn {
namespace {

constexpr int kAsmU = 4;

struct AsmRow {
    const uint32_t* addr;
    const uint8_t* gpu;
    int64_t kg;
    const uint8_t* host;
    int64_t kh;
    const uint8_t* chunk;
    int64_t cr;
    int64_t row_bytes;
    uint8_t* out;
    int* err;
    __device__ __forceinline__ bool operator()(int64_t j, const uint8_t*& s, uint8_t*& d) const {
        const uint32_t a = addr[j];
        const uint32_t tier = a >> DGNN_TIER_SHIFT;
        const int64_t slot = a & DGNN_SLOT_MASK;
        d = out + j * row_bytes;
        if (tier == DGNN_TIER_GPU && slot < kg) s = gpu + slot * row_bytes;
        else if (tier == DGNN_TIER_HOST && slot < kh) s = host + slot * row_bytes;
        else if (tier == DGNN_TIER_DISK && slot < cr) s = chunk + slot * row_bytes;
        else {
            atomicOr(err, DEVERR_ADDR_RANGE);
            s = nullptr;
            return false;
        }
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256) k_assemble(AsmRow fn, int64_t n) {
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(n, fn.row_bytes, fn, warp, nwarps);
}

// A run of consecutive batches in one launch: row j belongs to batch b =
// segment(node_off, j); its DISK slot indexes that batch's chunk at
// chunk_base + chunk_off[b] (chunks of consecutive batches are contiguous in
// the disk tier, so one staging copy brings the whole run).
constexpr int kMaxSeg = 1024;

struct AsmGroupRow {
    const uint32_t* addr;
    const int64_t* node_off;   // [nb+1] relative to addr (smem copy)
    const int64_t* chunk_off;  // [nb+1] byte offsets relative to chunk_base
    const int64_t* chunk_rows; // [nb+1] exclusive prefix of packed rows
    int nb;
    const uint8_t* gpu;
    int64_t kg;
    const uint8_t* host;
    int64_t kh;
    const uint8_t* chunk_base;
    int64_t row_bytes;
    uint8_t* out;
    int* err;
    __device__ __forceinline__ bool operator()(int64_t j, const uint8_t*& s, uint8_t*& d) const {
        const uint32_t a = addr[j];
        const uint32_t tier = a >> DGNN_TIER_SHIFT;
        const int64_t slot = a & DGNN_SLOT_MASK;
        d = out + j * row_bytes;
        if (tier == DGNN_TIER_GPU && slot < kg) {
            s = gpu + slot * row_bytes;
        } else if (tier == DGNN_TIER_HOST && slot < kh) {
            s = host + slot * row_bytes;
        } else if (tier == DGNN_TIER_DISK) {
            const int b = segment_of(node_off, nb + 1, j);
            if (slot >= chunk_rows[b + 1] - chunk_rows[b]) {
                atomicOr(err, DEVERR_ADDR_RANGE);
                s = nullptr;
                return false;
            }
            s = chunk_base + chunk_off[b] + slot * row_bytes;
        } else {
            atomicOr(err, DEVERR_ADDR_RANGE);
            s = nullptr;
            return false;
        }
        return true;
    }
};

template <class V>
__global__ void __launch_bounds__(256) k_assemble_group(AsmGroupRow fn, int64_t n) {
    __shared__ int64_t s_no[kMaxSeg + 1], s_co[kMaxSeg + 1], s_cr[kMaxSeg + 1];
    if (fn.nb <= kMaxSeg) {
        for (int i = threadIdx.x; i <= fn.nb; i += blockDim.x) {
            s_no[i] = fn.node_off[i];
            s_co[i] = fn.chunk_off[i];
            s_cr[i] = fn.chunk_rows[i];
        }
        __syncthreads();
        fn.node_off = s_no;
        fn.chunk_off = s_co;
        fn.chunk_rows = s_cr;
    }
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    copy_rows_warp<kAsmU, V>(n, fn.row_bytes, fn, warp, nwarps);
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_assemble(dgnn_ctx* c, const uint32_t* addr, int64_t n, const void* gpu_tier, int64_t k_gpu,
                                     const void* host_tier, int64_t k_host, const void* chunk, int64_t chunk_rows,
                                     int64_t row_bytes, void* out) {
    DGNN_REQUIRE(c && (n == 0 || (addr && out)), "dgnn_assemble: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0 && k_gpu >= 0 && k_host >= 0 && chunk_rows >= 0,
                 "dgnn_assemble: bad sizes");
    DGNN_REQUIRE((k_gpu == 0 || gpu_tier) && (k_host == 0 || host_tier) && (chunk_rows == 0 || chunk),
                 "dgnn_assemble: a non-empty source is NULL");
    if (n == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(gpu_tier) && al16(host_tier) && al16(chunk) && al16(out);
    AsmRow fn{addr,        (const uint8_t*)gpu_tier, k_gpu,     (const uint8_t*)host_tier, k_host, (const uint8_t*)chunk,
              chunk_rows,  row_bytes,                (uint8_t*)out, c->dev_err};
    const int grid = grid_for(c, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_assemble_group(dgnn_ctx* c, const uint32_t* addr, const int64_t* node_off, int64_t nb,
                                           int64_t n, const void* gpu_tier, int64_t k_gpu, const void* host_tier,
                                           int64_t k_host, const void* chunk_base, const int64_t* chunk_off,
                                           const int64_t* chunk_rows, int64_t row_bytes, void* out) {
    DGNN_REQUIRE(c && (n == 0 || (addr && out && node_off && chunk_off && chunk_rows)),
                 "dgnn_assemble_group: NULL argument");
    DGNN_REQUIRE(row_bytes > 0 && row_bytes % 4 == 0 && n >= 0 && nb >= 0 && nb < (1 << 30) && k_gpu >= 0 &&
                     k_host >= 0, "dgnn_assemble_group: bad sizes");
    DGNN_REQUIRE((k_gpu == 0 || gpu_tier) && (k_host == 0 || host_tier), "dgnn_assemble_group: NULL tier");
    if (n == 0 || nb == 0) return DGNN_OK;
    DGNN_CK(cudaSetDevice(c->device));
    const bool v16 = row_bytes % 16 == 0 && al16(gpu_tier) && al16(host_tier) && al16(chunk_base) && al16(out);
    AsmGroupRow fn{addr,    node_off, chunk_off, chunk_rows, (int)nb,  (const uint8_t*)gpu_tier, k_gpu,
                   (const uint8_t*)host_tier, k_host, (const uint8_t*)chunk_base, row_bytes, (uint8_t*)out,
                   c->dev_err};
    const int grid = grid_for(c, n * 32 / kAsmU, 256, c->assemble_blocks_per_sm);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble_group<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble_group<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}
