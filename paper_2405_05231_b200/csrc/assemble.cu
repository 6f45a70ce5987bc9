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
    const int grid = grid_for(c, n * 32 / kAsmU, 256, 8);
    launch(c, DGNN_K_ASSEMBLE, (double)n * (2.0 * row_bytes + 4.0), [&] {
        if (v16) k_assemble<uint4><<<grid, 256, 0, c->stream>>>(fn, n);
        else k_assemble<uint32_t><<<grid, 256, 0, c->stream>>>(fn, n);
    });
    DGNN_CK_LAUNCH();
    return DGNN_OK;
}
