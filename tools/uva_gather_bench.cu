// uva_gather_bench.cu -- microbenchmark for the a9 design choice: how fast can
// SMs gather random rows out of pinned host memory over PCIe (UVA)?
//   (a) LDG: warp per row, 16 B per lane, U rows in flight per warp
//   (b) TMA: cp.async.bulk global->shared of whole rows (1-D bulk copies),
//       then a bulk shared->global store of the staged tile
//   (c) copy engine: cudaMemcpyAsync of one contiguous block (the ceiling)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o uva tools/uva_gather_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void __launch_bounds__(256) ldg_gather(const uint4* __restrict__ src, const int* __restrict__ idx, int64_t n,
                                                  int vec_per_row, uint4* __restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = warp * U; r0 < n; r0 += nw * U) {
        for (int q0 = 0; q0 < vec_per_row; q0 += 32) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t r = r0 + u;
                if (r < n && q0 + lane < vec_per_row) v[u] = __ldg(src + (int64_t)idx[r] * vec_per_row + q0 + lane);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t r = r0 + u;
                if (r < n && q0 + lane < vec_per_row) __stcs(dst + r * vec_per_row + q0 + lane, v[u]);
            }
        }
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(bar)),
        "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
                 "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// one CTA = one warp; per stage: T rows of row_bytes each, double buffered
template <int T>
__global__ void __launch_bounds__(32) tma_gather(const uint8_t* __restrict__ src, const int* __restrict__ idx,
                                                 int64_t n, int row_bytes, uint8_t* __restrict__ dst) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[2];
    const int lane = threadIdx.x;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    uint32_t phase[2] = {0, 0};
    const int64_t tiles = (n + T - 1) / T;
    int s = 0;
    int64_t prev = -1;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t r0 = t * T;
        const int rows = (int)min((int64_t)T, n - r0);
        uint8_t* buf = smem + (size_t)s * T * row_bytes;
        if (lane == 0) {
            bulk_wait_read0();  // buffer s was last stored from 2 tiles ago
            mbar_expect_tx(&bar[s], rows * row_bytes);
        }
        __syncwarp();
        for (int r = lane; r < rows; r += 32) bulk_g2s(buf + (size_t)r * row_bytes, src + (int64_t)idx[r0 + r] * row_bytes,
                                                       row_bytes, &bar[s]);
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
        if (lane == 0) bulk_s2g(dst + r0 * row_bytes, buf, rows * row_bytes);
        s ^= 1;
        prev = t;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const int64_t table_rows = 11'100'000;
    std::vector<int> row_sizes = {512, 1024, 4096};
    for (int rb : row_sizes) {
        const int64_t trows = table_rows * 512 / rb;
        const int64_t n = (int64_t)(2LL << 30) / rb;  // 2 GiB gathered
        uint8_t* host;
        CK(cudaHostAlloc((void**)&host, trows * rb, cudaHostAllocMapped | cudaHostAllocPortable));
        memset(host, 1, trows * rb);
        std::vector<int> hidx(n);
        srand(1);
        for (int64_t i = 0; i < n; ++i) hidx[i] = (int)(((uint64_t)rand() * 2654435761ULL) % trows);
        int* idx;
        uint8_t* dst;
        CK(cudaMalloc(&idx, n * 4));
        CK(cudaMalloc(&dst, n * rb));
        CK(cudaMemcpy(idx, hidx.data(), n * 4, cudaMemcpyHostToDevice));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms;
        auto report = [&](const char* name) {
            cudaEventElapsedTime(&ms, a, b);
            printf("rb=%5d %-28s %7.2f GB/s\n", rb, name, n * (double)rb / (ms / 1e3) / 1e9);
        };
        for (int bps : {1, 2, 4, 8}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                ldg_gather<4><<<148 * bps, 256>>>((const uint4*)host, idx, n, rb / 16, (uint4*)dst);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
            }
            char nm[64];
            snprintf(nm, 64, "LDG U=4 %d CTA/SM", bps);
            report(nm);
        }
        for (int ctas : {148 * 4, 148 * 8, 148 * 16}) {
            const int T = 16;
            size_t sm = (size_t)2 * T * rb;
            CK(cudaFuncSetAttribute(tma_gather<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                tma_gather<16><<<ctas, 32, sm>>>(host, idx, n, rb, dst);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                CK(cudaGetLastError());
            }
            char nm[64];
            snprintf(nm, 64, "TMA bulk T=16 ctas=%d", ctas);
            report(nm);
        }
        cudaEventRecord(a);
        CK(cudaMemcpyAsync(dst, host, n * rb, cudaMemcpyHostToDevice));
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        report("copy engine contiguous");
        if (rb == 512) {
            // interference: the gather (H2D reads) while a D2H copy engine stream writes host memory
            uint8_t* hd2h;
            const size_t d2h_bytes = (size_t)4 << 30;
            uint8_t* dsrc;
            CK(cudaHostAlloc((void**)&hd2h, d2h_bytes, cudaHostAllocPortable));
            CK(cudaMalloc(&dsrc, d2h_bytes));
            cudaStream_t s1, s2;
            cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
            cudaEvent_t c0, c1;
            cudaEventCreate(&c0);
            cudaEventCreate(&c1);
            for (int bps : {2, 8}) {
                cudaEventRecord(c0, s2);
                CK(cudaMemcpyAsync(hd2h, dsrc, d2h_bytes, cudaMemcpyDeviceToHost, s2));
                cudaEventRecord(c1, s2);
                cudaEventRecord(a, s1);
                ldg_gather<4><<<148 * bps, 256, 0, s1>>>((const uint4*)host, idx, n, rb / 16, (uint4*)dst);
                cudaEventRecord(b, s1);
                CK(cudaDeviceSynchronize());
                float ms2;
                cudaEventElapsedTime(&ms2, c0, c1);
                char nm[64];
                snprintf(nm, 64, "LDG %d CTA/SM + D2H copy", bps);
                report(nm);
                printf("          concurrent D2H copy %7.2f GB/s\n", d2h_bytes / (ms2 / 1e3) / 1e9);
            }
            cudaFreeHost(hd2h);
            cudaFree(dsrc);
        }
        // correctness spot check of the TMA path
        std::vector<uint8_t> chk(rb);
        CK(cudaMemcpy(chk.data(), dst + (n / 2) * rb, rb, cudaMemcpyDeviceToHost));
        if (chk[0] != 1 || chk[rb - 1] != 1) printf("TMA/copy result mismatch\n");
        cudaFree(idx);
        cudaFree(dst);
        cudaFreeHost(host);
    }
    return 0;
}
