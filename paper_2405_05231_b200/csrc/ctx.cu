#include <algorithm>
// ctx.cu -- context, errors, allocation, statistics and the a8 staging runtime.
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace dgnn {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

dgnn_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e), what, file, line);
    return e == cudaErrorMemoryAllocation ? DGNN_ENOMEM : DGNN_ECUDA;
}

void* dev_alloc(dgnn_ctx* c, size_t bytes) {
    if (c->has_alloc) return c->alloc.alloc(bytes, (void*)c->stream, c->alloc.user);
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, c->stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void dev_free(dgnn_ctx* c, void* p, size_t bytes) {
    if (!p) return;
    if (c->has_alloc) c->alloc.free(p, bytes, (void*)c->stream, c->alloc.user);
    else cudaFreeAsync(p, c->stream);
}

void* keep_take(dgnn_ctx* c, size_t need, size_t* got) {
    if (need == 0) need = 1;
    int best = -1;
    for (int i = 0; i < (int)c->kept.size(); ++i) {
        const size_t b = c->kept[i].bytes;
        if (b >= need && b <= 2 * need + ((size_t)256 << 20) && (best < 0 || b < c->kept[best].bytes)) best = i;
    }
    if (best >= 0) {
        void* p = c->kept[best].p;
        *got = c->kept[best].bytes;
        c->kept_bytes -= *got;
        c->kept.erase(c->kept.begin() + best);
        return p;
    }
    void* p = dev_alloc(c, need);
    if (!p) {
        // the kept buffers are the first thing to give back under memory pressure
        keep_trim(c, 0);
        p = dev_alloc(c, need);
    }
    *got = p ? need : 0;
    return p;
}

void keep_trim(dgnn_ctx* c, size_t limit) {
    while (!c->kept.empty() && c->kept_bytes > limit) {
        dev_free(c, c->kept.front().p, c->kept.front().bytes);
        c->kept_bytes -= c->kept.front().bytes;
        c->kept.erase(c->kept.begin());
    }
}

void keep_put(dgnn_ctx* c, void* p, size_t bytes) {
    if (!p) return;
    if (bytes > c->kept_limit) {
        dev_free(c, p, bytes);
        return;
    }
    c->kept.push_back({p, bytes});
    c->kept_bytes += bytes;
    keep_trim(c, c->kept_limit);
}

cudaEvent_t take_event(dgnn_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void fold_pending(dgnn_ctx* c, bool sync) {
    if (sync) cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            c->stat_ms[p.kid] += ms;
            c->stat_bytes[p.kid] += p.bytes;
            c->stat_n[p.kid] += 1;
        } else {
            cudaGetLastError();
        }
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.clear();
}

dgnn_status memset_async(dgnn_ctx* c, void* p, int value, size_t bytes) {
    if (!bytes) return DGNN_OK;
    DGNN_CK(cudaMemsetAsync(p, value, bytes, c->stream));
    return DGNN_OK;
}

void* pinned_scratch(dgnn_ctx* c, size_t bytes) {
    if (bytes > c->pinned_bytes) {
        if (c->pinned) cudaFreeHost(c->pinned);
        c->pinned = nullptr;
        c->pinned_bytes = 0;
        const size_t n = bytes + bytes / 2 + 4096;
        if (cudaHostAlloc(&c->pinned, n, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            c->pinned = nullptr;
            return nullptr;
        }
        c->pinned_bytes = n;
    }
    return c->pinned;
}

extern std::atomic<int> g_io_error;

namespace {
// word-wise copy into mapped pinned host memory; SM stores go out as posted PCIe writes
__global__ void k_readback(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t nw) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nw; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    __threadfence_system();
}
bool readback_by_copy() {
    static const bool v = [] {
        const char* e = std::getenv("DGNN_SMALL_D2H");
        return e && std::string(e) == "copy";
    }();
    return v;
}
}  // namespace

dgnn_status readback_reserve(dgnn_ctx* c, size_t bytes) {
    if (bytes <= c->rb_bytes) return DGNN_OK;
    if (c->rb) DGNN_CK(cudaFreeHost(c->rb));
    c->rb = nullptr;
    c->rb_bytes = 0;
    const size_t n = std::max<size_t>(bytes + bytes / 2, 64 << 10);
    DGNN_CK(cudaHostAlloc(&c->rb, n, cudaHostAllocMapped | cudaHostAllocPortable));
    c->rb_bytes = n;
    return DGNN_OK;
}

dgnn_status readback_enqueue(dgnn_ctx* c, size_t off, const void* src_dev, size_t n) {
    if (!n) return DGNN_OK;
    if (off + n > c->rb_bytes || (off | n | (size_t)src_dev) % 4) {
        set_error("readback_enqueue: %zu bytes at %zu outside the reserved %zu (or misaligned)", n, off, c->rb_bytes);
        return DGNN_EINVAL;
    }
    uint8_t* dst = static_cast<uint8_t*>(c->rb) + off;
    if (readback_by_copy()) {
        DGNN_CK(cudaMemcpyAsync(dst, src_dev, n, cudaMemcpyDeviceToHost, c->stream));
        return DGNN_OK;
    }
    uint32_t* ddst = nullptr;
    DGNN_CK(cudaHostGetDevicePointer((void**)&ddst, dst, 0));
    const size_t nw = n / 4;
    const int grid = (int)std::min<size_t>((nw + 1023) / 1024, (size_t)c->num_sms);
    k_readback<<<std::max(grid, 1), 256, 0, c->stream>>>(ddst, static_cast<const uint32_t*>(src_dev), nw);
    DGNN_CK(cudaGetLastError());
    return DGNN_OK;
}

constexpr int kUploadChunk = 4000;  // bytes per launch (kernel parameter space)
struct UploadChunk {
    uint8_t b[kUploadChunk];
};
__global__ void k_upload(uint8_t* __restrict__ dst, const UploadChunk chunk, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = chunk.b[i];
}

dgnn_status upload_small(dgnn_ctx* c, void* dst_dev, const void* src_host, size_t n) {
    if (!n) return DGNN_OK;
    if (n > kUploadMax || readback_by_copy()) {
        DGNN_CK(cudaMemcpyAsync(dst_dev, src_host, n, cudaMemcpyHostToDevice, c->stream));
        return DGNN_OK;
    }
    UploadChunk ch;
    for (size_t off = 0; off < n; off += kUploadChunk) {
        const int len = (int)std::min<size_t>(kUploadChunk, n - off);
        std::memcpy(ch.b, static_cast<const uint8_t*>(src_host) + off, (size_t)len);
        k_upload<<<1, 256, 0, c->stream>>>(static_cast<uint8_t*>(dst_dev) + off, ch, len);
        DGNN_CK(cudaGetLastError());
    }
    return DGNN_OK;
}

dgnn_status read_small(dgnn_ctx* c, void* dst_host, const void* src_dev, size_t n) {
    if (!n) return DGNN_OK;
    const size_t n4 = (n + 3) & ~(size_t)3;
    DGNN_TRY(readback_reserve(c, n4));
    if (n % 4 || (size_t)src_dev % 4) {  // (odd sizes: the copy engine)
        DGNN_CK(cudaMemcpyAsync(c->rb, src_dev, n, cudaMemcpyDeviceToHost, c->stream));
    } else {
        DGNN_TRY(readback_enqueue(c, 0, src_dev, n));
    }
    DGNN_CK(cudaStreamSynchronize(c->stream));
    std::memcpy(dst_host, c->rb, n);
    return DGNN_OK;
}

dgnn_status read_dev_err(dgnn_ctx* c, int* flags) {
    DGNN_TRY(readback_reserve(c, 64));
    DGNN_TRY(readback_enqueue(c, 0, c->dev_err, sizeof(int)));
    DGNN_CK(cudaStreamSynchronize(c->stream));
    *flags = *reinterpret_cast<volatile int*>(c->rb);
    if (*flags) DGNN_CK(cudaMemsetAsync(c->dev_err, 0, sizeof(int), c->stream));
    return DGNN_OK;
}

namespace scan {
dgnn_status scratch(dgnn_ctx* c, size_t bytes, unsigned long long** status) {
    if (c->scan_bytes < bytes) {
        if (c->scan_buf) {
            DGNN_CK(cudaStreamSynchronize(c->stream));  // (growth is rare: the old buffer may be in use)
            DGNN_CK(cudaFree(c->scan_buf));
            c->scan_buf = nullptr;
        }
        const size_t want = std::max<size_t>(bytes + bytes / 2, (size_t)1 << 20);
        if (cudaMalloc(&c->scan_buf, want) != cudaSuccess) {
            cudaGetLastError();
            c->scan_bytes = 0;
            set_error("scan scratch allocation of %zu bytes failed", want);
            return DGNN_ENOMEM;
        }
        c->scan_bytes = want;
    }
    *status = static_cast<unsigned long long*>(c->scan_buf);
    return DGNN_OK;
}
}  // namespace scan

dgnn_status dev_err_status(int h) {
    if (!h) return DGNN_OK;
    if (h & DEVERR_SEED_RANGE) { set_error("a seed is outside [0, num_nodes)"); return DGNN_EINVAL; }
    if (h & DEVERR_SEED_DUP) { set_error("a seed appears twice within one batch (reading c12)"); return DGNN_EINVAL; }
    if (h & DEVERR_ADDR_RANGE) { set_error("unresolvable node address (slot beyond its tier)"); return DGNN_ERANGE; }
    if (h & DEVERR_TABLE) { set_error("internal: sampling hash table overflow"); return DGNN_ECUDA; }
    if (h & DEVERR_PART) { set_error("internal: partitioned dedup bucket overflow"); return DGNN_ECUDA; }
    set_error("internal: device capacity overflow (flags %d)", h);
    return DGNN_ECUDA;
}

dgnn_status check_dev_err(dgnn_ctx* c) {
    int h = 0;
    DGNN_TRY(read_dev_err(c, &h));
    if (g_io_error.exchange(0)) {
        set_error("file staging: a pread/pwrite failed or hit end of file");
        return DGNN_EIO;
    }
    return dev_err_status(h);
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

const char* dgnn_last_error(void) { return g_err; }

dgnn_status dgnn_ctx_create(int device, void* stream, const dgnn_allocator* allocator, dgnn_ctx** out) {
    DGNN_REQUIRE(out != nullptr, "dgnn_ctx_create: out is NULL");
    *out = nullptr;
    int ndev = 0;
    DGNN_CK(cudaGetDeviceCount(&ndev));
    DGNN_REQUIRE(device >= 0 && device < ndev, "dgnn_ctx_create: device %d not present (%d devices)", device, ndev);
    DGNN_CK(cudaSetDevice(device));
    auto* c = new dgnn_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    // NULL = the legacy default stream (what frameworks call "the default stream"), so
    // work enqueued by the caller on it is ordered with the library's kernels
    c->stream = stream ? (cudaStream_t)stream : cudaStreamLegacy;
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        set_error("cudaStreamCreate (side) failed");
        return DGNN_ECUDA;
    }
    if (allocator && allocator->alloc && allocator->free) {
        c->alloc = *allocator;
        c->has_alloc = true;
    } else {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming);
    if (cudaMalloc(&c->dev_err, sizeof(int)) != cudaSuccess || cudaMemset(c->dev_err, 0, sizeof(int)) != cudaSuccess) {
        dgnn_ctx_destroy(c);
        set_error("cudaMalloc of the error word failed");
        return DGNN_ECUDA;
    }
    *out = c;
    return DGNN_OK;
}

void dgnn_ctx_destroy(dgnn_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    fold_pending(c, false);
    keep_trim(c, 0);
    for (auto e : c->event_pool) cudaEventDestroy(e);
    for (int i = 0; i < dgnn_ctx::kStageRing; ++i)
        if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    if (c->order_ev) cudaEventDestroy(c->order_ev);
    if (c->dev_err) cudaFree(c->dev_err);
    if (c->scan_buf) cudaFree(c->scan_buf);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->pinned_err) cudaFreeHost(c->pinned_err);
    if (c->rb) cudaFreeHost(c->rb);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

dgnn_status dgnn_ctx_set_stream(dgnn_ctx* c, void* stream) {
    DGNN_REQUIRE(c && stream, "dgnn_ctx_set_stream: NULL argument");
    if (c->own_stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
        c->own_stream = false;
    }
    c->stream = (cudaStream_t)stream;
    return DGNN_OK;
}

void* dgnn_ctx_stream(const dgnn_ctx* c) { return c ? (void*)c->stream : nullptr; }
void* dgnn_ctx_side_stream(const dgnn_ctx* c) { return c ? (void*)c->side : nullptr; }

dgnn_status dgnn_ctx_sync(dgnn_ctx* c) {
    DGNN_REQUIRE(c, "dgnn_ctx_sync: NULL ctx");
    DGNN_CK(cudaSetDevice(c->device));
    DGNN_CK(cudaStreamSynchronize(c->side));
    return check_dev_err(c);
}

dgnn_status dgnn_upload(dgnn_ctx* c, void* dst_dev, const void* src_host, int64_t bytes) {
    DGNN_REQUIRE(c && bytes >= 0 && (bytes == 0 || (dst_dev && src_host)), "dgnn_upload: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    return upload_small(c, dst_dev, src_host, (size_t)bytes);
}

dgnn_status dgnn_ctx_set_sample_group(dgnn_ctx* c, int32_t batches) {
    DGNN_REQUIRE(c && batches >= 0 && batches <= 1024, "dgnn_ctx_set_sample_group: bad argument");
    c->sample_group = batches;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_set_keep_limit(dgnn_ctx* c, int64_t bytes) {
    DGNN_REQUIRE(c && bytes >= 0, "dgnn_ctx_set_keep_limit: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    c->kept_limit = (size_t)bytes;
    keep_trim(c, c->kept_limit);
    return DGNN_OK;
}

int64_t dgnn_ctx_kept_bytes(const dgnn_ctx* c) { return c ? (int64_t)c->kept_bytes : 0; }

dgnn_status dgnn_ctx_set_sample_budget(dgnn_ctx* c, int64_t bytes) {
    DGNN_REQUIRE(c && bytes >= ((int64_t)16 << 20), "dgnn_ctx_set_sample_budget: budget below 16 MiB");
    c->sample_budget = (size_t)bytes;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_set_grid_cap(dgnn_ctx* c, int32_t max_blocks) {
    DGNN_REQUIRE(c && max_blocks >= 0, "dgnn_ctx_set_grid_cap: bad argument");
    c->grid_cap = max_blocks;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_set_sample_mode(dgnn_ctx* c, int32_t mode) {
    DGNN_REQUIRE(c && (mode == DGNN_SAMPLE_NODEWISE || mode == DGNN_SAMPLE_BLOCKS),
                 "dgnn_ctx_set_sample_mode: bad argument");
    c->sample_mode = mode;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_set_assemble_occupancy(dgnn_ctx* c, int32_t blocks_per_sm) {
    DGNN_REQUIRE(c && blocks_per_sm >= 1 && blocks_per_sm <= 32, "dgnn_ctx_set_assemble_occupancy: bad argument");
    c->assemble_blocks_per_sm = blocks_per_sm;
    return DGNN_OK;
}

int64_t dgnn_ctx_launches(const dgnn_ctx* c) { return c ? c->launches : 0; }

dgnn_status dgnn_ctx_set_timing(dgnn_ctx* c, int enable) {
    DGNN_REQUIRE(c, "dgnn_ctx_set_timing: NULL ctx");
    c->timing = enable != 0;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_set_timing_mask(dgnn_ctx* c, uint64_t mask) {
    DGNN_REQUIRE(c, "dgnn_ctx_set_timing_mask: NULL ctx");
    c->timing_mask = mask;
    return DGNN_OK;
}

dgnn_status dgnn_ctx_kernel_stats(dgnn_ctx* c, int32_t kid, dgnn_kernel_stat* out) {
    DGNN_REQUIRE(c && out && kid >= 0 && kid < DGNN_K_NUM, "dgnn_ctx_kernel_stats: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    fold_pending(c, true);
    out->launches = c->stat_n[kid];
    out->ms = c->stat_ms[kid];
    out->bytes = c->stat_bytes[kid];
    return DGNN_OK;
}

dgnn_status dgnn_ctx_reset_stats(dgnn_ctx* c) {
    DGNN_REQUIRE(c, "dgnn_ctx_reset_stats: NULL ctx");
    fold_pending(c, true);
    for (int k = 0; k < DGNN_K_NUM; ++k) {
        c->stat_ms[k] = 0;
        c->stat_bytes[k] = 0;
        c->stat_n[k] = 0;
    }
    return DGNN_OK;
}

const char* dgnn_kernel_name(int32_t kid) {
    static const char* names[DGNN_K_NUM] = {"scan",           "sample_seed",   "sample_hop",    "sample_order",
                                            "sample_remap",   "sample_compact", "sample_setup", "cache_hist",
                                            "cache_select",   "classify",      "pack_gather",   "tier_gather",
                                            "assemble",       "misc",          "sort",          "disk_plan",
                                            "disk_gather",   "train",
                                            "host_window",    "host_gather",   "tier_gather_pcie",
                                            "graph_io",       "sample_dedup",  "sample_count"};
    return (kid >= 0 && kid < DGNN_K_NUM) ? names[kid] : "?";
}

// ---------------------------------------------------------------- staging
dgnn_status dgnn_stage_copy(dgnn_ctx* c, void* dst, const void* src, int64_t bytes, int32_t kind, int64_t* ticket) {
    DGNN_REQUIRE(c && ticket && bytes >= 0 && kind >= 0 && kind <= 2 && (bytes == 0 || (dst && src)),
                 "dgnn_stage_copy: bad argument");
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t t = c->stage_next++;
    cudaEvent_t& slot = c->stage_ev[t % dgnn_ctx::kStageRing];
    if (!slot) DGNN_CK(cudaEventCreateWithFlags(&slot, cudaEventDisableTiming));
    cudaEvent_t ev = slot;
    if (t >= dgnn_ctx::kStageRing) DGNN_CK(cudaEventSynchronize(ev));  // slot reuse: the older copy must be done
    // order after everything already on the ctx stream
    DGNN_CK(cudaEventRecord(c->order_ev, c->stream));
    DGNN_CK(cudaStreamWaitEvent(c->side, c->order_ev, 0));
    static const cudaMemcpyKind kinds[3] = {cudaMemcpyDeviceToHost, cudaMemcpyHostToDevice, cudaMemcpyDeviceToDevice};
    if (bytes) DGNN_CK(cudaMemcpyAsync(dst, src, (size_t)bytes, kinds[kind], c->side));
    DGNN_CK(cudaEventRecord(ev, c->side));
    *ticket = t;
    return DGNN_OK;
}

dgnn_status dgnn_stage_wait(dgnn_ctx* c, int64_t ticket) {
    DGNN_REQUIRE(c && ticket >= 0 && ticket < c->stage_next, "dgnn_stage_wait: bad ticket");
    if (c->stage_next - ticket > dgnn_ctx::kStageRing) return DGNN_OK;  // long since complete (slot was reused)
    DGNN_CK(cudaStreamWaitEvent(c->stream, c->stage_ev[ticket % dgnn_ctx::kStageRing], 0));
    return DGNN_OK;
}

dgnn_status dgnn_stage_wait_stream(dgnn_ctx* c, int64_t ticket, void* stream) {
    DGNN_REQUIRE(c && ticket >= 0 && ticket < c->stage_next, "dgnn_stage_wait_stream: bad ticket");
    if (c->stage_next - ticket > dgnn_ctx::kStageRing) return DGNN_OK;
    DGNN_CK(cudaStreamWaitEvent(stream ? (cudaStream_t)stream : cudaStreamLegacy,
                                c->stage_ev[ticket % dgnn_ctx::kStageRing], 0));
    return DGNN_OK;
}

dgnn_status dgnn_stage_sync(dgnn_ctx* c, int64_t ticket) {
    DGNN_REQUIRE(c && ticket >= 0 && ticket < c->stage_next, "dgnn_stage_sync: bad ticket");
    if (c->stage_next - ticket > dgnn_ctx::kStageRing) return DGNN_OK;
    DGNN_CK(cudaEventSynchronize(c->stage_ev[ticket % dgnn_ctx::kStageRing]));
    return DGNN_OK;
}

dgnn_status dgnn_host_alloc(int64_t bytes, void** out) {
    DGNN_REQUIRE(out && bytes >= 0, "dgnn_host_alloc: bad argument");
    *out = nullptr;
    DGNN_CK(cudaHostAlloc(out, (size_t)(bytes ? bytes : 1), cudaHostAllocPortable | cudaHostAllocMapped));
    return DGNN_OK;
}

dgnn_status dgnn_host_free(void* p) {
    if (p) DGNN_CK(cudaFreeHost(p));
    return DGNN_OK;
}

}  // extern "C"
