// file.cu -- a8 with the disk tier as a file on local storage: packed chunks are
// written with pwrite and read back with pread (O_DIRECT when requested, as in the
// paper's I/O engine) through a pinned bounce buffer.  The copies and the
// syscalls are issued in stream order on the ctx side stream: each piece is a
// cudaMemcpyAsync plus a cudaLaunchHostFunc that runs the syscall, so a staging
// ticket completes exactly when its bytes are on disk (write) or in HBM (read).
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <thread>
#include <vector>

#include "internal.cuh"

struct dgnn_file {
    int fd = -1;
    bool direct = false;
};

namespace dgnn {

std::atomic<int> g_io_error{0};

namespace {

struct IoOp {
    int fd;
    bool write;
    uint8_t* buf;
    int64_t bytes;
    int64_t off;
};

void CUDART_CB io_host_fn(void* p) {
    IoOp* op = static_cast<IoOp*>(p);
    int64_t done = 0;
    while (done < op->bytes) {
        const ssize_t r = op->write ? pwrite(op->fd, op->buf + done, (size_t)(op->bytes - done), op->off + done)
                                    : pread(op->fd, op->buf + done, (size_t)(op->bytes - done), op->off + done);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) {
            g_io_error.store(1);
            break;
        }
        done += r;
    }
    delete op;
}

dgnn_status stage_file(dgnn_ctx* c, dgnn_file* f, int64_t file_off, uint8_t* dev, int64_t bytes, uint8_t* bounce,
                       int64_t chunk, bool write, int64_t* ticket) {
    DGNN_REQUIRE(c && f && f->fd >= 0 && ticket && bytes >= 0 && file_off >= 0 && (bytes == 0 || (dev && bounce)),
                 "dgnn_stage_file: bad argument");
    DGNN_REQUIRE(chunk > 0, "dgnn_stage_file: chunk_bytes must be positive");
    if (f->direct)
        DGNN_REQUIRE(file_off % 4096 == 0 && bytes % 4096 == 0 && chunk % 4096 == 0 && ((uintptr_t)bounce % 4096) == 0,
                     "dgnn_stage_file: O_DIRECT needs 4096-aligned offsets, sizes and bounce buffer");
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t t = c->stage_next++;
    cudaEvent_t& slot = c->stage_ev[t % dgnn_ctx::kStageRing];
    if (!slot) DGNN_CK(cudaEventCreateWithFlags(&slot, cudaEventDisableTiming));
    if (t >= dgnn_ctx::kStageRing) DGNN_CK(cudaEventSynchronize(slot));
    DGNN_CK(cudaEventRecord(c->order_ev, c->stream));
    DGNN_CK(cudaStreamWaitEvent(c->side, c->order_ev, 0));
    for (int64_t pos = 0; pos < bytes; pos += chunk) {
        const int64_t n = std::min(chunk, bytes - pos);
        if (write) {
            DGNN_CK(cudaMemcpyAsync(bounce, dev + pos, (size_t)n, cudaMemcpyDeviceToHost, c->side));
            DGNN_CK(cudaLaunchHostFunc(c->side, io_host_fn, new IoOp{f->fd, true, bounce, n, file_off + pos}));
        } else {
            DGNN_CK(cudaLaunchHostFunc(c->side, io_host_fn, new IoOp{f->fd, false, bounce, n, file_off + pos}));
            DGNN_CK(cudaMemcpyAsync(dev + pos, bounce, (size_t)n, cudaMemcpyHostToDevice, c->side));
        }
    }
    DGNN_CK(cudaEventRecord(slot, c->side));
    *ticket = t;
    return DGNN_OK;
}

// Disk-cache page reads (the paper issues them with io_uring from 4 threads): the
// listed 4 KiB pages land back to back in the bounce buffer; runs of consecutive pages are
// one pread each, and the runs are split over `threads` threads.
struct PageReadOp {
    int fd;
    uint8_t* buf;
    std::vector<int64_t> run_off, run_bytes, run_dst;  // file offset, length, offset in buf
    int threads;
};

void CUDART_CB pages_host_fn(void* p) {
    PageReadOp* op = static_cast<PageReadOp*>(p);
    const int64_t nr = (int64_t)op->run_off.size();
    auto work = [op, nr](int64_t t, int64_t T) {
        for (int64_t r = t; r < nr; r += T) {
            int64_t done = 0;
            while (done < op->run_bytes[r]) {
                const ssize_t k = pread(op->fd, op->buf + op->run_dst[r] + done, (size_t)(op->run_bytes[r] - done),
                                        op->run_off[r] + done);
                if (k < 0 && errno == EINTR) continue;
                if (k <= 0) {
                    g_io_error.store(1);
                    break;
                }
                done += k;
            }
        }
    };
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(op->threads, nr));
    if (T == 1) {
        work(0, 1);
    } else {
        std::vector<std::thread> pool;
        for (int64_t t = 1; t < T; ++t) pool.emplace_back(work, t, T);
        work(0, T);
        for (auto& th : pool) th.join();
    }
    delete op;
}

}  // namespace
}  // namespace dgnn

using namespace dgnn;

extern "C" dgnn_status dgnn_stage_file_read_pages(dgnn_ctx* c, dgnn_file* f, int64_t base_off, const int32_t* pages,
                                                  int64_t n_pages, void* dev_dst, void* bounce, int64_t bounce_bytes,
                                                  int32_t threads, int64_t* ticket) {
    constexpr int64_t kPage = 4096;
    DGNN_REQUIRE(c && f && f->fd >= 0 && ticket && n_pages >= 0 && base_off >= 0 && threads >= 1 &&
                     (n_pages == 0 || (pages && dev_dst && bounce && bounce_bytes >= kPage)),
                 "dgnn_stage_file_read_pages: bad argument");
    DGNN_REQUIRE(base_off % kPage == 0 && ((uintptr_t)bounce % kPage) == 0,
                 "dgnn_stage_file_read_pages: the cache region and the bounce buffer must be page-aligned");
    DGNN_CK(cudaSetDevice(c->device));
    const int64_t t = c->stage_next++;
    cudaEvent_t& slot = c->stage_ev[t % dgnn_ctx::kStageRing];
    if (!slot) DGNN_CK(cudaEventCreateWithFlags(&slot, cudaEventDisableTiming));
    if (t >= dgnn_ctx::kStageRing) DGNN_CK(cudaEventSynchronize(slot));
    DGNN_CK(cudaEventRecord(c->order_ev, c->stream));
    DGNN_CK(cudaStreamWaitEvent(c->side, c->order_ev, 0));
    const int64_t per = bounce_bytes / kPage;  // pages per bounce fill
    for (int64_t p0 = 0; p0 < n_pages; p0 += per) {
        const int64_t p1 = std::min(n_pages, p0 + per);
        auto* op = new PageReadOp{f->fd, (uint8_t*)bounce, {}, {}, {}, threads};
        for (int64_t i = p0; i < p1; ++i) {
            const int64_t off = base_off + (int64_t)pages[i] * kPage;
            if (i > p0 && pages[i] == pages[i - 1] + 1) {
                op->run_bytes.back() += kPage;  // extends the current run
            } else {
                op->run_off.push_back(off);
                op->run_bytes.push_back(kPage);
                op->run_dst.push_back((i - p0) * kPage);
            }
        }
        DGNN_CK(cudaLaunchHostFunc(c->side, pages_host_fn, op));
        DGNN_CK(cudaMemcpyAsync((uint8_t*)dev_dst + p0 * kPage, bounce, (size_t)((p1 - p0) * kPage),
                                cudaMemcpyHostToDevice, c->side));
    }
    DGNN_CK(cudaEventRecord(slot, c->side));
    *ticket = t;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_file_open(const char* path, int32_t direct, int32_t create, int64_t size, dgnn_file** out) {
    DGNN_REQUIRE(path && out && size >= 0, "dgnn_file_open: bad argument");
    *out = nullptr;
    int flags = O_RDWR | (create ? O_CREAT | O_TRUNC : 0);
#ifdef O_DIRECT
    if (direct) flags |= O_DIRECT;
#endif
    const int fd = open(path, flags, 0644);
    if (fd < 0) {
        set_error("dgnn_file_open: open(%s) failed: %s", path, strerror(errno));
        return DGNN_EIO;
    }
    if (create && size > 0 && ftruncate(fd, size) != 0) {
        set_error("dgnn_file_open: ftruncate(%s, %lld) failed: %s", path, (long long)size, strerror(errno));
        close(fd);
        return DGNN_EIO;
    }
    auto* f = new dgnn_file();
    f->fd = fd;
    f->direct = direct != 0;
    *out = f;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_file_close(dgnn_file* f) {
    if (!f) return DGNN_OK;
    const int r = f->fd >= 0 ? close(f->fd) : 0;
    delete f;
    if (r != 0) {
        set_error("dgnn_file_close: %s", strerror(errno));
        return DGNN_EIO;
    }
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_stage_file_write(dgnn_ctx* c, dgnn_file* f, int64_t file_off, const void* dev_src,
                                             int64_t bytes, void* bounce, int64_t chunk_bytes, int64_t* ticket) {
    return stage_file(c, f, file_off, (uint8_t*)dev_src, bytes, (uint8_t*)bounce, chunk_bytes, true, ticket);
}

extern "C" dgnn_status dgnn_stage_file_read(dgnn_ctx* c, dgnn_file* f, int64_t file_off, void* dev_dst, int64_t bytes,
                                            void* bounce, int64_t chunk_bytes, int64_t* ticket) {
    return stage_file(c, f, file_off, (uint8_t*)dev_dst, bytes, (uint8_t*)bounce, chunk_bytes, false, ticket);
}
