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

}  // namespace
}  // namespace dgnn

using namespace dgnn;

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
