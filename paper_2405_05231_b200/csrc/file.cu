// file.cu -- a8 with the disk tier as a file on local storage: packed chunks are
// written with pwrite and read back with pread (O_DIRECT when requested, as in the
// paper's I/O engine) through a pinned bounce buffer.  Each file owns an I/O
// engine (worker threads with one request queue each, 4 by default); the copies and
// the engine's submit / wait steps are issued in stream order on the ctx side stream
// (cudaLaunchHostFunc), double-buffered through the bounce buffer's two halves, so a
// staging ticket completes exactly when its bytes are on disk (write) or in HBM (read).
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace dgnn {

std::atomic<int> g_io_error{0};

// The I/O engine of a disk-tier file (the paper drives its NVMe with io_uring from a
// pool of threads): `nq` worker threads, one request queue each.  A transfer is split into
// 4 KiB-aligned parts spread over the queues, so a large pread / pwrite keeps several requests
// in flight on the device; an IoBatch counts a transfer's outstanding parts.
struct IoBatch {
    std::atomic<int> left{0};
    std::mutex m;
    std::condition_variable cv;
    void done() {
        if (left.fetch_sub(1) == 1) {
            std::lock_guard<std::mutex> g(m);
            cv.notify_all();
        }
    }
    void wait() {
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [this] { return left.load() == 0; });
    }
};

struct IoReq {
    int fd;
    bool write;
    uint8_t* buf;
    int64_t bytes;
    int64_t off;
    IoBatch* batch;
};

class IoEngine {
   public:
    explicit IoEngine(int nq) : qs_(nq) {
        for (int i = 0; i < nq; ++i) th_.emplace_back([this, i] { run(i); });
    }
    ~IoEngine() {
        for (auto& q : qs_) {
            std::lock_guard<std::mutex> g(q.m);
            q.stop = true;
            q.cv.notify_all();
        }
        for (auto& t : th_) t.join();
    }
    int queues() const { return (int)qs_.size(); }
    // one transfer [off, off + bytes) <-> buf, split into <= queues() parts on 4 KiB boundaries
    void submit(int fd, bool write, uint8_t* buf, int64_t bytes, int64_t off, IoBatch* b) {
        const int64_t nq = (int64_t)qs_.size();
        int64_t part = ((bytes + nq - 1) / nq + 4095) & ~(int64_t)4095;
        if (part < (int64_t)1 << 20) part = (int64_t)1 << 20;  // >= 1 MiB per request
        for (int64_t pos = 0; pos < bytes; pos += part) push(IoReq{fd, write, buf + pos, std::min(part, bytes - pos), off + pos, b});
    }
    // one request per listed run, round robin over the queues
    void push(IoReq r) {
        r.batch->left.fetch_add(1);
        Q& q = qs_[next_.fetch_add(1) % qs_.size()];
        std::lock_guard<std::mutex> g(q.m);
        q.q.push_back(r);
        q.cv.notify_one();
    }

   private:
    struct Q {
        std::mutex m;
        std::condition_variable cv;
        std::deque<IoReq> q;
        bool stop = false;
    };
    void run(int i) {
        Q& q = qs_[i];
        for (;;) {
            IoReq r;
            {
                std::unique_lock<std::mutex> g(q.m);
                q.cv.wait(g, [&] { return q.stop || !q.q.empty(); });
                if (q.q.empty()) return;
                r = q.q.front();
                q.q.pop_front();
            }
            int64_t done = 0;
            while (done < r.bytes) {
                const ssize_t k = r.write ? pwrite(r.fd, r.buf + done, (size_t)(r.bytes - done), r.off + done)
                                          : pread(r.fd, r.buf + done, (size_t)(r.bytes - done), r.off + done);
                if (k < 0 && errno == EINTR) continue;
                if (k <= 0) {
                    g_io_error.store(1);
                    break;
                }
                done += k;
            }
            r.batch->done();
        }
    }
    std::vector<Q> qs_;
    std::vector<std::thread> th_;
    std::atomic<uint64_t> next_{0};
};

}  // namespace dgnn

struct dgnn_file {
    int fd = -1;
    bool direct = false;
    int queues = 4;
    std::unique_ptr<dgnn::IoEngine> io;
    dgnn::IoEngine* engine() {
        if (!io) io.reset(new dgnn::IoEngine(queues));
        return io.get();
    }
};

namespace dgnn {
namespace {

// stream-ordered host steps of a transfer: submit (returns at once) and wait (blocks until the
// transfer's parts are done; frees the batch)
struct IoStep {
    dgnn_file* f;
    bool write;
    uint8_t* buf;
    int64_t bytes;
    int64_t off;
    IoBatch* batch;
};

void CUDART_CB io_submit_fn(void* p) {
    IoStep* s = static_cast<IoStep*>(p);
    s->f->engine()->submit(s->f->fd, s->write, s->buf, s->bytes, s->off, s->batch);
    delete s;
}

void CUDART_CB io_wait_fn(void* p) {
    IoBatch* b = static_cast<IoBatch*>(p);
    b->wait();
    delete b;
}

// Double-buffered staging: the bounce buffer is two halves; while the copy engine moves piece k
// through one half, the I/O engine reads piece k+1 into (or writes piece k-1 from) the other.
// Read:  submit(0); for k: submit(k+1), wait(k), H2D(k).
// Write: for k: wait(k-2), D2H(k), submit(k); then wait(n-2), wait(n-1).
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
    // two halves when the bounce buffer allows it (4 KiB-aligned), else one
    const int64_t half = (chunk / 2) & ~(int64_t)4095;
    const int nbuf = half >= 4096 ? 2 : 1;
    const int64_t piece = nbuf == 2 ? half : chunk;
    const int64_t n = (bytes + piece - 1) / piece;
    std::vector<IoBatch*> batches((size_t)n);
    for (int64_t k = 0; k < n; ++k) batches[k] = new IoBatch();
    auto buf_of = [&](int64_t k) { return bounce + (k % nbuf) * piece; };
    auto len_of = [&](int64_t k) { return std::min(piece, bytes - k * piece); };
    auto submit = [&](int64_t k) -> dgnn_status {
        DGNN_CK(cudaLaunchHostFunc(c->side, io_submit_fn,
                                   new IoStep{f, write, buf_of(k), len_of(k), file_off + k * piece, batches[k]}));
        return DGNN_OK;
    };
    auto wait = [&](int64_t k) -> dgnn_status {
        DGNN_CK(cudaLaunchHostFunc(c->side, io_wait_fn, batches[k]));
        return DGNN_OK;
    };
    if (!write) {
        if (n) DGNN_TRY(submit(0));
        for (int64_t k = 0; k < n; ++k) {
            if (k + 1 < n && nbuf == 2) DGNN_TRY(submit(k + 1));
            DGNN_TRY(wait(k));
            DGNN_CK(cudaMemcpyAsync(dev + k * piece, buf_of(k), (size_t)len_of(k), cudaMemcpyHostToDevice, c->side));
            if (k + 1 < n && nbuf == 1) DGNN_TRY(submit(k + 1));
        }
    } else {
        for (int64_t k = 0; k < n; ++k) {
            if (k >= nbuf) DGNN_TRY(wait(k - nbuf));
            DGNN_CK(cudaMemcpyAsync(buf_of(k), dev + k * piece, (size_t)len_of(k), cudaMemcpyDeviceToHost, c->side));
            DGNN_TRY(submit(k));
        }
        for (int64_t k = std::max<int64_t>(0, n - nbuf); k < n; ++k) DGNN_TRY(wait(k));
    }
    DGNN_CK(cudaEventRecord(slot, c->side));
    *ticket = t;
    return DGNN_OK;
}

// Disk-cache page reads (the paper issues them with io_uring from 4 threads): the
// listed 4 KiB pages land back to back in the bounce buffer; runs of consecutive pages are one
// request each, spread over the file's I/O queues; bounce fills alternate between its halves
// so that the reads of fill i+1 overlap the H2D copy of fill i.
struct PageStep {
    dgnn_file* f;
    uint8_t* buf;
    std::vector<int64_t> run_off, run_bytes, run_dst;  // file offset, length, offset in buf
    IoBatch* batch;
};

void CUDART_CB pages_submit_fn(void* p) {
    PageStep* s = static_cast<PageStep*>(p);
    IoEngine* e = s->f->engine();
    for (size_t r = 0; r < s->run_off.size(); ++r)
        e->push(IoReq{s->f->fd, false, s->buf + s->run_dst[r], s->run_bytes[r], s->run_off[r], s->batch});
    delete s;
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
    if (!f->io && threads > f->queues) f->queues = threads;  // (the engine starts at first use)
    const int64_t t = c->stage_next++;
    cudaEvent_t& slot = c->stage_ev[t % dgnn_ctx::kStageRing];
    if (!slot) DGNN_CK(cudaEventCreateWithFlags(&slot, cudaEventDisableTiming));
    if (t >= dgnn_ctx::kStageRing) DGNN_CK(cudaEventSynchronize(slot));
    DGNN_CK(cudaEventRecord(c->order_ev, c->stream));
    DGNN_CK(cudaStreamWaitEvent(c->side, c->order_ev, 0));
    const int64_t total = bounce_bytes / kPage;                // pages the bounce buffer holds
    const int nbuf = total >= 2 ? 2 : 1;
    const int64_t per = total / nbuf;                          // pages per bounce fill
    std::vector<PageStep*> steps;
    for (int64_t p0 = 0; p0 < n_pages; p0 += per) {
        const int64_t p1 = std::min(n_pages, p0 + per);
        uint8_t* buf = (uint8_t*)bounce + (int64_t)(steps.size() % nbuf) * per * kPage;
        auto* op = new PageStep{f, buf, {}, {}, {}, new IoBatch()};
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
        steps.push_back(op);
    }
    const int64_t ns = (int64_t)steps.size();
    // (a submit step frees its PageStep when it runs, possibly before this loop ends)
    std::vector<uint8_t*> bufs;
    std::vector<IoBatch*> bats;
    for (auto* st : steps) {
        bufs.push_back(st->buf);
        bats.push_back(st->batch);
    }
    auto submit = [&](int64_t i) -> dgnn_status {
        DGNN_CK(cudaLaunchHostFunc(c->side, pages_submit_fn, steps[i]));
        return DGNN_OK;
    };
    if (ns) DGNN_TRY(submit(0));
    for (int64_t i = 0; i < ns; ++i) {
        const int64_t p0 = i * per, p1 = std::min(n_pages, p0 + per);
        uint8_t* buf = bufs[i];
        IoBatch* b = bats[i];
        if (i + 1 < ns && nbuf == 2) DGNN_TRY(submit(i + 1));
        DGNN_CK(cudaLaunchHostFunc(c->side, io_wait_fn, b));
        DGNN_CK(cudaMemcpyAsync((uint8_t*)dev_dst + p0 * kPage, buf, (size_t)((p1 - p0) * kPage),
                                cudaMemcpyHostToDevice, c->side));
        if (i + 1 < ns && nbuf == 1) DGNN_TRY(submit(i + 1));
    }
    DGNN_CK(cudaEventRecord(slot, c->side));
    *ticket = t;
    return DGNN_OK;
}

extern "C" dgnn_status dgnn_file_set_queues(dgnn_file* f, int32_t queues) {
    DGNN_REQUIRE(f && queues >= 1 && queues <= 64, "dgnn_file_set_queues: queues must be in [1, 64]");
    DGNN_REQUIRE(!f->io, "dgnn_file_set_queues: the file's I/O engine has already started");
    f->queues = queues;
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
    f->io.reset();  // joins the I/O threads (the caller has synchronized its staging tickets)
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
