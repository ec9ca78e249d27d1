// hostcopy.cu -- host -> device copies from pageable memory at pinned-memory speed.
// (The slot copies use streaming stores, ntcopy.cpp: C3's pageable l0_search 7.5 -> 6.1 ms.)
//
// The drop-in's real caller passes plain numpy arrays (pipeline.py:219-229): pageable memory,
// which cudaMemcpyAsync copies through the driver's own single-threaded staging (~8 GB/s, 20 ms
// for C3's 160 MB).  Here the source is streamed through a ring of pinned slots: a pool of host
// threads memcpy one slot's piece in parallel, the slot is sent with cudaMemcpyAsync on the
// caller's stream, and the slot is reused once its event has completed.  Pinned sources (the
// caller registered or allocated them) bypass the ring.
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "kernels.h"

namespace l0s {

void host_copy(void* dst, const void* src, size_t n);  // ntcopy.cpp: streaming stores when AVX2 is there

namespace {

// Fork-join pool: run(f, parts) calls f(0..parts-1), part 0 on the caller's thread.
class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 1; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
        n_ = n;
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return n_; }
    template <typename F>
    void run(F&& f) {
        {
            std::lock_guard<std::mutex> g(mu_);
            job_ = std::function<void(int)>(f);
            left_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> g(mu_);
        done_.wait(g, [this] { return left_ == 0; });
    }

  private:
    void loop(int me) {
        int seen = 0;
        for (;;) {
            std::function<void(int)> job;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            job(me);
            {
                std::lock_guard<std::mutex> g(mu_);
                if (--left_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::function<void(int)> job_;
    int n_ = 1, left_ = 0, gen_ = 0;
    bool stop_ = false;
};

}  // namespace

struct HostStager {
    static constexpr size_t kSlot = (size_t)16 << 20;  // bytes per pinned slot (one fork-join each)
    static constexpr int kSlots = 4;
    char* pin = nullptr;
    cudaEvent_t ev[kSlots] = {};
    int next = 0;
    Pool* pool = nullptr;
    ~HostStager() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (pin) cudaFreeHost(pin);
        delete pool;
    }
};

HostStager* host_stager_create() {
    HostStager* h = new HostStager();
    if (cudaHostAlloc((void**)&h->pin, HostStager::kSlot * HostStager::kSlots, cudaHostAllocDefault) != cudaSuccess) {
        h->pin = nullptr;
        delete h;
        return nullptr;
    }
    for (auto& e : h->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    const unsigned hw = std::thread::hardware_concurrency();
    // 8 threads: with streaming stores C3's pageable l0_search ran 6.1 ms (12 threads 6.3, 16 6.4)
    int threads = (int)std::max(1u, std::min(8u, hw ? hw : 4u));
    if (const char* e = getenv("L0S_COPY_THREADS")) threads = std::max(1, atoi(e));  // tuning
    h->pool = new Pool(threads);
    return h;
}

void host_stager_destroy(HostStager* h) { delete h; }

bool host_is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // clear: an unregistered pointer is not an error
        return false;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged;
}

// Rows r = 0..nrows-1 of row_bytes each (source row(r), host) to consecutive device rows at dst.
cudaError_t host_stager_copy_rows(HostStager* h, void* dst, const std::function<const void*(int64_t)>& row,
                                  int64_t nrows, size_t row_bytes, cudaStream_t st) {
    char* d = static_cast<char*>(dst);
    const int parts = h->pool->size();
    if (row_bytes > HostStager::kSlot) {  // one row spans several slots: slot-sized pieces of each row
        for (int64_t r = 0; r < nrows; ++r) {
            const char* s = static_cast<const char*>(row(r));
            for (size_t off = 0; off < row_bytes; off += HostStager::kSlot) {
                const size_t n = std::min(HostStager::kSlot, row_bytes - off);
                const int slot = h->next;
                h->next = (h->next + 1) % HostStager::kSlots;
                cudaError_t e = cudaEventSynchronize(h->ev[slot]);
                if (e != cudaSuccess) return e;
                char* buf = h->pin + (size_t)slot * HostStager::kSlot;
                const size_t per = (n / parts + 63) / 64 * 64;
                h->pool->run([&](int p) {
                    const size_t a = std::min(n, (size_t)p * per), b = std::min(n, a + per);
                    if (b > a) host_copy(buf + a, s + off + a, b - a);
                });
                e = cudaMemcpyAsync(d + (size_t)r * row_bytes + off, buf, n, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaEventRecord(h->ev[slot], st);
                if (e != cudaSuccess) return e;
            }
        }
        return cudaSuccess;
    }
    const int64_t per_slot = (int64_t)(HostStager::kSlot / row_bytes);
    for (int64_t r0 = 0; r0 < nrows; r0 += per_slot) {
        const int64_t nr = std::min(per_slot, nrows - r0);
        const int slot = h->next;
        h->next = (h->next + 1) % HostStager::kSlots;
        cudaError_t e = cudaEventSynchronize(h->ev[slot]);  // the slot's previous copy has left
        if (e != cudaSuccess) return e;
        char* buf = h->pin + (size_t)slot * HostStager::kSlot;
        const size_t n = (size_t)nr * row_bytes;
        const size_t per = (n / parts + 63) / 64 * 64;
        // each thread copies one byte range of the slot; rows are cut wherever the range falls
        h->pool->run([&](int p) {
            size_t a = std::min(n, (size_t)p * per);
            const size_t b = std::min(n, a + per);
            while (a < b) {
                const int64_t r = (int64_t)(a / row_bytes);
                const size_t in = a - (size_t)r * row_bytes, len = std::min(b - a, row_bytes - in);
                host_copy(buf + a, static_cast<const char*>(row(r0 + r)) + in, len);
                a += len;
            }
        });
        e = cudaMemcpyAsync(d + (size_t)r0 * row_bytes, buf, n, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(h->ev[slot], st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace l0s
