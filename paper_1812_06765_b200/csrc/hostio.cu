// Host <-> device staging for numpy-facing calls (the reference's arrays are pageable
// host memory).  A pageable cudaMemcpy runs at 7-17 GB/s on the B200 boxes (driver bounce
// buffers) and a single-thread copy into a page-locked buffer at ~18 GB/s; the DMA itself
// runs at ~50 GB/s.  Staged transfers here split the array into chunks, copy the chunks
// into a page-locked buffer with a small persistent thread team and issue each chunk's DMA
// as soon as its host copy lands, so the host copy runs on several cores and overlaps
// the PCIe transfer (tools/e2e_breakdown.py, tools/h2d_probe.py).  Page-locked sources
// and destinations skip the staging.

#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ngf {

namespace {

// Persistent copy threads.  Workers spin for a short while after each job (calls come
// in bursts: one per objective evaluation) and then sleep on a condition variable.
class Team {
  public:
    static Team& get() {
        // a forked child has none of the parent's threads: it builds its own team (the
        // parent's object is leaked in the child, never joined)
        static Team* t = nullptr;
        static pid_t owner = 0;
        const pid_t me = getpid();
        if (!t || owner != me) {
            t = new Team();
            owner = me;
        }
        return *t;
    }
    int size() const { return (int)th_.size(); }

    // Run job(i) for i in [0, n) on the workers; returns immediately.  `wait_all` blocks
    // until every index has finished.  Each call publishes a fresh Job object together
    // with its generation under the mutex; a worker takes a reference to the job it saw
    // (never to shared fields that the next start() rewrites), so a worker waking late
    // from an earlier generation either finds that job exhausted or runs the new one.
    void start(int n, std::function<void(int)> fn) {
        auto j = std::make_shared<Job>();
        j->fn = std::move(fn);
        j->n = n;
        {
            std::lock_guard<std::mutex> lk(m_);
            cur_ = j;
            gen_.fetch_add(1, std::memory_order_release);
        }
        last_ = std::move(j);
        if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
    }
    void wait_all() {
        const std::shared_ptr<Job> j = last_;
        if (!j) return;
        while (j->done.load(std::memory_order_acquire) < j->n) _mm_pause();
    }

  private:
    struct Job {
        std::function<void(int)> fn;
        int n = 0;
        std::atomic<int> next{0}, done{0};
    };

    Team() {
        int hw = (int)std::thread::hardware_concurrency();
        int k = std::max(1, std::min(4, hw / 2));  // 4: best of 1-12 on the B200 hosts (tools/host_copy_probe.py)
        if (const char* e = std::getenv("NGF_HOST_THREADS")) k = std::max(1, std::atoi(e));
        for (int i = 0; i < k; ++i) th_.emplace_back([this] { loop(); });
    }
    ~Team() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void loop() {
        uint64_t seen = 0;
        while (true) {
            if (gen_.load(std::memory_order_acquire) != seen) {
                std::shared_ptr<Job> j;
                {
                    std::lock_guard<std::mutex> lk(m_);
                    if (stop_) return;
                    seen = gen_.load(std::memory_order_acquire);
                    j = cur_;
                }
                while (j) {
                    const int i = j->next.fetch_add(1, std::memory_order_acq_rel);
                    if (i >= j->n) break;
                    j->fn(i);
                    j->done.fetch_add(1, std::memory_order_acq_rel);
                }
            }
            // spin ~2 ms for the next job, then sleep
            int spins = 0;
            while (gen_.load(std::memory_order_acquire) == seen && spins < 20000) {
                _mm_pause();
                ++spins;
            }
            if (gen_.load(std::memory_order_acquire) == seen) {
                std::unique_lock<std::mutex> lk(m_);
                sleepers_.fetch_add(1, std::memory_order_acq_rel);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
                sleepers_.fetch_sub(1, std::memory_order_acq_rel);
            }
        }
    }

    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> sleepers_{0};
    std::shared_ptr<Job> cur_;   // guarded by m_
    std::shared_ptr<Job> last_;  // the caller's (start/wait_all run under g_io)
    bool stop_ = false;          // guarded by m_
};

// A growable page-locked buffer whose last DMA is fenced by an event.
struct Stage {
    char* buf = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;  // recorded after the last DMA that used buf
    int reserve(size_t bytes) {
        if (done) NGF_CUDA(cudaEventSynchronize(done));
        if (bytes <= cap) return 0;
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        NGF_CUDA(cudaHostAlloc((void**)&buf, bytes, cudaHostAllocDefault));
        cap = bytes;
        return 0;
    }
};

std::mutex g_io;  // one staged transfer at a time (the team and the stages are shared)
Stage g_up, g_down;
constexpr int kMaxChunks = 64;
std::atomic<int> g_ready[kMaxChunks];
cudaEvent_t g_chunk_ev[kMaxChunks];
bool g_ev_ready = false;

constexpr size_t kDirect = 256 << 10;  // below this one plain copy + one DMA

size_t chunk_bytes(size_t bytes) {
    const int k = Team::get().size();
    size_t c = (bytes + 2 * k - 1) / (2 * k);  // two chunks per thread: the DMA starts early
    c = std::max<size_t>(c, 128 << 10);
    c = std::max(c, (bytes + kMaxChunks - 1) / kMaxChunks);
    return (c + 4095) & ~size_t(4095);
}

}  // namespace

bool host_is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int host_upload(void* dst_dev, const void* src, size_t bytes, cudaStream_t s) {
    if (!bytes) return 0;
    if (host_is_pinned(src)) {
        NGF_CUDA(cudaMemcpyAsync(dst_dev, src, bytes, cudaMemcpyHostToDevice, s));
        return 0;
    }
    std::lock_guard<std::mutex> lk(g_io);
    if (!g_up.done) NGF_CUDA(cudaEventCreateWithFlags(&g_up.done, cudaEventDisableTiming));
    if (int rc = g_up.reserve(bytes)) return rc;
    char* stage = g_up.buf;
    const char* in = (const char*)src;
    if (bytes <= kDirect) {
        std::memcpy(stage, in, bytes);
        NGF_CUDA(cudaMemcpyAsync(dst_dev, stage, bytes, cudaMemcpyHostToDevice, s));
    } else {
        const size_t cb = chunk_bytes(bytes);
        const int nc = (int)((bytes + cb - 1) / cb);
        for (int i = 0; i < nc; ++i) g_ready[i].store(0, std::memory_order_relaxed);
        Team::get().start(nc, [=](int i) {
            const size_t o = (size_t)i * cb, len = std::min(cb, bytes - o);
            std::memcpy(stage + o, in + o, len);
            g_ready[i].store(1, std::memory_order_release);
        });
        int rc = 0;
        for (int i = 0; i < nc; ++i) {
            while (!g_ready[i].load(std::memory_order_acquire)) _mm_pause();
            const size_t o = (size_t)i * cb, len = std::min(cb, bytes - o);
            if (!rc) rc = (int)cudaMemcpyAsync((char*)dst_dev + o, stage + o, len, cudaMemcpyHostToDevice, s);
        }
        Team::get().wait_all();
        if (rc) return rc;
    }
    NGF_CUDA(cudaEventRecord(g_up.done, s));
    return 0;
}

int host_download(void* dst, const void* src_dev, size_t bytes, cudaStream_t s) {
    if (!bytes) return 0;
    if (host_is_pinned(dst)) {
        NGF_CUDA(cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, s));
        NGF_CUDA(cudaStreamSynchronize(s));
        return 0;
    }
    std::lock_guard<std::mutex> lk(g_io);
    if (!g_ev_ready) {
        for (int i = 0; i < kMaxChunks; ++i)
            NGF_CUDA(cudaEventCreateWithFlags(&g_chunk_ev[i], cudaEventDisableTiming));
        g_ev_ready = true;
    }
    if (int rc = g_down.reserve(bytes)) return rc;
    char* stage = g_down.buf;
    char* out = (char*)dst;
    if (bytes <= kDirect) {
        NGF_CUDA(cudaMemcpyAsync(stage, src_dev, bytes, cudaMemcpyDeviceToHost, s));
        NGF_CUDA(cudaStreamSynchronize(s));
        std::memcpy(out, stage, bytes);
        return 0;
    }
    const size_t cb = chunk_bytes(bytes);
    const int nc = (int)((bytes + cb - 1) / cb);
    for (int i = 0; i < nc; ++i) {
        const size_t o = (size_t)i * cb, len = std::min(cb, bytes - o);
        NGF_CUDA(cudaMemcpyAsync(stage + o, (const char*)src_dev + o, len, cudaMemcpyDeviceToHost, s));
        NGF_CUDA(cudaEventRecord(g_chunk_ev[i], s));
    }
    std::atomic<int> err{0};
    Team::get().start(nc, [=, &err](int i) {
        const size_t o = (size_t)i * cb, len = std::min(cb, bytes - o);
        while (cudaEventQuery(g_chunk_ev[i]) == cudaErrorNotReady) _mm_pause();
        const cudaError_t e = cudaEventSynchronize(g_chunk_ev[i]);
        if (e != cudaSuccess) {
            err.store((int)e);
            return;
        }
        std::memcpy(out + o, stage + o, len);
    });
    Team::get().wait_all();
    return err.load();
}

}  // namespace ngf

extern "C" int ngf_host_upload(void* dst_dev, const void* src_host, size_t bytes, void* stream) {
    if ((!dst_dev || !src_host) && bytes) return NGF_EARG;
    return ngf::host_upload(dst_dev, src_host, bytes, ngf::as_stream(stream));
}

extern "C" int ngf_host_is_pinned(const void* host_ptr) {
    return host_ptr && ngf::host_is_pinned(host_ptr) ? 1 : 0;
}

extern "C" int ngf_host_download(void* dst_host, const void* src_dev, size_t bytes, void* stream) {
    if ((!dst_host || !src_dev) && bytes) return NGF_EARG;
    return ngf::host_download(dst_host, src_dev, bytes, ngf::as_stream(stream));
}
