// Pinned staging for pageable host operands of ozk_gemm_host.
//
// The reference's callers hand over Matrix<T> storage, i.e. std::vector
// (pageable) memory (/root/reference/proj/include/crtgemm/matrix.hpp:14).
// cudaMemcpy from pageable memory stages through a driver buffer on the
// calling thread at ~11 GB/s and cannot overlap with the call's other copies;
// registering the caller's buffers (cudaHostRegister) costs more than the
// copy. Instead each direction gets a ring of pinned slots and a copy thread:
//   H2D: a slot is filled from the caller's buffer by a pool of host threads
//        (parallel memcpy), then DMA'd to the device on the copy stream while
//        the next slot fills; the slot is reused once its DMA event fired.
//   D2H: regions are DMA'd into slots as soon as the compute stream's event
//        for them is recorded, several chunks ahead, and copied out of each
//        slot into the caller's buffer by the host pool when its DMA is done.
// Events the compute stream waits on are recorded by the H2D thread; the
// caller blocks in wait_issued(ticket) until that has happened (a
// cudaStreamWaitEvent on a not-yet-recorded event would not wait).
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "ozk_internal.h"

namespace ozk {

bool host_is_pageable(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // older drivers flag unregistered pointers as an error
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

namespace {

// A fixed pool of host threads running one parallel-for at a time; the
// calling thread takes a share too.
class CopyPool {
  public:
    explicit CopyPool(int threads) {
        for (int t = 0; t < threads; ++t) th_.emplace_back([this, t] { worker(t + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int parts() const { return static_cast<int>(th_.size()) + 1; }
    // fn(part) for part in [0, parts())
    void run(const std::function<void(int)>& fn) {
        {
            std::lock_guard<std::mutex> l(m_);
            fn_ = &fn;
            pending_ = static_cast<int>(th_.size());
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> l(m_);
        done_cv_.wait(l, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void worker(int part) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* fn;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                fn = fn_;
            }
            (*fn)(part);
            {
                std::lock_guard<std::mutex> l(m_);
                if (--pending_ == 0) done_cv_.notify_all();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// dst/src pitched 2-D byte blocks (width bytes x height columns), split over
// the pool by columns (or, for one tall column, by byte ranges)
void pcopy2d(CopyPool& pool, char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
             size_t height) {
    const size_t total = width * height;
    if (total < (size_t(1) << 20) || pool.parts() == 1) {
        for (size_t j = 0; j < height; ++j) std::memcpy(dst + j * dpitch, src + j * spitch, width);
        return;
    }
    const int P = pool.parts();
    pool.run([&](int part) {
        // element range [lo, hi) of the flattened block, cut at whole bytes
        const size_t lo = total * part / P, hi = total * (part + 1) / P;
        size_t e = lo;
        while (e < hi) {
            const size_t j = e / width, i = e % width;
            const size_t n = std::min(width - i, hi - e);
            std::memcpy(dst + j * dpitch + i, src + j * spitch + i, n);
            e += n;
        }
    });
}

struct Chunk {  // one slot's worth of a 2-D copy: columns [j0, j0 + nj), bytes [i0, i0 + w)
    size_t j0, nj, i0, w;
};

std::vector<Chunk> chunks_of(size_t width, size_t height, size_t slot) {
    std::vector<Chunk> out;
    if (width == 0 || height == 0) return out;
    if (width <= slot) {
        const size_t per = std::max<size_t>(1, slot / width);
        for (size_t j = 0; j < height; j += per) out.push_back({j, std::min(per, height - j), 0, width});
    } else {
        for (size_t j = 0; j < height; ++j)
            for (size_t i = 0; i < width; i += slot) out.push_back({j, 1, i, std::min(slot, width - i)});
    }
    return out;
}

}  // namespace

struct HostStager::Impl {
    struct Job {
        char* dev;
        size_t dpitch;
        char* host;
        size_t hpitch, width, height;
        cudaEvent_t ev;  // H2D: record after; D2H: wait before
    };
    int device;
    size_t slot;
    int nslots;
    std::vector<char*> h2d_slot, d2h_slot;
    std::vector<cudaEvent_t> h2d_ev, d2h_ev;
    CopyPool h2d_pool, d2h_pool;
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;

    std::mutex m;
    std::condition_variable cv_job, cv_issued, cv_idle;
    std::deque<Job> h2d_q, d2h_q;
    int64_t issued = 0, queued_h2d = 0;
    int busy = 0;  // jobs taken by the threads and not finished
    bool stop = false;
    cudaError_t err = cudaSuccess;
    std::thread h2d_thread, d2h_thread;

    Impl(int dev, size_t slot_bytes, int slots, int threads)
        : device(dev), slot(slot_bytes), nslots(slots), h2d_pool(threads), d2h_pool(threads) {}

    void fail(cudaError_t e) {
        std::lock_guard<std::mutex> l(m);
        if (err == cudaSuccess) err = e;
        cv_issued.notify_all();
        cv_idle.notify_all();
    }
    bool failed() {
        std::lock_guard<std::mutex> l(m);
        return err != cudaSuccess;
    }

    void h2d_loop() {
        cudaSetDevice(device);
        int s = 0;
        for (;;) {
            Job J;
            {
                std::unique_lock<std::mutex> l(m);
                cv_job.wait(l, [&] { return stop || !h2d_q.empty(); });
                if (stop && h2d_q.empty()) return;
                J = h2d_q.front();
                h2d_q.pop_front();
                ++busy;
            }
            if (!failed()) {
                for (const Chunk& c : chunks_of(J.width, J.height, slot)) {
                    cudaError_t e = cudaEventSynchronize(h2d_ev[s]);  // the slot's previous DMA is done
                    if (e != cudaSuccess) {
                        fail(e);
                        break;
                    }
                    pcopy2d(h2d_pool, h2d_slot[s], c.w, J.host + c.j0 * J.hpitch + c.i0, J.hpitch, c.w, c.nj);
                    e = cudaMemcpy2DAsync(J.dev + c.j0 * J.dpitch + c.i0, J.dpitch, h2d_slot[s], c.w, c.w, c.nj,
                                          cudaMemcpyHostToDevice, h2d_stream);
                    if (e == cudaSuccess) e = cudaEventRecord(h2d_ev[s], h2d_stream);
                    if (e != cudaSuccess) {
                        fail(e);
                        break;
                    }
                    s = (s + 1) % nslots;
                }
                if (J.ev && !failed()) {
                    const cudaError_t e = cudaEventRecord(J.ev, h2d_stream);
                    if (e != cudaSuccess) fail(e);
                }
            }
            {
                std::lock_guard<std::mutex> l(m);
                ++issued;
                --busy;
            }
            cv_issued.notify_all();
            cv_idle.notify_all();
        }
    }

    void d2h_loop() {
        cudaSetDevice(device);
        struct InFlight {
            int s;
            Chunk c;
            Job J;
        };
        std::deque<InFlight> fl;
        int s = 0;
        auto drain_one = [&] {
            InFlight f = fl.front();
            fl.pop_front();
            const cudaError_t e = cudaEventSynchronize(d2h_ev[f.s]);
            if (e != cudaSuccess) {
                fail(e);
                return;
            }
            if (!failed())
                pcopy2d(d2h_pool, f.J.host + f.c.j0 * f.J.hpitch + f.c.i0, f.J.hpitch, d2h_slot[f.s], f.c.w, f.c.w,
                        f.c.nj);
        };
        for (;;) {
            Job J;
            {
                std::unique_lock<std::mutex> l(m);
                cv_job.wait(l, [&] { return stop || !d2h_q.empty(); });
                if (stop && d2h_q.empty()) return;
                J = d2h_q.front();
                d2h_q.pop_front();
                ++busy;
            }
            if (!failed()) {
                cudaError_t e = J.ev ? cudaStreamWaitEvent(d2h_stream, J.ev, 0) : cudaSuccess;
                if (e != cudaSuccess) fail(e);
                for (const Chunk& c : chunks_of(J.width, J.height, slot)) {
                    if (failed()) break;
                    if (static_cast<int>(fl.size()) == nslots) drain_one();  // free the oldest slot
                    e = cudaMemcpy2DAsync(d2h_slot[s], c.w, J.dev + c.j0 * J.dpitch + c.i0, J.dpitch, c.w, c.nj,
                                          cudaMemcpyDeviceToHost, d2h_stream);
                    if (e == cudaSuccess) e = cudaEventRecord(d2h_ev[s], d2h_stream);
                    if (e != cudaSuccess) {
                        fail(e);
                        break;
                    }
                    fl.push_back({s, c, J});
                    s = (s + 1) % nslots;
                }
            }
            bool more;
            {
                std::lock_guard<std::mutex> l(m);
                more = !d2h_q.empty();
            }
            if (!more)
                while (!fl.empty()) drain_one();
            {
                std::lock_guard<std::mutex> l(m);
                --busy;
            }
            cv_idle.notify_all();
        }
    }
};

HostStager::HostStager(int device) {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    int threads = static_cast<int>(std::min(8u, std::max(1u, hw / 2 - 1)));  // helpers per direction
    if (const char* e = std::getenv("OZK_HOST_STAGE_THREADS")) threads = std::max(0, std::atoi(e));
    size_t slot = size_t(16) << 20;
    if (const char* e = std::getenv("OZK_HOST_STAGE_SLOT")) {  // tests: small slots split columns
        const long long v = std::atoll(e);
        if (v > 0) slot = static_cast<size_t>(v);
    }
    impl_ = new Impl(device, slot, 8, threads);
}

HostStager::~HostStager() {
    if (!impl_) return;
    {
        std::lock_guard<std::mutex> l(impl_->m);
        impl_->stop = true;
    }
    impl_->cv_job.notify_all();
    if (impl_->h2d_thread.joinable()) impl_->h2d_thread.join();
    if (impl_->d2h_thread.joinable()) impl_->d2h_thread.join();
    cudaSetDevice(impl_->device);
    for (char* p : impl_->h2d_slot) cudaFreeHost(p);
    for (char* p : impl_->d2h_slot) cudaFreeHost(p);
    for (cudaEvent_t e : impl_->h2d_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : impl_->d2h_ev) cudaEventDestroy(e);
    delete impl_;
}

cudaError_t HostStager::begin(cudaStream_t h2d, cudaStream_t d2h) {
    Impl& I = *impl_;
    if (I.h2d_slot.empty()) {
        for (int s = 0; s < I.nslots; ++s) {
            char* p = nullptr;
            cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p), I.slot);
            if (e != cudaSuccess) return e;
            I.h2d_slot.push_back(p);
            e = cudaMallocHost(reinterpret_cast<void**>(&p), I.slot);
            if (e != cudaSuccess) return e;
            I.d2h_slot.push_back(p);
            cudaEvent_t ev;
            e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
            I.h2d_ev.push_back(ev);
            e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
            I.d2h_ev.push_back(ev);
        }
        I.h2d_thread = std::thread([&I] { I.h2d_loop(); });
        I.d2h_thread = std::thread([&I] { I.d2h_loop(); });
    }
    std::lock_guard<std::mutex> l(I.m);
    I.h2d_stream = h2d;
    I.d2h_stream = d2h;
    I.err = cudaSuccess;
    I.issued = I.queued_h2d = 0;
    return cudaSuccess;
}

int64_t HostStager::h2d(void* dev, size_t dpitch, const void* host, size_t hpitch, size_t width, size_t height,
                        cudaEvent_t done) {
    Impl& I = *impl_;
    int64_t ticket;
    {
        std::lock_guard<std::mutex> l(I.m);
        I.h2d_q.push_back({static_cast<char*>(dev), dpitch, const_cast<char*>(static_cast<const char*>(host)), hpitch,
                           width, height, done});
        ticket = ++I.queued_h2d;
    }
    I.cv_job.notify_all();
    return ticket;
}

cudaError_t HostStager::wait_issued(int64_t ticket) {
    Impl& I = *impl_;
    std::unique_lock<std::mutex> l(I.m);
    I.cv_issued.wait(l, [&] { return I.issued >= ticket || I.err != cudaSuccess; });
    return I.err;
}

void HostStager::d2h(void* host, size_t hpitch, const void* dev, size_t dpitch, size_t width, size_t height,
                     cudaEvent_t ready) {
    Impl& I = *impl_;
    {
        std::lock_guard<std::mutex> l(I.m);
        I.d2h_q.push_back({const_cast<char*>(static_cast<const char*>(dev)), dpitch, static_cast<char*>(host), hpitch,
                           width, height, ready});
    }
    I.cv_job.notify_all();
}

cudaError_t HostStager::finish() {
    Impl& I = *impl_;
    std::unique_lock<std::mutex> l(I.m);
    I.cv_idle.wait(l, [&] { return (I.h2d_q.empty() && I.d2h_q.empty() && I.busy == 0) || I.err != cudaSuccess; });
    if (I.err != cudaSuccess) {
        // let the threads drop what is queued, then report
        I.h2d_q.clear();
        I.d2h_q.clear();
        I.cv_idle.wait(l, [&] { return I.busy == 0; });
    }
    return I.err;
}

}  // namespace ozk
