// Pageable host <-> device copies through pinned staging buffers (host side
// of libpolycast_cuda.so; used by the C-ABI's host-pointer entry points).
//
// cudaMemcpy from pageable memory runs at ~11 GB/s on the B200 boxes (the
// driver's own single-threaded staging); pinned memory DMAs at ~45-50 GB/s.
// A Stager keeps two pinned chunks per device and fills / drains them with a
// small pool of host threads while the copy engine moves the other chunk, so
// a pageable transfer approaches the pinned rate.  Sources that are already
// pinned (cudaHostAlloc / cudaHostRegister) go straight to cudaMemcpyAsync.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pch {

// Fixed worker threads; run(n, fn) calls fn(0) .. fn(n-1) on the workers and
// the caller, and returns when all are done.
class Pool {
  public:
    explicit Pool(int workers) {
        for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return (int)th_.size() + 1; }
    void run(int n, const std::function<void(int)>& fn) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return done_ == n_; });
        fn_ = nullptr;
    }

  private:
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* f;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!fn_ || next_ >= n_) return;
                i = next_++;
                f = fn_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (++done_ == n_) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

inline bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

class Stager {
  public:
    static constexpr size_t kChunk = 16u << 20;  // bytes per staging chunk
    static constexpr size_t kDirect = 4u << 20;  // smaller copies: plain cudaMemcpyAsync

    ~Stager() { release(); }

    // dst (device) <- src (host).  Returns once src may be reused; the last
    // chunk's DMA may still be in flight on `st`.
    cudaError_t h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
        if (n < kDirect || is_pinned(src)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
        cudaError_t e = ensure();
        for (size_t off = 0, k = 0; e == cudaSuccess && off < n; off += kChunk, ++k) {
            const size_t m = std::min(kChunk, n - off);
            const int b = (int)(k & 1);
            if (used_[b] && (e = cudaEventSynchronize(ev_[b])) != cudaSuccess) break;
            pcopy(pin_[b], static_cast<const char*>(src) + off, m);
            e = cudaMemcpyAsync(static_cast<char*>(dst) + off, pin_[b], m, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaEventRecord(ev_[b], st);
            used_[b] = true;
        }
        return e;
    }

    // dst (host) <- src (device), after the work queued on `st`; complete on return.
    cudaError_t d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
        if (n < kDirect || is_pinned(dst)) {
            cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
            return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
        }
        cudaError_t e = ensure();
        const size_t chunks = (n + kChunk - 1) / kChunk;
        for (size_t k = 0; e == cudaSuccess && k <= chunks; ++k) {
            if (k < chunks) { // queue chunk k into buffer k & 1 (free: drained two steps ago)
                const size_t off = k * kChunk, m = std::min(kChunk, n - off);
                e = cudaMemcpyAsync(pin_[k & 1], static_cast<const char*>(src) + off, m, cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaEventRecord(ev_[k & 1], st);
                used_[k & 1] = true;
            }
            if (k > 0 && e == cudaSuccess) { // drain chunk k - 1 while chunk k is in flight
                const size_t off = (k - 1) * kChunk, m = std::min(kChunk, n - off);
                const int b = (int)((k - 1) & 1);
                if ((e = cudaEventSynchronize(ev_[b])) != cudaSuccess) break;
                pcopy(static_cast<char*>(dst) + off, pin_[b], m);
            }
        }
        return e;
    }

    void release() {
        for (int b = 0; b < 2; ++b) {
            if (used_[b]) cudaEventSynchronize(ev_[b]);
            if (pin_[b]) cudaFreeHost(pin_[b]);
            if (ev_[b]) cudaEventDestroy(ev_[b]);
            pin_[b] = nullptr;
            ev_[b] = nullptr;
            used_[b] = false;
        }
        delete pool_;
        pool_ = nullptr;
    }

  private:
    cudaError_t ensure() {
        for (int b = 0; b < 2; ++b) {
            if (!pin_[b]) {
                cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&pin_[b]), kChunk);
                if (e != cudaSuccess) return e;
            }
            if (!ev_[b]) {
                cudaError_t e = cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming);
                if (e != cudaSuccess) return e;
            }
        }
        if (!pool_) {
            const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
            pool_ = new Pool((int)std::min(8u, hw) - 1);
        }
        return cudaSuccess;
    }
    void pcopy(char* dst, const char* src, size_t m) {
        const int parts = pool_->size();
        const size_t per = ((m + parts - 1) / parts + 63) & ~size_t(63);
        pool_->run(parts, [&](int i) {
            const size_t lo = std::min(m, (size_t)i * per), hi = std::min(m, lo + per);
            if (hi > lo) std::memcpy(dst + lo, src + lo, hi - lo);
        });
    }
    char* pin_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    bool used_[2] = {false, false};
    Pool* pool_ = nullptr;
};

} // namespace pch
