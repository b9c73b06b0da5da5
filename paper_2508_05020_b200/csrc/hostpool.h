// hostpool.h -- a small persistent host thread pool for the O(active) loops of the regrid plan (build_plan):
// run(n, f) calls f(k) for every chunk k in [0, n) on the pool's workers and the calling thread and returns when
// all chunks are done.  Workers are created once (first use) and park on a condition variable between jobs, so a
// parallel region costs a wake-up, not a thread start.  Chunks write disjoint outputs; results are merged by the
// caller in chunk order, so they do not depend on the thread count.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace amr {

class HostPool {
  public:
    static HostPool& get() {
        static HostPool p;
        return p;
    }
    int threads() const { return (int)th_.size() + 1; }
    void run(int n, const std::function<void(int)>& f) {
        if (n <= 1 || th_.empty()) {
            for (int k = 0; k < n; ++k) f(k);
            return;
        }
        std::unique_lock<std::mutex> lk(m_);
        job_ = &f;
        n_ = n;
        next_.store(0);
        pending_ = (int)th_.size();
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        work();
        lk.lock();
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

  private:
    HostPool() {
        const char* e = getenv("AMR_HOST_THREADS");   // default: up to 8 (the plan loops are ~10^4 items)
        int want = e ? atoi(e) : std::min(8, (int)std::thread::hardware_concurrency());
        for (int k = 1; k < want; ++k) th_.emplace_back([this] { loop(); });
    }
    void work() {
        for (int k; (k = next_.fetch_add(1)) < n_;) (*job_)(k);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            if (stop_) return;
            lk.unlock();
            work();
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    int n_ = 0, pending_ = 0;
    std::atomic<int> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace amr
