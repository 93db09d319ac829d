// hostpool.h — a small persistent pool of host threads for the result
// assembly of tsk_search (search.cu): the id columns of a compact result
// are expanded from (entry, query) ordinals on the host while the next
// chunk is still crossing PCIe.
#pragma once

#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace tsk {

class HostPool {
  public:
    static HostPool &get() {
        static HostPool pool;
        return pool;
    }
    int size() const { return (int)workers_.size() + 1; }

    // fn(part, parts) for part = 0..parts-1, parts = size(); the caller runs
    // part 0 and returns when every part is done.
    void run(const std::function<void(int, int)> &fn) {
        std::lock_guard<std::mutex> one(run_mu_);  // one job at a time (calls from several host threads)
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &fn;
        pending_ = (int)workers_.size();
        ++gen_;
        cv_.notify_all();
        lk.unlock();
        fn(0, size());
        lk.lock();
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    HostPool() {
        unsigned hw = std::thread::hardware_concurrency();
        int n = hw ? (int)hw : 8;
        if (n > 16) n = 16;
        for (int w = 1; w < n; ++w) workers_.emplace_back([this, w] { loop(w); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            cv_.notify_all();
        }
        for (auto &t : workers_) t.join();
    }
    void loop(int w) {
        unsigned long seen = 0;
        for (;;) {
            const std::function<void(int, int)> *job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            (*job)(w, size());
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int, int)> *job_ = nullptr;
    unsigned long gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

}  // namespace tsk
