#include "host_util.hpp"

#include <algorithm>
#include <cmath>

#include "rng.hpp"

namespace pg {

ThreadPool::ThreadPool(int n) {
  for (int i = 1; i < std::max(1, n); ++i) workers_.emplace_back([this] { loop(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop() {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(int)>* job;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      job = job_;
      ++active_;
    }
    for (;;) {
      int i;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (next_ >= n_) break;
        i = next_++;
      }
      (*job)(i);
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      --active_;
    }
    done_cv_.notify_all();
  }
}

void ThreadPool::parallel_for(int n, const std::function<void(int)>& f) {
  if (n <= 0) return;
  if (workers_.empty() || n == 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = &f;
    n_ = n;
    next_ = 0;
    ++gen_;
  }
  cv_.notify_all();
  for (;;) {
    int i;
    {
      std::lock_guard<std::mutex> g(mu_);
      if (next_ >= n_) break;
      i = next_++;
    }
    f(i);
  }
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return active_ == 0 && next_ >= n_; });
  job_ = nullptr;
}

void cosine_label(long C, long H, long W, long per_label, uint64_t seed, int label, double* out) {
  Rng rng(derive_seed(seed, static_cast<uint64_t>(label)));
  const double two_pi = 6.283185307179586476925286766559;
  const long HW = H * W;
  std::vector<double> field(static_cast<size_t>(C * HW));
  for (long c = 0; c < C; ++c) {
    double u[8], v[8], a[8], ph[8];
    for (int t = 0; t < 8; ++t) {
      u[t] = static_cast<double>(static_cast<long>(rng.index(7)) - 3);
      v[t] = static_cast<double>(static_cast<long>(rng.index(7)) - 3);
      a[t] = rng.normal();
      ph[t] = two_pi * rng.uniform();
    }
    double peak = 0;
    double* f = field.data() + c * HW;
    for (long y = 0; y < H; ++y)
      for (long x = 0; x < W; ++x) {
        double s = 0;
        for (int t = 0; t < 8; ++t)
          s += a[t] * std::cos(two_pi * (u[t] * static_cast<double>(x) / static_cast<double>(W) +
                                         v[t] * static_cast<double>(y) / static_cast<double>(H)) + ph[t]);
        f[y * W + x] = s;
        peak = std::max(peak, std::abs(s));
      }
    if (peak > 0)
      for (long t = 0; t < HW; ++t) f[t] /= peak;
  }
  const long S = C * HW;
  for (long j = 0; j < per_label; ++j) {
    double* o = out + j * S;
    for (long t = 0; t < S; ++t) {
      double val = field[static_cast<size_t>(t)] + 0.1 * rng.normal();
      o[t] = (std::min(1.0, std::max(-1.0, val)) + 1.0) * 0.5;
    }
  }
}

}  // namespace pg
