// Host-side helpers: a persistent worker pool (per-label RNG work is spread
// over host threads so latent sampling never throttles the GPU), the
// label-sharding rule used across GPUs, and the cosine-field dataset.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace pg {

class ThreadPool {
 public:
  explicit ThreadPool(int n);
  ~ThreadPool();
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // runs f(i) for i in [0, n); the caller thread participates; blocks until done
  void parallel_for(int n, const std::function<void(int)>& f);

 private:
  void loop();
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, next_ = 0, active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// GPU g of P owns labels [shard_begin(g), shard_begin(g+1)): balanced
// contiguous blocks whose sizes differ by at most one.
inline int shard_begin(int n_labels, int n_gpus, int g) {
  return static_cast<int>((static_cast<long long>(g) * n_labels) / n_gpus);
}

// One label of the cosine-field synthetic dataset ([per_label][C][H][W] in
// [0,1], f64).  Definition (shared with the test oracle):
// stream Rng(derive_seed(seed, label)); per channel 8 terms
//   u = index(7)-3, v = index(7)-3, a = normal(), phi = 2 pi uniform();
// F(y,x) = sum a cos(2 pi (u x/W + v y/H) + phi) scaled by 1/max|F|; then per
// sample and pixel ([C][H][W] order) clamp(F + 0.1 normal(), -1, 1) -> (v+1)/2.
void cosine_label(long C, long H, long W, long per_label, uint64_t seed, int label, double* out);

}  // namespace pg
