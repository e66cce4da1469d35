// Engine selection for the implicit GEMMs, launch accounting and the
// optional per-GEMM event timing used by bench.py's roofline figure.
#include <atomic>
#include <mutex>
#include <vector>

#include "kernels.hpp"

namespace pg {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_timing{false};
std::mutex g_mu;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
}  // namespace

cudaError_t launched() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

long long launch_count() { return g_launches.load(); }

void gemm_timing_enable(bool on) {
  std::lock_guard<std::mutex> g(g_mu);
  for (auto& e : g_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_events.clear();
  g_timing = on;
}

double gemm_timing_read_ms() {
  std::lock_guard<std::mutex> g(g_mu);
  double total = 0;
  for (auto& e : g_events) {
    cudaEventSynchronize(e.second);
    float ms = 0;
    cudaEventElapsedTime(&ms, e.first, e.second);
    total += ms;
  }
  return total;
}

cudaError_t launch_gemm(const GemmArgs& a, int math, cudaStream_t st) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  cudaError_t r = (math != MATH_FP32_SIMT && gemm_tc_supported(a)) ? launch_gemm_tc(a, math, st)
                                                                    : launch_gemm_simt(a, st);
  if (g_timing) {
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> g(g_mu);
    g_events.emplace_back(e0, e1);
  }
  return r;
}

}  // namespace pg
