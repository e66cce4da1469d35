// Engine selection for the implicit GEMMs, launch accounting and the
// optional per-GEMM event timing used by bench.py's roofline figure.
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <mutex>
#include <vector>
#include <map>

#include "device_cache.hpp"
#include "kernels.hpp"

namespace pg {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_timing{false};
std::mutex g_mu;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
std::vector<std::string> g_tags;
// PG_NO_LOWERED bit 1: im2col FPROP, bit 2: column-GEMM + col2im DGRAD (A/B only)
bool lowered_enabled(const GemmArgs& a) {
  static const int off = [] {
    const char* e = std::getenv("PG_NO_LOWERED");
    return e ? std::atoi(e) : 0;
  }();
  return !(off & (a.kind == GEMM_FPROP ? 1 : 2));
}
// PG_DENSE_WIDE=0: the wide dense layers on the previous engines (A/B timing)
bool dense_wide_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_DENSE_WIDE");
    return !(e && e[0] == '0');
  }();
  return on;
}
// FPROP shapes the SIMT thin kernels also accept but the pair engine runs
// faster: the 4-channel image side (direct TMA gather, KIND_F4) and wide dense
// layers with a small K (the generator's latent projection, K = 100)
bool image_side_direct(const GemmArgs& a) {
  if (a.kind != GEMM_FPROP) return false;
  const ConvGeo& g = a.g;
  const bool dense = g.k == 1 && g.SH == 1 && g.SW == 1 && g.GH == 1 && g.GW == 1;
  return (g.CG == 4 || (dense && g.CS >= 64)) && gemm_pair_supported(a);
}
}  // namespace

std::string gemm_timing_report() {
  std::lock_guard<std::mutex> g(g_mu);
  std::string out;
  char buf[64];
  for (size_t i = 0; i < g_events.size(); ++i) {
    cudaEventSynchronize(g_events[i].second);
    float ms = 0;
    cudaEventElapsedTime(&ms, g_events[i].first, g_events[i].second);
    std::snprintf(buf, sizeof(buf), " %.4f\n", ms);
    out += g_tags[i] + buf;
  }
  return out;
}

// grow-only device scratch per (device, stream, slot): the split-K paths
// (SCRATCH_GEMM) and the pair engine's pre-split weight lo parts (SCRATCH_BLO;
// a separate slot because the lowered paths hand SCRATCH_GEMM pointers to that
// engine as operands)
namespace {
struct ScratchKey {
  int dev;
  cudaStream_t st;
  int slot;
  bool operator<(const ScratchKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (st != o.st) return st < o.st;
    return slot < o.slot;
  }
};
struct ScratchBuf {
  float* p = nullptr;
  size_t cap = 0;
};
std::mutex g_scratch_mu;
std::map<ScratchKey, ScratchBuf> g_scratch;
}  // namespace

float* stream_scratch(int slot, size_t floats, cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  ScratchBuf& b = g_scratch[ScratchKey{cur_device(), st, slot}];
  if (floats > b.cap) {
    if (b.p) {
      cudaStreamSynchronize(st);
      cudaFree(b.p);
    }
    b.p = nullptr;
    b.cap = 0;
    if (cudaMalloc(&b.p, floats * sizeof(float)) != cudaSuccess) {
      b.p = nullptr;
      return nullptr;
    }
    b.cap = floats;
  }
  return b.p;
}

void release_stream_scratch(cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  const int dev = cur_device();
  for (auto it = g_scratch.begin(); it != g_scratch.end();) {
    if (it->first.st == st && it->first.dev == dev) {
      cudaStreamSynchronize(st);
      cudaFree(it->second.p);
      it = g_scratch.erase(it);
    } else {
      ++it;
    }
  }
}

float* gemm_scratch(size_t floats, cudaStream_t st) { return stream_scratch(SCRATCH_GEMM, floats, st); }

cudaError_t launched() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

long long launch_count() { return g_launches.load(); }
void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool gemm_timing_on() { return g_timing.load(); }

void gemm_timing_enable(bool on) {
  std::lock_guard<std::mutex> g(g_mu);
  for (auto& e : g_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_events.clear();
  g_tags.clear();
  g_timing = on;
}

cudaEvent_t timing_start(cudaStream_t st) {
  if (!g_timing) return nullptr;
  cudaEvent_t e0 = nullptr;
  cudaEventCreate(&e0);
  cudaEventRecord(e0, st);
  return e0;
}

void timing_stop(cudaEvent_t e0, cudaStream_t st, const std::string& tag) {
  if (!e0) return;
  cudaEvent_t e1 = nullptr;
  cudaEventCreate(&e1);
  cudaEventRecord(e1, st);
  std::lock_guard<std::mutex> g(g_mu);
  g_events.emplace_back(e0, e1);
  g_tags.emplace_back(tag);
}

// summed device time of the implicit-GEMM launches (the "hbm ..." tagged
// elementwise launches of the same report are excluded)
double gemm_timing_read_ms() {
  std::lock_guard<std::mutex> g(g_mu);
  double total = 0;
  for (size_t i = 0; i < g_events.size(); ++i) {
    if (g_tags[i].rfind("hbm", 0) == 0) continue;
    const auto& e = g_events[i];
    cudaEventSynchronize(e.second);
    float ms = 0;
    cudaEventElapsedTime(&ms, e.first, e.second);
    total += ms;
  }
  return total;
}

int gemm_stat_slots(const GemmArgs& a, int math, int* npack) {
  if (npack) *npack = 1;
  if (math == MATH_FP32_SIMT) return 0;
  if (dense_wide_enabled() && dense_wide_supported(a)) return dense_wide_stat_slots(a);
  if (lowered_enabled(a) && gemm_lowered_supported(a)) return gemm_lowered_stat_slots(a);
  if (image_side_direct(a)) return gemm_pair_stat_slots(a, npack);
  if (gemm_thin_supported(a)) return 0;
  return gemm_pair_stat_slots(a, npack);
}

cudaError_t launch_gemm(const GemmArgs& a, int math, cudaStream_t st) {
  if (a.stat_mode != STAT_NONE && gemm_stat_slots(a, math) == 0) return cudaErrorInvalidValue;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  cudaError_t r;
  if (dense_wide_enabled() && dense_wide_supported(a)) r = launch_dense_wide(a, st);  // latent projection
  else if (math != MATH_FP32_SIMT && lowered_enabled(a) && gemm_lowered_supported(a)) r = launch_gemm_lowered(a, math, st);
  else if (math != MATH_FP32_SIMT && image_side_direct(a)) r = launch_gemm_pair(a, math, st);  // 4-channel FPROP
  else if (gemm_thin_supported(a)) r = launch_gemm_thin(a, st, math);  // image-side / dense-head shapes
  else if (math != MATH_FP32_SIMT && gemm_pair_supported(a)) r = launch_gemm_pair(a, math, st);  // big conv GEMMs
  else if (math != MATH_FP32_SIMT && gemm_tma_supported(a)) r = launch_gemm_tma(a, math, st);  // conv GEMMs
  else if (math != MATH_FP32_SIMT && gemm_tc_supported(a)) r = launch_gemm_tc(a, math, st);
  else r = launch_gemm_simt(a, st);
  if (g_timing) {
    cudaEventRecord(e1, st);
    char tag[160];
    std::snprintf(tag, sizeof(tag), "%s L=%d M=%d N=%d K=%d phases=%d CS=%d CG=%d S=%dx%d G=%dx%d k=%d",
                  a.kind == GEMM_FPROP ? "fprop" : a.kind == GEMM_DGRAD ? "dgrad" : "wgrad", a.L, gemm_max_m(a),
                  gemm_n(a),
                  a.kind == GEMM_FPROP ? a.g.k * a.g.k * a.g.CG
                                       : a.kind == GEMM_WGRAD ? a.g.B * a.g.SH * a.g.SW : a.g.k * a.g.k * a.g.CS / (a.g.s * a.g.s),
                  a.kind == GEMM_DGRAD ? a.g.s * a.g.s : 1, a.g.CS, a.g.CG, a.g.SH, a.g.SW, a.g.GH, a.g.GW, a.g.k);
    std::lock_guard<std::mutex> g(g_mu);
    g_events.emplace_back(e0, e1);
    g_tags.emplace_back(tag);
  }
  return r;
}

}  // namespace pg
