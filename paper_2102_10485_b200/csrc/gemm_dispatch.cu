// Engine selection for the implicit GEMMs, launch accounting and the
// optional per-GEMM event timing used by bench.py's roofline figure.
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <mutex>
#include <vector>
#include <map>
#include <stdexcept>

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

// caller-owned workspace of a stream (pg_set_workspace): SCRATCH_GEMM is
// carved from its start, SCRATCH_BLO from its end; both are live within one
// GEMM call, so a request fails loudly when the two would overlap
struct UserWs {
  char* p = nullptr;
  size_t bytes = 0;
  size_t used[SCRATCH_SLOTS] = {};  // bytes requested per slot in the current GEMM call
};
std::map<std::pair<int, cudaStream_t>, UserWs> g_user_ws;
size_t ws_round(size_t b) { return (b + 255) / 256 * 256; }
}  // namespace

void set_stream_workspace(cudaStream_t st, void* p, size_t bytes) {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  const auto key = std::make_pair(cur_device(), st);
  if (!p) {
    g_user_ws.erase(key);
    return;
  }
  if (reinterpret_cast<uintptr_t>(p) % 256) throw std::invalid_argument("workspace must be 256-byte aligned");
  UserWs w;
  w.p = static_cast<char*>(p);
  w.bytes = bytes / 256 * 256;
  g_user_ws[key] = w;
}

void scratch_call_begin(cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  auto it = g_user_ws.find(std::make_pair(cur_device(), st));
  if (it != g_user_ws.end())
    for (size_t& u : it->second.used) u = 0;
}

float* stream_scratch(int slot, size_t floats, cudaStream_t st) {
  std::lock_guard<std::mutex> g(g_scratch_mu);
  auto uw = g_user_ws.find(std::make_pair(cur_device(), st));
  if (uw != g_user_ws.end()) {
    UserWs& w = uw->second;
    const size_t need = ws_round(floats * sizeof(float));
    size_t other = 0;
    for (int s = 0; s < SCRATCH_SLOTS; ++s)
      if (s != slot) other += w.used[s];
    if (need + other > w.bytes)
      throw std::invalid_argument("workspace too small: this call needs " + std::to_string(need + other) +
                                  " bytes (pg_workspace_size), the stream has " + std::to_string(w.bytes));
    w.used[slot] = need;
    return reinterpret_cast<float*>(slot == SCRATCH_GEMM ? w.p : w.p + (w.bytes - need));
  }
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
  g_user_ws.erase(std::make_pair(dev, st));
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

GemmWorkspace gemm_workspace(const GemmArgs& a, int math) {
  GemmWorkspace w;
  if (dense_wide_enabled() && dense_wide_supported(a)) return w;
  if (math != MATH_FP32_SIMT && dgrad4_supported(a, math)) return w;
  if (math != MATH_FP32_SIMT && lowered_enabled(a) && gemm_lowered_supported(a)) return gemm_lowered_workspace(a, math);
  if (math != MATH_FP32_SIMT && image_side_direct(a)) return w;
  if (gemm_thin_supported(a)) {
    w.gemm = gemm_thin_workspace_floats(a);
    return w;
  }
  if (math != MATH_FP32_SIMT && gemm_pair_supported(a)) w.blo = gemm_pair_blo_floats(a, math);
  return w;
}

cudaError_t launch_gemm(const GemmArgs& a, int math, cudaStream_t st) {
  scratch_call_begin(st);
  if (a.stat_mode != STAT_NONE && (a.kind == GEMM_WGRAD || gemm_stat_slots(a, math) == 0)) return cudaErrorInvalidValue;
  // the input-side activation backward exists only in the 4-channel image-side kernels
  if (a.in_act != ACT_NONE && !(a.kind == GEMM_WGRAD ? wgrad4_supported(a, math) : dgrad4_supported(a, math)))
    return cudaErrorInvalidValue;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  cudaError_t r;
  if (dense_wide_enabled() && dense_wide_supported(a)) r = launch_dense_wide(a, st);  // latent projection
  else if (math != MATH_FP32_SIMT && dgrad4_supported(a, math)) r = launch_dgrad4(a, math, st);  // 4-channel DGRAD
  else if (math != MATH_FP32_SIMT && lowered_enabled(a) && gemm_lowered_supported(a)) r = launch_gemm_lowered(a, math, st);
  else if (math != MATH_FP32_SIMT && fprop4_supported(a, math)) r = launch_fprop4(a, math, st);  // 4-channel FPROP
  else if (math != MATH_FP32_SIMT && image_side_direct(a)) r = launch_gemm_pair(a, math, st);  // 4-channel FPROP + stats
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
