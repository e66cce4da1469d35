// extern "C" surface of include/pg_network.h: one device network behind the
// reference's build_network / forward / infer / backward (network.cpp:308-480)
// and adam_step on host vectors (optim.cpp:20-34).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pg_network.h"
#include "capi_util.hpp"
#include "device_cache.hpp"
#include "net.hpp"

struct pg_net {
  int device = 0, math = 0;
  std::string spec;
  std::vector<long> in_shape;
  std::unique_ptr<pg::DevNet> net;
  int bmax = 0;
  cudaStream_t st = nullptr;
};

struct pg_trace {
  pg_net* owner = nullptr;
  int B = 0;
  bool consumed = false;
  pg::Trace t;
};

namespace {

using pg::check_cuda;
using pg::guard;

std::string shape_str(long B, const std::vector<long>& s) {
  std::string r = "[" + std::to_string(B);
  for (long d : s) r += "x" + std::to_string(d);
  return r + "]";
}

// the per-sample reference shape of a device map: [C,H,W] for spatial maps, [F] for flat ones
void to_device_layout(const pg::Map& m, bool spatial, int B, const double* ref, std::vector<float>& dev) {
  dev.assign(static_cast<size_t>(B) * m.numel(), 0.f);
  const long C = m.C, H = m.H, W = m.W, Cp = m.Cp;
  for (long b = 0; b < B; ++b)
    for (long c = 0; c < C; ++c)
      for (long y = 0; y < H; ++y)
        for (long x = 0; x < W; ++x)
          dev[static_cast<size_t>(b * m.numel() + (y * W + x) * Cp + c)] =
              static_cast<float>(ref[((b * C + c) * H + y) * W + x]);
  (void)spatial;
}

void from_device_layout(const pg::Map& m, int B, const std::vector<float>& dev, double* ref) {
  const long C = m.C, H = m.H, W = m.W, Cp = m.Cp;
  for (long b = 0; b < B; ++b)
    for (long c = 0; c < C; ++c)
      for (long y = 0; y < H; ++y)
        for (long x = 0; x < W; ++x)
          ref[((b * C + c) * H + y) * W + x] =
              static_cast<double>(dev[static_cast<size_t>(b * m.numel() + (y * W + x) * Cp + c)]);
}

void set_dev(const pg_net* n) { check_cuda(cudaSetDevice(n->device), "cudaSetDevice"); }

// device buffers sized for at least B samples (parameters and buffers carried over)
void ensure_batch(pg_net* n, int B) {
  if (B < 1) throw std::invalid_argument("batch size must be positive");
  if (n->net && B <= n->bmax) return;
  auto fresh = std::make_unique<pg::DevNet>(n->spec, n->in_shape, 1, B, n->math);
  if (n->net) {
    check_cuda(cudaStreamSynchronize(n->st), "sync");
    check_cuda(cudaMemcpy(fresh->params.p, n->net->params.p, sizeof(float) * n->net->P(), cudaMemcpyDeviceToDevice),
               "params");
    check_cuda(cudaMemcpy(fresh->running.p, n->net->running.p,
                          sizeof(float) * std::max<long long>(n->net->Bf(), 4), cudaMemcpyDeviceToDevice),
               "buffers");
  }
  n->net = std::move(fresh);
  n->bmax = B;
}

std::vector<long> out_shape(const pg_net* n) { return n->net->ref_out_shape(); }

}  // namespace

extern "C" {

int pg_net_create(const char* spec, const long* in_shape, int in_rank, uint64_t seed, double init_std, int math,
                  int device, pg_net** out) {
  return guard([&] {
    if (!spec || !in_shape || !out) throw std::invalid_argument("null argument");
    if (in_rank != 1 && in_rank != 3) throw std::invalid_argument("input shape must be [F] or [C,H,W]");
    *out = nullptr;
    auto n = std::make_unique<pg_net>();
    n->device = device;
    if (math < PG_MATH_FP32_SIMT || math > PG_MATH_BF16) throw std::invalid_argument("unknown math mode");
    n->math = math;
    n->spec = spec;
    n->in_shape.assign(in_shape, in_shape + in_rank);
    set_dev(n.get());
    check_cuda(cudaStreamCreateWithFlags(&n->st, cudaStreamNonBlocking), "stream");
    ensure_batch(n.get(), 1);
    // build_network's draws (network.cpp:308-343), then the fp32 device layout
    auto p = n->net->init_ref_params(seed, init_std);
    auto b = n->net->init_ref_buffers();
    std::vector<float> hp(static_cast<size_t>(n->net->P())), hb(static_cast<size_t>(std::max<long long>(n->net->Bf(), 4)));
    n->net->import_params(p.data(), hp.data());
    n->net->import_buffers(b.data(), hb.data());
    check_cuda(cudaMemcpy(n->net->params.p, hp.data(), hp.size() * sizeof(float), cudaMemcpyHostToDevice), "params");
    check_cuda(cudaMemcpy(n->net->running.p, hb.data(), hb.size() * sizeof(float), cudaMemcpyHostToDevice), "buffers");
    *out = n.release();
  });
}

void pg_net_destroy(pg_net* n) {
  if (!n) return;
  cudaSetDevice(n->device);
  if (n->st) {
    cudaStreamSynchronize(n->st);
    pg::release_stream_scratch(n->st);
  }
  n->net.reset();
  if (n->st) cudaStreamDestroy(n->st);
  delete n;
}

long pg_net_param_count(const pg_net* n) { return n ? n->net->ref_params() : -1; }
long pg_net_buffer_count(const pg_net* n) { return n ? n->net->ref_buffers() : -1; }

int pg_net_out_shape(const pg_net* n, long* shape, int* rank) {
  return guard([&] {
    if (!n || !shape || !rank) throw std::invalid_argument("null argument");
    auto s = out_shape(n);
    *rank = static_cast<int>(s.size());
    for (size_t i = 0; i < s.size() && i < 4; ++i) shape[i] = s[i];
  });
}

int pg_net_get_params(pg_net* n, double* out) {
  return guard([&] {
    set_dev(n);
    check_cuda(cudaStreamSynchronize(n->st), "sync");
    std::vector<float> h(static_cast<size_t>(n->net->P()));
    check_cuda(cudaMemcpy(h.data(), n->net->params.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost), "params");
    n->net->export_params(h.data(), out);
  });
}

int pg_net_set_params(pg_net* n, const double* in) {
  return guard([&] {
    set_dev(n);
    check_cuda(cudaStreamSynchronize(n->st), "sync");
    std::vector<float> h(static_cast<size_t>(n->net->P()));
    n->net->import_params(in, h.data());
    check_cuda(cudaMemcpy(n->net->params.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice), "params");
  });
}

int pg_net_get_buffers(pg_net* n, double* out) {
  return guard([&] {
    set_dev(n);
    check_cuda(cudaStreamSynchronize(n->st), "sync");
    std::vector<float> h(static_cast<size_t>(std::max<long long>(n->net->Bf(), 4)));
    check_cuda(cudaMemcpy(h.data(), n->net->running.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost), "buffers");
    n->net->export_buffers(h.data(), out);
  });
}

int pg_net_set_buffers(pg_net* n, const double* in) {
  return guard([&] {
    set_dev(n);
    check_cuda(cudaStreamSynchronize(n->st), "sync");
    std::vector<float> h(static_cast<size_t>(std::max<long long>(n->net->Bf(), 4)));
    n->net->import_buffers(in, h.data());
    check_cuda(cudaMemcpy(n->net->running.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice), "buffers");
  });
}

int pg_net_forward(pg_net* n, const double* x, int B, int train, double* y, pg_trace** trace) {
  return guard([&] {
    if (!n || !x) throw std::invalid_argument("null argument");
    if (trace) *trace = nullptr;
    set_dev(n);
    ensure_batch(n, B);
    pg::DevNet& net = *n->net;
    auto tr = std::make_unique<pg_trace>();
    tr->owner = n;
    tr->B = B;
    tr->t = net.make_trace(false);
    std::vector<float> h;
    to_device_layout(net.in_map(), n->in_shape.size() == 3, B, x, h);
    check_cuda(cudaMemcpyAsync(tr->t.act[0], h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, n->st),
               "input H2D");
    net.forward(tr->t, B, train != 0, train != 0, n->st);
    if (y) {
      const pg::Map& om = net.out_map();
      std::vector<float> o(static_cast<size_t>(B) * om.numel());
      check_cuda(cudaMemcpyAsync(o.data(), tr->t.act[static_cast<size_t>(net.blocks())], o.size() * sizeof(float),
                                 cudaMemcpyDeviceToHost, n->st),
                 "output D2H");
      check_cuda(cudaStreamSynchronize(n->st), "forward");
      from_device_layout(om, B, o, y);
    }
    check_cuda(cudaStreamSynchronize(n->st), "forward");
    if (trace) *trace = tr.release();
  });
}

int pg_net_backward(pg_net* n, pg_trace* tr, const double* gy, int B, double* gparams, double* gx) {
  return guard([&] {
    if (!n || !gy) throw std::invalid_argument("null argument");
    // the reference's checks and messages (network.cpp:430-440)
    if (!tr || tr->owner != n) throw std::invalid_argument("trace does not belong to this network");
    if (tr->consumed) throw std::invalid_argument("trace already consumed by a previous backward call");
    tr->consumed = true;
    if (B != tr->B)
      throw std::invalid_argument("output gradient shape " + shape_str(B, out_shape(n)) +
                                  " does not match network output " + shape_str(tr->B, out_shape(n)));
    set_dev(n);
    pg::DevNet& net = *n->net;
    const pg::Map& om = net.out_map();
    const pg::Map& im = net.in_map();
    std::vector<float> h;
    to_device_layout(om, false, B, gy, h);
    pg::DeviceBuf dgy(h.size()), dgx(static_cast<size_t>(B) * im.numel());
    check_cuda(cudaMemcpyAsync(dgy.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, n->st), "gy H2D");
    net.backward(tr->t, B, dgy.p, true, false, dgx.p, n->st);
    check_cuda(cudaStreamSynchronize(n->st), "backward");
    if (gparams) {
      std::vector<float> g(static_cast<size_t>(net.P()));
      check_cuda(cudaMemcpy(g.data(), net.grads.p, g.size() * sizeof(float), cudaMemcpyDeviceToHost), "grads");
      net.export_params(g.data(), gparams);
    }
    if (gx) {
      std::vector<float> g(dgx.n);
      check_cuda(cudaMemcpy(g.data(), dgx.p, g.size() * sizeof(float), cudaMemcpyDeviceToHost), "gx");
      from_device_layout(im, B, g, gx);
    }
  });
}

void pg_trace_destroy(pg_trace* tr) {
  if (!tr) return;
  if (tr->owner) cudaSetDevice(tr->owner->device);
  delete tr;
}

int pg_adam_step_host(long n, double* params, const double* grads, double* m, double* v, long* t, double lr,
                      double beta1, double beta2, double eps, int device) {
  return guard([&] {
    if (n < 0 || (n > 0 && (!params || !grads || !m || !v)) || !t) throw std::invalid_argument("null argument");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    const long long P = (n + 3) / 4 * 4;  // the Adam kernel walks float4 groups
    // [p | g | m | v] in one staging buffer
    std::vector<float> h(static_cast<size_t>(4 * P), 0.f);
    for (long i = 0; i < n; ++i) {
      h[static_cast<size_t>(i)] = static_cast<float>(params[i]);
      h[static_cast<size_t>(P + i)] = static_cast<float>(grads[i]);
      h[static_cast<size_t>(2 * P + i)] = static_cast<float>(m[i]);
      h[static_cast<size_t>(3 * P + i)] = static_cast<float>(v[i]);
    }
    cudaStream_t st = nullptr;
    check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } sg{st};
    pg::DeviceBuf d(static_cast<size_t>(4 * P));
    int* flags = nullptr;
    long long* tt = nullptr;
    check_cuda(cudaMalloc(&flags, sizeof(int)), "malloc");
    struct Free {
      void* p;
      ~Free() { cudaFree(p); }
    } f1{flags};
    check_cuda(cudaMalloc(&tt, sizeof(long long)), "malloc");
    Free f2{tt};
    const long long t0 = *t;
    int flag = 0;
    check_cuda(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemcpyAsync(flags, &flag, sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemcpyAsync(tt, &t0, sizeof(long long), cudaMemcpyHostToDevice, st), "H2D");
    float* dp = d.p;
    check_cuda(pg::launch_nonfinite_check(1, P, dp + P, flags, st), "nonfinite");
    check_cuda(pg::launch_adam_tick(1, flags, tt, st), "tick");
    check_cuda(pg::launch_adam(1, P, dp, dp + P, dp + 2 * P, dp + 3 * P, tt, flags, static_cast<float>(lr), beta1, beta2,
                               static_cast<float>(eps), st),
               "adam");
    check_cuda(cudaMemcpyAsync(&flag, flags, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "adam");
    // the reference rejects before touching state (optim.cpp:21-25)
    if (flag) throw pg::NonFiniteError("adam_step: non-finite gradient rejected");
    check_cuda(cudaMemcpyAsync(h.data(), d.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "adam");
    for (long i = 0; i < n; ++i) {
      params[i] = h[static_cast<size_t>(i)];
      m[i] = h[static_cast<size_t>(2 * P + i)];
      v[i] = h[static_cast<size_t>(3 * P + i)];
    }
    *t = t0 + 1;
  });
}

}  // extern "C"
