// Device network: block compilation, parameter-arena mapping, and the
// label-batched forward / backward passes.  See net.hpp.
#include "net.hpp"

#include <algorithm>
#include <cstdlib>
#include <sstream>

#include "rng.hpp"

namespace pg {

// PG_DEBUG_SYNC=1: synchronize after every checked call so an asynchronous
// fault is attributed to the launch that caused it.
static const bool g_debug_sync = std::getenv("PG_DEBUG_SYNC") != nullptr;

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess && g_debug_sync) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

DeviceBuf::DeviceBuf(size_t count) : n(count) {
  if (count) {
    check_cuda(cudaMalloc(&p, count * sizeof(float)), "cudaMalloc");
    check_cuda(cudaMemset(p, 0, count * sizeof(float)), "cudaMemset");
  }
}
DeviceBuf::~DeviceBuf() {
  if (p) cudaFree(p);
}
DeviceBuf& DeviceBuf::operator=(DeviceBuf&& o) noexcept {
  if (this != &o) {
    if (p) cudaFree(p);
    p = o.p;
    n = o.n;
    o.p = nullptr;
    o.n = 0;
  }
  return *this;
}

// ---------------------------------------------------------------------------
// layer grammar (the same text form the tests use on the oracle side)
// ---------------------------------------------------------------------------
const char* layer_name(LK k) {
  switch (k) {
    case LK::Dense: return "dense";
    case LK::Conv: return "conv2d";
    case LK::ConvT: return "conv_transpose2d";
    case LK::BN: return "batch_norm";
    case LK::Upsample: return "upsample";
    case LK::Dropout: return "dropout";
    case LK::ReLU: return "relu";
    case LK::LReLU: return "leaky_relu";
    case LK::Tanh: return "tanh";
    case LK::Sigmoid: return "sigmoid";
    case LK::Reshape: return "reshape";
  }
  return "?";
}

std::vector<LayerSpec> parse_layers(const std::string& text) {
  std::vector<LayerSpec> out;
  std::stringstream all(text);
  std::string item;
  while (std::getline(all, item, ';')) {
    std::stringstream ss(item);
    std::string name;
    if (!(ss >> name)) continue;
    std::vector<double> a;
    double v;
    while (ss >> v) a.push_back(v);
    auto need = [&](size_t n) {
      if (a.size() < n) throw std::invalid_argument("layer spec '" + item + "' needs " + std::to_string(n) + " numbers");
    };
    LayerSpec l;
    auto I = [&](size_t i) { return static_cast<long>(a[i]); };
    if (name == "dense") { need(2); l.kind = LK::Dense; l.in = I(0); l.out = I(1); }
    else if (name == "conv2d" || name == "convT2d") {
      need(5);
      l.kind = name == "conv2d" ? LK::Conv : LK::ConvT;
      l.in = I(0); l.out = I(1); l.k = I(2); l.s = I(3); l.p = I(4);
    } else if (name == "bn") {
      need(1);
      l.kind = LK::BN; l.in = l.out = I(0);
      if (a.size() > 1) l.eps = a[1];
      if (a.size() > 2) l.momentum = a[2];
    } else if (name == "upsample") { need(1); l.kind = LK::Upsample; l.scale = I(0); }
    else if (name == "dropout") { need(1); l.kind = LK::Dropout; l.rate = a[0]; }
    else if (name == "relu") l.kind = LK::ReLU;
    else if (name == "lrelu") { l.kind = LK::LReLU; l.slope = a.empty() ? 0.2 : a[0]; }
    else if (name == "tanh") l.kind = LK::Tanh;
    else if (name == "sigmoid") l.kind = LK::Sigmoid;
    else if (name == "reshape") {
      need(1);
      l.kind = LK::Reshape;
      for (size_t i = 0; i < a.size(); ++i) l.target.push_back(I(i));
    } else {
      throw std::invalid_argument("unknown layer '" + name + "'");
    }
    out.push_back(l);
  }
  return out;
}

std::vector<long> parse_shape(const std::string& text) {
  std::stringstream ss(text);
  std::vector<long> s;
  long v;
  while (ss >> v) s.push_back(v);
  return s;
}

static long numel(const std::vector<long>& s) {
  long n = 1;
  for (long d : s) n *= d;
  return n;
}

static std::string shape_str(const std::vector<long>& s) {
  std::string r = "[";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? "x" : "") + std::to_string(s[i]);
  return r + "]";
}

[[noreturn]] static void layer_fail(size_t i, const LayerSpec& l, const std::string& what) {
  throw std::invalid_argument("layer " + std::to_string(i) + " (" + layer_name(l.kind) + "): " + what);
}

long ref_param_count(const LayerSpec& l) {
  switch (l.kind) {
    case LK::Dense: return l.in * l.out + l.out;
    case LK::Conv:
    case LK::ConvT: return l.in * l.out * l.k * l.k + l.out;
    case LK::BN: return 2 * l.in;
    default: return 0;
  }
}

long ref_buffer_count(const LayerSpec& l) { return l.kind == LK::BN ? 2 * l.in : 0; }

// layers.cpp:70-104 shape algebra (+ ConvTranspose2d: (in-1)s - 2p + k)
std::vector<long> ref_out_shape(const LayerSpec& l, const std::vector<long>& in, size_t i) {
  switch (l.kind) {
    case LK::Dense:
      if (l.in < 1 || l.out < 1) layer_fail(i, l, "dimensions must be positive");
      if (in.size() != 1 || in[0] != l.in) layer_fail(i, l, "expects input [" + std::to_string(l.in) + "], got " + shape_str(in));
      return {l.out};
    case LK::Conv:
    case LK::ConvT: {
      if (l.in < 1 || l.out < 1) layer_fail(i, l, "channel counts must be positive");
      if (l.k < 1 || l.s < 1 || l.p < 0) layer_fail(i, l, "invalid kernel/stride/padding");
      if (in.size() != 3 || in[0] != l.in)
        layer_fail(i, l, "expects input [" + std::to_string(l.in) + " x H x W], got " + shape_str(in));
      if (l.kind == LK::Conv) {
        if (in[1] + 2 * l.p < l.k || in[2] + 2 * l.p < l.k) layer_fail(i, l, "kernel larger than padded input " + shape_str(in));
        return {l.out, (in[1] + 2 * l.p - l.k) / l.s + 1, (in[2] + 2 * l.p - l.k) / l.s + 1};
      }
      long oh = (in[1] - 1) * l.s - 2 * l.p + l.k, ow = (in[2] - 1) * l.s - 2 * l.p + l.k;
      if (oh < 1 || ow < 1) layer_fail(i, l, "non-positive output extent");
      return {l.out, oh, ow};
    }
    case LK::BN:
      if (in.empty() || in[0] != l.in) layer_fail(i, l, "expects " + std::to_string(l.in) + " channels, got input " + shape_str(in));
      return in;
    case LK::Upsample:
      if (in.size() != 3) layer_fail(i, l, "expects input [C x H x W]");
      return {in[0], in[1] * l.scale, in[2] * l.scale};
    case LK::Reshape:
      if (numel(in) != numel(l.target)) layer_fail(i, l, "cannot reshape " + shape_str(in) + " to " + shape_str(l.target));
      return l.target;
    default:
      return in;
  }
}

static bool is_act(LK k) { return k == LK::ReLU || k == LK::LReLU || k == LK::Tanh || k == LK::Sigmoid; }
static int act_code(LK k) {
  switch (k) {
    case LK::ReLU: return ACT_RELU;
    case LK::LReLU: return ACT_LRELU;
    case LK::Tanh: return ACT_TANH;
    case LK::Sigmoid: return ACT_SIGMOID;
    default: return ACT_NONE;
  }
}

static Map map_of(const std::vector<long>& s) {
  Map m;
  if (s.size() == 3) {
    m.C = s[0];
    m.H = s[1];
    m.W = s[2];
  } else {
    m.C = numel(s);
  }
  m.Cp = pad4(m.C);
  return m;
}

static long long align4(long long x) { return (x + 3) / 4 * 4; }

// ---------------------------------------------------------------------------
// block compilation
// ---------------------------------------------------------------------------
DevNet::DevNet(const std::string& spec, const std::vector<long>& in_shape, int L, int max_batch, int math)
    : L_(L), Bmax_(max_batch), math_(math), layers_(parse_layers(spec)) {
  if (layers_.empty()) throw std::invalid_argument("network spec list is empty");
  if (in_shape.empty()) throw std::invalid_argument("network input shape is empty");
  if (L < 1 || max_batch < 1) throw std::invalid_argument("label count and batch must be positive");
  ref_shapes_.push_back(in_shape);
  ref_off_.push_back(0);
  ref_boff_.push_back(0);
  for (size_t i = 0; i < layers_.size(); ++i) {
    ref_shapes_.push_back(pg::ref_out_shape(layers_[i], ref_shapes_.back(), i));
    ref_off_.push_back(ref_off_.back() + ref_param_count(layers_[i]));
    ref_boff_.push_back(ref_boff_.back() + ref_buffer_count(layers_[i]));
  }
  ref_P_ = ref_off_.back();
  ref_Bf_ = ref_boff_.back();

  Map cur = map_of(in_shape);
  size_t i = 0;
  const size_t n = layers_.size();
  while (i < n) {
    Block b;
    b.first_layer = static_cast<int>(i);
    b.in = cur;
    if (layers_[i].kind == LK::Reshape && i + 1 < n && layers_[i + 1].kind == LK::Dense && ref_shapes_[i].size() == 3) {
      b.in_from_chw = true;
      b.in_chw = ref_shapes_[i];
      ++i;
    } else if (layers_[i].kind == LK::Reshape && i + 1 < n && layers_[i + 1].kind == LK::Dense &&
               ref_shapes_[i].size() == 1) {
      ++i;  // [F] -> [F]: identity
    }
    const LayerSpec& lin = layers_[i];
    if (lin.kind != LK::Dense && lin.kind != LK::Conv && lin.kind != LK::ConvT)
      throw std::invalid_argument("layer " + std::to_string(i) + " (" + layer_name(lin.kind) +
                                  "): not supported on the device path here (blocks must start with dense, conv2d or "
                                  "conv_transpose2d; upsample/dropout are outside the BASELINE architectures)");
    if (lin.kind == LK::Dense && !b.in_from_chw && b.in.H * b.in.W != 1)
      throw std::invalid_argument("layer " + std::to_string(i) + " (dense): input must be flat");
    b.L = lin;
    b.lin = lin.kind;
    b.ref_lin = ref_off_[i];
    ++i;
    if (b.lin == LK::Dense && i < n && layers_[i].kind == LK::Reshape) {
      if (ref_shapes_[i + 1].size() == 3) {
        b.out_to_chw = true;
        b.out_chw = ref_shapes_[i + 1];
      }
      ++i;
    }
    if (i < n && layers_[i].kind == LK::BN) {
      b.has_bn = true;
      b.bn = layers_[i];
      b.ref_bn = ref_off_[i];
      b.ref_buf = ref_boff_[i];
      ++i;
    }
    if (i < n && is_act(layers_[i].kind)) {
      b.act = act_code(layers_[i].kind);
      b.slope = static_cast<float>(layers_[i].slope);
      ++i;
    }
    b.last_layer = static_cast<int>(i) - 1;
    b.out = map_of(ref_shapes_[i]);

    ConvGeo& g = b.geo;
    g.B = 0;
    if (b.lin == LK::Dense) {
      g.SH = g.SW = g.GH = g.GW = 1;
      g.k = g.s = 1;
      g.p = 0;
      g.CS = static_cast<int>(b.out.numel());
      g.CG = static_cast<int>(b.in.numel());
    } else if (b.lin == LK::Conv) {
      g.GH = static_cast<int>(b.in.H); g.GW = static_cast<int>(b.in.W); g.CG = static_cast<int>(b.in.Cp);
      g.SH = static_cast<int>(b.out.H); g.SW = static_cast<int>(b.out.W); g.CS = static_cast<int>(b.out.Cp);
      g.k = static_cast<int>(lin.k); g.s = static_cast<int>(lin.s); g.p = static_cast<int>(lin.p);
    } else {
      g.SH = static_cast<int>(b.in.H); g.SW = static_cast<int>(b.in.W); g.CS = static_cast<int>(b.in.Cp);
      g.GH = static_cast<int>(b.out.H); g.GW = static_cast<int>(b.out.W); g.CG = static_cast<int>(b.out.Cp);
      g.k = static_cast<int>(lin.k); g.s = static_cast<int>(lin.s); g.p = static_cast<int>(lin.p);
    }
    b.n_w = static_cast<long long>(g.CS) * g.k * g.k * g.CG;
    b.n_b = b.lin == LK::ConvT ? g.CG : g.CS;
    b.off_w = P_;
    P_ = align4(P_ + b.n_w);
    b.off_b = P_;
    P_ = align4(P_ + b.n_b);
    if (b.has_bn) {
      b.off_bn = P_;
      P_ = align4(P_ + 2 * b.bn.in);
      b.off_run = Bf_;
      Bf_ = align4(Bf_ + 2 * b.bn.in);
    }
    blocks_.push_back(b);
    cur = b.out;
  }
  P_ = align4(P_);
  params = DeviceBuf(static_cast<size_t>(L_) * P_);
  grads = DeviceBuf(static_cast<size_t>(L_) * P_);
  adam_m = DeviceBuf(static_cast<size_t>(L_) * P_);
  adam_v = DeviceBuf(static_cast<size_t>(L_) * P_);
  running = DeviceBuf(static_cast<size_t>(L_) * std::max<long long>(Bf_, 4));

  size_t mx = max_map_floats();
  gscratch_[0] = DeviceBuf(mx);
  gscratch_[1] = DeviceBuf(mx);
  gz_ = DeviceBuf(mx);
  size_t part = 0, coef = 0;
  for (auto& b : blocks_) {
    long R = static_cast<long>(Bmax_) * b.out.H * b.out.W;
    ChannelMap cm{L_, static_cast<int>(R), static_cast<int>(b.out.Cp), static_cast<int>(b.out.C), 0};
    part = std::max(part, reduce_partial_floats(cm));
    part = std::max(part, static_cast<size_t>(L_) * 4 * b.out.Cp);  // launch_slot_sum output
    // bias reductions over the linear output map
    ChannelMap cb{L_, static_cast<int>(static_cast<long>(Bmax_) * (b.lin == LK::ConvT ? b.geo.GH * b.geo.GW : b.geo.SH * b.geo.SW)),
                  b.lin == LK::ConvT ? b.geo.CG : b.geo.CS, 0, 0};
    part = std::max(part, reduce_partial_floats(cb));
    coef = std::max(coef, static_cast<size_t>(L_) * b.out.Cp * 3);
  }
  partial_ = DeviceBuf(std::max<size_t>(part, 4));
  coef_ = DeviceBuf(std::max<size_t>(coef, 4));
}

size_t DevNet::max_map_floats() const {
  size_t mx = 4;
  for (auto& b : blocks_) {
    mx = std::max(mx, static_cast<size_t>(L_) * Bmax_ * b.in.numel());
    mx = std::max(mx, static_cast<size_t>(L_) * Bmax_ * b.out.numel());
  }
  return mx;
}

// f(ref_index, dev_index) over every real (non-padding) parameter of a block
template <class F>
void DevNet::map_params(const Block& b, F f) const {
  const LayerSpec& l = b.L;
  const ConvGeo& g = b.geo;
  if (b.lin == LK::Conv) {
    for (long co = 0; co < l.out; ++co)
      for (long ci = 0; ci < l.in; ++ci)
        for (long ki = 0; ki < l.k; ++ki)
          for (long kj = 0; kj < l.k; ++kj)
            f(b.ref_lin + ((co * l.in + ci) * l.k + ki) * l.k + kj, b.off_w + ((co * l.k + ki) * l.k + kj) * g.CG + ci);
    for (long co = 0; co < l.out; ++co) f(b.ref_lin + l.out * l.in * l.k * l.k + co, b.off_b + co);
  } else if (b.lin == LK::ConvT) {
    for (long ci = 0; ci < l.in; ++ci)
      for (long co = 0; co < l.out; ++co)
        for (long ki = 0; ki < l.k; ++ki)
          for (long kj = 0; kj < l.k; ++kj)
            f(b.ref_lin + ((ci * l.out + co) * l.k + ki) * l.k + kj, b.off_w + ((ci * l.k + ki) * l.k + kj) * g.CG + co);
    for (long co = 0; co < l.out; ++co) f(b.ref_lin + l.in * l.out * l.k * l.k + co, b.off_b + co);
  } else {
    auto dout = [&](long o) -> long {
      if (!b.out_to_chw) return o;
      long hw = b.out_chw[1] * b.out_chw[2];
      return (o % hw) * b.out.Cp + o / hw;
    };
    auto din = [&](long i) -> long {
      if (!b.in_from_chw) return i;
      long hw = b.in_chw[1] * b.in_chw[2];
      return (i % hw) * b.in.Cp + i / hw;
    };
    for (long o = 0; o < l.out; ++o) {
      long od = dout(o);
      for (long i = 0; i < l.in; ++i) f(b.ref_lin + o * l.in + i, b.off_w + od * g.CG + din(i));
    }
    for (long o = 0; o < l.out; ++o) f(b.ref_lin + l.out * l.in + o, b.off_b + dout(o));
  }
  if (b.has_bn)
    for (long c = 0; c < 2 * b.bn.in; ++c) f(b.ref_bn + c, b.off_bn + c);
}

void DevNet::import_params(const double* ref, float* dev) const {
  std::fill(dev, dev + P_, 0.f);
  for (auto& b : blocks_) map_params(b, [&](long r, long long d) { dev[d] = static_cast<float>(ref[r]); });
}
void DevNet::export_params(const float* dev, double* ref) const {
  std::fill(ref, ref + ref_P_, 0.0);
  for (auto& b : blocks_) map_params(b, [&](long r, long long d) { ref[r] = static_cast<double>(dev[d]); });
}
void DevNet::import_buffers(const double* ref, float* dev) const {
  std::fill(dev, dev + Bf_, 0.f);
  for (auto& b : blocks_)
    if (b.has_bn)
      for (long c = 0; c < 2 * b.bn.in; ++c) dev[b.off_run + c] = static_cast<float>(ref[b.ref_buf + c]);
}
void DevNet::export_buffers(const float* dev, double* ref) const {
  std::fill(ref, ref + ref_Bf_, 0.0);
  for (auto& b : blocks_)
    if (b.has_bn)
      for (long c = 0; c < 2 * b.bn.in; ++c) ref[b.ref_buf + c] = static_cast<double>(dev[b.off_run + c]);
}

std::vector<double> DevNet::init_ref_params(uint64_t seed, double init_std) const {
  std::vector<double> p(static_cast<size_t>(ref_P_), 0.0);
  Rng rng(seed);
  for (size_t i = 0; i < layers_.size(); ++i) {
    const LayerSpec& l = layers_[i];
    double* q = p.data() + ref_off_[i];
    if (l.kind == LK::Dense || l.kind == LK::Conv || l.kind == LK::ConvT) {
      long nw = ref_param_count(l) - l.out;
      for (long j = 0; j < nw; ++j) q[j] = rng.normal() * init_std;
    } else if (l.kind == LK::BN) {
      for (long c = 0; c < l.in; ++c) q[c] = 1.0;
    }
  }
  return p;
}

std::vector<double> DevNet::init_ref_buffers() const {
  std::vector<double> b(static_cast<size_t>(ref_Bf_), 0.0);
  for (size_t i = 0; i < layers_.size(); ++i)
    if (layers_[i].kind == LK::BN)
      for (long c = 0; c < layers_[i].in; ++c) b[static_cast<size_t>(ref_boff_[i] + layers_[i].in + c)] = 1.0;
  return b;
}

Trace DevNet::make_trace(bool alias_input) const {
  Trace t;
  const size_t nb = blocks_.size();
  t.act.assign(nb + 1, nullptr);
  t.own.resize(nb + 1);
  t.pre.resize(nb);
  t.mean.resize(nb);
  t.istd.resize(nb);
  if (!alias_input) {
    t.own[0] = DeviceBuf(static_cast<size_t>(L_) * Bmax_ * blocks_[0].in.numel());
    t.act[0] = t.own[0].p;
  }
  for (size_t i = 0; i < nb; ++i) {
    const Block& b = blocks_[i];
    t.own[i + 1] = DeviceBuf(static_cast<size_t>(L_) * Bmax_ * b.out.numel());
    t.act[i + 1] = t.own[i + 1].p;
    if (b.has_bn) {
      t.pre[i] = DeviceBuf(static_cast<size_t>(L_) * Bmax_ * b.out.numel());
      t.mean[i] = DeviceBuf(static_cast<size_t>(L_) * b.out.Cp);
      t.istd[i] = DeviceBuf(static_cast<size_t>(L_) * b.out.Cp);
    }
  }
  return t;
}

ConvGeo DevNet::geo_for(const Block& b, int B) const {
  ConvGeo g = b.geo;
  g.B = B;
  return g;
}

// Fused epilogue statistics.  bit 1: forward BN moments (default on: saves two
// reads of every pre-BN map, measured -2 ms/step on c4), bit 2: backward
// act/BN sums (default off: the y / z reads in the epilogue stall the MMA
// pipeline more than the separate reduce pass costs, +2.7 ms/step).
// PG_FUSE overrides the bit set (A/B timing).
// PG_WG_ACT=0: the discriminator conv1's activation backward as its own pass (A/B timing)
static bool wg_act_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_WG_ACT");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool fuse_enabled(int bit) {
  static const int on = [] {
    const char* e = std::getenv("PG_FUSE");
    return e ? std::atoi(e) : 1;
  }();
  return on & bit;
}

float* DevNet::stat_buf(size_t floats, cudaStream_t st) {
  if (stat_.n < floats) {
    check_cuda(cudaStreamSynchronize(st), "stat buffer grow");
    stat_ = DeviceBuf(floats);
  }
  return stat_.p;
}

void DevNet::linear_fwd(const Block& b, int B, const float* x, float* y, bool with_epilogue, cudaStream_t st) {
  check_cuda(launch_gemm(linear_args(b, B, x, y, with_epilogue), math_, st), "linear forward");
}

GemmArgs DevNet::linear_args(const Block& b, int B, const float* x, float* y, bool with_epilogue) const {
  GemmArgs a{};
  a.g = geo_for(b, B);
  a.L = L_;
  a.kind = b.lin == LK::ConvT ? GEMM_DGRAD : GEMM_FPROP;
  if (a.kind == GEMM_FPROP) {
    a.big = x;
    a.big_ls = static_cast<long long>(B) * b.in.numel();
  } else {
    a.small = x;
    a.small_ls = static_cast<long long>(B) * b.in.numel();
  }
  a.w = params.p + b.off_w;
  a.w_ls = P_;
  a.out = y;
  a.out_ls = static_cast<long long>(B) * b.out.numel();
  a.bias = params.p + b.off_b;
  a.bias_ls = P_;
  a.act = with_epilogue ? b.act : ACT_NONE;
  a.slope = b.slope;
  a.c_valid = static_cast<int>(b.out.C);
  a.c_pad = static_cast<int>(b.out.Cp);
  return a;
}

void DevNet::forward(Trace& t, int B, bool train, bool update_running, cudaStream_t st) {
  if (B < 1 || B > Bmax_) throw std::invalid_argument("batch size outside [1, max_batch]");
  t.train = train;
  for (size_t i = 0; i < blocks_.size(); ++i) {
    const Block& b = blocks_[i];
    if (!b.has_bn) {
      linear_fwd(b, B, t.act[i], t.act[i + 1], true, st);
      continue;
    }
    float* z = t.pre[i].p;
    GemmArgs a = linear_args(b, B, t.act[i], z, false);
    ChannelMap cm{L_, static_cast<int>(static_cast<long>(B) * b.out.H * b.out.W), static_cast<int>(b.out.Cp),
                  static_cast<int>(b.out.C), static_cast<long long>(B) * b.out.numel()};
    int npack = 1;
    const int slots = train && fuse_enabled(1) ? gemm_stat_slots(a, math_, &npack) : 0;
    // a dense layer reshaped to [C][H][W] before BatchNorm: GEMM column n is
    // (pixel, channel) -> H*W statistic columns per channel
    if (npack == 1) npack = gemm_n(a) / static_cast<int>(b.out.Cp);
    if (slots > 0) {
      // batch statistics fused into the GEMM epilogue (per 32-row slot), merged here
      a.stat_mode = STAT_FWD;
      a.stat = stat_buf(static_cast<size_t>(L_) * slots * 4 * npack * b.out.Cp, st);
      check_cuda(launch_gemm(a, math_, st), "linear forward");
      cm.nslot = slots;
      cm.npack = npack;
      check_cuda(launch_bn_stats_finalize(cm, a.stat, t.mean[i].p, t.istd[i].p, running.p + b.off_run, Bf_,
                                          static_cast<float>(b.bn.eps), static_cast<float>(b.bn.momentum),
                                          update_running ? 1 : 0, st),
                 "bn stats finalize");
      cm.nslot = 0;
      cm.npack = 1;
    } else {
      check_cuda(launch_gemm(a, math_, st), "linear forward");
    }
    if (train && slots == 0) {
      check_cuda(launch_channel_reduce(cm, RED_SUM, z, nullptr, nullptr, nullptr, 0, 0.f, partial_.p, st), "bn sum");
      check_cuda(launch_bn_finalize_mean(cm, partial_.p, t.mean[i].p, st), "bn mean");
      check_cuda(launch_channel_reduce(cm, RED_SQDEV, z, nullptr, nullptr, t.mean[i].p, 0, 0.f, partial_.p, st), "bn var");
      check_cuda(launch_bn_finalize_var(cm, partial_.p, t.mean[i].p, t.istd[i].p, running.p + b.off_run, Bf_,
                                        static_cast<float>(b.bn.eps), static_cast<float>(b.bn.momentum),
                                        update_running ? 1 : 0, st),
                 "bn finalize");
    } else if (!train) {
      check_cuda(launch_bn_eval_stats(cm, running.p + b.off_run, Bf_, static_cast<float>(b.bn.eps), t.mean[i].p,
                                      t.istd[i].p, st),
                 "bn eval stats");
    }
    check_cuda(launch_bn_apply(cm, z, t.mean[i].p, t.istd[i].p, params.p + b.off_bn, P_, b.act, b.slope,
                               t.act[i + 1], st),
               "bn apply");
  }
}

void DevNet::backward(Trace& t, int B, const float* gy_ext, bool param_grads, bool accumulate, float* gx_ext,
                      cudaStream_t st) {
  const int nb = static_cast<int>(blocks_.size());
  const float* gy = gy_ext;
  int fused = 0;  // > 0: gy already is act_bwd(gy, y) and its channel sums sit in stat_ (that many slots)
  int fused_pack = 1;
  for (int i = nb - 1; i >= 0; --i) {
    const Block& b = blocks_[static_cast<size_t>(i)];
    const long long out_ls = static_cast<long long>(B) * b.out.numel();
    const long long in_ls = static_cast<long long>(B) * b.in.numel();
    ChannelMap cm{L_, static_cast<int>(static_cast<long>(B) * b.out.H * b.out.W), static_cast<int>(b.out.Cp),
                  static_cast<int>(b.out.C), out_ls};
    // 1) gradient w.r.t. the linear output (through activation and BatchNorm)
    const float* gz = gy;
    float* dbias = param_grads ? grads.p + b.off_b : nullptr;
    bool bias_done = false;
    // a conv layer with an activation, no BatchNorm and no input gradient to
    // produce (the discriminator's conv1 in its own update): its weight-gradient
    // kernel applies the activation backward to gy on the fly and sums the bias
    // gradient, so the act_bwd + bias-sum pass over (gy, y) and the g1 map drop out
    bool wg_act = param_grads && !fused && !b.has_bn && b.act != ACT_NONE && b.lin == LK::Conv && i == 0 && !gx_ext &&
                  wg_act_enabled();
    if (wg_act) {  // only the tcgen05 4-channel weight gradient (wgrad4.cu) fuses it
      GemmArgs probe{};
      probe.kind = GEMM_WGRAD;
      probe.g = geo_for(b, B);
      probe.L = L_;
      probe.small = gy;
      probe.small_ls = out_ls;
      probe.big = t.act[static_cast<size_t>(i)];
      probe.big_ls = in_ls;
      wg_act = wgrad4_supported(probe, math_);
    }
    if (b.has_bn) {
      // bn_bwd_apply takes the activation mask from (pre-BN map, BN coefficients), not the stored y
      static const bool yfree = [] {
        const char* e = std::getenv("PG_YFREE");  // 0: read the stored y (A/B timing)
        return !(e && e[0] == '0');
      }();
      const BnCoef bnc = yfree ? BnCoef{t.istd[i].p, params.p + b.off_bn, P_} : BnCoef{};
      ChannelMap cs = cm;
      if (fused) {
        // sums from the producing GEMM's epilogue, pre-reduced over its slots
        cs.nslot = fused;
        cs.npack = fused_pack;
        check_cuda(launch_slot_sum(cs, stat_.p, partial_.p, st), "bn bwd slot sum");
        cs.nslot = 1;
        cs.npack = 1;
      } else {
        static const bool yfree_red = [] {
          const char* e = std::getenv("PG_YFREE_RED");  // 0: read the stored y (A/B timing)
          return !(e && e[0] == '0');
        }();
        check_cuda(launch_channel_reduce(cm, RED_BN_BWD, t.pre[i].p, gy, t.act[i + 1], t.mean[i].p, b.act, b.slope,
                                         partial_.p, st, nullptr, yfree_red ? bnc : BnCoef{}),
                   "bn bwd reduce");
      }
      bool closed_form_bias = b.bias_per_bn_channel();
      check_cuda(launch_bn_bwd_finalize(cs, partial_.p, t.istd[i].p, params.p + b.off_bn, P_,
                                        param_grads ? grads.p + b.off_bn : nullptr, P_,
                                        closed_form_bias ? dbias : nullptr, P_, accumulate ? 1 : 0, t.train ? 1 : 0,
                                        coef_.p, st),
                 "bn bwd finalize");
      bias_done = closed_form_bias;
      check_cuda(launch_bn_bwd_apply(cm, gy, t.act[i + 1], t.pre[i].p, t.mean[i].p, coef_.p, fused ? ACT_NONE : b.act,
                                     b.slope, gz_.p, st, bnc),
                 "bn bwd apply");
      gz = gz_.p;
    } else if (wg_act) {
      bias_done = true;  // both come out of the weight-gradient launch below
    } else if (b.act != ACT_NONE && !fused) {
      if (param_grads) {
        // activation backward and the bias sums in one pass over (gy, y)
        check_cuda(launch_channel_reduce(cm, RED_ACT_G, nullptr, gy, t.act[i + 1], nullptr, b.act, b.slope, partial_.p,
                                         st, gz_.p),
                   "act bwd + bias reduce");
        check_cuda(launch_bias_finalize(cm, partial_.p, dbias, P_, accumulate ? 1 : 0, st), "bias finalize");
        bias_done = true;
      } else {
        check_cuda(launch_act_bwd(cm, gy, t.act[i + 1], b.act, b.slope, gz_.p, st), "act bwd");
      }
      gz = gz_.p;
    }
    if (param_grads && !bias_done && fused && !b.has_bn) {
      ChannelMap cb = cm;
      cb.nslot = fused;
      cb.npack = fused_pack;
      check_cuda(launch_slot_sum(cb, stat_.p, partial_.p, st), "bias slot sum");
      cb.nslot = 1;
      cb.npack = 1;
      check_cuda(launch_bias_finalize(cb, partial_.p, dbias, P_, accumulate ? 1 : 0, st), "bias finalize");
      bias_done = true;
    }
    if (param_grads && !bias_done) {
      // bias gradient = column sums of gz over the linear output rows
      ChannelMap cb;
      cb.L = L_;
      cb.ls = out_ls;
      if (b.lin == LK::ConvT) {
        cb.R = B * b.geo.GH * b.geo.GW;
        cb.Cp = b.geo.CG;
        cb.C = static_cast<int>(b.L.out);
      } else if (b.lin == LK::Conv) {
        cb.R = B * b.geo.SH * b.geo.SW;
        cb.Cp = b.geo.CS;
        cb.C = static_cast<int>(b.L.out);
      } else {
        cb.R = B;
        cb.Cp = b.geo.CS;
        cb.C = b.out_to_chw ? b.geo.CS : static_cast<int>(b.L.out);
      }
      check_cuda(launch_channel_reduce(cb, RED_SUM, gz, nullptr, nullptr, nullptr, 0, 0.f, partial_.p, st), "bias reduce");
      check_cuda(launch_bias_finalize(cb, partial_.p, dbias, P_, accumulate ? 1 : 0, st), "bias finalize");
    }
    // 2) weight gradient
    if (param_grads) {
      GemmArgs a{};
      a.kind = GEMM_WGRAD;
      a.g = geo_for(b, B);
      a.L = L_;
      if (b.lin == LK::ConvT) {
        a.small = t.act[i];
        a.small_ls = in_ls;
        a.big = gz;
        a.big_ls = out_ls;
      } else {
        a.small = gz;
        a.small_ls = out_ls;
        a.big = t.act[i];
        a.big_ls = in_ls;
      }
      a.out = grads.p + b.off_w;
      a.out_ls = P_;
      a.accumulate = accumulate ? 1 : 0;
      if (wg_act) {
        a.in_act = b.act;
        a.in_slope = b.slope;
        a.in_y = t.act[static_cast<size_t>(i) + 1];
        a.in_dbias = dbias;  // [L] x C bias gradient, label stride P_ (= out_ls)
      }
      check_cuda(launch_gemm(a, math_, st), "wgrad");
    }
    // 3) input gradient
    float* gx = nullptr;
    if (i > 0) gx = gscratch_[i % 2].p;
    else gx = gx_ext;
    fused = 0;
    if (gx) {
      GemmArgs a{};
      a.g = geo_for(b, B);
      a.L = L_;
      a.w = params.p + b.off_w;
      a.w_ls = P_;
      a.out = gx;
      a.out_ls = in_ls;
      a.act = ACT_NONE;
      a.c_valid = static_cast<int>(b.in.C);
      a.c_pad = static_cast<int>(b.in.Cp);
      if (b.lin == LK::ConvT) {
        a.kind = GEMM_FPROP;
        a.big = gz;
        a.big_ls = out_ls;
      } else {
        a.kind = GEMM_DGRAD;
        a.small = gz;
        a.small_ls = out_ls;
      }
      if (i > 0) {
        // the previous block's activation backward and BatchNorm / bias sums ride
        // on this GEMM's epilogue when its engine supports it
        const Block& pb = blocks_[static_cast<size_t>(i - 1)];
        int npack = 1;
        const int slots =
            (pb.has_bn || pb.act != ACT_NONE) && fuse_enabled(2) ? gemm_stat_slots(a, math_, &npack) : 0;
        if (slots > 0) {
          a.stat_mode = pb.has_bn ? STAT_BWD_BN : STAT_BWD_ACT;
          a.stat = stat_buf(static_cast<size_t>(L_) * slots * 4 * npack * b.in.Cp, st);
          fused_pack = npack;
          a.stat_y = t.act[static_cast<size_t>(i)];
          a.stat_z = pb.has_bn ? t.pre[static_cast<size_t>(i - 1)].p : nullptr;
          a.stat_mu = pb.has_bn ? t.mean[static_cast<size_t>(i - 1)].p : nullptr;
          a.stat_act = pb.act;
          a.stat_slope = pb.slope;
          fused = slots;
        }
      }
      check_cuda(launch_gemm(a, math_, st), "dgrad");
    }
    gy = gx;
  }
}

}  // namespace pg
