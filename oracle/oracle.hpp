// oracle/oracle.hpp — TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
// baseline). Nothing in the product (paper_2102_10485_b200/) includes, links or
// calls this file. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may use the shared library built from it.
//
// A CPU restatement of the reference `partgan` training path
// (/root/reference/proj, C++20 + Eigen, f64), templated on the arithmetic type
// so it runs both in f64 (the reference's precision, "truth") and in f32
// ("same-precision" parity for the fp32 GPU path).  Eigen is not available in
// this image, so every matrix product is a plain fixed-order loop (see gemm_*
// below); results are deterministic and independent of the thread count.
//
// Reference correspondence (file:line under /root/reference/proj):
//   splitmix64 / derive_seed / Rng ........ include/partgan/rng.hpp:9-46
//   Layer set, counts, shape algebra ...... include/partgan/layers.hpp:12-53, src/layers.cpp:33-104
//   build_network (init order) ............. src/network.cpp:308-343
//   dense fwd/bwd .......................... src/network.cpp:28-45
//   im2col + conv fwd/bwd .................. src/network.cpp:49-144
//   batch norm fwd/bwd ..................... src/network.cpp:151-271
//   upsample, dropout, activations ......... src/network.cpp:275-300, 374-393, 463-472
//   forward / infer / backward / grad_check  src/network.cpp:402-516
//   adam ................................... src/optim.cpp:9-34
//   losses + gradients ..................... src/gan.cpp:86-132
//   make_gan_pair / sample_latent .......... src/gan.cpp:27-84
//   train_step (step_impl) ................. src/gan.cpp:136-182
//   generate ............................... src/gan.cpp:190-201
//   partition_by_label / estimate_priors ... src/partition.cpp:40-74
//   run_worker / train_distributed ......... src/partition.cpp:78-180
//   mixture_sample ......................... src/partition.cpp:182-227
//   Dataset::gather ........................ src/data.cpp:13-23
// Additions required by BASELINE.json: ConvTranspose2d
// (restated from the conv_bwd / conv_fwd identities), the c1..c4 architecture
// builders, and the per-label cosine-field synthetic dataset.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <numeric>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace oracle {

using Shape = std::vector<long>;

inline long shape_numel(const Shape& s) {
  long n = 1;
  for (long d : s) n *= d;
  return n;
}

inline std::string shape_str(const Shape& s) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < s.size(); ++i) os << (i ? "x" : "") << s[i];
  os << "]";
  return os.str();
}

// ---------------------------------------------------------------------------
// seeds and random streams (rng.hpp:9-46).  The engine and both distributions
// are the libstdc++ ones, so every draw is bit-identical to the reference's;
// the normal_distribution object persists inside the stream (its cached second
// polar value carries over between calls exactly as in the reference).
// ---------------------------------------------------------------------------
inline uint64_t splitmix64(uint64_t& state) {
  state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = state;
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline uint64_t derive_seed(uint64_t base, uint64_t stream) {
  uint64_t st = base;
  uint64_t first = splitmix64(st);
  st = first ^ (stream * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
  return splitmix64(st);
}

class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double normal() { return nd_(eng_); }
  double uniform() { return ud_(eng_); }
  size_t index(size_t n) { return std::uniform_int_distribution<size_t>(0, n - 1)(eng_); }
  std::mt19937_64& engine() { return eng_; }

 private:
  std::mt19937_64 eng_;
  std::normal_distribution<double> nd_{0.0, 1.0};
  std::uniform_real_distribution<double> ud_{0.0, 1.0};
};

// ---------------------------------------------------------------------------
// tensors
// ---------------------------------------------------------------------------
template <class R>
struct Tensor {
  Shape shape;
  std::vector<R> data;
  Tensor() = default;
  explicit Tensor(Shape s) : shape(std::move(s)) {
    for (long d : shape)
      if (d <= 0) throw std::invalid_argument("tensor extents must be positive, got " + shape_str(shape));
    data.assign(static_cast<size_t>(shape_numel(shape)), R(0));
  }
  Tensor(Shape s, std::vector<R> d) : shape(std::move(s)), data(std::move(d)) {
    if (static_cast<long>(data.size()) != shape_numel(shape))
      throw std::invalid_argument("tensor shape " + shape_str(shape) + " does not match data length");
  }
  long size() const { return static_cast<long>(data.size()); }
  long dim(size_t i) const { return shape.at(i); }
  R& operator[](long i) { return data[static_cast<size_t>(i)]; }
  R operator[](long i) const { return data[static_cast<size_t>(i)]; }
  bool finite() const {
    for (R v : data)
      if (!std::isfinite(static_cast<double>(v))) return false;
    return true;
  }
};

// ---------------------------------------------------------------------------
// layers (layers.hpp:12-53 plus ConvTranspose2d)
// ---------------------------------------------------------------------------
enum class Kind { Dense, Conv2d, ConvT2d, BatchNorm, Upsample, Dropout, ReLU, LeakyReLU, Tanh, Sigmoid, Reshape };

struct Layer {
  Kind kind = Kind::ReLU;
  long in = 0, out = 0;     // dense dims or channels
  long k = 3, s = 1, p = 0; // conv geometry
  double eps = 1e-5, momentum = 0.1;
  long scale = 2;
  double rate = 0.5;
  double slope = 0.2;
  Shape target;

  static Layer dense(long i, long o) { Layer l; l.kind = Kind::Dense; l.in = i; l.out = o; return l; }
  static Layer conv(long i, long o, long k, long s, long p) {
    Layer l; l.kind = Kind::Conv2d; l.in = i; l.out = o; l.k = k; l.s = s; l.p = p; return l;
  }
  static Layer convT(long i, long o, long k, long s, long p) {
    Layer l; l.kind = Kind::ConvT2d; l.in = i; l.out = o; l.k = k; l.s = s; l.p = p; return l;
  }
  static Layer bn(long c, double eps = 1e-5, double mom = 0.1) {
    Layer l; l.kind = Kind::BatchNorm; l.in = l.out = c; l.eps = eps; l.momentum = mom; return l;
  }
  static Layer upsample(long f) { Layer l; l.kind = Kind::Upsample; l.scale = f; return l; }
  static Layer dropout(double r) { Layer l; l.kind = Kind::Dropout; l.rate = r; return l; }
  static Layer relu() { Layer l; l.kind = Kind::ReLU; return l; }
  static Layer lrelu(double sl = 0.2) { Layer l; l.kind = Kind::LeakyReLU; l.slope = sl; return l; }
  static Layer tanh_() { Layer l; l.kind = Kind::Tanh; return l; }
  static Layer sigmoid() { Layer l; l.kind = Kind::Sigmoid; return l; }
  static Layer reshape(Shape t) { Layer l; l.kind = Kind::Reshape; l.target = std::move(t); return l; }
};

inline const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Dense: return "dense";
    case Kind::Conv2d: return "conv2d";
    case Kind::ConvT2d: return "conv_transpose2d";
    case Kind::BatchNorm: return "batch_norm";
    case Kind::Upsample: return "upsample";
    case Kind::Dropout: return "dropout";
    case Kind::ReLU: return "relu";
    case Kind::LeakyReLU: return "leaky_relu";
    case Kind::Tanh: return "tanh";
    case Kind::Sigmoid: return "sigmoid";
    case Kind::Reshape: return "reshape";
  }
  return "?";
}

[[noreturn]] inline void layer_fail(size_t idx, const Layer& l, const std::string& what) {
  throw std::invalid_argument("layer " + std::to_string(idx) + " (" + kind_name(l.kind) + "): " + what);
}

inline void validate_layer(const Layer& l, size_t i) {
  switch (l.kind) {
    case Kind::Dense:
      if (l.in < 1 || l.out < 1) layer_fail(i, l, "dimensions must be positive");
      break;
    case Kind::Conv2d:
    case Kind::ConvT2d:
      if (l.in < 1 || l.out < 1) layer_fail(i, l, "channel counts must be positive");
      if (l.k < 1) layer_fail(i, l, "kernel must be >= 1");
      if (l.s < 1) layer_fail(i, l, "stride must be >= 1");
      if (l.p < 0) layer_fail(i, l, "padding must be >= 0");
      break;
    case Kind::BatchNorm:
      if (l.in < 1) layer_fail(i, l, "channels must be positive");
      if (!(l.eps > 0)) layer_fail(i, l, "epsilon must be > 0");
      if (l.momentum < 0 || l.momentum > 1) layer_fail(i, l, "momentum must be in [0, 1]");
      break;
    case Kind::Upsample:
      if (l.scale < 1) layer_fail(i, l, "scale_factor must be >= 1");
      break;
    case Kind::Dropout:
      if (l.rate < 0 || l.rate >= 1) layer_fail(i, l, "rate must be in [0, 1)");
      break;
    case Kind::LeakyReLU:
      if (!(l.slope > 0)) layer_fail(i, l, "slope must be > 0");
      break;
    case Kind::Reshape:
      if (l.target.empty()) layer_fail(i, l, "target_shape must be non-empty");
      for (long d : l.target)
        if (d < 1) layer_fail(i, l, "target_shape extents must be positive");
      break;
    default:
      break;
  }
}

inline long param_count(const Layer& l) {
  switch (l.kind) {
    case Kind::Dense: return l.in * l.out + l.out;
    case Kind::Conv2d:
    case Kind::ConvT2d: return l.in * l.out * l.k * l.k + l.out;
    case Kind::BatchNorm: return 2 * l.in;
    default: return 0;
  }
}

inline long buffer_count(const Layer& l) { return l.kind == Kind::BatchNorm ? 2 * l.in : 0; }

inline Shape out_shape(const Layer& l, const Shape& in, size_t i) {
  switch (l.kind) {
    case Kind::Dense:
      if (in.size() != 1 || in[0] != l.in)
        layer_fail(i, l, "expects input [" + std::to_string(l.in) + "], got " + shape_str(in));
      return {l.out};
    case Kind::Conv2d: {
      if (in.size() != 3 || in[0] != l.in)
        layer_fail(i, l, "expects input [" + std::to_string(l.in) + " x H x W], got " + shape_str(in));
      if (in[1] + 2 * l.p < l.k || in[2] + 2 * l.p < l.k)
        layer_fail(i, l, "kernel larger than padded input " + shape_str(in));
      return {l.out, (in[1] + 2 * l.p - l.k) / l.s + 1, (in[2] + 2 * l.p - l.k) / l.s + 1};
    }
    case Kind::ConvT2d: {
      if (in.size() != 3 || in[0] != l.in)
        layer_fail(i, l, "expects input [" + std::to_string(l.in) + " x H x W], got " + shape_str(in));
      long oh = (in[1] - 1) * l.s - 2 * l.p + l.k, ow = (in[2] - 1) * l.s - 2 * l.p + l.k;
      if (oh < 1 || ow < 1) layer_fail(i, l, "non-positive output extent for input " + shape_str(in));
      return {l.out, oh, ow};
    }
    case Kind::BatchNorm:
      if (in.empty() || in[0] != l.in)
        layer_fail(i, l, "expects " + std::to_string(l.in) + " channels, got input " + shape_str(in));
      return in;
    case Kind::Upsample:
      if (in.size() != 3) layer_fail(i, l, "expects input [C x H x W], got " + shape_str(in));
      return {in[0], in[1] * l.scale, in[2] * l.scale};
    case Kind::Reshape:
      if (shape_numel(in) != shape_numel(l.target))
        layer_fail(i, l, "cannot reshape " + shape_str(in) + " to " + shape_str(l.target));
      return l.target;
    default:
      return in;
  }
}

// ---------------------------------------------------------------------------
// fixed-order matrix kernels (stand-in for the reference's Eigen products)
// ---------------------------------------------------------------------------
// C[M][N] (+)= A[M][K] * B[K][N], all row-major, i-k-j order.
template <class R>
void gemm_nn(long M, long N, long K, const R* A, const R* B, R* C, bool acc) {
  if (!acc) std::fill(C, C + M * N, R(0));
  for (long i = 0; i < M; ++i) {
    R* c = C + i * N;
    const R* a = A + i * K;
    for (long k = 0; k < K; ++k) {
      const R av = a[k];
      const R* b = B + k * N;
      for (long j = 0; j < N; ++j) c[j] += av * b[j];
    }
  }
}
// C[M][N] (+)= A[M][K] * B[N][K]^T.  B is transposed once into a scratch
// [K][N] copy so the inner loop runs contiguously over N (i-k-j order).
template <class R>
void gemm_nt(long M, long N, long K, const R* A, const R* B, R* C, bool acc) {
  std::vector<R> bt(static_cast<size_t>(K * N));
  for (long j = 0; j < N; ++j)
    for (long k = 0; k < K; ++k) bt[static_cast<size_t>(k * N + j)] = B[j * K + k];
  gemm_nn(M, N, K, A, bt.data(), C, acc);
}
// C[M][N] (+)= A[K][M]^T * B[K][N].
template <class R>
void gemm_tn(long M, long N, long K, const R* A, const R* B, R* C, bool acc) {
  if (!acc) std::fill(C, C + M * N, R(0));
  for (long k = 0; k < K; ++k) {
    const R* a = A + k * M;
    const R* b = B + k * N;
    for (long i = 0; i < M; ++i) {
      const R av = a[i];
      R* c = C + i * N;
      for (long j = 0; j < N; ++j) c[j] += av * b[j];
    }
  }
}

// Convolution geometry seen from the "large" side: the large map (ch x H x W)
// is sampled by the small map (OH x OW) at row oh*s - p + ki.
struct Geo {
  long ch, h, w, oh, ow, k, s, p;
  long rows() const { return ch * k * k; }
  long cols() const { return oh * ow; }
};

// col[(c*k+ki)*k+kj][oh*OW+ow] = big[c][oh*s-p+ki][ow*s-p+kj] (0 outside).
template <class R>
void unfold(const Geo& g, const R* big, R* col) {
  for (long c = 0; c < g.ch; ++c)
    for (long ki = 0; ki < g.k; ++ki)
      for (long kj = 0; kj < g.k; ++kj) {
        R* dst = col + ((c * g.k + ki) * g.k + kj) * g.cols();
        for (long oi = 0; oi < g.oh; ++oi) {
          long y = oi * g.s - g.p + ki;
          for (long oj = 0; oj < g.ow; ++oj) {
            long x = oj * g.s - g.p + kj;
            dst[oi * g.ow + oj] = (y >= 0 && y < g.h && x >= 0 && x < g.w) ? big[(c * g.h + y) * g.w + x] : R(0);
          }
        }
      }
}

// Adjoint of unfold: big[...] += col[...].
template <class R>
void fold_add(const Geo& g, const R* col, R* big) {
  for (long c = 0; c < g.ch; ++c)
    for (long ki = 0; ki < g.k; ++ki)
      for (long kj = 0; kj < g.k; ++kj) {
        const R* src = col + ((c * g.k + ki) * g.k + kj) * g.cols();
        for (long oi = 0; oi < g.oh; ++oi) {
          long y = oi * g.s - g.p + ki;
          if (y < 0 || y >= g.h) continue;
          for (long oj = 0; oj < g.ow; ++oj) {
            long x = oj * g.s - g.p + kj;
            if (x < 0 || x >= g.w) continue;
            big[(c * g.h + y) * g.w + x] += src[oi * g.ow + oj];
          }
        }
      }
}

// ---------------------------------------------------------------------------
// network (network.hpp:20-107)
// ---------------------------------------------------------------------------
enum class Mode { train, eval };

template <class R>
struct Network {
  std::vector<Layer> layers;
  std::vector<Shape> shapes;  // layers.size() + 1 per-sample shapes
  std::vector<long> poff, boff;
  std::vector<R> params, buffers;
  const Shape& in_shape() const { return shapes.front(); }
  const Shape& out_shape_() const { return shapes.back(); }
  long n_params() const { return static_cast<long>(params.size()); }
  bool stochastic() const {
    for (const auto& l : layers)
      if (l.kind == Kind::Dropout) return true;
    return false;
  }
};

// build_network (network.cpp:308-343): weights ~ N(0,1)*init_std drawn in layer
// order from one stream; biases 0; BN gamma 1, beta 0, running mean 0, var 1.
template <class R>
Network<R> build_network(std::vector<Layer> specs, Shape input, uint64_t seed, double init_std = 0.02) {
  if (specs.empty()) throw std::invalid_argument("network spec list is empty");
  if (input.empty()) throw std::invalid_argument("network input shape is empty");
  for (long d : input)
    if (d < 1) throw std::invalid_argument("network input shape extents must be positive");
  Network<R> net;
  net.layers = std::move(specs);
  net.shapes.push_back(std::move(input));
  net.poff.push_back(0);
  net.boff.push_back(0);
  for (size_t i = 0; i < net.layers.size(); ++i) {
    validate_layer(net.layers[i], i);
    net.shapes.push_back(out_shape(net.layers[i], net.shapes.back(), i));
    net.poff.push_back(net.poff.back() + param_count(net.layers[i]));
    net.boff.push_back(net.boff.back() + buffer_count(net.layers[i]));
  }
  net.params.assign(static_cast<size_t>(net.poff.back()), R(0));
  net.buffers.assign(static_cast<size_t>(net.boff.back()), R(0));
  Rng rng(seed);
  for (size_t i = 0; i < net.layers.size(); ++i) {
    const Layer& l = net.layers[i];
    R* p = net.params.data() + net.poff[i];
    if (l.kind == Kind::Dense || l.kind == Kind::Conv2d || l.kind == Kind::ConvT2d) {
      long nw = param_count(l) - l.out;
      for (long j = 0; j < nw; ++j) p[j] = static_cast<R>(rng.normal() * init_std);
    } else if (l.kind == Kind::BatchNorm) {
      for (long c = 0; c < l.in; ++c) p[c] = R(1);
      R* b = net.buffers.data() + net.boff[i];
      for (long c = 0; c < l.in; ++c) b[l.in + c] = R(1);
    }
  }
  return net;
}

template <class R>
struct LayerTrace {
  Tensor<R> input, output, xhat, mask;
  std::vector<R> mean, inv_std;
  std::vector<uint8_t> amask;  // forced ReLU / LeakyReLU mask (MaskTape), empty = the sign test
};

// MaskTape — parity instrumentation, not reference behaviour.  When a tape is
// installed on the calling thread, every train-mode ReLU / LeakyReLU layer
// takes its mask (1 = positive branch) from the tape, in call order, instead
// of the sign test of network.cpp:384-391 / 463-470, and counts where the
// tape disagrees with that sign test ("forced flips").  Used to replay a
// device step's activation decisions: a pre-activation within rounding of
// zero may take either branch in any fp32 summation order, and the tape
// removes that discontinuity so gradients can be compared at 1e-4.
struct MaskTape {
  const uint8_t* m = nullptr;
  long n = 0, at = 0, flips = 0;
  std::vector<uint8_t>* record = nullptr;  // non-null: record the sign-test masks instead of forcing
};
inline MaskTape*& mask_tape() {
  thread_local MaskTape* t = nullptr;
  return t;
}

template <class R>
struct Trace {
  const Network<R>* net = nullptr;
  Mode mode = Mode::eval;
  long batch = 0;
  std::vector<LayerTrace<R>> layers;
  bool consumed = false;
};

template <class R>
struct Grads {
  std::vector<R> params;
  Tensor<R> input;
};

namespace detail {

inline Shape with_batch(long n, const Shape& s) {
  Shape r{n};
  r.insert(r.end(), s.begin(), s.end());
  return r;
}

template <class R>
Tensor<R> dense_fwd(const Layer& l, const R* p, const Tensor<R>& x) {
  long n = x.dim(0);
  Tensor<R> y(with_batch(n, {l.out}));
  gemm_nt(n, l.out, l.in, x.data.data(), p, y.data.data(), false);
  const R* b = p + l.out * l.in;
  for (long i = 0; i < n; ++i)
    for (long o = 0; o < l.out; ++o) y[i * l.out + o] += b[o];
  return y;
}

template <class R>
void dense_bwd(const Layer& l, const R* p, const Tensor<R>& x, const Tensor<R>& gy, R* gp, Tensor<R>& gx) {
  long n = x.dim(0);
  gemm_tn(l.out, l.in, n, gy.data.data(), x.data.data(), gp, false);  // gW = gy^T x
  R* gb = gp + l.out * l.in;
  for (long o = 0; o < l.out; ++o) {
    R s = 0;
    for (long i = 0; i < n; ++i) s += gy[i * l.out + o];
    gb[o] = s;
  }
  gemm_nn(n, l.in, l.out, gy.data.data(), p, gx.data.data(), false);  // gx = gy W
}

template <class R>
Tensor<R> conv_fwd(const Layer& l, const R* p, const Tensor<R>& x, const Shape& in, const Shape& out) {
  long n = x.dim(0);
  Geo g{l.in, in[1], in[2], out[1], out[2], l.k, l.s, l.p};
  Tensor<R> y(with_batch(n, out));
  std::vector<R> col(static_cast<size_t>(g.rows() * g.cols()));
  const R* b = p + l.out * g.rows();
  long xs = shape_numel(in), ys = shape_numel(out);
  for (long i = 0; i < n; ++i) {
    unfold(g, x.data.data() + i * xs, col.data());
    R* yo = y.data.data() + i * ys;
    gemm_nn(l.out, g.cols(), g.rows(), p, col.data(), yo, false);
    for (long o = 0; o < l.out; ++o)
      for (long j = 0; j < g.cols(); ++j) yo[o * g.cols() + j] += b[o];
  }
  return y;
}

template <class R>
void conv_bwd(const Layer& l, const R* p, const Tensor<R>& x, const Shape& in, const Shape& out, const Tensor<R>& gy,
              R* gp, Tensor<R>& gx) {
  long n = x.dim(0);
  Geo g{l.in, in[1], in[2], out[1], out[2], l.k, l.s, l.p};
  std::vector<R> col(static_cast<size_t>(g.rows() * g.cols())), gcol(col.size());
  R* gw = gp;
  R* gb = gp + l.out * g.rows();
  std::fill(gp, gp + param_count(l), R(0));
  std::fill(gx.data.begin(), gx.data.end(), R(0));
  long xs = shape_numel(in), ys = shape_numel(out);
  for (long i = 0; i < n; ++i) {
    unfold(g, x.data.data() + i * xs, col.data());
    const R* go = gy.data.data() + i * ys;
    gemm_nt(l.out, g.rows(), g.cols(), go, col.data(), gw, true);  // gW += go col^T
    for (long o = 0; o < l.out; ++o) {
      R s = 0;
      for (long j = 0; j < g.cols(); ++j) s += go[o * g.cols() + j];
      gb[o] += s;
    }
    gemm_tn(g.rows(), g.cols(), l.out, p, go, gcol.data(), false);  // gcol = W^T go
    fold_add(g, gcol.data(), gx.data.data() + i * xs);
  }
}

// ConvTranspose2d, weight [Cin][Cout*k*k] (PyTorch layout), bias [Cout].
// Forward = fold(W^T x) with conv geometry (large side = output); backward
// data = W unfold(gy); backward weight = x unfold(gy)^T.
template <class R>
Tensor<R> convT_fwd(const Layer& l, const R* p, const Tensor<R>& x, const Shape& in, const Shape& out) {
  long n = x.dim(0);
  Geo g{l.out, out[1], out[2], in[1], in[2], l.k, l.s, l.p};
  Tensor<R> y(with_batch(n, out));
  std::vector<R> col(static_cast<size_t>(g.rows() * g.cols()));
  const R* b = p + l.in * g.rows();
  long xs = shape_numel(in), ys = shape_numel(out), hw = out[1] * out[2];
  for (long i = 0; i < n; ++i) {
    gemm_tn(g.rows(), g.cols(), l.in, p, x.data.data() + i * xs, col.data(), false);
    R* yo = y.data.data() + i * ys;
    fold_add(g, col.data(), yo);
    for (long o = 0; o < l.out; ++o)
      for (long j = 0; j < hw; ++j) yo[o * hw + j] += b[o];
  }
  return y;
}

template <class R>
void convT_bwd(const Layer& l, const R* p, const Tensor<R>& x, const Shape& in, const Shape& out, const Tensor<R>& gy,
               R* gp, Tensor<R>& gx) {
  long n = x.dim(0);
  Geo g{l.out, out[1], out[2], in[1], in[2], l.k, l.s, l.p};
  std::vector<R> col(static_cast<size_t>(g.rows() * g.cols()));
  R* gw = gp;
  R* gb = gp + l.in * g.rows();
  std::fill(gp, gp + param_count(l), R(0));
  long xs = shape_numel(in), ys = shape_numel(out), hw = out[1] * out[2];
  for (long i = 0; i < n; ++i) {
    const R* go = gy.data.data() + i * ys;
    unfold(g, go, col.data());
    const R* xi = x.data.data() + i * xs;
    gemm_nt(l.in, g.rows(), g.cols(), xi, col.data(), gw, true);             // gW += x col^T
    gemm_nn(l.in, g.cols(), g.rows(), p, col.data(), gx.data.data() + i * xs, false);  // gx = W col
    for (long o = 0; o < l.out; ++o) {
      R s = 0;
      for (long j = 0; j < hw; ++j) s += go[o * hw + j];
      gb[o] += s;
    }
  }
}

// batch norm (network.cpp:151-271): stats per channel over batch x spatial;
// biased variance normalizes, the running variance stores the unbiased one.
template <class R>
Tensor<R> bn_fwd(const Layer& l, const R* p, const R* buf_read, R* buf_write, const Tensor<R>& x, Mode mode,
                 LayerTrace<R>* tr) {
  long n = x.dim(0), C = x.dim(1), S = x.size() / (n * C);
  const R* gamma = p;
  const R* beta = p + C;
  std::vector<R> mean(static_cast<size_t>(C)), var(static_cast<size_t>(C));
  if (mode == Mode::train) {
    R m = static_cast<R>(n * S);
    for (long c = 0; c < C; ++c) {
      R sum = 0;
      for (long i = 0; i < n; ++i)
        for (long t = 0; t < S; ++t) sum += x[(i * C + c) * S + t];
      R mu = sum / m;
      R sq = 0;
      for (long i = 0; i < n; ++i)
        for (long t = 0; t < S; ++t) {
          R d = x[(i * C + c) * S + t] - mu;
          sq += d * d;
        }
      mean[c] = mu;
      var[c] = sq / m;
    }
    if (buf_write) {
      R unbias = m > 1 ? m / (m - 1) : R(1);
      R mom = static_cast<R>(l.momentum);
      for (long c = 0; c < C; ++c) {
        buf_write[c] = (1 - mom) * buf_write[c] + mom * mean[c];
        buf_write[C + c] = (1 - mom) * buf_write[C + c] + mom * var[c] * unbias;
      }
    }
  } else {
    for (long c = 0; c < C; ++c) {
      mean[c] = buf_read[c];
      var[c] = buf_read[C + c];
    }
  }
  std::vector<R> istd(static_cast<size_t>(C));
  for (long c = 0; c < C; ++c) istd[c] = R(1) / std::sqrt(var[c] + static_cast<R>(l.eps));
  Tensor<R> y(x.shape), xh(x.shape);
  for (long i = 0; i < n; ++i)
    for (long c = 0; c < C; ++c)
      for (long t = 0; t < S; ++t) {
        long o = (i * C + c) * S + t;
        R h = (x[o] - mean[c]) * istd[c];
        xh[o] = h;
        y[o] = gamma[c] * h + beta[c];
      }
  if (tr) {
    tr->mean = std::move(mean);
    tr->inv_std = std::move(istd);
    tr->xhat = std::move(xh);
  }
  return y;
}

template <class R>
void bn_bwd(const Layer&, const R* p, const LayerTrace<R>& tr, const Tensor<R>& x, const Tensor<R>& gy, Mode mode,
            R* gp, Tensor<R>& gx) {
  long n = x.dim(0), C = x.dim(1), S = x.size() / (n * C);
  const R* gamma = p;
  R* dgamma = gp;
  R* dbeta = gp + C;
  for (long c = 0; c < C; ++c) dgamma[c] = dbeta[c] = 0;
  for (long i = 0; i < n; ++i)
    for (long c = 0; c < C; ++c)
      for (long t = 0; t < S; ++t) {
        long o = (i * C + c) * S + t;
        dgamma[c] += gy[o] * tr.xhat[o];
        dbeta[c] += gy[o];
      }
  if (mode == Mode::eval) {
    for (long i = 0; i < n; ++i)
      for (long c = 0; c < C; ++c)
        for (long t = 0; t < S; ++t) {
          long o = (i * C + c) * S + t;
          gx[o] = gy[o] * gamma[c] * tr.inv_std[c];
        }
    return;
  }
  R m = static_cast<R>(n * S);
  for (long c = 0; c < C; ++c) {
    R is = tr.inv_std[c], mu = tr.mean[c];
    R dvar = 0, dmean = 0, csum = 0;
    for (long i = 0; i < n; ++i)
      for (long t = 0; t < S; ++t) {
        long o = (i * C + c) * S + t;
        R dxh = gy[o] * gamma[c];
        R cen = x[o] - mu;
        dvar += dxh * cen;
        dmean -= dxh;
        csum += cen;
      }
    dvar *= R(-0.5) * is * is * is;
    dmean = dmean * is + dvar * (R(-2) / m) * csum;
    for (long i = 0; i < n; ++i)
      for (long t = 0; t < S; ++t) {
        long o = (i * C + c) * S + t;
        gx[o] = gy[o] * gamma[c] * is + dvar * R(2) * (x[o] - mu) / m + dmean / m;
      }
  }
}

template <class R>
Tensor<R> upsample_fwd(long f, const Tensor<R>& x, const Shape& in) {
  long n = x.dim(0), C = in[0], H = in[1], W = in[2];
  Tensor<R> y(with_batch(n, {C, H * f, W * f}));
  for (long i = 0; i < n * C; ++i)
    for (long a = 0; a < H * f; ++a)
      for (long b = 0; b < W * f; ++b) y[(i * H * f + a) * W * f + b] = x[(i * H + a / f) * W + b / f];
  return y;
}

template <class R>
void upsample_bwd(long f, const Shape& in, const Tensor<R>& gy, Tensor<R>& gx) {
  long n = gy.dim(0), C = in[0], H = in[1], W = in[2];
  std::fill(gx.data.begin(), gx.data.end(), R(0));
  for (long i = 0; i < n * C; ++i)
    for (long a = 0; a < H * f; ++a)
      for (long b = 0; b < W * f; ++b) gx[(i * H + a / f) * W + b / f] += gy[(i * H * f + a) * W * f + b];
}

template <class R>
void check_batch(const Network<R>& net, const Tensor<R>& x) {
  const Shape& in = net.in_shape();
  bool ok = x.shape.size() == in.size() + 1 && x.dim(0) >= 1;
  for (size_t i = 0; ok && i < in.size(); ++i) ok = x.dim(i + 1) == in[i];
  if (!ok)
    throw std::invalid_argument("batch shape " + shape_str(x.shape) + " does not match network input " +
                                shape_str(in));
}

// ReLU (leaky = false) / LeakyReLU forward with the mask taken from the tape
template <class R>
Tensor<R> forced_act(MaskTape& tp, const Tensor<R>& x, bool leaky, R sl, LayerTrace<R>& tr) {
  Tensor<R> y(x.shape);
  if (tp.record) {
    for (long j = 0; j < y.size(); ++j) {
      const bool on = leaky ? x[j] >= R(0) : x[j] > R(0);
      tp.record->push_back(on);
      y[j] = on ? x[j] : (leaky ? x[j] * sl : R(0));
    }
    return y;
  }
  if (tp.at + x.size() > tp.n) throw std::invalid_argument("mask tape exhausted");
  tr.amask.assign(tp.m + tp.at, tp.m + tp.at + x.size());
  for (long j = 0; j < y.size(); ++j) {
    const bool own = leaky ? x[j] >= R(0) : x[j] > R(0);
    const bool on = tr.amask[static_cast<size_t>(j)] != 0;
    tp.flips += own != on;
    y[j] = on ? x[j] : (leaky ? x[j] * sl : R(0));
  }
  tp.at += x.size();
  return y;
}

template <class R>
Tensor<R> run_layer(const Network<R>& net, size_t i, const Tensor<R>& x, Mode mode, Rng* rng, LayerTrace<R>* tr,
                    std::vector<R>* bufs) {
  const Layer& l = net.layers[i];
  const R* p = net.params.data() + net.poff[i];
  const Shape& in = net.shapes[i];
  const Shape& out = net.shapes[i + 1];
  switch (l.kind) {
    case Kind::Dense: return dense_fwd(l, p, x);
    case Kind::Conv2d: return conv_fwd(l, p, x, in, out);
    case Kind::ConvT2d: return convT_fwd(l, p, x, in, out);
    case Kind::BatchNorm: {
      const R* br = net.buffers.data() + net.boff[i];
      R* bw = (mode == Mode::train && bufs) ? bufs->data() + net.boff[i] : nullptr;
      return bn_fwd(l, p, br, bw, x, mode, tr);
    }
    case Kind::Upsample: return upsample_fwd(l.scale, x, in);
    case Kind::Dropout: {
      if (mode != Mode::train) return x;
      Tensor<R> mask(x.shape);
      R keep = static_cast<R>(1.0 / (1.0 - l.rate));
      for (long j = 0; j < mask.size(); ++j) mask[j] = (rng->uniform() >= l.rate) ? keep : R(0);
      Tensor<R> y(x.shape);
      for (long j = 0; j < y.size(); ++j) y[j] = x[j] * mask[j];
      if (tr) tr->mask = std::move(mask);
      return y;
    }
    case Kind::ReLU: {
      Tensor<R> y(x.shape);
      if (MaskTape* tp = mode == Mode::train && tr ? mask_tape() : nullptr)
        return forced_act(*tp, x, false, R(0), *tr);
      for (long j = 0; j < y.size(); ++j) y[j] = x[j] > R(0) ? x[j] : R(0);
      return y;
    }
    case Kind::LeakyReLU: {
      Tensor<R> y(x.shape);
      R sl = static_cast<R>(l.slope);
      if (MaskTape* tp = mode == Mode::train && tr ? mask_tape() : nullptr) return forced_act(*tp, x, true, sl, *tr);
      for (long j = 0; j < y.size(); ++j) y[j] = x[j] >= R(0) ? x[j] : x[j] * sl;
      return y;
    }
    case Kind::Tanh: {
      Tensor<R> y(x.shape);
      for (long j = 0; j < y.size(); ++j) y[j] = std::tanh(x[j]);
      return y;
    }
    case Kind::Sigmoid: {
      Tensor<R> y(x.shape);
      for (long j = 0; j < y.size(); ++j) y[j] = R(1) / (std::exp(-x[j]) + R(1));
      return y;
    }
    case Kind::Reshape: return Tensor<R>(with_batch(x.dim(0), out), x.data);
  }
  throw std::logic_error("unhandled layer");
}

}  // namespace detail

// forward (network.cpp:402-419): train mode updates BN running stats and draws
// dropout masks from rng; the trace keeps every layer input plus the extras.
template <class R>
std::pair<Tensor<R>, Trace<R>> forward(Network<R>& net, const Tensor<R>& batch, Mode mode, Rng& rng) {
  detail::check_batch(net, batch);
  Trace<R> tr;
  tr.net = &net;
  tr.mode = mode;
  tr.batch = batch.dim(0);
  tr.layers.resize(net.layers.size());
  Tensor<R> x = batch;
  for (size_t i = 0; i < net.layers.size(); ++i) {
    Tensor<R> y = detail::run_layer(net, i, x, mode, &rng, &tr.layers[i], &net.buffers);
    Kind k = net.layers[i].kind;
    if (k == Kind::Tanh || k == Kind::Sigmoid) tr.layers[i].output = y;
    tr.layers[i].input = std::move(x);
    x = std::move(y);
  }
  return {std::move(x), std::move(tr)};
}

template <class R>
Tensor<R> infer(const Network<R>& net, const Tensor<R>& batch) {
  detail::check_batch(net, batch);
  Tensor<R> x = batch;
  for (size_t i = 0; i < net.layers.size(); ++i) x = detail::run_layer<R>(net, i, x, Mode::eval, nullptr, nullptr, nullptr);
  return x;
}

// backward (network.cpp:429-480): exact reverse mode, returns fresh gradients.
template <class R>
Grads<R> backward(const Network<R>& net, Trace<R>& tr, const Tensor<R>& gout) {
  if (tr.net != &net || tr.layers.size() != net.layers.size())
    throw std::invalid_argument("trace does not belong to this network");
  if (tr.consumed) throw std::invalid_argument("trace already consumed by a previous backward call");
  tr.consumed = true;
  Shape want = detail::with_batch(tr.batch, net.out_shape_());
  if (gout.shape != want)
    throw std::invalid_argument("output gradient shape " + shape_str(gout.shape) + " does not match network output " +
                                shape_str(want));
  Grads<R> g;
  g.params.assign(net.params.size(), R(0));
  Tensor<R> gy = gout;
  for (size_t idx = net.layers.size(); idx-- > 0;) {
    const Layer& l = net.layers[idx];
    const LayerTrace<R>& t = tr.layers[idx];
    const R* p = net.params.data() + net.poff[idx];
    R* gp = g.params.data() + net.poff[idx];
    Tensor<R> gx(t.input.shape);
    switch (l.kind) {
      case Kind::Dense: detail::dense_bwd(l, p, t.input, gy, gp, gx); break;
      case Kind::Conv2d: detail::conv_bwd(l, p, t.input, net.shapes[idx], net.shapes[idx + 1], gy, gp, gx); break;
      case Kind::ConvT2d: detail::convT_bwd(l, p, t.input, net.shapes[idx], net.shapes[idx + 1], gy, gp, gx); break;
      case Kind::BatchNorm: detail::bn_bwd(l, p, t, t.input, gy, tr.mode, gp, gx); break;
      case Kind::Upsample: detail::upsample_bwd(l.scale, net.shapes[idx], gy, gx); break;
      case Kind::Dropout:
        for (long j = 0; j < gx.size(); ++j) gx[j] = tr.mode == Mode::train ? gy[j] * t.mask[j] : gy[j];
        break;
      case Kind::ReLU:
        for (long j = 0; j < gx.size(); ++j)
          gx[j] = (t.amask.empty() ? t.input[j] > R(0) : t.amask[static_cast<size_t>(j)] != 0) ? gy[j] : R(0);
        break;
      case Kind::LeakyReLU: {
        R sl = static_cast<R>(l.slope);
        for (long j = 0; j < gx.size(); ++j)
          gx[j] = (t.amask.empty() ? t.input[j] >= R(0) : t.amask[static_cast<size_t>(j)] != 0) ? gy[j] : gy[j] * sl;
        break;
      }
      case Kind::Tanh:
        for (long j = 0; j < gx.size(); ++j) gx[j] = gy[j] * (R(1) - t.output[j] * t.output[j]);
        break;
      case Kind::Sigmoid:
        for (long j = 0; j < gx.size(); ++j) gx[j] = gy[j] * t.output[j] * (R(1) - t.output[j]);
        break;
      case Kind::Reshape: gx.data = gy.data; break;
    }
    gy = std::move(gx);
  }
  g.input = std::move(gy);
  return g;
}

template <class R>
struct LossFn {
  std::function<double(const Tensor<R>&)> value;
  std::function<Tensor<R>(const Tensor<R>&)> grad;
};

// grad_check (network.cpp:482-516): central differences on sampled coordinates.
template <class R>
double grad_check(const Network<R>& net, const Tensor<R>& input, const LossFn<R>& loss, int n_coords, double step,
                  Mode mode, Rng& rng) {
  if (net.n_params() == 0) return 0.0;
  if (mode == Mode::train && net.stochastic())
    throw std::invalid_argument(
        "grad_check requires a deterministic forward; run networks containing dropout in eval mode");
  Network<R> work = net;
  Rng unused(0);
  auto fw = forward(work, input, mode, unused);
  Grads<R> g = backward(work, fw.second, loss.grad(fw.first));
  std::vector<long> coords(static_cast<size_t>(net.n_params()));
  std::iota(coords.begin(), coords.end(), 0L);
  if (n_coords < static_cast<int>(coords.size())) {
    std::shuffle(coords.begin(), coords.end(), rng.engine());
    coords.resize(static_cast<size_t>(n_coords));
  }
  double worst = 0;
  for (long c : coords) {
    R saved = work.params[c];
    work.params[c] = static_cast<R>(saved + step);
    double fp = loss.value(forward(work, input, mode, unused).first);
    work.params[c] = static_cast<R>(saved - step);
    double fm = loss.value(forward(work, input, mode, unused).first);
    work.params[c] = saved;
    double num = (fp - fm) / (2 * step);
    double ana = static_cast<double>(g.params[c]);
    double rel = std::abs(ana - num) / std::max({std::abs(ana), std::abs(num), 1e-8});
    worst = std::max(worst, rel);
  }
  return worst;
}

// ---------------------------------------------------------------------------
// Adam (optim.hpp:7-29, optim.cpp:9-34)
// ---------------------------------------------------------------------------
struct AdamConfig {
  double lr = 2e-4, beta1 = 0.5, beta2 = 0.999, eps = 1e-8;
};

template <class R>
struct AdamState {
  std::vector<R> m, v;
  long t = 0;
  double lr = 2e-4, beta1 = 0.5, beta2 = 0.999, eps = 1e-8;
  static AdamState create(long n, const AdamConfig& c) {
    AdamState s;
    s.m.assign(static_cast<size_t>(n), R(0));
    s.v.assign(static_cast<size_t>(n), R(0));
    s.lr = c.lr;
    s.beta1 = c.beta1;
    s.beta2 = c.beta2;
    s.eps = c.eps;
    return s;
  }
};

// Same update as the reference; in f32 the moments and step are evaluated in
// f32 with the bias corrections formed in f64 (the GPU kernel does the same).
template <class R>
void adam_step(AdamState<R>& st, std::vector<R>& params, const std::vector<R>& grads) {
  if (params.size() != st.m.size() || grads.size() != st.m.size())
    throw std::invalid_argument("adam_step: length mismatch (params " + std::to_string(params.size()) + ", grads " +
                                std::to_string(grads.size()) + ", state " + std::to_string(st.m.size()) + ")");
  for (R g : grads)
    if (!std::isfinite(static_cast<double>(g))) throw std::invalid_argument("adam_step: non-finite gradient rejected");
  st.t += 1;
  const R b1 = static_cast<R>(st.beta1), b2 = static_cast<R>(st.beta2);
  const R c1 = static_cast<R>(1.0 - std::pow(st.beta1, static_cast<double>(st.t)));
  const R c2 = static_cast<R>(1.0 - std::pow(st.beta2, static_cast<double>(st.t)));
  const R lr = static_cast<R>(st.lr), eps = static_cast<R>(st.eps);
  for (size_t i = 0; i < params.size(); ++i) {
    R g = grads[i];
    st.m[i] = b1 * st.m[i] + (R(1) - b1) * g;
    st.v[i] = b2 * st.v[i] + (R(1) - b2) * g * g;
    params[i] -= lr * (st.m[i] / c1) / (std::sqrt(st.v[i] / c2) + eps);
  }
}

// ---------------------------------------------------------------------------
// GAN pair, losses, step (gan.hpp, gan.cpp)
// ---------------------------------------------------------------------------
struct StepReport {
  double j_d = 0, j_g = 0, d_real_mean = 0, d_fake_mean = 0;
};

template <class R>
struct GanPair {
  Network<R> gen, disc;
  long d_z = 100, d_y = 0;
  AdamState<R> opt_g, opt_d;
  double clamp = 1e-7;
  long steps = 0;
  // gradients of the last step (kept for parity checks)
  std::vector<R> last_grad_g, last_grad_d;
};

inline void check_clamp(double c) {
  if (!(c > 0.0 && c < 0.5))
    throw std::invalid_argument("probability clamp must lie in (0, 0.5), got " + std::to_string(c));
}

template <class R>
GanPair<R> make_gan_pair(std::vector<Layer> g_arch, std::vector<Layer> d_arch, Shape image, long d_z, long d_y,
                         const AdamConfig& adam, uint64_t seed, double init_std = 0.02, double clamp = 1e-7) {
  check_clamp(clamp);
  if (d_z < 1) throw std::invalid_argument("latent dimension must be positive");
  if (d_y < 0) throw std::invalid_argument("label embedding dimension must be non-negative");
  GanPair<R> pr;
  pr.d_z = d_z;
  pr.d_y = d_y;
  pr.clamp = clamp;
  pr.gen = build_network<R>(std::move(g_arch), {d_z + d_y}, derive_seed(seed, 1), init_std);
  pr.disc = build_network<R>(std::move(d_arch), image, derive_seed(seed, 2), init_std);
  if (pr.gen.out_shape_() != image)
    throw std::invalid_argument("generator emits " + shape_str(pr.gen.out_shape_()) + " but images are " +
                                shape_str(image));
  if (shape_numel(pr.disc.out_shape_()) != 1)
    throw std::invalid_argument("discriminator must emit a scalar, got " + shape_str(pr.disc.out_shape_()));
  pr.opt_g = AdamState<R>::create(pr.gen.n_params(), adam);
  pr.opt_d = AdamState<R>::create(pr.disc.n_params(), adam);
  return pr;
}

template <class R>
Tensor<R> sample_latent(long d_z, long d_y, std::optional<int> cls, long n, Rng& rng) {
  if (n < 1) throw std::invalid_argument("sample_latent: batch size must be positive");
  int k = 0;
  if (d_y > 0) {
    if (!cls) throw std::invalid_argument("sample_latent: class id required when conditioning is enabled");
    k = *cls;
    if (k < 0 || k >= d_y)
      throw std::out_of_range("class id " + std::to_string(k) + " out of range [0, " + std::to_string(d_y) + ")");
  }
  long w = d_z + d_y;
  Tensor<R> z({n, w});
  for (long i = 0; i < n; ++i) {
    for (long j = 0; j < d_z; ++j) z[i * w + j] = static_cast<R>(rng.normal());
    if (d_y > 0) z[i * w + d_z + k] = R(1);
  }
  return z;
}

inline double clampd(double p, double c) { return std::min(std::max(p, c), 1.0 - c); }
inline bool inside(double p, double c) { return p > c && p < 1.0 - c; }

template <class R>
double discriminator_loss(const Tensor<R>& pr, const Tensor<R>& pf, double c) {
  check_clamp(c);
  if (pr.size() == 0 || pf.size() == 0) throw std::invalid_argument("discriminator_loss: empty batch");
  double sr = 0, sf = 0;
  for (long i = 0; i < pr.size(); ++i) sr += std::log(clampd(pr[i], c));
  for (long i = 0; i < pf.size(); ++i) sf += std::log(1.0 - clampd(pf[i], c));
  return -0.5 * sr / static_cast<double>(pr.size()) - 0.5 * sf / static_cast<double>(pf.size());
}

template <class R>
double generator_loss(const Tensor<R>& pf, double c) {
  check_clamp(c);
  if (pf.size() == 0) throw std::invalid_argument("generator_loss: empty batch");
  double s = 0;
  for (long i = 0; i < pf.size(); ++i) s += std::log(clampd(pf[i], c));
  return 0.5 * s / static_cast<double>(pf.size());
}

// which: 0 = d J_D / d p_real, 1 = d J_D / d p_fake, 2 = d(-J_G)/d p_fake.
template <class R>
Tensor<R> loss_grad(const Tensor<R>& p, double c, int which) {
  check_clamp(c);
  if (p.size() == 0) throw std::invalid_argument("loss gradient: empty batch");
  Tensor<R> g(p.shape);
  double n = static_cast<double>(p.size());
  for (long i = 0; i < p.size(); ++i) {
    double v = p[i];
    double r = 0;
    if (inside(v, c)) r = which == 1 ? 0.5 / (n * (1.0 - v)) : -0.5 / (n * v);
    g[i] = static_cast<R>(r);
  }
  return g;
}

// train_step (gan.cpp:136-182).  `latent` yields z1 then z2; the default
// (train_step) samples them from rng, so the stream order is z1, [dropout
// masks of the D-step forwards], z2, [masks] exactly as in the reference.
template <class R>
StepReport step_core(GanPair<R>& pr, const Tensor<R>& real01, const std::function<Tensor<R>()>& latent, Rng& rng) {
  if (real01.size() == 0) throw std::invalid_argument("train_step: empty batch");
  double c = pr.clamp;
  Tensor<R> real(real01.shape);
  for (long i = 0; i < real.size(); ++i) real[i] = real01[i] * R(2) - R(1);

  Tensor<R> z1 = latent();
  Tensor<R> fake = forward(pr.gen, z1, Mode::train, rng).first;
  auto fr = forward(pr.disc, real, Mode::train, rng);
  auto ff = forward(pr.disc, fake, Mode::train, rng);
  double j_d = discriminator_loss(fr.first, ff.first, c);
  Grads<R> gr = backward(pr.disc, fr.second, loss_grad(fr.first, c, 0));
  Grads<R> gf = backward(pr.disc, ff.second, loss_grad(ff.first, c, 1));
  std::vector<R> dg(gr.params.size());
  for (size_t i = 0; i < dg.size(); ++i) dg[i] = gr.params[i] + gf.params[i];
  adam_step(pr.opt_d, pr.disc.params, dg);

  Tensor<R> z2 = latent();
  auto fg = forward(pr.gen, z2, Mode::train, rng);
  auto fd = forward(pr.disc, fg.first, Mode::train, rng);
  double j_g = generator_loss(fd.first, c);
  Grads<R> gd = backward(pr.disc, fd.second, loss_grad(fd.first, c, 2));
  Grads<R> gg = backward(pr.gen, fg.second, gd.input);
  adam_step(pr.opt_g, pr.gen.params, gg.params);

  pr.last_grad_d = std::move(dg);
  pr.last_grad_g = std::move(gg.params);
  pr.steps += 1;
  StepReport rep;
  rep.j_d = j_d;
  rep.j_g = j_g;
  double sr = 0, sf = 0;
  for (long i = 0; i < fr.first.size(); ++i) sr += fr.first[i];
  for (long i = 0; i < ff.first.size(); ++i) sf += ff.first[i];
  rep.d_real_mean = sr / static_cast<double>(fr.first.size());
  rep.d_fake_mean = sf / static_cast<double>(ff.first.size());
  return rep;
}

template <class R>
StepReport train_step(GanPair<R>& pr, const Tensor<R>& real01, std::optional<int> cls, Rng& rng) {
  if (real01.size() == 0) throw std::invalid_argument("train_step: empty batch");
  long n = real01.dim(0);
  return step_core<R>(pr, real01, [&]() { return sample_latent<R>(pr.d_z, pr.d_y, cls, n, rng); }, rng);
}

// generate (gan.cpp:197-201): eval-mode generator, tanh range -> [0,1].
template <class R>
Tensor<R> generate(const GanPair<R>& pr, std::optional<int> cls, long n, Rng& rng) {
  Tensor<R> z = sample_latent<R>(pr.d_z, pr.d_y, cls, n, rng);
  Tensor<R> out = infer(pr.gen, z);
  for (auto& v : out.data) v = (v + R(1)) * R(0.5);
  return out;
}

// ---------------------------------------------------------------------------
// data (data.hpp, data.cpp) + the cosine-field synthetic kind
// ---------------------------------------------------------------------------
struct Dataset {
  std::vector<double> images;  // [m][C][H][W] in [0,1]
  long m = 0, C = 0, H = 0, W = 0;
  std::vector<int> labels;
  int k = 0;
  Shape sample_shape() const { return {C, H, W}; }
  template <class R>
  Tensor<R> gather(const std::vector<long>& idx) const {
    if (idx.empty()) throw std::invalid_argument("gather: empty index list");
    long s = C * H * W;
    Tensor<R> out({static_cast<long>(idx.size()), C, H, W});
    for (size_t i = 0; i < idx.size(); ++i) {
      long j = idx[i];
      if (j < 0 || j >= m) throw std::out_of_range("gather: index " + std::to_string(j));
      for (long t = 0; t < s; ++t) out[static_cast<long>(i) * s + t] = static_cast<R>(images[j * s + t]);
    }
    return out;
  }
};

// Cosine-field dataset (this build's definition, shared bit-for-bit with the
// product's generator).  Label l draws from
// Rng(derive_seed(seed, l)):
//   per channel c, 8 terms: u = index(7)-3, v = index(7)-3, a = normal(), phi = 2*pi*uniform();
//   F(y,x) = sum a*cos(2*pi*(u*x/W + v*y/H) + phi), scaled by 1/max|F| into [-1,1];
//   then per sample, per pixel in [C][H][W] order: clamp(F + 0.1*normal(), -1, 1) -> (v+1)/2.
// Rows are label-blocked: sample j of label l is row l*per_label + j.
struct CosineSpec {
  int k = 10;
  long per_label = 64;
  long C = 1, H = 28, W = 28;
  uint64_t seed = 1;
  int first_label = 0;  // generate labels [first_label, first_label + k)
};

inline void cosine_label(const CosineSpec& sp, int label, double* out /* per_label*C*H*W */) {
  Rng rng(derive_seed(sp.seed, static_cast<uint64_t>(label)));
  const long HW = sp.H * sp.W;
  std::vector<double> field(static_cast<size_t>(sp.C * HW));
  const double two_pi = 6.283185307179586476925286766559;
  for (long c = 0; c < sp.C; ++c) {
    double u[8], v[8], a[8], ph[8];
    for (int t = 0; t < 8; ++t) {
      u[t] = static_cast<double>(static_cast<long>(rng.index(7)) - 3);
      v[t] = static_cast<double>(static_cast<long>(rng.index(7)) - 3);
      a[t] = rng.normal();
      ph[t] = two_pi * rng.uniform();
    }
    double mx = 0;
    for (long y = 0; y < sp.H; ++y)
      for (long x = 0; x < sp.W; ++x) {
        double f = 0;
        for (int t = 0; t < 8; ++t)
          f += a[t] * std::cos(two_pi * (u[t] * static_cast<double>(x) / static_cast<double>(sp.W) +
                                         v[t] * static_cast<double>(y) / static_cast<double>(sp.H)) + ph[t]);
        field[static_cast<size_t>(c * HW + y * sp.W + x)] = f;
        mx = std::max(mx, std::abs(f));
      }
    if (mx > 0)
      for (long t = 0; t < HW; ++t) field[static_cast<size_t>(c * HW + t)] /= mx;
  }
  const long S = sp.C * HW;
  for (long j = 0; j < sp.per_label; ++j)
    for (long t = 0; t < S; ++t) {
      double val = field[static_cast<size_t>(t)] + 0.1 * rng.normal();
      val = std::min(1.0, std::max(-1.0, val));
      out[j * S + t] = (val + 1.0) * 0.5;
    }
}

inline Dataset make_cosine_dataset(const CosineSpec& sp) {
  if (sp.k < 1 || sp.per_label < 1) throw std::invalid_argument("cosine dataset needs k >= 1 and per_label >= 1");
  Dataset ds;
  ds.k = sp.first_label + sp.k;
  ds.C = sp.C;
  ds.H = sp.H;
  ds.W = sp.W;
  ds.m = sp.k * sp.per_label;
  const long S = sp.C * sp.H * sp.W;
  ds.images.assign(static_cast<size_t>(ds.m * S), 0.0);
  ds.labels.resize(static_cast<size_t>(ds.m));
  for (int l = 0; l < sp.k; ++l) {
    cosine_label(sp, sp.first_label + l, ds.images.data() + static_cast<long>(l) * sp.per_label * S);
    for (long j = 0; j < sp.per_label; ++j) ds.labels[static_cast<size_t>(l * sp.per_label + j)] = sp.first_label + l;
  }
  return ds;
}

// ---------------------------------------------------------------------------
// architectures for BASELINE.json c1..c4
// ---------------------------------------------------------------------------
struct Arch {
  std::vector<Layer> gen, disc;
  Shape image;
  long d_z = 100;
};

// cfg 1: 28x28x1; cfg 2/3: 32x32x3; cfg 4: 64x64x3.
inline Arch baseline_arch(int cfg, long d_z = 100) {
  Arch a;
  a.d_z = d_z;
  auto tail = [](std::vector<Layer>& g, std::vector<long> ch, long out_c) {
    for (size_t i = 0; i + 1 < ch.size(); ++i) {
      g.push_back(Layer::convT(ch[i], ch[i + 1], 4, 2, 1));
      g.push_back(Layer::bn(ch[i + 1]));
      g.push_back(Layer::relu());
    }
    g.push_back(Layer::convT(ch.back(), out_c, 4, 2, 1));
    g.push_back(Layer::tanh_());
  };
  auto dnet = [](std::vector<Layer>& d, long in_c, std::vector<long> ch, long side) {
    d.push_back(Layer::conv(in_c, ch[0], 4, 2, 1));
    d.push_back(Layer::lrelu(0.2));
    for (size_t i = 1; i < ch.size(); ++i) {
      d.push_back(Layer::conv(ch[i - 1], ch[i], 4, 2, 1));
      d.push_back(Layer::bn(ch[i]));
      d.push_back(Layer::lrelu(0.2));
    }
    long f = ch.back() * side * side;
    d.push_back(Layer::reshape({f}));
    d.push_back(Layer::dense(f, 1));
    d.push_back(Layer::sigmoid());
  };
  if (cfg == 1) {
    a.image = {1, 28, 28};
    a.gen = {Layer::dense(d_z, 128 * 7 * 7), Layer::reshape({128, 7, 7}), Layer::bn(128), Layer::relu()};
    tail(a.gen, {128, 64}, 1);
    dnet(a.disc, 1, {64, 128}, 7);
  } else if (cfg == 2 || cfg == 3) {
    a.image = {3, 32, 32};
    a.gen = {Layer::dense(d_z, 256 * 4 * 4), Layer::reshape({256, 4, 4}), Layer::bn(256), Layer::relu()};
    tail(a.gen, {256, 128, 64}, 3);
    dnet(a.disc, 3, {64, 128, 256}, 4);
  } else if (cfg == 4) {
    a.image = {3, 64, 64};
    a.gen = {Layer::dense(d_z, 512 * 4 * 4), Layer::reshape({512, 4, 4}), Layer::bn(512), Layer::relu()};
    tail(a.gen, {512, 256, 128, 64}, 3);
    dnet(a.disc, 3, {64, 128, 256, 512}, 4);
  } else {
    throw std::invalid_argument("baseline_arch: config must be 1..4");
  }
  return a;
}

// ---------------------------------------------------------------------------
// partition / coordinator (partition.hpp, partition.cpp)
// ---------------------------------------------------------------------------
struct ClassShard {
  int class_id = 0;
  std::vector<long> indices;
};

inline std::vector<ClassShard> partition_by_label(const std::vector<int>& labels, int k) {
  if (k < 1) throw std::invalid_argument("partition_by_label: k must be >= 1");
  if (labels.empty()) throw std::invalid_argument("partition_by_label: empty label vector");
  std::vector<ClassShard> sh(static_cast<size_t>(k));
  for (int j = 0; j < k; ++j) sh[static_cast<size_t>(j)].class_id = j;
  for (size_t i = 0; i < labels.size(); ++i) {
    int l = labels[i];
    if (l < 0 || l >= k)
      throw std::out_of_range("label " + std::to_string(l) + " at index " + std::to_string(i) + " outside [0, " +
                              std::to_string(k) + ")");
    sh[static_cast<size_t>(l)].indices.push_back(static_cast<long>(i));
  }
  for (const auto& s : sh)
    if (s.indices.empty()) throw std::invalid_argument("class " + std::to_string(s.class_id) + " has no samples");
  return sh;
}

struct ClassPrior {
  std::vector<long> counts;
  std::vector<double> probabilities;
};

inline ClassPrior estimate_priors(const std::vector<ClassShard>& sh) {
  if (sh.empty()) throw std::invalid_argument("estimate_priors: no shards");
  ClassPrior pr;
  pr.counts.assign(sh.size(), 0);
  long total = 0;
  for (const auto& s : sh) {
    if (s.class_id < 0 || s.class_id >= static_cast<int>(sh.size()))
      throw std::invalid_argument("shard class id " + std::to_string(s.class_id) + " out of range");
    if (s.indices.empty()) throw std::invalid_argument("class " + std::to_string(s.class_id) + " has no samples");
    pr.counts[static_cast<size_t>(s.class_id)] = static_cast<long>(s.indices.size());
    total += static_cast<long>(s.indices.size());
  }
  for (long c : pr.counts) pr.probabilities.push_back(static_cast<double>(c) / static_cast<double>(total));
  return pr;
}

struct WorkerConfig {
  int class_id = 0;
  uint64_t seed = 0;
  int epochs = 1;
  long batch_size = 64;
  std::vector<Layer> gen_arch, disc_arch;
  Shape image;
  long d_z = 100, d_y = 0;
  AdamConfig adam;
  double clamp = 1e-7, init_std = 0.02;
};

// The worker protocol of run_worker (partition.cpp:78-112) as a steppable
// object: one stream drives shuffle, z1, z2 in that order; contiguous batches
// over the shuffled shard including the partial tail batch.
template <class R>
struct Worker {
  WorkerConfig cfg;
  Rng rng;
  GanPair<R> pair;
  std::vector<long> order;
  int epoch = 0;
  size_t at = 0;
  bool fresh_epoch = true;
  std::vector<StepReport> reports;
  std::vector<long> last_batch;

  Worker(const WorkerConfig& c, const ClassShard& sh)
      : cfg(c), rng(c.seed),
        pair(make_gan_pair<R>(c.gen_arch, c.disc_arch, c.image, c.d_z, c.d_y, c.adam, c.seed, c.init_std, c.clamp)),
        order(sh.indices) {}

  bool done() const { return epoch >= cfg.epochs; }

  // next batch indices (drawing the epoch shuffle first when one starts)
  std::vector<long> next_batch() {
    if (fresh_epoch) {
      std::shuffle(order.begin(), order.end(), rng.engine());
      fresh_epoch = false;
      at = 0;
    }
    size_t end = std::min(order.size(), at + static_cast<size_t>(cfg.batch_size));
    std::vector<long> b(order.begin() + static_cast<long>(at), order.begin() + static_cast<long>(end));
    at = end;
    if (at >= order.size()) {
      epoch += 1;
      fresh_epoch = true;
    }
    return b;
  }

  StepReport step(const Dataset& ds) {
    last_batch = next_batch();
    std::optional<int> cid;
    if (pair.d_y > 0) cid = cfg.class_id;
    StepReport r = train_step(pair, ds.gather<R>(last_batch), cid, rng);
    reports.push_back(r);
    return r;
  }
};

template <class R>
struct WorkerResult {
  int class_id = 0;
  uint64_t seed = 0;
  GanPair<R> pair;
  std::vector<StepReport> reports;
  double duration_s = 0, start_s = 0, end_s = 0;
};

class TrainError : public std::runtime_error {
 public:
  TrainError(const std::string& m, std::vector<int> f, std::vector<int> c)
      : std::runtime_error(m), failed_classes(std::move(f)), completed_classes(std::move(c)) {}
  std::vector<int> failed_classes, completed_classes;
};

template <class R>
struct TrainingRun {
  std::vector<WorkerResult<R>> workers;
  ClassPrior priors;
  double coordinator_duration_s = 0;
};

// train_distributed (partition.cpp:116-180): bounded pool, atomic work index,
// per-worker failure capture, results in config order.
template <class R>
TrainingRun<R> train_distributed(const Dataset& ds, const std::vector<ClassShard>& shards,
                                 const std::vector<WorkerConfig>& cfgs, int pool_size) {
  using Clock = std::chrono::steady_clock;
  if (shards.empty()) throw std::invalid_argument("train_distributed: no shards");
  if (shards.size() != cfgs.size())
    throw std::invalid_argument("train_distributed: " + std::to_string(shards.size()) + " shards but " +
                                std::to_string(cfgs.size()) + " worker configs");
  size_t k = shards.size();
  int pool = pool_size > 0 ? pool_size : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  size_t nthreads = std::min<size_t>(static_cast<size_t>(pool), k);
  std::vector<std::optional<WorkerResult<R>>> res(k);
  std::vector<std::string> errs(k);
  std::atomic<size_t> next{0};
  auto t0 = Clock::now();
  auto since = [&](Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); };
  auto body = [&]() {
    for (;;) {
      size_t i = next.fetch_add(1);
      if (i >= k) break;
      try {
        WorkerResult<R> r;
        r.class_id = cfgs[i].class_id;
        r.seed = cfgs[i].seed;
        r.start_s = since(t0);
        auto b = Clock::now();
        Worker<R> w(cfgs[i], shards[i]);
        while (!w.done()) w.step(ds);
        r.pair = std::move(w.pair);
        r.reports = std::move(w.reports);
        r.duration_s = std::max(since(b), 1e-9);
        r.end_s = since(t0);
        res[i] = std::move(r);
      } catch (const std::exception& e) {
        errs[i] = e.what();
      } catch (...) {
        errs[i] = "unknown worker error";
      }
    }
  };
  if (nthreads <= 1) {
    body();
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < nthreads; ++t) th.emplace_back(body);
    for (auto& t : th) t.join();
  }
  double total = since(t0);
  std::vector<int> failed, done;
  std::string detail;
  for (size_t i = 0; i < k; ++i) {
    if (res[i]) {
      done.push_back(cfgs[i].class_id);
    } else {
      failed.push_back(cfgs[i].class_id);
      detail += " class " + std::to_string(cfgs[i].class_id) + ": " + errs[i] + ";";
    }
  }
  if (!failed.empty())
    throw TrainError("training failed for " + std::to_string(failed.size()) + " of " + std::to_string(k) +
                         " workers (" + std::to_string(done.size()) + " completed):" + detail,
                     failed, done);
  TrainingRun<R> run;
  run.coordinator_duration_s = std::max(total, 1e-9);
  run.priors = estimate_priors(shards);
  for (size_t i = 0; i < k; ++i) run.workers.push_back(std::move(*res[i]));
  return run;
}

// mixture_sample (partition.cpp:182-227): class ids drawn first from one
// stream, then class by class generation from the same stream.
template <class R>
std::pair<Tensor<R>, std::vector<int>> mixture_sample(const std::vector<const GanPair<R>*>& pairs,
                                                      const ClassPrior& pri, long n, Rng& rng) {
  if (pairs.empty()) throw std::invalid_argument("mixture_sample: no generator pairs");
  if (n < 1) throw std::invalid_argument("mixture_sample: n must be >= 1");
  size_t k = pairs.size();
  if (pri.probabilities.size() != k) throw std::invalid_argument("mixture_sample: prior length does not match pair count");
  if (k == 1) return {generate(*pairs[0], 0, n, rng), std::vector<int>(static_cast<size_t>(n), 0)};
  std::vector<double> cdf(k);
  double acc = 0;
  for (size_t j = 0; j < k; ++j) cdf[j] = (acc += pri.probabilities[j]);
  std::vector<int> ids(static_cast<size_t>(n));
  for (auto& id : ids) {
    double u = rng.uniform();
    size_t j = 0;
    while (j + 1 < k && u >= cdf[j]) ++j;
    id = static_cast<int>(j);
  }
  Shape smp = pairs[0]->gen.out_shape_();
  for (const auto* p : pairs)
    if (p->gen.out_shape_() != smp) throw std::invalid_argument("mixture_sample: pairs emit different sample shapes");
  Tensor<R> out(detail::with_batch(n, smp));
  long st = shape_numel(smp);
  for (size_t j = 0; j < k; ++j) {
    std::vector<long> where;
    for (long i = 0; i < n; ++i)
      if (ids[static_cast<size_t>(i)] == static_cast<int>(j)) where.push_back(i);
    if (where.empty()) continue;
    Tensor<R> s = generate(*pairs[j], static_cast<int>(j), static_cast<long>(where.size()), rng);
    for (size_t w = 0; w < where.size(); ++w)
      std::copy(s.data.begin() + static_cast<long>(w) * st, s.data.begin() + static_cast<long>(w + 1) * st,
                out.data.begin() + where[w] * st);
  }
  return {std::move(out), std::move(ids)};
}

}  // namespace oracle
