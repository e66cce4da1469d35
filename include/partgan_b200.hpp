// partgan_b200.hpp — C++ mirror of partgan's public API (/root/reference/proj
// include/partgan/{tensor,rng,layers,network,optim,gan,data,partition}.hpp)
// over the B200 C-ABI (pg_network.h, pg_trainer.h).  Header-only; link
// libpartgan_b200.so.  A reference user swaps `partgan::` for
// `partgan_b200::`: the names, argument meaning, call order of the random
// streams and the error types / message text are the reference's.
//
// Deliberate differences (device-resident storage, no Eigen in this image):
//   - Tensor holds std::vector<double> (row-major, last index fastest) instead
//     of Eigen::ArrayXd; Network::params()/buffers() return copies, with
//     set_params()/set_buffers() to write (the values live in HBM, fp32);
//   - arithmetic is fp32 on the device (PG_MATH_TF32X3 by default: tcgen05
//     3xTF32, fp32-accurate), so results match the reference to the tolerances
//     stated in DESIGN.md §5, not bit for bit;
//   - layer lists must be the device block form [Reshape] Dense|Conv2d|
//     ConvTranspose2d [Reshape] [BatchNorm] [activation] (every BASELINE
//     architecture); Upsample / Dropout and conditional pairs (LabelSpec d_y > 0)
//     raise std::invalid_argument;
//   - train_distributed's pool_size counts GPUs, not threads (0 = every visible
//     GPU): labels are sharded in contiguous blocks, one host thread and one
//     label group per GPU; results are bitwise independent of the sharding.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <variant>
#include <vector>

#include "pg_network.h"
#include "pg_trainer.h"

namespace partgan_b200 {

using Index = long;
using Shape = std::vector<Index>;

// ---------------------------------------------------------------- errors
namespace detail {
inline void check(int rc) {
  if (rc == PG_OK) return;
  const std::string msg = pg_last_error();
  if (rc == PG_EINVAL || rc == PG_ENONFINITE) {
    if (msg.find("out of range") != std::string::npos || msg.find("label index") == 0) throw std::out_of_range(msg);
    throw std::invalid_argument(msg);
  }
  throw std::runtime_error(msg);
}
}  // namespace detail

// ---------------------------------------------------------------- tensor.hpp
inline std::string shape_to_string(const Shape& s) {
  std::string r = "[";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? "x" : "") + std::to_string(s[i]);
  return r + "]";
}
inline Index shape_size(const Shape& s) {
  Index n = 1;
  for (Index d : s) n *= d;
  return n;
}

// Dense row-major numeric array (tensor.hpp:17-48).
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(Shape shape) : shape_(std::move(shape)) {
    for (Index d : shape_)
      if (d <= 0) throw std::invalid_argument("tensor extents must be positive, got " + shape_to_string(shape_));
    data_.assign(static_cast<size_t>(shape_size(shape_)), 0.0);
  }
  Tensor(Shape shape, std::vector<double> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (static_cast<Index>(data_.size()) != shape_size(shape_))
      throw std::invalid_argument("tensor data size does not match shape " + shape_to_string(shape_));
  }
  static Tensor zeros(Shape shape) { return Tensor(std::move(shape)); }
  static Tensor constant(Shape shape, double v) {
    Tensor t(std::move(shape));
    std::fill(t.data_.begin(), t.data_.end(), v);
    return t;
  }
  const Shape& shape() const { return shape_; }
  Index dim(size_t i) const { return shape_.at(i); }
  size_t rank() const { return shape_.size(); }
  Index size() const { return static_cast<Index>(data_.size()); }
  std::vector<double>& data() { return data_; }
  const std::vector<double>& data() const { return data_; }
  double operator[](Index i) const { return data_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return data_[static_cast<size_t>(i)]; }
  Tensor reshaped(Shape target) const {
    if (shape_size(target) != size())
      throw std::invalid_argument("cannot reshape " + shape_to_string(shape_) + " to " + shape_to_string(target));
    return Tensor(std::move(target), data_);
  }
  bool all_finite() const {
    return std::all_of(data_.begin(), data_.end(), [](double v) { return std::isfinite(v); });
  }

 private:
  Shape shape_;
  std::vector<double> data_;
};

// ---------------------------------------------------------------- rng.hpp
inline uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t derive_seed(uint64_t base_seed, uint64_t stream_id) { return pg_derive_seed(base_seed, stream_id); }

// The reference stream (rng.hpp:27-46): mt19937_64 + libstdc++ distributions.
class Rng {
 public:
  explicit Rng(uint64_t seed) : engine_(seed) {}
  double normal() { return normal_(engine_); }
  double uniform() { return uniform_(engine_); }
  size_t index(size_t n) {
    std::uniform_int_distribution<size_t> d(0, n - 1);
    return d(engine_);
  }
  std::mt19937_64& engine() { return engine_; }

 private:
  std::mt19937_64 engine_;
  std::normal_distribution<double> normal_{0.0, 1.0};
  std::uniform_real_distribution<double> uniform_{0.0, 1.0};
};

// ---------------------------------------------------------------- layers.hpp
struct Dense {
  Index in_dim = 0, out_dim = 0;
};
struct Conv2d {
  Index in_ch = 0, out_ch = 0, kernel = 3, stride = 1, padding = 0;
};
// the BASELINE generators' transposed convolution (weight [Cin][Cout][k][k])
struct ConvTranspose2d {
  Index in_ch = 0, out_ch = 0, kernel = 4, stride = 2, padding = 1;
};
struct BatchNorm {
  Index channels = 0;
  double epsilon = 1e-5;
  double momentum = 0.1;
};
struct Upsample {
  Index scale_factor = 2;
};
struct Dropout {
  double rate = 0.5;
};
struct ReLU {};
struct LeakyReLU {
  double slope = 0.2;
};
struct Tanh {};
struct Sigmoid {};
struct Reshape {
  Shape target_shape;
};
using LayerSpec = std::variant<Dense, Conv2d, ConvTranspose2d, BatchNorm, Upsample, Dropout, ReLU, LeakyReLU, Tanh,
                               Sigmoid, Reshape>;

namespace detail {
inline std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}
inline std::string layer_text(const LayerSpec& l) {
  struct V {
    std::string operator()(const Dense& d) const { return "dense " + std::to_string(d.in_dim) + " " + std::to_string(d.out_dim); }
    std::string operator()(const Conv2d& c) const {
      return "conv2d " + std::to_string(c.in_ch) + " " + std::to_string(c.out_ch) + " " + std::to_string(c.kernel) +
             " " + std::to_string(c.stride) + " " + std::to_string(c.padding);
    }
    std::string operator()(const ConvTranspose2d& c) const {
      return "convT2d " + std::to_string(c.in_ch) + " " + std::to_string(c.out_ch) + " " + std::to_string(c.kernel) +
             " " + std::to_string(c.stride) + " " + std::to_string(c.padding);
    }
    std::string operator()(const BatchNorm& b) const {
      return "bn " + std::to_string(b.channels) + " " + num(b.epsilon) + " " + num(b.momentum);
    }
    std::string operator()(const Upsample& u) const { return "upsample " + std::to_string(u.scale_factor); }
    std::string operator()(const Dropout& d) const { return "dropout " + num(d.rate); }
    std::string operator()(const ReLU&) const { return "relu"; }
    std::string operator()(const LeakyReLU& l) const { return "lrelu " + num(l.slope); }
    std::string operator()(const Tanh&) const { return "tanh"; }
    std::string operator()(const Sigmoid&) const { return "sigmoid"; }
    std::string operator()(const Reshape& r) const {
      std::string s = "reshape";
      for (Index d : r.target_shape) s += " " + std::to_string(d);
      return s;
    }
  };
  return std::visit(V{}, l);
}
inline std::string spec_text(const std::vector<LayerSpec>& ls) {
  std::string s;
  for (size_t i = 0; i < ls.size(); ++i) s += (i ? "; " : "") + layer_text(ls[i]);
  return s;
}
}  // namespace detail

// ---------------------------------------------------------------- network.hpp
enum class Mode { train, eval };

// Device-side options of a network / pair (not in the reference API).
struct DeviceOptions {
  int math = PG_MATH_TF32X3;  // PG_MATH_{FP32_SIMT, TF32X3 (fp32-accurate), TF32, BF16} (pg_kernels.h)
  int device = 0;
};

// A device-resident network (network.hpp:20-54).  Copying makes an
// independent device copy (parameters and buffers), like the reference's
// value semantics.
class Network {
 public:
  Network() = default;
  Network(const Network& o) { *this = o; }
  Network& operator=(const Network& o) {
    if (this == &o) return *this;
    layers_ = o.layers_;
    input_ = o.input_;
    seed_ = o.seed_;
    init_std_ = o.init_std_;
    opt_ = o.opt_;
    h_.reset();
    if (o.h_) {
      create();
      set_params(o.params());
      set_buffers(o.buffers());
    }
    return *this;
  }
  Network(Network&&) noexcept = default;
  Network& operator=(Network&&) noexcept = default;

  const std::vector<LayerSpec>& layers() const { return layers_; }
  size_t layer_count() const { return layers_.size(); }
  const Shape& input_shape() const { return input_; }
  Shape output_shape() const {
    long s[4] = {0, 0, 0, 0};
    int r = 0;
    detail::check(pg_net_out_shape(h(), s, &r));
    return Shape(s, s + r);
  }
  Index param_count() const { return pg_net_param_count(h()); }
  Index buffer_count() const { return pg_net_buffer_count(h()); }
  std::vector<double> params() const {
    std::vector<double> p(static_cast<size_t>(param_count()));
    detail::check(pg_net_get_params(h(), p.data()));
    return p;
  }
  void set_params(const std::vector<double>& p) {
    if (static_cast<Index>(p.size()) != param_count()) throw std::invalid_argument("set_params: length mismatch");
    detail::check(pg_net_set_params(h(), p.data()));
  }
  std::vector<double> buffers() const {
    std::vector<double> b(static_cast<size_t>(std::max<Index>(buffer_count(), 1)));
    detail::check(pg_net_get_buffers(h(), b.data()));
    b.resize(static_cast<size_t>(buffer_count()));
    return b;
  }
  void set_buffers(const std::vector<double>& b) {
    if (static_cast<Index>(b.size()) != buffer_count()) throw std::invalid_argument("set_buffers: length mismatch");
    if (!b.empty()) detail::check(pg_net_set_buffers(h(), b.data()));
  }
  pg_net* handle() const { return h(); }

 private:
  friend Network build_network(std::vector<LayerSpec>, Shape, uint64_t, double, DeviceOptions);
  struct Del {
    void operator()(pg_net* p) const { pg_net_destroy(p); }
  };
  std::vector<LayerSpec> layers_;
  Shape input_;
  uint64_t seed_ = 0;
  double init_std_ = 0.02;
  DeviceOptions opt_;
  std::unique_ptr<pg_net, Del> h_;

  pg_net* h() const {
    if (!h_) throw std::invalid_argument("network is empty (use build_network)");
    return h_.get();
  }
  void create() {
    const std::string text = detail::spec_text(layers_);
    std::vector<long> in(input_.begin(), input_.end());
    pg_net* p = nullptr;
    detail::check(
        pg_net_create(text.c_str(), in.data(), static_cast<int>(in.size()), seed_, init_std_, opt_.math, opt_.device, &p));
    h_.reset(p);
  }
};

// build_network (network.cpp:308-343): the reference's init draws, in order.
inline Network build_network(std::vector<LayerSpec> specs, Shape input_shape, uint64_t seed, double init_std = 0.02,
                             DeviceOptions opt = {}) {
  if (specs.empty()) throw std::invalid_argument("network spec list is empty");
  Network n;
  n.layers_ = std::move(specs);
  n.input_ = std::move(input_shape);
  n.seed_ = seed;
  n.init_std_ = init_std;
  n.opt_ = opt;
  n.create();
  return n;
}

// One trace per forward call; backward consumes it exactly once (network.hpp:71-77).
struct ForwardTrace {
  const Network* net = nullptr;
  Mode mode = Mode::eval;
  Index batch = 0;
  bool consumed = false;
  struct Del {
    void operator()(pg_trace* t) const { pg_trace_destroy(t); }
  };
  std::unique_ptr<pg_trace, Del> device;
};

struct Gradients {
  std::vector<double> params;
  Tensor input;
};

namespace detail {
inline void check_batch(const Network& net, const Tensor& batch) {
  Shape want = net.input_shape();
  Shape got(batch.shape().begin() + (batch.rank() ? 1 : 0), batch.shape().end());
  if (batch.rank() == 0 || got != want)
    throw std::invalid_argument("input shape " + shape_to_string(batch.shape()) + " does not match network input " +
                                shape_to_string(want));
}
inline Shape with_batch(Index n, Shape s) {
  s.insert(s.begin(), n);
  return s;
}
}  // namespace detail

// forward (network.cpp:402-419).  rng feeds dropout masks in the reference;
// the device block form has none, so it is not drawn from.
inline std::pair<Tensor, ForwardTrace> forward(Network& net, const Tensor& batch, Mode mode, Rng& rng) {
  (void)rng;
  detail::check_batch(net, batch);
  const Index B = batch.dim(0);
  Tensor y(detail::with_batch(B, net.output_shape()));
  pg_trace* t = nullptr;
  detail::check(pg_net_forward(net.handle(), batch.data().data(), static_cast<int>(B), mode == Mode::train ? 1 : 0,
                               y.data().data(), &t));
  ForwardTrace tr;
  tr.net = &net;
  tr.mode = mode;
  tr.batch = B;
  tr.device.reset(t);
  return {std::move(y), std::move(tr)};
}

// infer (network.cpp:421-427): eval-mode forward, no trace, no state touched.
inline Tensor infer(const Network& net, const Tensor& batch) {
  detail::check_batch(net, batch);
  const Index B = batch.dim(0);
  Tensor y(detail::with_batch(B, net.output_shape()));
  detail::check(pg_net_forward(net.handle(), batch.data().data(), static_cast<int>(B), 0, y.data().data(), nullptr));
  return y;
}

// backward (network.cpp:429-480): fresh gradients of the traced computation.
inline Gradients backward(const Network& net, ForwardTrace& trace, const Tensor& output_grad) {
  if (trace.net != &net) throw std::invalid_argument("trace does not belong to this network");
  if (trace.consumed) throw std::invalid_argument("trace already consumed by a previous backward call");
  const Shape want = detail::with_batch(trace.batch, net.output_shape());
  trace.consumed = true;
  if (output_grad.shape() != want)
    throw std::invalid_argument("output gradient shape " + shape_to_string(output_grad.shape()) +
                                " does not match network output " + shape_to_string(want));
  Gradients g;
  g.params.assign(static_cast<size_t>(net.param_count()), 0.0);
  g.input = Tensor(detail::with_batch(trace.batch, net.input_shape()));
  detail::check(pg_net_backward(net.handle(), trace.device.get(), output_grad.data().data(),
                                static_cast<int>(trace.batch), g.params.data(), g.input.data().data()));
  return g;
}

struct LossFn {
  std::function<double(const Tensor&)> value;
  std::function<Tensor(const Tensor&)> grad;
};

// grad_check (network.cpp:482-516): backprop vs central differences on
// n_coords sampled coordinates (same coordinate draw as the reference).  The
// forwards run in fp32 on the device, so `step` should be ~1e-2.
inline double grad_check(const Network& net, const Tensor& input, const LossFn& loss, int n_coords, double step,
                         Mode mode, Rng& rng) {
  if (net.param_count() == 0) return 0.0;
  Network work = net;
  Rng unused(0);
  auto fw = forward(work, input, mode, unused);
  Tensor gout = loss.grad(fw.first);
  Gradients g = backward(work, fw.second, gout);
  std::vector<Index> coords(static_cast<size_t>(net.param_count()));
  std::iota(coords.begin(), coords.end(), Index{0});
  if (n_coords < static_cast<int>(coords.size())) {
    std::shuffle(coords.begin(), coords.end(), rng.engine());
    coords.resize(static_cast<size_t>(n_coords));
  }
  const std::vector<double> base = work.params();
  const std::vector<double> bufs = work.buffers();
  double max_rel = 0.0;
  for (Index c : coords) {
    std::vector<double> p = base;
    p[static_cast<size_t>(c)] = base[static_cast<size_t>(c)] + step;
    work.set_params(p);
    work.set_buffers(bufs);
    double f_plus = loss.value(forward(work, input, mode, unused).first);
    p[static_cast<size_t>(c)] = base[static_cast<size_t>(c)] - step;
    work.set_params(p);
    work.set_buffers(bufs);
    double f_minus = loss.value(forward(work, input, mode, unused).first);
    double numeric = (f_plus - f_minus) / (2.0 * step);
    double analytic = g.params[static_cast<size_t>(c)];
    double rel = std::abs(analytic - numeric) / std::max({std::abs(analytic), std::abs(numeric), 1e-8});
    max_rel = std::max(max_rel, rel);
  }
  return max_rel;
}

// ---------------------------------------------------------------- optim.hpp
struct AdamConfig {
  double lr = 2e-4, beta1 = 0.5, beta2 = 0.999, eps = 1e-8;
};
struct AdamState {
  std::vector<double> m, v;
  long t = 0;
  double lr = 2e-4, beta1 = 0.5, beta2 = 0.999, eps = 1e-8;
  static AdamState create(Index n, const AdamConfig& cfg) {
    AdamState s;
    s.m.assign(static_cast<size_t>(n), 0.0);
    s.v.assign(static_cast<size_t>(n), 0.0);
    s.lr = cfg.lr;
    s.beta1 = cfg.beta1;
    s.beta2 = cfg.beta2;
    s.eps = cfg.eps;
    return s;
  }
};

// adam_step (optim.cpp:20-34) on the device, fp32 state arithmetic.
inline void adam_step(AdamState& st, std::vector<double>& params, const std::vector<double>& grads, int device = 0) {
  if (params.size() != st.m.size() || grads.size() != st.m.size())
    throw std::invalid_argument("adam_step: length mismatch (params " + std::to_string(params.size()) + ", grads " +
                                std::to_string(grads.size()) + ", state " + std::to_string(st.m.size()) + ")");
  if (params.empty()) {
    for (double g : grads)
      if (!std::isfinite(g)) throw std::invalid_argument("adam_step: non-finite gradient rejected");
    st.t += 1;
    return;
  }
  detail::check(pg_adam_step_host(static_cast<long>(params.size()), params.data(), grads.data(), st.m.data(),
                                  st.v.data(), &st.t, st.lr, st.beta1, st.beta2, st.eps, device));
}

// ---------------------------------------------------------------- gan.hpp
struct LatentSpec {
  Index d_z = 100;
};
struct LabelSpec {
  Index d_y = 0;
};
struct StepReport {
  double j_d = 0, j_g = 0, d_real_mean = 0, d_fake_mean = 0;
};

namespace detail {
// One label group on one device; GanPairs reference (group, label index).
struct Group {
  pg_group* g = nullptr;
  std::vector<int> class_ids;
  std::vector<uint64_t> seeds;
  std::string gen, disc;
  Shape image;
  Index d_z = 100;
  int batch = 0;
  long per_label = 0;
  AdamConfig adam;
  double clamp = 1e-7, init_std = 0.02;
  DeviceOptions opt;
  int epochs = 1;
  ~Group() {
    if (g) pg_group_destroy(g);
  }
};
inline std::shared_ptr<Group> make_group(const std::string& gen, const std::string& disc, const Shape& image, Index d_z,
                                         const std::vector<int>& class_ids, const std::vector<uint64_t>& seeds,
                                         int batch, long per_label, int epochs, const AdamConfig& adam, double clamp,
                                         double init_std, DeviceOptions opt) {
  auto G = std::make_shared<Group>();
  G->class_ids = class_ids;
  G->seeds = seeds;
  G->gen = gen;
  G->disc = disc;
  G->image = image;
  G->d_z = d_z;
  G->batch = batch;
  G->per_label = per_label;
  G->adam = adam;
  G->clamp = clamp;
  G->init_std = init_std;
  G->opt = opt;
  G->epochs = epochs;
  if (image.size() != 3) throw std::invalid_argument("image shape must be [C, H, W]");
  pg_group_config c{};
  c.gen_spec = G->gen.c_str();
  c.disc_spec = G->disc.c_str();
  c.C = static_cast<int>(image[0]);
  c.H = static_cast<int>(image[1]);
  c.W = static_cast<int>(image[2]);
  c.d_z = static_cast<int>(d_z);
  c.n_labels = static_cast<int>(G->class_ids.size());
  c.class_ids = G->class_ids.data();
  c.base_seed = 0;
  c.batch = batch;
  c.epochs = epochs;
  c.per_label = per_label;
  c.lr = adam.lr;
  c.beta1 = adam.beta1;
  c.beta2 = adam.beta2;
  c.eps = adam.eps;
  c.clamp = clamp;
  c.init_std = init_std;
  c.math = opt.math;
  c.threads = 8;
  c.device = opt.device;
  c.seeds = G->seeds.data();
  detail::check(pg_group_create(&c, &G->g));
  return G;
}
inline std::vector<double> get(pg_group* g, int l, int field) {
  long n = pg_group_get(g, l, field, nullptr, 0);
  if (n < 0) check(static_cast<int>(n));
  std::vector<double> v(static_cast<size_t>(n));
  if (n) check(pg_group_get(g, l, field, v.data(), n) < 0 ? PG_EINVAL : PG_OK);
  return v;
}
inline void set(pg_group* g, int l, int field, const std::vector<double>& v) {
  check(pg_group_set(g, l, field, v.data(), static_cast<long>(v.size())));
}
}  // namespace detail

// A generator/discriminator pair with its optimizer states (gan.hpp:25-34),
// device-resident: one label of a label group.  Stepping a pair that shares
// its group with other labels (a train_distributed result) first moves it to
// a group of its own (its state copied), so pairs keep value semantics.
class GanPair {
 public:
  LatentSpec latent;
  LabelSpec label;
  double prob_clamp = 1e-7;

  long steps() const { return static_cast<long>(detail::get(grp_->g, idx_, PG_F_COUNTERS)[2]); }
  long opt_g_t() const { return static_cast<long>(detail::get(grp_->g, idx_, PG_F_COUNTERS)[0]); }
  long opt_d_t() const { return static_cast<long>(detail::get(grp_->g, idx_, PG_F_COUNTERS)[1]); }
  std::vector<double> generator_params() const { return detail::get(grp_->g, idx_, PG_F_GEN_PARAMS); }
  std::vector<double> discriminator_params() const { return detail::get(grp_->g, idx_, PG_F_DISC_PARAMS); }
  std::vector<double> generator_buffers() const { return detail::get(grp_->g, idx_, PG_F_GEN_BUFFERS); }
  std::vector<double> discriminator_buffers() const { return detail::get(grp_->g, idx_, PG_F_DISC_BUFFERS); }
  std::vector<double> field(int pg_field) const { return detail::get(grp_->g, idx_, pg_field); }
  Shape image_shape() const { return grp_->image; }
  pg_group* group() const { return grp_->g; }
  int label_index() const { return idx_; }
  // reference checkpoint format (checkpoint.cpp:91-194)
  void save(const std::string& path) const { detail::check(pg_group_save_checkpoint(grp_->g, idx_, path.c_str())); }
  void load(const std::string& path) { detail::check(pg_group_load_checkpoint(grp_->g, idx_, path.c_str())); }

  // a group of its own with capacity for batches of n
  void own(int n) {
    if (grp_->class_ids.size() == 1 && grp_->batch >= n) return;
    const int cap = std::max(n, grp_->batch);
    auto G = detail::make_group(grp_->gen, grp_->disc, grp_->image, grp_->d_z, {grp_->class_ids[static_cast<size_t>(idx_)]},
                                {grp_->seeds[static_cast<size_t>(idx_)]}, cap, cap, 1, grp_->adam, grp_->clamp,
                                grp_->init_std, grp_->opt);
    for (int f : {PG_F_GEN_PARAMS, PG_F_DISC_PARAMS, PG_F_GEN_BUFFERS, PG_F_DISC_BUFFERS, PG_F_GEN_ADAM_M,
                  PG_F_GEN_ADAM_V, PG_F_DISC_ADAM_M, PG_F_DISC_ADAM_V, PG_F_COUNTERS})
      detail::set(G->g, 0, f, detail::get(grp_->g, idx_, f));
    grp_ = std::move(G);
    idx_ = 0;
  }

 private:
  friend GanPair make_gan_pair(std::vector<LayerSpec>, std::vector<LayerSpec>, Shape, LatentSpec, LabelSpec,
                               const AdamConfig&, uint64_t, double, double, DeviceOptions);
  friend struct PairAccess;
  std::shared_ptr<detail::Group> grp_;
  int idx_ = 0;
};

struct PairAccess {
  static GanPair make(std::shared_ptr<detail::Group> g, int idx) {
    GanPair p;
    p.latent.d_z = g->d_z;
    p.prob_clamp = g->clamp;
    p.grp_ = std::move(g);
    p.idx_ = idx;
    return p;
  }
};

// make_gan_pair (gan.cpp:27-52): G from derive_seed(seed, 1), D from derive_seed(seed, 2).
inline GanPair make_gan_pair(std::vector<LayerSpec> gen_arch, std::vector<LayerSpec> disc_arch, Shape image_shape,
                             LatentSpec latent, LabelSpec label, const AdamConfig& adam, uint64_t seed,
                             double init_std = 0.02, double prob_clamp = 1e-7, DeviceOptions opt = {}) {
  if (!(prob_clamp > 0.0 && prob_clamp < 0.5))
    throw std::invalid_argument("probability clamp must lie in (0, 0.5), got " + std::to_string(prob_clamp));
  if (latent.d_z < 1) throw std::invalid_argument("latent dimension must be positive");
  if (label.d_y < 0) throw std::invalid_argument("label embedding dimension must be non-negative");
  if (label.d_y > 0)
    throw std::invalid_argument("conditional pairs (LabelSpec d_y > 0) are not on the B200 path: the label-partitioned "
                                "step trains unconditional pairs");
  auto G = detail::make_group(detail::spec_text(gen_arch), detail::spec_text(disc_arch), image_shape, latent.d_z, {0},
                              {seed}, 64, 64, 1, adam, prob_clamp, init_std, opt);
  GanPair p = PairAccess::make(std::move(G), 0);
  p.label = label;
  return p;
}

// sample_latent (gan.cpp:54-84): n rows of d_z normals, row-major.
inline Tensor sample_latent(const LatentSpec& latent, const LabelSpec& label, std::optional<int> class_id, Index n,
                            Rng& rng) {
  if (n < 1) throw std::invalid_argument("sample_latent: batch size must be positive");
  if (label.d_y > 0 && !class_id)
    throw std::invalid_argument("sample_latent: class id required when conditioning is enabled");
  const Index w = latent.d_z + label.d_y;
  Tensor z(Shape{n, w});
  for (Index i = 0; i < n; ++i) {
    for (Index j = 0; j < latent.d_z; ++j) z[i * w + j] = rng.normal();
    if (label.d_y > 0) {
      const int k = *class_id;
      if (k < 0 || k >= label.d_y)
        throw std::out_of_range("class id " + std::to_string(k) + " out of range [0, " + std::to_string(label.d_y) + ")");
      z[i * w + latent.d_z + k] = 1.0;
    }
  }
  return z;
}

namespace detail {
inline std::vector<float> to_f32(const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); }
}  // namespace detail

// train_step (gan.cpp:136-182): z1 then z2 from rng (no dropout in the device
// block form, so nothing else is drawn in between), D step then G step.
inline StepReport train_step(GanPair& pair, const Tensor& real_batch, std::optional<int> class_id, Rng& rng) {
  if (real_batch.size() == 0) throw std::invalid_argument("train_step: empty batch");
  const Shape img = pair.image_shape();
  if (real_batch.rank() != 4 || Shape(real_batch.shape().begin() + 1, real_batch.shape().end()) != img)
    throw std::invalid_argument("input shape " + shape_to_string(real_batch.shape()) + " does not match network input " +
                                shape_to_string(img));
  const Index n = real_batch.dim(0);
  pair.own(static_cast<int>(n));
  Tensor z1 = sample_latent(pair.latent, pair.label, class_id, n, rng);
  Tensor z2 = sample_latent(pair.latent, pair.label, class_id, n, rng);
  const auto r = detail::to_f32(real_batch.data()), a = detail::to_f32(z1.data()), b = detail::to_f32(z2.data());
  double rep[4];
  detail::check(pg_group_train_step_inputs(pair.group(), r.data(), a.data(), b.data(), static_cast<int>(n), rep));
  return StepReport{rep[0], rep[1], rep[2], rep[3]};
}

// generate (gan.cpp:197-201): eval-mode generator, (v+1)/2.
inline Tensor generate(const GanPair& pair, std::optional<int> class_id, Index n, Rng& rng) {
  Tensor z = sample_latent(pair.latent, pair.label, class_id, n, rng);
  const Shape img = pair.image_shape();
  GanPair solo = pair;  // a group of its own (a shared group would run every label's generator)
  solo.own(1);
  const auto zf = detail::to_f32(z.data());
  std::vector<float> o(static_cast<size_t>(n * shape_size(img)));
  detail::check(pg_group_generate_latents(solo.group(), zf.data(), static_cast<long>(n), o.data()));
  return Tensor(detail::with_batch(n, img), std::vector<double>(o.begin(), o.end()));
}

// ---------------------------------------------------------------- data.hpp / partition.hpp
struct Dataset {
  Tensor images;            // [m, C, H, W] in [0, 1]
  std::vector<int> labels;  // in [0, k)
  int k = 0;
  Index count() const { return images.dim(0); }
  Index channels() const { return images.dim(1); }
  Index height() const { return images.dim(2); }
  Index width() const { return images.dim(3); }
  Shape sample_shape() const { return {channels(), height(), width()}; }
  // Dataset::gather (data.cpp:13-23)
  Tensor gather(const std::vector<Index>& indices) const {
    if (indices.empty()) throw std::invalid_argument("gather: empty index list");
    const Index S = shape_size(sample_shape());
    Tensor out(Shape{static_cast<Index>(indices.size()), channels(), height(), width()});
    for (size_t i = 0; i < indices.size(); ++i) {
      const Index idx = indices[i];
      if (idx < 0 || idx >= count()) throw std::out_of_range("gather: index " + std::to_string(idx));
      std::copy(images.data().begin() + idx * S, images.data().begin() + (idx + 1) * S,
                out.data().begin() + static_cast<Index>(i) * S);
    }
    return out;
  }
};

struct ClassShard {
  int class_id = 0;
  std::vector<Index> indices;
};

// partition_by_label (partition.cpp:40-56)
inline std::vector<ClassShard> partition_by_label(const std::vector<int>& labels, int k) {
  if (k < 1) throw std::invalid_argument("partition_by_label: k must be >= 1");
  if (labels.empty()) throw std::invalid_argument("partition_by_label: empty label vector");
  std::vector<ClassShard> out(static_cast<size_t>(k));
  for (int c = 0; c < k; ++c) out[static_cast<size_t>(c)].class_id = c;
  for (size_t i = 0; i < labels.size(); ++i) {
    const int l = labels[i];
    if (l < 0 || l >= k)
      throw std::out_of_range("label " + std::to_string(l) + " at index " + std::to_string(i) + " outside [0, " +
                              std::to_string(k) + ")");
    out[static_cast<size_t>(l)].indices.push_back(static_cast<Index>(i));
  }
  for (auto& s : out)
    if (s.indices.empty()) throw std::invalid_argument("class " + std::to_string(s.class_id) + " has no samples");
  return out;
}

struct ClassPrior {
  std::vector<Index> counts;
  std::vector<double> probabilities;
};

// estimate_priors (partition.cpp:58-74)
inline ClassPrior estimate_priors(const std::vector<ClassShard>& shards) {
  if (shards.empty()) throw std::invalid_argument("estimate_priors: no shards");
  ClassPrior p;
  p.counts.assign(shards.size(), 0);
  Index total = 0;
  for (const auto& s : shards) {
    if (s.class_id < 0 || s.class_id >= static_cast<int>(shards.size()))
      throw std::invalid_argument("shard class id " + std::to_string(s.class_id) + " out of range");
    if (s.indices.empty()) throw std::invalid_argument("class " + std::to_string(s.class_id) + " has no samples");
    p.counts[static_cast<size_t>(s.class_id)] = static_cast<Index>(s.indices.size());
    total += static_cast<Index>(s.indices.size());
  }
  for (Index c : p.counts) p.probabilities.push_back(static_cast<double>(c) / static_cast<double>(total));
  return p;
}

struct WorkerConfig {
  int class_id = 0;
  uint64_t seed = 0;
  int epochs = 1;
  Index batch_size = 64;
  std::vector<LayerSpec> gen_arch, disc_arch;
  Shape image_shape;
  LatentSpec latent;
  LabelSpec label;
  AdamConfig adam;
  double prob_clamp = 1e-7;
  double init_std = 0.02;
  bool conditional_labels = false;
  DeviceOptions device;  // math mode (device ordinal is chosen by train_distributed)
};

struct WorkerResult {
  int class_id = 0;
  uint64_t seed = 0;
  GanPair pair;
  std::vector<StepReport> reports;
  double duration_s = 0, start_s = 0, end_s = 0;
};

struct TrainingRun {
  std::vector<WorkerResult> workers;  // config order
  ClassPrior priors;
  double coordinator_duration_s = 0;
};

class TrainError : public std::runtime_error {
 public:
  TrainError(const std::string& msg, std::vector<int> failed, std::vector<int> completed)
      : std::runtime_error(msg), failed_classes(std::move(failed)), completed_classes(std::move(completed)) {}
  std::vector<int> failed_classes;
  std::vector<int> completed_classes;
};

// train_distributed (partition.cpp:116-180) on the visible GPUs: workers
// whose configs differ only in class_id / seed and whose shards have equal
// size form one label group per GPU (contiguous blocks, pg_shard_begin); one
// host thread per GPU runs run_worker's protocol for all its labels in
// lockstep (per-label Rng(seed): epoch shuffle of the shard, contiguous
// batches with the partial tail, train_step).  pool_size = GPUs to use
// (0 = all).  Failed labels (non-finite gradients) raise TrainError after
// every worker finished, listing failed and completed classes.
inline TrainingRun train_distributed(const Dataset& dataset, const std::vector<ClassShard>& shards,
                                     const std::vector<WorkerConfig>& configs, int pool_size = 0) {
  using Clock = std::chrono::steady_clock;
  if (shards.empty()) throw std::invalid_argument("train_distributed: no shards");
  if (shards.size() != configs.size())
    throw std::invalid_argument("train_distributed: " + std::to_string(shards.size()) + " shards but " +
                                std::to_string(configs.size()) + " worker configs");
  const size_t k = shards.size();
  int ngpu = pg_device_count();
  if (ngpu < 1) throw std::runtime_error("train_distributed: no CUDA device");
  if (pool_size > 0) ngpu = std::min(ngpu, pool_size);
  for (const auto& c : configs) {
    if (c.conditional_labels || c.label.d_y > 0)
      throw std::invalid_argument("conditional pairs (LabelSpec d_y > 0) are not on the B200 path");
  }
  // buckets of uniform workers
  auto key = [&](size_t i) {
    const WorkerConfig& c = configs[i];
    return detail::spec_text(c.gen_arch) + "|" + detail::spec_text(c.disc_arch) + "|" + shape_to_string(c.image_shape) +
           "|" + std::to_string(c.latent.d_z) + "|" + std::to_string(c.epochs) + "|" + std::to_string(c.batch_size) +
           "|" + detail::num(c.adam.lr) + detail::num(c.adam.beta1) + detail::num(c.adam.beta2) +
           detail::num(c.adam.eps) + "|" + detail::num(c.prob_clamp) + detail::num(c.init_std) + "|" +
           std::to_string(c.device.math) + "|" + std::to_string(shards[i].indices.size());
  };
  std::vector<std::vector<size_t>> buckets;
  std::vector<std::string> keys;
  for (size_t i = 0; i < k; ++i) {
    const std::string kk = key(i);
    auto it = std::find(keys.begin(), keys.end(), kk);
    if (it == keys.end()) {
      keys.push_back(kk);
      buckets.push_back({i});
    } else {
      buckets[static_cast<size_t>(it - keys.begin())].push_back(i);
    }
  }
  struct Job {
    std::vector<size_t> workers;
    int device = 0;
    std::shared_ptr<detail::Group> grp;
    double start = 0, end = 0;
    std::string error;
  };
  std::vector<Job> jobs;
  for (const auto& b : buckets) {
    const int n = static_cast<int>(b.size());
    for (int gpu = 0; gpu < ngpu; ++gpu) {
      const int lo = pg_shard_begin(n, ngpu, gpu), hi = pg_shard_begin(n, ngpu, gpu + 1);
      if (hi <= lo) continue;
      Job j;
      j.device = gpu;
      j.workers.assign(b.begin() + lo, b.begin() + hi);
      jobs.push_back(std::move(j));
    }
  }
  const auto t0 = Clock::now();
  auto secs = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
  auto run_job = [&](Job& j) {
    try {
      const WorkerConfig& c0 = configs[j.workers.front()];
      const long per = static_cast<long>(shards[j.workers.front()].indices.size());
      std::vector<int> ids;
      std::vector<uint64_t> seeds;
      for (size_t w : j.workers) {
        ids.push_back(configs[w].class_id);
        seeds.push_back(configs[w].seed);
      }
      DeviceOptions opt = c0.device;
      opt.device = j.device;
      j.start = secs();
      j.grp = detail::make_group(detail::spec_text(c0.gen_arch), detail::spec_text(c0.disc_arch), c0.image_shape,
                                 c0.latent.d_z, ids, seeds, static_cast<int>(c0.batch_size), per, c0.epochs, c0.adam,
                                 c0.prob_clamp, c0.init_std, opt);
      // the labels' shards, label-blocked in shard order (position j <-> shard.indices[j])
      const Index S = shape_size(dataset.sample_shape());
      std::vector<float> img(static_cast<size_t>(j.workers.size() * per * S));
      for (size_t l = 0; l < j.workers.size(); ++l) {
        const auto& idx = shards[j.workers[l]].indices;
        for (long p = 0; p < per; ++p) {
          const Index src = idx[static_cast<size_t>(p)];
          if (src < 0 || src >= dataset.count()) throw std::out_of_range("gather: index " + std::to_string(src));
          std::copy(dataset.images.data().begin() + src * S, dataset.images.data().begin() + (src + 1) * S,
                    img.begin() + static_cast<Index>((l * per + p) * S));
        }
      }
      detail::check(pg_group_set_dataset(j.grp->g, img.data()));
      for (;;) {
        const int ran = pg_group_train_steps(j.grp->g, 64);
        if (ran < 0) detail::check(ran);
        if (ran < 64) break;
      }
      j.end = secs();
    } catch (const std::exception& e) {
      j.error = e.what();
    }
  };
  std::vector<std::thread> th;
  for (int gpu = 0; gpu < ngpu; ++gpu)
    th.emplace_back([&, gpu] {
      for (auto& j : jobs)
        if (j.device == gpu) run_job(j);
    });
  for (auto& t : th) t.join();
  const double total = secs();

  std::vector<int> failed, completed;
  std::string detail_msg;
  std::vector<std::optional<WorkerResult>> results(k);
  for (auto& j : jobs) {
    std::vector<int> bad(j.workers.size(), 0);
    if (j.error.empty()) detail::check(pg_group_failed(j.grp->g, bad.data()));
    for (size_t l = 0; l < j.workers.size(); ++l) {
      const size_t w = j.workers[l];
      if (!j.error.empty() || bad[l]) {
        failed.push_back(configs[w].class_id);
        detail_msg += " class " + std::to_string(configs[w].class_id) + ": " +
                      (j.error.empty() ? std::string("adam_step: non-finite gradient rejected") : j.error) + ";";
        continue;
      }
      WorkerResult r;
      r.class_id = configs[w].class_id;
      r.seed = configs[w].seed;
      r.pair = PairAccess::make(j.grp, static_cast<int>(l));
      const auto rep = detail::get(j.grp->g, static_cast<int>(l), PG_F_REPORTS);
      for (size_t s = 0; s + 3 < rep.size(); s += 4) r.reports.push_back(StepReport{rep[s], rep[s + 1], rep[s + 2], rep[s + 3]});
      r.start_s = j.start;
      r.end_s = j.end;
      r.duration_s = std::max(j.end - j.start, 1e-9);
      results[w] = std::move(r);
    }
  }
  for (size_t i = 0; i < k; ++i)
    if (results[i]) completed.push_back(configs[i].class_id);
  if (!failed.empty())
    throw TrainError("training failed for " + std::to_string(failed.size()) + " of " + std::to_string(k) +
                         " workers (" + std::to_string(completed.size()) + " completed):" + detail_msg,
                     std::move(failed), std::move(completed));
  TrainingRun run;
  run.coordinator_duration_s = std::max(total, 1e-9);
  run.priors = estimate_priors(shards);
  for (size_t i = 0; i < k; ++i) run.workers.push_back(std::move(*results[i]));
  return run;
}

// mixture_sample (partition.cpp:182-227): class ids from rng first, then class
// by class generate() from the same stream.
inline std::pair<Tensor, std::vector<int>> mixture_sample(const std::vector<const GanPair*>& pairs,
                                                          const ClassPrior& priors, Index n, Rng& rng) {
  if (pairs.empty()) throw std::invalid_argument("mixture_sample: no generator pairs");
  if (n < 1) throw std::invalid_argument("mixture_sample: n must be >= 1");
  const size_t k = pairs.size();
  if (priors.probabilities.size() != k)
    throw std::invalid_argument("mixture_sample: prior length does not match pair count");
  if (k == 1) return {generate(*pairs[0], 0, n, rng), std::vector<int>(static_cast<size_t>(n), 0)};
  std::vector<double> cdf(k);
  double acc = 0;
  for (size_t j = 0; j < k; ++j) cdf[j] = (acc += priors.probabilities[j]);
  std::vector<int> ids(static_cast<size_t>(n));
  for (auto& id : ids) {
    const double u = rng.uniform();
    size_t j = 0;
    while (j + 1 < k && u >= cdf[j]) ++j;
    id = static_cast<int>(j);
  }
  const Shape sample = pairs[0]->image_shape();
  for (const auto* p : pairs)
    if (p->image_shape() != sample) throw std::invalid_argument("mixture_sample: pairs emit different sample shapes");
  Tensor out(detail::with_batch(n, sample));
  const Index stride = shape_size(sample);
  for (size_t j = 0; j < k; ++j) {
    std::vector<Index> where;
    for (Index i = 0; i < n; ++i)
      if (ids[static_cast<size_t>(i)] == static_cast<int>(j)) where.push_back(i);
    if (where.empty()) continue;
    Tensor s = generate(*pairs[j], static_cast<int>(j), static_cast<Index>(where.size()), rng);
    for (size_t w = 0; w < where.size(); ++w)
      std::copy(s.data().begin() + static_cast<Index>(w) * stride, s.data().begin() + static_cast<Index>(w + 1) * stride,
                out.data().begin() + where[w] * stride);
  }
  return {std::move(out), std::move(ids)};
}

}  // namespace partgan_b200
