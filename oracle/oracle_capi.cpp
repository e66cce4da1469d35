// oracle/oracle_capi.cpp — TEST INFRASTRUCTURE ONLY.  C-ABI over the CPU
// restatement (oracle.hpp) so the Python tests and bench.py's cpu_baseline leg
// can drive it through ctypes.  Never linked into the product.
#include "oracle.hpp"
#include "spec.hpp"

#include <chrono>
#include <cstring>
#include <memory>

using namespace oracle;

namespace {

thread_local std::string g_err;

struct GroupBase {
  virtual ~GroupBase() = default;
  virtual void step(int n, int threads) = 0;
  virtual long get(int l, int what, double* out, long cap) = 0;
  virtual void set(int l, int what, const double* in, long n) = 0;
  virtual void step_inputs(int l, const double* real01, const double* z1, const double* z2, long B, double* rep) = 0;
  virtual int labels() const = 0;
  // MaskTape for the label's next step (consumed by it); flips of the last taped step
  virtual void set_masks(int l, const uint8_t* m, long n) = 0;
  virtual long mask_flips(int l) const = 0;
  // record the label's next step's own masks instead (read with get_masks)
  virtual void record_masks(int l) = 0;
  virtual long get_masks(int l, uint8_t* out, long cap) = 0;
  // mixture_sample (partition.cpp:182-227) over the group's pairs in label order
  virtual void mixture(const double* priors, long n, uint64_t seed, double* out, int* ids) = 0;
};

template <class R>
long put(const std::vector<R>& v, double* out, long cap) {
  long n = static_cast<long>(v.size());
  if (out) {
    if (cap < n) throw std::invalid_argument("output buffer too small");
    for (long i = 0; i < n; ++i) out[i] = static_cast<double>(v[static_cast<size_t>(i)]);
  }
  return n;
}

template <class R>
void take(std::vector<R>& v, const double* in, long n) {
  if (n != static_cast<long>(v.size())) throw std::invalid_argument("length mismatch on set");
  for (long i = 0; i < n; ++i) v[static_cast<size_t>(i)] = static_cast<R>(in[i]);
}

template <class R>
struct Group : GroupBase {
  Dataset ds;
  std::vector<std::unique_ptr<Worker<R>>> w;
  std::vector<std::vector<uint8_t>> masks, recorded;
  std::vector<long> flips;
  std::vector<char> recording;
  int labels() const override { return static_cast<int>(w.size()); }

  void set_masks(int l, const uint8_t* m, long n) override {
    masks.resize(w.size());
    flips.resize(w.size(), 0);
    masks.at(static_cast<size_t>(l)).assign(m, m + n);
  }
  long mask_flips(int l) const override {
    return static_cast<size_t>(l) < flips.size() ? flips[static_cast<size_t>(l)] : 0;
  }

  void record_masks(int l) override {
    recording.resize(w.size(), 0);
    recorded.resize(w.size());
    recording.at(static_cast<size_t>(l)) = 1;
  }
  long get_masks(int l, uint8_t* out, long cap) override {
    if (static_cast<size_t>(l) >= recorded.size()) return 0;
    const auto& r = recorded[static_cast<size_t>(l)];
    const long n = static_cast<long>(r.size());
    if (out) {
      if (cap < n) throw std::invalid_argument("output buffer too small");
      std::memcpy(out, r.data(), r.size());
    }
    return n;
  }

  // run f() with label i's mask tape installed (if one is set), then check it was used up
  template <class F>
  void taped(size_t i, F f) {
    if (i < recording.size() && recording[i]) {
      MaskTape tp;
      recorded[i].clear();
      tp.record = &recorded[i];
      mask_tape() = &tp;
      try {
        f();
      } catch (...) {
        mask_tape() = nullptr;
        throw;
      }
      mask_tape() = nullptr;
      recording[i] = 0;
      return;
    }
    if (i >= masks.size() || masks[i].empty()) {
      f();
      return;
    }
    MaskTape tp;
    tp.m = masks[i].data();
    tp.n = static_cast<long>(masks[i].size());
    mask_tape() = &tp;
    try {
      f();
    } catch (...) {
      mask_tape() = nullptr;
      throw;
    }
    mask_tape() = nullptr;
    masks[i].clear();
    flips[i] = tp.flips;
    if (tp.at != tp.n)
      throw std::invalid_argument("mask tape length " + std::to_string(tp.n) + " but the step used " +
                                  std::to_string(tp.at));
  }

  void step(int n, int threads) override {
    std::atomic<size_t> next{0};
    std::vector<std::string> errs(w.size());
    auto body = [&] {
      for (;;) {
        size_t i = next.fetch_add(1);
        if (i >= w.size()) break;
        try {
          for (int s = 0; s < n; ++s) taped(i, [&] { w[i]->step(ds); });
        } catch (const std::exception& e) {
          errs[i] = e.what();
        }
      }
    };
    int nt = std::max(1, std::min<int>(threads, static_cast<int>(w.size())));
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(body);
    body();
    for (auto& t : th) t.join();
    for (size_t i = 0; i < errs.size(); ++i)
      if (!errs[i].empty()) throw std::runtime_error("label index " + std::to_string(i) + ": " + errs[i]);
  }

  long get(int l, int what, double* out, long cap) override {
    Worker<R>& k = *w.at(static_cast<size_t>(l));
    GanPair<R>& p = k.pair;
    switch (what) {
      case 0: return put(p.gen.params, out, cap);
      case 1: return put(p.disc.params, out, cap);
      case 2: return put(p.gen.buffers, out, cap);
      case 3: return put(p.disc.buffers, out, cap);
      case 4: return put(p.last_grad_g, out, cap);
      case 5: return put(p.last_grad_d, out, cap);
      case 6: return put(p.opt_g.m, out, cap);
      case 7: return put(p.opt_g.v, out, cap);
      case 8: return put(p.opt_d.m, out, cap);
      case 9: return put(p.opt_d.v, out, cap);
      case 10: {
        std::vector<double> r;
        for (auto& s : k.reports) r.insert(r.end(), {s.j_d, s.j_g, s.d_real_mean, s.d_fake_mean});
        return put(r, out, cap);
      }
      case 11: {
        std::vector<double> r(k.last_batch.begin(), k.last_batch.end());
        return put(r, out, cap);
      }
      case 12: return put(std::vector<double>{double(p.opt_g.t), double(p.opt_d.t), double(p.steps)}, out, cap);
    }
    throw std::invalid_argument("unknown field code " + std::to_string(what));
  }

  void set(int l, int what, const double* in, long n) override {
    GanPair<R>& p = w.at(static_cast<size_t>(l))->pair;
    switch (what) {
      case 0: take(p.gen.params, in, n); return;
      case 1: take(p.disc.params, in, n); return;
      case 2: take(p.gen.buffers, in, n); return;
      case 3: take(p.disc.buffers, in, n); return;
      case 6: take(p.opt_g.m, in, n); return;
      case 7: take(p.opt_g.v, in, n); return;
      case 8: take(p.opt_d.m, in, n); return;
      case 9: take(p.opt_d.v, in, n); return;
      case 12:
        // Adam step counters {t_g, t_d, steps} (pg_group_set COUNTERS)
        if (n != 3) throw std::invalid_argument("length mismatch on set");
        p.opt_g.t = static_cast<long>(in[0]);
        p.opt_d.t = static_cast<long>(in[1]);
        p.steps = static_cast<long>(in[2]);
        return;
    }
    throw std::invalid_argument("field not settable: " + std::to_string(what));
  }

  void mixture(const double* priors, long n, uint64_t seed, double* out, int* ids) override {
    std::vector<const GanPair<R>*> pairs;
    for (auto& k : w) pairs.push_back(&k->pair);
    ClassPrior pri;
    pri.probabilities.assign(priors, priors + w.size());
    Rng rng(seed);
    auto ms = mixture_sample<R>(pairs, pri, n, rng);
    for (long i = 0; i < ms.first.size(); ++i) out[i] = static_cast<double>(ms.first[i]);
    for (long i = 0; i < n; ++i) ids[i] = ms.second[static_cast<size_t>(i)];
  }

  void step_inputs(int l, const double* real01, const double* z1, const double* z2, long B, double* rep) override {
    Worker<R>& k = *w.at(static_cast<size_t>(l));
    Shape img = k.cfg.image;
    Shape rs{B};
    rs.insert(rs.end(), img.begin(), img.end());
    Tensor<R> real(rs);
    for (long i = 0; i < real.size(); ++i) real[i] = static_cast<R>(real01[i]);
    long dz = k.pair.d_z;
    Tensor<R> a({B, dz}), b({B, dz});
    for (long i = 0; i < B * dz; ++i) {
      a[i] = static_cast<R>(z1[i]);
      b[i] = static_cast<R>(z2[i]);
    }
    int calls = 0;
    StepReport r;
    taped(static_cast<size_t>(l), [&] { r = step_core<R>(k.pair, real, [&]() { return calls++ == 0 ? a : b; }, k.rng); });
    k.reports.push_back(r);
    if (rep) {
      rep[0] = r.j_d;
      rep[1] = r.j_g;
      rep[2] = r.d_real_mean;
      rep[3] = r.d_fake_mean;
    }
  }
};

template <class R>
GroupBase* make_group(const Arch& a, int n_labels, int first_label, long per_label, uint64_t data_seed,
                      uint64_t base_seed, long batch, int epochs, double lr, int threads) {
  auto g = std::make_unique<Group<R>>();
  CosineSpec sp;
  sp.k = n_labels;
  sp.first_label = first_label;
  sp.per_label = per_label;
  sp.C = a.image[0];
  sp.H = a.image[1];
  sp.W = a.image[2];
  sp.seed = data_seed;
  // generate labels in parallel (each label owns its stream)
  g->ds.k = first_label + n_labels;
  g->ds.C = sp.C;
  g->ds.H = sp.H;
  g->ds.W = sp.W;
  g->ds.m = n_labels * per_label;
  long S = sp.C * sp.H * sp.W;
  g->ds.images.assign(static_cast<size_t>(g->ds.m * S), 0.0);
  g->ds.labels.resize(static_cast<size_t>(g->ds.m));
  {
    std::atomic<int> next{0};
    auto body = [&] {
      for (;;) {
        int l = next.fetch_add(1);
        if (l >= n_labels) break;
        cosine_label(sp, first_label + l, g->ds.images.data() + static_cast<long>(l) * per_label * S);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < std::max(1, std::min(threads, n_labels)); ++t) th.emplace_back(body);
    body();
    for (auto& t : th) t.join();
  }
  for (int l = 0; l < n_labels; ++l)
    for (long j = 0; j < per_label; ++j) g->ds.labels[static_cast<size_t>(l * per_label + j)] = first_label + l;
  for (int l = 0; l < n_labels; ++l) {
    WorkerConfig c;
    c.class_id = first_label + l;
    c.seed = derive_seed(base_seed, static_cast<uint64_t>(c.class_id));
    c.epochs = epochs;
    c.batch_size = batch;
    c.gen_arch = a.gen;
    c.disc_arch = a.disc;
    c.image = a.image;
    c.d_z = a.d_z;
    c.adam.lr = lr;
    ClassShard sh;
    sh.class_id = c.class_id;
    for (long j = 0; j < per_label; ++j) sh.indices.push_back(l * per_label + j);
    g->w.push_back(std::make_unique<Worker<R>>(c, sh));
  }
  return g.release();
}

template <class F>
int guard(F f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

// cfg 1..4 = BASELINE.json architectures; cfg 0 = custom (gen_spec/disc_spec/image).
void* or_group_create(int prec, int cfg, const char* gen_spec, const char* disc_spec, const char* image, long d_z,
                      int n_labels, int first_label, long per_label, uint64_t data_seed, uint64_t base_seed,
                      long batch, int epochs, double lr, int threads) {
  GroupBase* out = nullptr;
  int rc = guard([&] {
    Arch a;
    if (cfg >= 1) {
      a = baseline_arch(cfg, d_z);
    } else {
      a.gen = parse_layers(gen_spec);
      a.disc = parse_layers(disc_spec);
      a.image = parse_shape(image);
      a.d_z = d_z;
    }
    if (a.image.size() != 3) throw std::invalid_argument("image shape must be C H W");
    if (prec == 64)
      out = make_group<double>(a, n_labels, first_label, per_label, data_seed, base_seed, batch, epochs, lr, threads);
    else
      out = make_group<float>(a, n_labels, first_label, per_label, data_seed, base_seed, batch, epochs, lr, threads);
  });
  return rc == 0 ? out : nullptr;
}

int or_group_step(void* h, int n, int threads) {
  return guard([&] { static_cast<GroupBase*>(h)->step(n, threads); });
}

long or_group_get(void* h, int label_idx, int what, double* out, long cap) {
  long n = -1;
  if (guard([&] { n = static_cast<GroupBase*>(h)->get(label_idx, what, out, cap); }) != 0) return -1;
  return n;
}

int or_group_set(void* h, int label_idx, int what, const double* in, long n) {
  return guard([&] { static_cast<GroupBase*>(h)->set(label_idx, what, in, n); });
}

int or_group_step_inputs(void* h, int label_idx, const double* real01, const double* z1, const double* z2, long B,
                         double* report4) {
  return guard([&] { static_cast<GroupBase*>(h)->step_inputs(label_idx, real01, z1, z2, B, report4); });
}

// n samples [n][C][H][W] in [0,1] and their class indices (group label order)
int or_group_mixture(void* h, const double* priors, long n, uint64_t seed, double* out, int* ids) {
  return guard([&] { static_cast<GroupBase*>(h)->mixture(priors, n, seed, out, ids); });
}

void or_group_destroy(void* h) { delete static_cast<GroupBase*>(h); }

// Parity instrumentation: force the ReLU / LeakyReLU masks of label l's next
// step (bytes in the order the step evaluates them: G fwd z1, D fwd real,
// D fwd fake, G fwd z2, D fwd fake; each layer [B][C][H][W]); returns via
// or_group_mask_flips how many of them disagreed with the oracle's own sign test.
int or_group_set_masks(void* h, int label_idx, const uint8_t* masks, long n) {
  return guard([&] { static_cast<GroupBase*>(h)->set_masks(label_idx, masks, n); });
}
long or_group_mask_flips(void* h, int label_idx) { return static_cast<GroupBase*>(h)->mask_flips(label_idx); }
// record the label's next step's own masks (same order); read them with or_group_get_masks
int or_group_record_masks(void* h, int label_idx) {
  return guard([&] { static_cast<GroupBase*>(h)->record_masks(label_idx); });
}
long or_group_get_masks(void* h, int label_idx, uint8_t* out, long cap) {
  long n = -1;
  if (guard([&] { n = static_cast<GroupBase*>(h)->get_masks(label_idx, out, cap); }) != 0) return -1;
  return n;
}

// One label of the cosine-field dataset, [per_label][C][H][W] in [0,1].
int or_dataset_label(long C, long H, long W, int label, long per_label, uint64_t seed, double* out) {
  return guard([&] {
    CosineSpec sp;
    sp.C = C;
    sp.H = H;
    sp.W = W;
    sp.per_label = per_label;
    sp.seed = seed;
    cosine_label(sp, label, out);
  });
}

int or_derive_seed(uint64_t base, uint64_t stream, uint64_t* out) {
  *out = derive_seed(base, stream);
  return 0;
}

// partition_by_label: counts[k] and indices (concatenated by class).
int or_partition(const int* labels, long n, int k, long* counts, long* indices) {
  return guard([&] {
    auto sh = partition_by_label(std::vector<int>(labels, labels + n), k);
    long at = 0;
    for (auto& s : sh) {
      counts[s.class_id] = static_cast<long>(s.indices.size());
      for (long i : s.indices) indices[at++] = i;
    }
  });
}

// Per-layer-network forward/backward on the oracle (for kernel parity tests).
// x: [n][in_shape] f64; gy: [n][out_shape]; outputs y, gx, gparams (fresh).
int or_net_fwd_bwd(int prec, const char* spec, const char* in_shape, uint64_t seed, double init_std, int train,
                   long n, const double* x, const double* gy, double* params_out, double* y, double* gx,
                   double* gparams, double* buffers_out) {
  return guard([&] {
    auto run = [&](auto tag) {
      using R = decltype(tag);
      auto net = build_network<R>(parse_layers(spec), parse_shape(in_shape), seed, init_std);
      Shape xs{n};
      for (long d : net.in_shape()) xs.push_back(d);
      Tensor<R> xt(xs);
      for (long i = 0; i < xt.size(); ++i) xt[i] = static_cast<R>(x[i]);
      Rng r(0);
      if (params_out) {
        std::vector<R> pin(net.params.size());
        for (size_t i = 0; i < pin.size(); ++i) pin[i] = static_cast<R>(params_out[i]);
        net.params = pin;  // caller-provided parameters (NaN-free contract)
      }
      auto fw = forward(net, xt, train ? Mode::train : Mode::eval, r);
      for (long i = 0; i < fw.first.size(); ++i) y[i] = static_cast<double>(fw.first[i]);
      if (buffers_out)
        for (size_t i = 0; i < net.buffers.size(); ++i) buffers_out[i] = static_cast<double>(net.buffers[i]);
      if (gy) {
        Tensor<R> g(fw.first.shape);
        for (long i = 0; i < g.size(); ++i) g[i] = static_cast<R>(gy[i]);
        auto gr = backward(net, fw.second, g);
        for (long i = 0; i < gr.input.size(); ++i) gx[i] = static_cast<double>(gr.input[i]);
        for (size_t i = 0; i < gr.params.size(); ++i) gparams[i] = static_cast<double>(gr.params[i]);
      }
    };
    if (prec == 64) run(double{});
    else run(float{});
  });
}

// Number of params / buffers / output elements per sample for a spec.
int or_net_info(const char* spec, const char* in_shape, long* n_params, long* n_buffers, long* out_numel) {
  return guard([&] {
    auto net = build_network<double>(parse_layers(spec), parse_shape(in_shape), 1);
    *n_params = net.n_params();
    *n_buffers = static_cast<long>(net.buffers.size());
    *out_numel = shape_numel(net.out_shape_());
  });
}

// Initial parameters exactly as build_network draws them.
int or_net_init(const char* spec, const char* in_shape, uint64_t seed, double init_std, double* params) {
  return guard([&] {
    auto net = build_network<double>(parse_layers(spec), parse_shape(in_shape), seed, init_std);
    for (size_t i = 0; i < net.params.size(); ++i) params[i] = net.params[i];
  });
}

// CPU baseline: n_labels workers of config cfg, each runs `steps` train steps on
// a pool of `threads` threads (train_distributed semantics).  Returns wall
// seconds of the stepping only (dataset generation and init excluded).
double or_bench_steps(int cfg, int prec, int n_labels, long batch, int steps, int threads) {
  double secs = -1;
  guard([&] {
    Arch a = baseline_arch(cfg);
    std::unique_ptr<GroupBase> g(prec == 64 ? make_group<double>(a, n_labels, 0, batch * steps, 1, 2, batch, 1, 2e-4, threads)
                                            : make_group<float>(a, n_labels, 0, batch * steps, 1, 2, batch, 1, 2e-4, threads));
    auto t0 = std::chrono::steady_clock::now();
    g->step(steps, threads);
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}

}  // extern "C"
