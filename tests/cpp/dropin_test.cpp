// A C++ caller of the B200 library through include/partgan_b200.hpp (the
// reference-API mirror over pg_network.h / pg_trainer.h): the INTEGRATION.md §2
// loop plus ports of the reference's own unit tests for the API it mirrors
// (tests/test_optim.cpp, test_gan.cpp, test_partition.cpp, test_nn.cpp under
// /root/reference/proj), run on the GPU.  Test infrastructure: compiled by
// tests/test_cpp_dropin.py, prints one PASS / FAIL line per case and exits
// non-zero on any failure.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "partgan_b200.hpp"

using namespace partgan_b200;

static int g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("  check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);   \
      ok = false;                                                                \
    }                                                                            \
  } while (0)

template <class F>
static void run_case(const char* name, F f) {
  bool ok = true;
  try {
    f(ok);
  } catch (const std::exception& e) {
    std::printf("  exception: %s\n", e.what());
    ok = false;
  }
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", name);
  if (!ok) ++g_fail;
}

template <class E, class F>
static bool throws_with(F f, const std::string& substr) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()).find(substr) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

// BASELINE configs[0] (c1) layer lists in the reference's variant form
static std::vector<LayerSpec> c1_gen() {
  return {Dense{100, 128 * 7 * 7}, Reshape{{128, 7, 7}}, BatchNorm{128}, ReLU{}, ConvTranspose2d{128, 64, 4, 2, 1},
          BatchNorm{64},          ReLU{},               ConvTranspose2d{64, 1, 4, 2, 1}, Tanh{}};
}
static std::vector<LayerSpec> c1_disc() {
  return {Conv2d{1, 64, 4, 2, 1}, LeakyReLU{0.2}, Conv2d{64, 128, 4, 2, 1}, BatchNorm{128}, LeakyReLU{0.2},
          Reshape{{128 * 7 * 7}},  Dense{128 * 7 * 7, 1}, Sigmoid{}};
}

// k labels x per images of the cosine-field dataset, label-blocked
static Dataset cosine_dataset(int k, long per, uint64_t seed) {
  Dataset ds;
  ds.k = k;
  ds.images = Tensor(Shape{k * per, 1, 28, 28});
  const long S = 28 * 28;
  for (int c = 0; c < k; ++c) {
    std::vector<double> buf(static_cast<size_t>(per * S));
    if (pg_cosine_label(1, 28, 28, per, seed, c, buf.data()) != PG_OK) throw std::runtime_error(pg_last_error());
    std::copy(buf.begin(), buf.end(), ds.images.data().begin() + c * per * S);
    for (long j = 0; j < per; ++j) ds.labels.push_back(c);
  }
  return ds;
}

static WorkerConfig worker(int cls, uint64_t base, int epochs, long batch) {
  WorkerConfig w;
  w.class_id = cls;
  w.seed = derive_seed(base, static_cast<uint64_t>(cls));
  w.epochs = epochs;
  w.batch_size = batch;
  w.gen_arch = c1_gen();
  w.disc_arch = c1_disc();
  w.image_shape = {1, 28, 28};
  return w;
}

int main() {
  std::printf("devices: %d\n", pg_device_count());

  // ---- optim (tests/test_optim.cpp) ----
  run_case("adam: zero gradient leaves params, t advances [test_optim.cpp:29-37]", [](bool& ok) {
    AdamState s = AdamState::create(3, {});
    std::vector<double> p = {0.5, -1.25, 3.0}, before = p;
    adam_step(s, p, std::vector<double>(3, 0.0));
    CHECK(p == before);
    CHECK(s.t == 1);
  });
  run_case("adam: first step analytic value -lr [test_optim.cpp:39-48] (fp32 state: 1e-9 abs)", [](bool& ok) {
    AdamConfig cfg;
    AdamState s = AdamState::create(1, cfg);
    std::vector<double> p = {0.0}, g = {1.0};
    adam_step(s, p, g);
    CHECK(std::abs(p[0] + 2e-4) < 1e-9);
  });
  run_case("adam: five constant-gradient steps vs the scalar formula [test_optim.cpp:50-71] (fp32 state: 2e-6 abs)",
           [](bool& ok) {
             AdamConfig cfg;
             cfg.lr = 0.05;
             AdamState s = AdamState::create(2, cfg);
             std::vector<double> p = {1.0, -2.0}, g = {1.0, -0.3};
             double e[2] = {1.0, -2.0}, m[2] = {0, 0}, v[2] = {0, 0};
             for (int step = 1; step <= 5; ++step) {
               adam_step(s, p, g);
               for (int i = 0; i < 2; ++i) {
                 m[i] = 0.5 * m[i] + 0.5 * g[i];
                 v[i] = 0.999 * v[i] + 0.001 * g[i] * g[i];
                 const double c1 = 1 - std::pow(0.5, step), c2 = 1 - std::pow(0.999, step);
                 e[i] -= cfg.lr * (m[i] / c1) / (std::sqrt(v[i] / c2) + cfg.eps);
                 CHECK(std::abs(p[static_cast<size_t>(i)] - e[i]) < 2e-6);
               }
             }
             CHECK(s.t == 5);
           });
  run_case("adam: rejects bad inputs without touching state [test_optim.cpp:92-105]", [](bool& ok) {
    AdamState s = AdamState::create(2, {});
    std::vector<double> p = {1.0, 2.0};
    CHECK(throws_with<std::invalid_argument>([&] { adam_step(s, p, std::vector<double>(3, 0.0)); },
                                             "adam_step: length mismatch"));
    std::vector<double> bad = {1.0, std::nan("")};
    CHECK(throws_with<std::invalid_argument>([&] { adam_step(s, p, bad); }, "adam_step: non-finite gradient rejected"));
    CHECK(p[0] == 1.0 && p[1] == 2.0);
    CHECK(s.t == 0);
    CHECK(s.m[0] == 0.0 && s.m[1] == 0.0);
  });

  // ---- network (tests/test_nn.cpp) ----
  run_case("network: build/forward/backward shapes, counts, trace single-use [test_nn.cpp:136-180,320-336]",
           [](bool& ok) {
             Network d = build_network(c1_disc(), {1, 28, 28}, 5);
             CHECK(d.param_count() == 138817);
             CHECK(d.output_shape() == Shape{1});
             Rng rng(1);
             Tensor x(Shape{8, 1, 28, 28});
             for (auto& v : x.data()) v = rng.uniform() * 2 - 1;
             auto [y, tr] = forward(d, x, Mode::train, rng);
             CHECK(y.shape() == (Shape{8, 1}));
             for (double v : y.data()) CHECK(v > 0.0 && v < 1.0);
             Tensor gy = Tensor::constant({8, 1}, 1.0 / 8);
             Gradients g = backward(d, tr, gy);
             CHECK(static_cast<Index>(g.params.size()) == d.param_count());
             CHECK(g.input.shape() == x.shape());
             CHECK(throws_with<std::invalid_argument>([&] { backward(d, tr, gy); },
                                                      "trace already consumed by a previous backward call"));
             auto fw2 = forward(d, x, Mode::train, rng);
             CHECK(throws_with<std::invalid_argument>([&] { backward(d, fw2.second, Tensor::constant({4, 1}, 1.0)); },
                                                      "does not match network output"));
             Network other = build_network(c1_disc(), {1, 28, 28}, 5);
             auto fw3 = forward(d, x, Mode::train, rng);
             CHECK(throws_with<std::invalid_argument>([&] { backward(other, fw3.second, gy); },
                                                      "trace does not belong to this network"));
           });
  run_case("network: build_network init is the reference draw order (seeded twice = equal, weights ~N(0,0.02))",
           [](bool& ok) {
             Network a = build_network(c1_gen(), {100}, 9), b = build_network(c1_gen(), {100}, 9);
             auto pa = a.params(), pb = b.params();
             CHECK(pa == pb);
             CHECK(a.param_count() == 766017);
             double s2 = 0;
             for (int i = 0; i < 10000; ++i) s2 += pa[static_cast<size_t>(i)] * pa[static_cast<size_t>(i)];
             CHECK(std::abs(std::sqrt(s2 / 10000) - 0.02) < 0.002);
           });
  run_case("network: infer touches no state; eval forward uses running stats [test_nn.cpp:306-319]", [](bool& ok) {
    Network g = build_network(c1_gen(), {100}, 3);
    Rng rng(2);
    Tensor z(Shape{16, 100});
    for (auto& v : z.data()) v = rng.normal();
    auto b0 = g.buffers();
    Tensor a = infer(g, z), b = infer(g, z);
    CHECK(a.data() == b.data());
    CHECK(g.buffers() == b0);
    forward(g, z, Mode::train, rng);
    CHECK(g.buffers() != b0);  // running statistics moved
  });
  run_case("network: grad_check (central differences on device forwards) [test_nn.cpp:196-261]", [](bool& ok) {
    // a smooth net (tanh / sigmoid, no kinks for the finite differences to cross);
    // fp32 device forwards, so the step is 1e-2 instead of the f64 reference's 1e-5
    Network n = build_network({Dense{16, 12}, Tanh{}, Dense{12, 1}, Sigmoid{}}, {16}, 7, 0.3);
    Rng rng(4);
    Tensor x(Shape{6, 16});
    for (auto& v : x.data()) v = rng.normal();
    LossFn loss;
    loss.value = [](const Tensor& y) {
      double s = 0;
      for (double v : y.data()) s += v * v;
      return s;
    };
    loss.grad = [](const Tensor& y) {
      Tensor g(y.shape());
      for (Index i = 0; i < y.size(); ++i) g[i] = 2 * y[i];
      return g;
    };
    const double rel = grad_check(n, x, loss, 40, 1e-2, Mode::eval, rng);
    std::printf("  grad_check max rel %.3e\n", rel);
    CHECK(rel < 1e-2);
  });

  // ---- gan (tests/test_gan.cpp) ----
  run_case("gan: lr zero leaves parameters bitwise unchanged with finite losses [test_gan.cpp:211-222]", [](bool& ok) {
    AdamConfig cfg;
    cfg.lr = 0.0;
    GanPair pair = make_gan_pair(c1_gen(), c1_disc(), {1, 28, 28}, {100}, {0}, cfg, 11);
    auto g0 = pair.generator_params(), d0 = pair.discriminator_params();
    Rng rng(3);
    Tensor real = Tensor::constant({4, 1, 28, 28}, 0.7);
    StepReport rep = train_step(pair, real, std::nullopt, rng);
    CHECK(pair.generator_params() == g0);
    CHECK(pair.discriminator_params() == d0);
    CHECK(std::isfinite(rep.j_d) && std::isfinite(rep.j_g));
    CHECK(pair.steps() == 1);
  });
  run_case("gan: make_gan_pair validation messages [gan.cpp:27-52]", [](bool& ok) {
    CHECK(throws_with<std::invalid_argument>(
        [] { make_gan_pair(c1_gen(), c1_disc(), {1, 28, 28}, {100}, {0}, {}, 1, 0.02, 0.7); },
        "probability clamp must lie in (0, 0.5)"));
    auto g2 = c1_gen();
    g2[7] = ConvTranspose2d{64, 2, 4, 2, 1};
    CHECK(throws_with<std::invalid_argument>([&] { make_gan_pair(g2, c1_disc(), {1, 28, 28}, {100}, {0}, {}, 1); },
                                             "generator emits [2x28x28] but images are [1x28x28]"));
    CHECK(throws_with<std::invalid_argument>([] { make_gan_pair(c1_gen(), c1_disc(), {1, 28, 28}, {0}, {0}, {}, 1); },
                                             "latent dimension must be positive"));
  });
  run_case("gan: generate range and determinism; single-pair mixture equals generate [test_partition.cpp:196-210]",
           [](bool& ok) {
             GanPair pair = make_gan_pair(c1_gen(), c1_disc(), {1, 28, 28}, {100}, {0}, {}, 5);
             Rng r1(8), r2(8), r3(8);
             Tensor a = generate(pair, std::nullopt, 20, r1), b = generate(pair, std::nullopt, 20, r2);
             CHECK(a.data() == b.data());
             for (double v : a.data()) CHECK(v >= 0.0 && v <= 1.0);
             ClassPrior pri;
             pri.probabilities = {1.0};
             auto ms = mixture_sample({&pair}, pri, 20, r3);
             CHECK(ms.first.data() == a.data());
             for (int id : ms.second) CHECK(id == 0);
           });

  // ---- partition / coordinator (tests/test_partition.cpp) ----
  run_case("partition: stable shards, priors, error text [test_partition.cpp:47-82]", [](bool& ok) {
    auto sh = partition_by_label({2, 0, 1, 0, 2, 2}, 3);
    CHECK(sh[0].indices == (std::vector<Index>{1, 3}));
    CHECK(sh[2].indices == (std::vector<Index>{0, 4, 5}));
    auto pri = estimate_priors(sh);
    CHECK(std::abs(pri.probabilities[2] - 0.5) < 1e-15);
    CHECK(throws_with<std::invalid_argument>([] { partition_by_label({0, 0, 2}, 3); }, "class 1 has no samples"));
    CHECK(throws_with<std::out_of_range>([] { partition_by_label({0, 5}, 3); }, "label 5 at index 1"));
  });
  run_case("train_distributed: K=1 equals a hand-rolled single-GAN loop bitwise [test_partition.cpp:96-120]",
           [](bool& ok) {
             Dataset ds = cosine_dataset(1, 40, 3);
             auto shards = partition_by_label(ds.labels, 1);
             WorkerConfig cfg = worker(0, 123, 2, 16);  // 2 epochs of 16 + 16 + 8 (partial tail)
             TrainingRun run = train_distributed(ds, shards, {cfg}, 1);
             Rng rng(cfg.seed);
             GanPair pair = make_gan_pair(cfg.gen_arch, cfg.disc_arch, cfg.image_shape, cfg.latent, cfg.label, cfg.adam,
                                          cfg.seed, cfg.init_std, cfg.prob_clamp);
             std::vector<Index> order = shards[0].indices;
             for (int e = 0; e < cfg.epochs; ++e) {
               std::shuffle(order.begin(), order.end(), rng.engine());
               for (size_t at = 0; at < order.size(); at += static_cast<size_t>(cfg.batch_size)) {
                 const size_t end = std::min(order.size(), at + static_cast<size_t>(cfg.batch_size));
                 std::vector<Index> batch(order.begin() + static_cast<std::ptrdiff_t>(at),
                                          order.begin() + static_cast<std::ptrdiff_t>(end));
                 train_step(pair, ds.gather(batch), std::nullopt, rng);
               }
             }
             CHECK(run.workers[0].reports.size() == 6);
             CHECK(run.workers[0].pair.generator_params() == pair.generator_params());
             CHECK(run.workers[0].pair.discriminator_params() == pair.discriminator_params());
             CHECK(run.workers[0].pair.generator_buffers() == pair.generator_buffers());
           });
  run_case("train_distributed: 5 workers, config order, priors, per-worker reports; rerun bitwise "
           "[test_partition.cpp:122-162]",
           [](bool& ok) {
             Dataset ds = cosine_dataset(5, 32, 4);
             auto shards = partition_by_label(ds.labels, 5);
             std::vector<WorkerConfig> cfgs;
             for (int c : {3, 1, 4, 0, 2}) cfgs.push_back(worker(c, 77, 1, 16));
             std::vector<ClassShard> sh;
             for (int c : {3, 1, 4, 0, 2}) sh.push_back(shards[static_cast<size_t>(c)]);
             TrainingRun a = train_distributed(ds, sh, cfgs, 0);
             TrainingRun b = train_distributed(ds, sh, cfgs, 1);
             CHECK(a.workers.size() == 5);
             for (size_t i = 0; i < 5; ++i) {
               CHECK(a.workers[i].class_id == cfgs[i].class_id);
               CHECK(a.workers[i].reports.size() == 2);
               CHECK(a.workers[i].pair.generator_params() == b.workers[i].pair.generator_params());
               CHECK(a.workers[i].pair.discriminator_params() == b.workers[i].pair.discriminator_params());
             }
             CHECK(std::abs(a.priors.probabilities[0] - 0.2) < 1e-15);
             // a worker trained alone (its class's images as a 1-class dataset, same seed)
             // equals the same worker trained among others
             Dataset one;
             one.k = 1;
             one.images = ds.gather(sh[2].indices);
             one.labels.assign(sh[2].indices.size(), 0);
             WorkerConfig c = cfgs[2];
             c.class_id = 0;
             TrainingRun solo = train_distributed(one, partition_by_label(one.labels, 1), {c}, 1);
             CHECK(solo.workers[0].pair.generator_params() == a.workers[2].pair.generator_params());
             CHECK(solo.workers[0].pair.discriminator_params() == a.workers[2].pair.discriminator_params());
             // mixture over the trained pairs: ids in range, samples in [0, 1]
             std::vector<const GanPair*> pairs;
             for (auto& w : a.workers) pairs.push_back(&w.pair);
             ClassPrior pri;
             pri.probabilities = {0.2, 0.2, 0.2, 0.2, 0.2};
             Rng rng(5);
             auto ms = mixture_sample(pairs, pri, 30, rng);
             for (int id : ms.second) CHECK(id >= 0 && id < 5);
             for (double v : ms.first.data()) CHECK(v >= 0.0 && v <= 1.0);
           });
  run_case("train_distributed: shard/config count mismatch message [partition.cpp:119-123]", [](bool& ok) {
    Dataset ds = cosine_dataset(2, 8, 1);
    auto shards = partition_by_label(ds.labels, 2);
    CHECK(throws_with<std::invalid_argument>([&] { train_distributed(ds, shards, {worker(0, 1, 1, 8)}, 1); },
                                             "train_distributed: 2 shards but 1 worker configs"));
  });

  std::printf("%s: %d failed\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
