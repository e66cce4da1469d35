// oracle/kat.cpp — TEST INFRASTRUCTURE ONLY.  Pins the oracle against every
// known-answer test the reference ships for this path, re-run
// here on the restatement.  Each case names the reference test it ports
// (file:line under /root/reference/proj/tests).  Prints one "PASS name" /
// "FAIL name: detail" line per case; exit status = number of failures.
// tests/test_oracle_kat.py runs this binary.
#include "oracle.hpp"

#include <array>
#include <cstdio>
#include <iostream>
#include <map>
#include <memory>
#include <set>

using namespace oracle;

namespace {

int g_failures = 0;
std::string g_case;
int g_case_fail = 0;

#define CHECK(cond)                                                                              \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      if (!g_case_fail) std::printf("FAIL %s: %s (line %d)\n", g_case.c_str(), #cond, __LINE__); \
      g_case_fail++;                                                                             \
    }                                                                                            \
  } while (0)

template <class F>
bool throws(F f) {
  try {
    f();
  } catch (...) {
    return true;
  }
  return false;
}

template <class E, class F>
std::string throws_msg(F f) {
  try {
    f();
  } catch (const E& e) {
    return std::string("!") + e.what();
  } catch (...) {
    return "wrong-type";
  }
  return "";
}

void run(const std::string& name, const std::function<void()>& body) {
  g_case = name;
  g_case_fail = 0;
  try {
    body();
  } catch (const std::exception& e) {
    std::printf("FAIL %s: exception %s\n", name.c_str(), e.what());
    g_case_fail++;
  }
  if (g_case_fail) g_failures++;
  else std::printf("PASS %s\n", name.c_str());
}

using T = Tensor<double>;
using Net = Network<double>;

T rand_t(Shape s, Rng& r, double sc = 1.0) {
  T t(std::move(s));
  for (auto& v : t.data) v = r.normal() * sc;
  return t;
}
T off_kink(Shape s, Rng& r) {
  T t = rand_t(std::move(s), r, 0.6);
  for (auto& v : t.data) v += v >= 0 ? 0.1 : -0.1;
  return t;
}
LossFn<double> quad_loss() {
  LossFn<double> l;
  l.value = [](const T& y) {
    double s = 0;
    for (double v : y.data) s += v * v;
    return 0.5 * s / static_cast<double>(y.size());
  };
  l.grad = [](const T& y) {
    T g(y.shape);
    for (long i = 0; i < y.size(); ++i) g[i] = y[i] / static_cast<double>(y.size());
    return g;
  };
  return l;
}
LossFn<double> target_loss(const Shape& s, Rng& r) {
  auto tgt = std::make_shared<T>(rand_t(s, r));
  LossFn<double> l;
  l.value = [tgt](const T& y) {
    double s2 = 0;
    for (long i = 0; i < y.size(); ++i) s2 += (y[i] - (*tgt)[i]) * (y[i] - (*tgt)[i]);
    return 0.5 * s2 / static_cast<double>(y.size());
  };
  l.grad = [tgt](const T& y) {
    T g(y.shape);
    for (long i = 0; i < y.size(); ++i) g[i] = (y[i] - (*tgt)[i]) / static_cast<double>(y.size());
    return g;
  };
  return l;
}
bool kink_safe(const Net& net, const T& x) {
  Net w = net;
  Rng f(0);
  auto fw = forward(w, x, Mode::eval, f);
  for (size_t i = 0; i < net.layers.size(); ++i) {
    Kind k = net.layers[i].kind;
    if (k == Kind::ReLU || k == Kind::LeakyReLU)
      for (double v : fw.second.layers[i].input.data)
        if (std::abs(v) <= 0.02) return false;
  }
  return true;
}

// reference arch fixtures used by the ported tests (archs.cpp:5-111)
std::vector<Layer> gen_dense(long dz, const Shape& s, long h) {
  return {Layer::dense(dz, h), Layer::relu(), Layer::dense(h, shape_numel(s)), Layer::tanh_(), Layer::reshape(s)};
}
std::vector<Layer> disc_dense(const Shape& s, long h) {
  long f = shape_numel(s);
  return {Layer::reshape({f}), Layer::dense(f, h), Layer::lrelu(0.2), Layer::dropout(0.25), Layer::dense(h, 1),
          Layer::sigmoid()};
}
std::vector<Layer> disc_dc32(long c) {
  return {Layer::conv(c, 16, 3, 2, 1), Layer::lrelu(0.2), Layer::dropout(0.25), Layer::conv(16, 32, 3, 2, 1),
          Layer::lrelu(0.2), Layer::dropout(0.25), Layer::bn(32), Layer::conv(32, 64, 3, 2, 1), Layer::lrelu(0.2),
          Layer::dropout(0.25), Layer::bn(64), Layer::conv(64, 128, 3, 2, 1), Layer::lrelu(0.2), Layer::dropout(0.25),
          Layer::bn(128), Layer::reshape({512}), Layer::dense(512, 1), Layer::sigmoid()};
}

// gaussian_blobs_1d (data.cpp:54-118) as a test fixture
Dataset blobs(int k, long per, double sd, uint64_t seed) {
  std::vector<double> means;
  for (int j = 0; j < k; ++j) means.push_back(k == 1 ? 0.0 : -1.0 + 2.0 * j / (k - 1));
  double lo = *std::min_element(means.begin(), means.end()) - 5 * sd;
  double hi = *std::max_element(means.begin(), means.end()) + 5 * sd;
  Dataset ds;
  ds.k = k;
  ds.C = ds.H = ds.W = 1;
  ds.m = k * per;
  ds.images.resize(static_cast<size_t>(ds.m));
  ds.labels.resize(static_cast<size_t>(ds.m));
  Rng r(seed);
  long row = 0;
  for (int j = 0; j < k; ++j)
    for (long i = 0; i < per; ++i, ++row) {
      ds.labels[static_cast<size_t>(row)] = j;
      double x = means[static_cast<size_t>(j)] + sd * r.normal();
      ds.images[static_cast<size_t>(row)] = std::clamp((x - lo) / (hi - lo), 0.0, 1.0);
    }
  return ds;
}

WorkerConfig dense_worker(int cid, uint64_t seed, const Shape& s, int epochs, long batch, long dz = 2, long hid = 16,
                          double lr = 1e-3) {
  WorkerConfig w;
  w.class_id = cid;
  w.seed = seed;
  w.epochs = epochs;
  w.batch_size = batch;
  w.image = s;
  w.d_z = dz;
  w.adam.lr = lr;
  w.gen_arch = gen_dense(dz, s, hid);
  w.disc_arch = disc_dense(s, hid);
  return w;
}

GanPair<double> toy_pair(double lr, uint64_t seed) {
  AdamConfig a;
  a.lr = lr;
  return make_gan_pair<double>({Layer::dense(1, 1)}, {Layer::dense(1, 1), Layer::sigmoid()}, {1}, 1, 0, a, seed, 0.5);
}

struct ScalarAdam {
  double m = 0, v = 0;
  int t = 0;
  double lr, b1, b2, eps;
  double step(double p, double g) {
    t += 1;
    m = b1 * m + (1 - b1) * g;
    v = b2 * v + (1 - b2) * g * g;
    return p - lr * (m / (1 - std::pow(b1, t))) / (std::sqrt(v / (1 - std::pow(b2, t))) + eps);
  }
};

double sigm(double z) { return 1.0 / (1.0 + std::exp(-z)); }

// Direct (scatter) definition of ConvTranspose2d used to pin the fold-based
// restatement: y[co][ih*s-p+ki][iw*s-p+kj] += x[ci][ih][iw] * W[ci][co][ki][kj].
T convT_direct(const Layer& l, const std::vector<double>& p, const T& x) {
  long n = x.dim(0), H = x.dim(2), W = x.dim(3);
  long OH = (H - 1) * l.s - 2 * l.p + l.k, OW = (W - 1) * l.s - 2 * l.p + l.k;
  T y({n, l.out, OH, OW});
  for (long b = 0; b < n; ++b)
    for (long co = 0; co < l.out; ++co)
      for (long i = 0; i < OH * OW; ++i) y[(b * l.out + co) * OH * OW + i] = p[static_cast<size_t>(l.in * l.out * l.k * l.k + co)];
  for (long b = 0; b < n; ++b)
    for (long ci = 0; ci < l.in; ++ci)
      for (long ih = 0; ih < H; ++ih)
        for (long iw = 0; iw < W; ++iw)
          for (long co = 0; co < l.out; ++co)
            for (long ki = 0; ki < l.k; ++ki)
              for (long kj = 0; kj < l.k; ++kj) {
                long oy = ih * l.s - l.p + ki, ox = iw * l.s - l.p + kj;
                if (oy < 0 || oy >= OH || ox < 0 || ox >= OW) continue;
                y[((b * l.out + co) * OH + oy) * OW + ox] +=
                    x[((b * l.in + ci) * H + ih) * W + iw] * p[static_cast<size_t>(((ci * l.out + co) * l.k + ki) * l.k + kj)];
              }
  return y;
}

}  // namespace

int main() {
  // ---------------- test_optim.cpp ----------------
  run("optim.zero_grad_bitwise_unchanged [test_optim.cpp:29-37]", [] {
    auto s = AdamState<double>::create(3, {});
    std::vector<double> p{0.5, -1.25, 3.0}, b = p;
    adam_step(s, p, std::vector<double>(3, 0.0));
    CHECK(p == b);
    CHECK(s.t == 1);
  });
  run("optim.first_step_analytic [test_optim.cpp:39-48]", [] {
    AdamConfig c;
    auto s = AdamState<double>::create(1, c);
    std::vector<double> p{0.0};
    adam_step(s, p, {1.0});
    CHECK(std::abs(p[0] - (-2e-4)) <= 1e-7 * 2e-4 + 1e-18);
    CHECK(std::abs(std::abs(p[0]) - c.lr) < 1e-9);
  });
  run("optim.five_steps_scalar_oracle_1e-12 [test_optim.cpp:50-71]", [] {
    AdamConfig c;
    c.lr = 0.05;
    auto s = AdamState<double>::create(2, c);
    std::vector<double> p{1.0, -2.0}, g{1.0, -0.3};
    ScalarAdam o0{0, 0, 0, c.lr, c.beta1, c.beta2, c.eps}, o1 = o0;
    double e0 = p[0], e1 = p[1];
    for (int i = 0; i < 5; ++i) {
      adam_step(s, p, g);
      e0 = o0.step(e0, g[0]);
      e1 = o1.step(e1, g[1]);
      CHECK(std::abs(p[0] - e0) < 1e-12);
      CHECK(std::abs(p[1] - e1) < 1e-12);
    }
    CHECK(s.t == 5);
  });
  run("optim.first_step_magnitude_and_sign [test_optim.cpp:73-90]", [] {
    Rng r(99);
    for (int rep = 0; rep < 50; ++rep) {
      double g = r.normal();
      if (std::abs(g) < 1e-12) continue;
      AdamConfig c;
      auto s = AdamState<double>::create(1, c);
      std::vector<double> p{0.0};
      adam_step(s, p, {g});
      CHECK(std::abs(std::abs(p[0]) - c.lr * std::abs(g) / (std::abs(g) + c.eps)) < 1e-15);
      CHECK(p[0] * g < 0.0);
    }
  });
  run("optim.rejects_without_touching_state [test_optim.cpp:92-105]", [] {
    auto s = AdamState<double>::create(2, {});
    std::vector<double> p{1.0, 2.0};
    CHECK(throws([&] { adam_step(s, p, std::vector<double>(3, 0.0)); }));
    CHECK(throws([&] { adam_step(s, p, {1.0, std::nan("")}); }));
    CHECK(p[0] == 1.0 && p[1] == 2.0);
    CHECK(s.t == 0);
    CHECK(s.m[0] == 0 && s.m[1] == 0);
  });

  // ---------------- test_gan.cpp ----------------
  run("gan.conditional_latent_one_hot [test_gan.cpp:38-46]", [] {
    Rng r(5);
    T z = sample_latent<double>(100, 10, 3, 4, r);
    CHECK((z.shape == Shape{4, 110}));
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 10; ++j) CHECK(z[i * 110 + 100 + j] == (j == 3 ? 1.0 : 0.0));
  });
  run("gan.latent_deterministic_and_validated [test_gan.cpp:54-62]", [] {
    Rng a(42), b(42);
    T za = sample_latent<double>(5, 4, 2, 6, a), zb = sample_latent<double>(5, 4, 2, 6, b);
    CHECK(za.data == zb.data);
    Rng c(1);
    CHECK(throws_msg<std::out_of_range>([&] { sample_latent<double>(5, 4, 4, 1, c); })[0] == '!');
    CHECK(throws_msg<std::invalid_argument>([&] { sample_latent<double>(5, 4, std::nullopt, 1, c); })[0] == '!');
  });
  run("gan.discriminator_loss_analytic [test_gan.cpp:64-75]", [] {
    double c = 1e-7;
    T half({4, 1}, std::vector<double>(4, 0.5));
    CHECK(std::abs(discriminator_loss(half, half, c) - 0.6931471805599453) < 1e-14 * 0.7);
    T good({4, 1}, std::vector<double>(4, 1 - c)), bad({4, 1}, std::vector<double>(4, c));
    CHECK(std::abs(discriminator_loss(good, bad, c)) < 1e-6);
    T pr({1, 1}, {0.8}), pf({1, 1}, {0.3});
    CHECK(std::abs(discriminator_loss(pr, pf, c) - 0.2899092476264711) < 1e-13 * 0.3);
  });
  run("gan.generator_loss_analytic [test_gan.cpp:77-85]", [] {
    double c = 1e-7;
    CHECK(std::abs(generator_loss(T({2, 1}, {0.5, 0.5}), c) - (-0.34657359027997264)) < 1e-14 * 0.35);
    CHECK(std::abs(generator_loss(T({2, 1}, {1 - c, 1 - c}), c)) < 1e-6);
    CHECK(std::abs(generator_loss(T({1, 1}, {0.3}), c) - (-0.6019864021629681)) < 1e-13 * 0.61);
  });
  run("gan.losses_vs_scalar_reference [test_gan.cpp:87-110]", [] {
    Rng r(123);
    for (int rep = 0; rep < 30; ++rep) {
      double c = 0.02;
      long n = 1 + static_cast<long>(r.index(8));
      T pr({n, 1}), pf({n, 1});
      for (long i = 0; i < n; ++i) {
        pr[i] = r.uniform();
        pf[i] = r.uniform();
      }
      double sr = 0, sf = 0, sg = 0;
      for (long i = 0; i < n; ++i) {
        double cr = std::min(std::max(pr[i], c), 1 - c), cf = std::min(std::max(pf[i], c), 1 - c);
        sr += std::log(cr);
        sf += std::log(1 - cf);
        sg += std::log(cf);
      }
      CHECK(std::abs(discriminator_loss(pr, pf, c) - (-0.5 * sr / n - 0.5 * sf / n)) < 1e-12);
      CHECK(std::abs(generator_loss(pf, c) - 0.5 * sg / n) < 1e-12);
    }
  });
  run("gan.losses_reject_empty_and_stay_finite [test_gan.cpp:112-122]", [] {
    T empty, ok({1, 1}, {0.5});
    CHECK(throws([&] { discriminator_loss(empty, ok, 1e-7); }));
    CHECK(throws([&] { generator_loss(empty, 1e-7); }));
    T z({3, 1}, {0, 0, 0}), o({3, 1}, {1, 1, 1});
    CHECK(std::isfinite(discriminator_loss(z, o, 1e-7)));
    CHECK(std::isfinite(generator_loss(z, 1e-7)));
  });
  run("gan.loss_grads_vs_fd [test_gan.cpp:124-147]", [] {
    Rng r(7);
    double c = 1e-3;
    long n = 5;
    T p({n, 1});
    for (long i = 0; i < n; ++i) p[i] = 0.1 + 0.8 * r.uniform();
    T fixed({n, 1}, std::vector<double>(5, 0.6));
    T gr = loss_grad(p, c, 0), gf = loss_grad(p, c, 1), gg = loss_grad(p, c, 2);
    double h = 1e-6;
    for (long i = 0; i < n; ++i) {
      T up = p, dn = p;
      up[i] += h;
      dn[i] -= h;
      double fr = (discriminator_loss(up, fixed, c) - discriminator_loss(dn, fixed, c)) / (2 * h);
      double ff = (discriminator_loss(fixed, up, c) - discriminator_loss(fixed, dn, c)) / (2 * h);
      double fg = (-generator_loss(up, c) + generator_loss(dn, c)) / (2 * h);
      CHECK(std::abs(gr[i] - fr) <= 1e-6 * std::abs(fr) + 1e-9);
      CHECK(std::abs(gf[i] - ff) <= 1e-6 * std::abs(ff) + 1e-9);
      CHECK(std::abs(gg[i] - fg) <= 1e-6 * std::abs(fg) + 1e-9);
    }
  });
  run("gan.train_step_matches_scalar_simulation_1e-10 [test_gan.cpp:149-209]", [] {
    double lr = 0.01;
    auto pair = toy_pair(lr, 2024);
    double wg = pair.gen.params[0], bg = pair.gen.params[1], wd = pair.disc.params[0], bd = pair.disc.params[1];
    Rng peek(99);
    double z1[2] = {peek.normal(), peek.normal()};
    double z2[2] = {peek.normal(), peek.normal()};
    T real01({2, 1}, {0.9, 0.2});
    Rng rng(99);
    StepReport rep = train_step(pair, real01, std::nullopt, rng);
    double r[2] = {0.9 * 2 - 1, 0.2 * 2 - 1};
    double f[2] = {wg * z1[0] + bg, wg * z1[1] + bg};
    double pr[2] = {sigm(wd * r[0] + bd), sigm(wd * r[1] + bd)};
    double pf[2] = {sigm(wd * f[0] + bd), sigm(wd * f[1] + bd)};
    double jd = -.25 * (std::log(pr[0]) + std::log(pr[1])) - .25 * (std::log(1 - pf[0]) + std::log(1 - pf[1]));
    double gwd = 0, gbd = 0;
    for (int i = 0; i < 2; ++i) {
      double dz = (-0.25 / pr[i]) * pr[i] * (1 - pr[i]);
      gwd += dz * r[i];
      gbd += dz;
    }
    for (int i = 0; i < 2; ++i) {
      double dz = (0.25 / (1 - pf[i])) * pf[i] * (1 - pf[i]);
      gwd += dz * f[i];
      gbd += dz;
    }
    ScalarAdam awd{0, 0, 0, lr, 0.5, 0.999, 1e-8}, abd = awd, awg = awd, abg = awd;
    double wd2 = awd.step(wd, gwd), bd2 = abd.step(bd, gbd);
    double f2[2] = {wg * z2[0] + bg, wg * z2[1] + bg};
    double p2[2] = {sigm(wd2 * f2[0] + bd2), sigm(wd2 * f2[1] + bd2)};
    double jg = .25 * (std::log(p2[0]) + std::log(p2[1]));
    double gwg = 0, gbg = 0;
    for (int i = 0; i < 2; ++i) {
      double dz = (-0.25 / p2[i]) * p2[i] * (1 - p2[i]);
      gwg += dz * wd2 * z2[i];
      gbg += dz * wd2;
    }
    double wg2 = awg.step(wg, gwg), bg2 = abg.step(bg, gbg);
    CHECK(std::abs(pair.disc.params[0] - wd2) < 1e-10);
    CHECK(std::abs(pair.disc.params[1] - bd2) < 1e-10);
    CHECK(std::abs(pair.gen.params[0] - wg2) < 1e-10);
    CHECK(std::abs(pair.gen.params[1] - bg2) < 1e-10);
    CHECK(std::abs(rep.j_d - jd) < 1e-10);
    CHECK(std::abs(rep.j_g - jg) < 1e-10);
    CHECK(std::abs(rep.d_real_mean - 0.5 * (pr[0] + pr[1])) < 1e-10);
    CHECK(std::abs(rep.d_fake_mean - 0.5 * (pf[0] + pf[1])) < 1e-10);
  });
  run("gan.lr_zero_bitwise [test_gan.cpp:211-222]", [] {
    auto pair = toy_pair(0.0, 11);
    auto g0 = pair.gen.params, d0 = pair.disc.params;
    Rng r(3);
    StepReport rep = train_step(pair, T({4, 1}, std::vector<double>(4, 0.7)), std::nullopt, r);
    CHECK(pair.gen.params == g0);
    CHECK(pair.disc.params == d0);
    CHECK(std::isfinite(rep.j_d) && std::isfinite(rep.j_g));
  });
  run("gan.parameter_isolation [test_gan.cpp:224-246]", [] {
    for (int frozen = 0; frozen < 2; ++frozen) {
      auto pair = toy_pair(0.05, 17);
      if (frozen == 0) pair.opt_d.lr = 0.0;
      else pair.opt_g.lr = 0.0;
      auto g0 = pair.gen.params, d0 = pair.disc.params;
      Rng r(19);
      train_step(pair, T({4, 1}, std::vector<double>(4, 0.8)), std::nullopt, r);
      if (frozen == 0) {
        CHECK(pair.disc.params == d0);
        CHECK(pair.gen.params != g0);
      } else {
        CHECK(pair.gen.params == g0);
        CHECK(pair.disc.params != d0);
      }
    }
  });
  run("gan.generator_objective_fd_through_DoG [test_gan.cpp:248-298]", [] {
    std::vector<Layer> gen = {Layer::dense(4, 16), Layer::relu(), Layer::reshape({4, 2, 2}), Layer::bn(4),
                              Layer::upsample(2), Layer::conv(4, 1, 3, 1, 1), Layer::tanh_()};
    std::vector<Layer> disc = {Layer::conv(1, 2, 3, 2, 1), Layer::lrelu(0.2), Layer::dropout(0.25),
                               Layer::reshape({8}), Layer::dense(8, 1), Layer::sigmoid()};
    auto pair = make_gan_pair<double>(gen, disc, {1, 4, 4}, 4, 0, AdamConfig{}, 31, 0.3);
    double c = pair.clamp;
    long n = 6;
    std::vector<double> ana;
    {
      Rng r(77);
      T z = sample_latent<double>(4, 0, std::nullopt, n, r);
      auto fg = forward(pair.gen, z, Mode::train, r);
      auto fd = forward(pair.disc, fg.first, Mode::train, r);
      auto gd = backward(pair.disc, fd.second, loss_grad(fd.first, c, 2));
      ana = backward(pair.gen, fg.second, gd.input).params;
    }
    auto loss_at = [&]() {
      Rng r(77);
      T z = sample_latent<double>(4, 0, std::nullopt, n, r);
      T fake = forward(pair.gen, z, Mode::train, r).first;
      T p = forward(pair.disc, fake, Mode::train, r).first;
      return -generator_loss(p, c);
    };
    Rng cr(5);
    double worst = 0;
    for (int rep = 0; rep < 100; ++rep) {
      long ci = static_cast<long>(cr.index(static_cast<size_t>(pair.gen.n_params())));
      double sv = pair.gen.params[ci], h = 1e-3;
      pair.gen.params[ci] = sv + h;
      double fp = loss_at();
      pair.gen.params[ci] = sv - h;
      double fm = loss_at();
      pair.gen.params[ci] = sv;
      double num = (fp - fm) / (2 * h);
      worst = std::max(worst, std::abs(ana[ci] - num) / std::max({std::abs(ana[ci]), std::abs(num), 1e-8}));
    }
    CHECK(worst < 1e-4);
  });
  run("gan.generate_unit_interval_deterministic [test_gan.cpp:300-315]", [] {
    auto pair = make_gan_pair<double>({Layer::dense(3, 8), Layer::tanh_(), Layer::dense(8, 2), Layer::tanh_(),
                                       Layer::reshape({2})},
                                      {Layer::reshape({2}), Layer::dense(2, 1), Layer::sigmoid()}, {2}, 3, 0,
                                      AdamConfig{}, 3, 0.5);
    Rng a(8), b(8);
    T s1 = generate(pair, std::nullopt, 1000, a), s2 = generate(pair, std::nullopt, 1000, b);
    bool in01 = true;
    double mean = 0;
    for (double v : s1.data) {
      in01 = in01 && v >= 0 && v <= 1;
      mean += v;
    }
    mean /= static_cast<double>(s1.size());
    double var = 0;
    for (double v : s1.data) var += (v - mean) * (v - mean);
    CHECK(in01);
    CHECK(s1.data == s2.data);
    CHECK(var > 0);
  });
  run("gan.generator_width_must_match [test_gan.cpp:317-322]", [] {
    CHECK(throws([] {
      make_gan_pair<double>({Layer::dense(5, 2), Layer::tanh_(), Layer::reshape({2})},
                            {Layer::reshape({2}), Layer::dense(2, 1), Layer::sigmoid()}, {2}, 5, 3, AdamConfig{}, 1);
    }));
  });

  // ---------------- test_nn.cpp ----------------
  run("nn.tensor_basics [test_nn.cpp:70-77]", [] {
    T t({2, 3});
    CHECK(t.size() == 6);
    CHECK(throws([] { T bad({2, 0}); }));
  });
  run("nn.build_rejects_empty_and_incompatible [test_nn.cpp:79-91]", [] {
    CHECK(throws_msg<std::invalid_argument>([] { build_network<double>({}, {4}, 1); }) == "!network spec list is empty");
    std::string m = throws_msg<std::invalid_argument>([] {
      build_network<double>({Layer::dense(4, 8), Layer::dense(4, 2)}, {4}, 1);
    });
    CHECK(m.find("layer 1") != std::string::npos && m.find("dense") != std::string::npos);
  });
  run("nn.build_deterministic_per_seed [test_nn.cpp:93-100]", [] {
    auto sp = [] { return std::vector<Layer>{Layer::dense(6, 5), Layer::relu(), Layer::dense(5, 2)}; };
    auto a = build_network<double>(sp(), {6}, 42), b = build_network<double>(sp(), {6}, 42),
         c = build_network<double>(sp(), {6}, 43);
    CHECK(a.params == b.params);
    CHECK(a.params != c.params);
  });
  run("nn.conv_shape_algebra_dc32 [test_nn.cpp:113-121]", [] {
    auto d = build_network<double>(disc_dc32(3), {3, 32, 32}, 7);
    CHECK((d.shapes[1] == Shape{16, 16, 16}));
    CHECK((d.shapes[4] == Shape{32, 8, 8}));
    CHECK((d.shapes[8] == Shape{64, 4, 4}));
    CHECK((d.shapes[12] == Shape{128, 2, 2}));
    CHECK((d.out_shape_() == Shape{1}));
  });
  run("nn.dense_identity [test_nn.cpp:136-144]", [] {
    auto net = build_network<double>({Layer::dense(3, 3)}, {3}, 1);
    std::fill(net.params.begin(), net.params.end(), 0.0);
    for (int i = 0; i < 3; ++i) net.params[static_cast<size_t>(i * 3 + i)] = 1.0;
    Rng r(1);
    T x = rand_t({4, 3}, r);
    CHECK(infer(net, x).data == x.data);
  });
  run("nn.activations_at_zero [test_nn.cpp:146-152]", [] {
    auto s = build_network<double>({Layer::sigmoid()}, {1}, 1);
    auto t = build_network<double>({Layer::tanh_()}, {1}, 1);
    T z({1, 1});
    CHECK(std::abs(infer(s, z)[0] - 0.5) < 1e-15);
    CHECK(std::abs(infer(t, z)[0]) < 1e-15);
  });
  run("nn.conv_stride2_halves [test_nn.cpp:154-157]", [] {
    auto net = build_network<double>({Layer::conv(1, 4, 3, 2, 1)}, {1, 32, 32}, 1);
    CHECK((net.out_shape_() == Shape{4, 16, 16}));
  });
  run("nn.single_dense_grad_equals_input [test_nn.cpp:159-170]", [] {
    auto net = build_network<double>({Layer::dense(3, 1)}, {3}, 1);
    Rng r(2), f(0);
    T x = rand_t({1, 3}, r);
    auto fw = forward(net, x, Mode::eval, f);
    auto g = backward(net, fw.second, T({1, 1}, {1.0}));
    for (int i = 0; i < 3; ++i) CHECK(std::abs(g.params[static_cast<size_t>(i)] - x[i]) <= 1e-15 * std::abs(x[i]));
    CHECK(g.params[3] == 1.0);
  });
  run("nn.lrelu_negative_slope_grad [test_nn.cpp:172-180]", [] {
    auto net = build_network<double>({Layer::lrelu(0.2)}, {1}, 1);
    Rng f(0);
    auto fw = forward(net, T({1, 1}, {-2.0}), Mode::eval, f);
    CHECK(std::abs(fw.first[0] + 0.4) < 1e-12);
    auto g = backward(net, fw.second, T({1, 1}, {1.0}));
    CHECK(std::abs(g.input[0] - 0.2) < 1e-15);
  });
  run("nn.trace_misuse_rejected [test_nn.cpp:182-194]", [] {
    auto net = build_network<double>({Layer::dense(2, 2)}, {2}, 1);
    auto other = build_network<double>({Layer::dense(2, 2)}, {2}, 1);
    Rng r(1), f(0);
    T x = rand_t({1, 2}, r);
    auto fw = forward(net, x, Mode::eval, f);
    CHECK(throws([&] { backward(other, fw.second, fw.first); }));
    backward(net, fw.second, fw.first);
    CHECK(throws_msg<std::invalid_argument>([&] { backward(net, fw.second, fw.first); }) ==
          "!trace already consumed by a previous backward call");
  });
  run("nn.fd_property_every_layer_type_incl_convT [test_nn.cpp:196-250]", [] {
    Rng rng(123);
    struct Case {
      std::vector<Layer> layers;
      Shape in;
      Mode mode;
    };
    std::vector<Case> cases = {
        {{Layer::dense(5, 4)}, {5}, Mode::eval},
        {{Layer::conv(2, 3, 3, 1, 1)}, {2, 5, 5}, Mode::eval},
        {{Layer::conv(2, 3, 3, 2, 1)}, {2, 6, 6}, Mode::eval},
        {{Layer::conv(1, 2, 2, 1, 0)}, {1, 4, 4}, Mode::eval},
        {{Layer::dense(4, 6), Layer::bn(6), Layer::dense(6, 2)}, {4}, Mode::eval},
        {{Layer::conv(2, 4, 3, 1, 1), Layer::bn(4)}, {2, 4, 4}, Mode::train},
        {{Layer::dense(4, 6), Layer::reshape({6, 1, 1}), Layer::bn(6), Layer::reshape({6})}, {4}, Mode::train},
        {{Layer::dense(3, 8), Layer::reshape({2, 2, 2}), Layer::upsample(2), Layer::conv(2, 1, 3, 1, 1)}, {3}, Mode::eval},
        {{Layer::dense(4, 4), Layer::relu(), Layer::dense(4, 2)}, {4}, Mode::eval},
        {{Layer::dense(4, 4), Layer::lrelu(0.2), Layer::dense(4, 2)}, {4}, Mode::eval},
        {{Layer::dense(4, 4), Layer::tanh_(), Layer::dense(4, 2)}, {4}, Mode::eval},
        {{Layer::dense(4, 4), Layer::sigmoid(), Layer::dense(4, 2)}, {4}, Mode::eval},
        {{Layer::dense(4, 6), Layer::dropout(0.25), Layer::dense(6, 2)}, {4}, Mode::eval},
        {{Layer::reshape({2, 2}), Layer::reshape({4}), Layer::dense(4, 2)}, {4}, Mode::eval},
        // new: ConvTranspose2d in the k4 s2 p1 and odd geometries
        {{Layer::convT(2, 3, 4, 2, 1)}, {2, 3, 3}, Mode::eval},
        {{Layer::convT(3, 2, 3, 2, 1)}, {3, 3, 3}, Mode::eval},
        {{Layer::convT(2, 2, 3, 1, 1)}, {2, 4, 4}, Mode::eval},
        {{Layer::convT(2, 4, 4, 2, 1), Layer::bn(4)}, {2, 2, 2}, Mode::train},
    };
    int total = 0;
    for (size_t ci = 0; ci < cases.size(); ++ci) {
      for (int rep = 0; rep < 8; ++rep) {
        long batch = 8 + static_cast<long>(rng.index(4));
        Shape in = cases[ci].in;
        in.insert(in.begin(), batch);
        bool checked = false;
        for (uint64_t nt = 0; nt < 10 && !checked; ++nt) {
          auto net = build_network<double>(cases[ci].layers, cases[ci].in,
                                           derive_seed(9, static_cast<uint64_t>(ci * 100 + rep) + 7919 * nt), 0.3);
          for (int it = 0; it < 20 && !checked; ++it) {
            T x = off_kink(in, rng);
            if (!kink_safe(net, x)) continue;
            Shape out = net.out_shape_();
            out.insert(out.begin(), batch);
            double err = grad_check(net, x, target_loss(out, rng), 12, 1e-3, cases[ci].mode, rng);
            if (!(err < 1e-4)) std::printf("  case %zu rep %d err %.3e\n", ci, rep, err);
            CHECK(err < 1e-4);
            total += 12;
            checked = true;
          }
        }
        CHECK(checked);
      }
    }
    CHECK(total >= 100);
  });
  run("nn.full_dc32_disc_fd [test_nn.cpp:252-261]", [] {
    auto d = build_network<double>(disc_dc32(3), {3, 32, 32}, 21, 0.1);
    Rng r(77);
    T x = rand_t({2, 3, 32, 32}, r, 0.5);
    CHECK(grad_check(d, x, quad_loss(), 100, 1e-3, Mode::eval, r) < 1e-4);
  });
  run("nn.grad_check_dense_near_exact [test_nn.cpp:263-269]", [] {
    auto net = build_network<double>({Layer::dense(6, 4), Layer::dense(4, 3)}, {6}, 5);
    Rng r(11);
    T x = rand_t({3, 6}, r);
    CHECK(grad_check(net, x, quad_loss(), 1000, 1e-3, Mode::eval, r) < 1e-6);
  });
  run("nn.grad_check_edge_cases [test_nn.cpp:271-280]", [] {
    Rng r(3);
    auto np = build_network<double>({Layer::relu(), Layer::tanh_()}, {4}, 1);
    T x = rand_t({2, 4}, r);
    CHECK(grad_check(np, x, quad_loss(), 10, 1e-3, Mode::eval, r) == 0.0);
    auto wd = build_network<double>({Layer::dense(4, 4), Layer::dropout(0.5)}, {4}, 1);
    CHECK(throws([&] { grad_check(wd, x, quad_loss(), 10, 1e-3, Mode::train, r); }));
  });
  run("nn.bn_train_output_mean_var_1e-10 [test_nn.cpp:282-304]", [] {
    auto net = build_network<double>({Layer::bn(3, 1e-12, 0.1)}, {3}, 1);
    net.params = {2.5, -1.5, 0.5, 0.7, 0.0, -2.0};
    Rng r(5), f(0);
    T x = rand_t({64, 3}, r, 3.0);
    T y = forward(net, x, Mode::train, f).first;
    for (int c = 0; c < 3; ++c) {
      double mean = 0, var = 0;
      for (int i = 0; i < 64; ++i) mean += y[i * 3 + c];
      mean /= 64;
      for (int i = 0; i < 64; ++i) var += (y[i * 3 + c] - mean) * (y[i * 3 + c] - mean);
      var /= 64;
      CHECK(std::abs(mean - net.params[static_cast<size_t>(3 + c)]) < 1e-10);
      CHECK(std::abs(var - net.params[static_cast<size_t>(c)] * net.params[static_cast<size_t>(c)]) < 1e-10);
    }
  });
  run("nn.bn_eval_uses_running_stats [test_nn.cpp:306-319]", [] {
    auto net = build_network<double>({Layer::dense(2, 4), Layer::bn(4), Layer::dropout(0.5)}, {2}, 8);
    Rng r(6), f(1);
    T x = rand_t({16, 2}, r);
    auto b0 = net.buffers;
    forward(net, x, Mode::train, f);
    CHECK(net.buffers != b0);
    auto b1 = net.buffers;
    T a = infer(net, x), b = infer(net, x);
    CHECK(net.buffers == b1);
    CHECK(a.data == b.data);
  });
  run("nn.dropout_mask_algebra [test_nn.cpp:321-336]", [] {
    auto net = build_network<double>({Layer::dropout(0.25)}, {8}, 1);
    Rng f(42), r(9);
    T x = off_kink({4, 8}, r);
    auto fw = forward(net, x, Mode::train, f);
    auto g = backward(net, fw.second, T({4, 8}, std::vector<double>(32, 1.0)));
    int dropped = 0;
    for (long i = 0; i < 32; ++i) {
      double m = fw.first[i] / x[i];
      CHECK((std::abs(m) < 1e-12 || std::abs(m - 1.0 / 0.75) < 1e-12));
      CHECK(std::abs(g.input[i] - m) < 1e-12);
      if (std::abs(m) < 1e-12) ++dropped;
    }
    CHECK(dropped > 0);
  });
  run("nn.eval_bitwise_deterministic_across_threads [test_nn.cpp:338-351]", [] {
    auto net = build_network<double>({Layer::conv(1, 8, 3, 2, 1), Layer::lrelu(0.2), Layer::reshape({512}),
                                      Layer::dense(512, 1), Layer::sigmoid()},
                                     {1, 16, 16}, 33);
    Rng r(4);
    T x = rand_t({3, 1, 16, 16}, r);
    T base = infer(net, x);
    std::vector<std::vector<double>> res(4);
    std::vector<std::thread> th;
    for (int t = 0; t < 4; ++t) th.emplace_back([&, t] { res[static_cast<size_t>(t)] = infer(net, x).data; });
    for (auto& t : th) t.join();
    for (auto& v : res) CHECK(v == base.data);
  });
  run("nn.forward_backward_finite_on_random_nets [test_nn.cpp:353-369]", [] {
    Rng r(1234);
    for (int rep = 0; rep < 20; ++rep) {
      auto net = build_network<double>({Layer::dense(6, 12), Layer::lrelu(0.2), Layer::reshape({3, 2, 2}), Layer::bn(3),
                                        Layer::upsample(2), Layer::conv(3, 2, 3, 1, 1), Layer::tanh_(),
                                        Layer::reshape({32}), Layer::dense(32, 1), Layer::sigmoid()},
                                       {6}, derive_seed(55, static_cast<uint64_t>(rep)), 0.5);
      T x = rand_t({4, 6}, r, 2.0);
      Rng f(7);
      auto fw = forward(net, x, Mode::train, f);
      CHECK(fw.first.finite());
      auto g = backward(net, fw.second, T({4, 1}, std::vector<double>(4, 1.0)));
      bool ok = true;
      for (double v : g.params) ok = ok && std::isfinite(v);
      CHECK(ok);
      CHECK(g.input.finite());
    }
  });
  run("nn.batch_shape_mismatch_rejected [test_nn.cpp:371-375]", [] {
    auto net = build_network<double>({Layer::dense(3, 2)}, {3}, 1);
    Rng r(1);
    T bad = rand_t({2, 4}, r);
    CHECK(throws([&] { infer(net, bad); }));
  });
  // new pins for the BASELINE additions
  run("new.convT_fold_equals_direct_scatter", [] {
    Rng r(17);
    for (auto geo : {std::array<long, 5>{3, 5, 4, 2, 1}, {2, 3, 3, 2, 1}, {4, 2, 3, 1, 0}, {2, 2, 5, 3, 2}}) {
      Layer l = Layer::convT(geo[0], geo[1], geo[2], geo[3], geo[4]);
      auto net = build_network<double>({l}, {geo[0], 4, 5}, 3, 0.5);
      for (long c = 0; c < geo[1]; ++c) net.params[net.params.size() - static_cast<size_t>(geo[1]) + static_cast<size_t>(c)] = 0.1 * static_cast<double>(c + 1);
      T x = rand_t({2, geo[0], 4, 5}, r);
      T y = infer(net, x), d = convT_direct(l, net.params, x);
      CHECK(y.shape == d.shape);
      double worst = 0;
      for (long i = 0; i < y.size(); ++i) worst = std::max(worst, std::abs(y[i] - d[i]));
      CHECK(worst < 1e-12);
    }
  });
  run("new.baseline_arch_param_counts [SURVEY 8a a3]", [] {
    long want[5][2] = {{0, 0}, {766017, 138817}, {1073219, 663745}, {1073219, 663745}, {3585347, 2766529}};
    for (int c = 1; c <= 4; ++c) {
      Arch a = baseline_arch(c);
      auto g = build_network<double>(a.gen, {a.d_z}, 1);
      auto d = build_network<double>(a.disc, a.image, 2);
      CHECK(g.n_params() == want[c][0]);
      CHECK(d.n_params() == want[c][1]);
      CHECK(g.out_shape_() == a.image);
      CHECK((d.out_shape_() == Shape{1}));
    }
  });
  run("new.cosine_dataset_bounds_determinism", [] {
    CosineSpec sp;
    sp.k = 3;
    sp.per_label = 5;
    sp.C = 3;
    sp.H = sp.W = 16;
    sp.seed = 7;
    Dataset a = make_cosine_dataset(sp), b = make_cosine_dataset(sp);
    CHECK(a.images == b.images);
    bool in01 = true;
    for (double v : a.images) in01 = in01 && v >= 0.0 && v <= 1.0;
    CHECK(in01);
    CHECK(a.labels[0] == 0 && a.labels[5] == 1 && a.labels[14] == 2);
    // a label's field is independent of which other labels are generated
    CosineSpec one = sp;
    one.k = 1;
    one.first_label = 2;
    Dataset c = make_cosine_dataset(one);
    CHECK(std::equal(c.images.begin(), c.images.end(), a.images.begin() + 10 * 768));
  });

  // ---------------- test_partition.cpp ----------------
  run("partition.basic_examples [test_partition.cpp:47-60]", [] {
    auto sh = partition_by_label({0, 1, 0, 1}, 2);
    CHECK(sh.size() == 2);
    CHECK((sh[0].indices == std::vector<long>{0, 2}));
    CHECK((sh[1].indices == std::vector<long>{1, 3}));
    CHECK((partition_by_label({0, 0, 0}, 1)[0].indices == std::vector<long>{0, 1, 2}));
    CHECK(throws_msg<std::out_of_range>([] { partition_by_label({0, 3}, 2); })[0] == '!');
    CHECK(throws_msg<std::invalid_argument>([] { partition_by_label({0, 0}, 2); }).find("class 1 has no samples") !=
          std::string::npos);
  });
  run("partition.disjoint_covering_10k [test_partition.cpp:62-82]", [] {
    Rng r(42);
    std::vector<int> labels(10000);
    std::vector<long> cnt(10, 0);
    for (auto& l : labels) {
      l = static_cast<int>(r.index(10));
      cnt[static_cast<size_t>(l)]++;
    }
    auto sh = partition_by_label(labels, 10);
    std::set<long> seen;
    long tot = 0;
    for (auto& s : sh) {
      CHECK(static_cast<long>(s.indices.size()) == cnt[static_cast<size_t>(s.class_id)]);
      for (long i : s.indices) {
        CHECK(seen.insert(i).second);
        CHECK(labels[static_cast<size_t>(i)] == s.class_id);
      }
      tot += static_cast<long>(s.indices.size());
    }
    CHECK(tot == 10000);
  });
  run("partition.priors_proportional [test_partition.cpp:84-94]", [] {
    auto p = estimate_priors(partition_by_label({0, 0, 0, 0, 0, 1, 1, 1, 1, 1}, 2));
    CHECK(std::abs(p.probabilities[0] - 0.5) < 1e-15);
    auto q = estimate_priors(partition_by_label({0, 1, 1, 1}, 2));
    CHECK(std::abs(q.probabilities[0] - 0.25) < 1e-15);
    CHECK(std::abs(q.probabilities[1] - 0.75) < 1e-15);
  });
  run("partition.K1_equals_hand_rolled_loop_bitwise [test_partition.cpp:96-120]", [] {
    Dataset ds = blobs(1, 64, 0.05, 7);
    auto sh = partition_by_label(ds.labels, 1);
    WorkerConfig cfg = dense_worker(0, derive_seed(123, 0), ds.sample_shape(), 3, 16);
    auto run1 = train_distributed<double>(ds, sh, {cfg}, 1);
    Rng rng(cfg.seed);
    auto pair = make_gan_pair<double>(cfg.gen_arch, cfg.disc_arch, cfg.image, cfg.d_z, cfg.d_y, cfg.adam, cfg.seed,
                                      cfg.init_std, cfg.clamp);
    std::vector<long> order = sh[0].indices;
    for (int e = 0; e < cfg.epochs; ++e) {
      std::shuffle(order.begin(), order.end(), rng.engine());
      for (size_t at = 0; at < order.size(); at += static_cast<size_t>(cfg.batch_size)) {
        size_t end = std::min(order.size(), at + static_cast<size_t>(cfg.batch_size));
        std::vector<long> b(order.begin() + static_cast<long>(at), order.begin() + static_cast<long>(end));
        train_step(pair, ds.gather<double>(b), std::nullopt, rng);
      }
    }
    CHECK(run1.workers[0].pair.gen.params == pair.gen.params);
    CHECK(run1.workers[0].pair.disc.params == pair.disc.params);
    CHECK(run1.workers[0].pair.gen.buffers == pair.gen.buffers);
  });
  run("partition.identical_seeds_identical_workers [test_partition.cpp:122-143]", [] {
    Dataset ds;
    ds.k = 2;
    ds.C = ds.H = ds.W = 1;
    ds.m = 64;
    ds.images.resize(64);
    ds.labels.resize(64);
    Rng v(9);
    for (int i = 0; i < 32; ++i) {
      double x = v.uniform();
      ds.images[static_cast<size_t>(i)] = ds.images[static_cast<size_t>(32 + i)] = x;
      ds.labels[static_cast<size_t>(i)] = 0;
      ds.labels[static_cast<size_t>(32 + i)] = 1;
    }
    auto sh = partition_by_label(ds.labels, 2);
    auto run2 = train_distributed<double>(
        ds, sh, {dense_worker(0, 555, ds.sample_shape(), 2, 8), dense_worker(1, 555, ds.sample_shape(), 2, 8)}, 2);
    CHECK(run2.workers[0].pair.gen.params == run2.workers[1].pair.gen.params);
    CHECK(run2.workers[0].pair.disc.params == run2.workers[1].pair.disc.params);
  });
  run("partition.serial_vs_concurrent_bitwise [test_partition.cpp:145-162]", [] {
    Dataset ds = blobs(4, 48, 0.05, 11);
    auto sh = partition_by_label(ds.labels, 4);
    std::vector<WorkerConfig> cf;
    for (int j = 0; j < 4; ++j)
      cf.push_back(dense_worker(j, derive_seed(321, static_cast<uint64_t>(j)), ds.sample_shape(), 2, 16));
    auto s = train_distributed<double>(ds, sh, cf, 1), p = train_distributed<double>(ds, sh, cf, 4);
    for (size_t j = 0; j < 4; ++j) {
      CHECK(s.workers[j].pair.gen.params == p.workers[j].pair.gen.params);
      CHECK(s.workers[j].pair.disc.params == p.workers[j].pair.disc.params);
      CHECK(s.workers[j].pair.gen.buffers == p.workers[j].pair.gen.buffers);
    }
  });
  run("partition.failure_attribution [test_partition.cpp:178-194]", [] {
    Dataset ds = blobs(3, 16, 0.05, 17);
    auto sh = partition_by_label(ds.labels, 3);
    std::vector<WorkerConfig> cf;
    for (int j = 0; j < 3; ++j)
      cf.push_back(dense_worker(j, derive_seed(77, static_cast<uint64_t>(j)), ds.sample_shape(), 1, 8));
    cf[1].gen_arch = gen_dense(2, {7}, 16);
    bool caught = false;
    try {
      train_distributed<double>(ds, sh, cf, 2);
    } catch (const TrainError& e) {
      caught = true;
      CHECK((e.failed_classes == std::vector<int>{1}));
      CHECK((e.completed_classes == std::vector<int>{0, 2}));
      CHECK(std::string(e.what()).find("class 1") != std::string::npos);
    }
    CHECK(caught);
  });
  run("partition.mixture_single_pair_equals_generate [test_partition.cpp:196-210]", [] {
    auto pair = make_gan_pair<double>(gen_dense(2, {1, 1, 1}, 8), disc_dense({1, 1, 1}, 8), {1, 1, 1}, 2, 0,
                                      AdamConfig{}, 3);
    ClassPrior pr;
    pr.counts = {10};
    pr.probabilities = {1.0};
    Rng a(21), b(21);
    auto ms = mixture_sample<double>({&pair}, pr, 50, a);
    T direct = generate(pair, 0, 50, b);
    CHECK(ms.first.data == direct.data);
    for (int i : ms.second) CHECK(i == 0);
  });
  run("partition.degenerate_priors_route_to_zero [test_partition.cpp:212-223]", [] {
    std::vector<GanPair<double>> pairs;
    for (int j = 0; j < 2; ++j)
      pairs.push_back(make_gan_pair<double>(gen_dense(2, {1, 1, 1}, 8), disc_dense({1, 1, 1}, 8), {1, 1, 1}, 2, 0,
                                            AdamConfig{}, derive_seed(9, static_cast<uint64_t>(j))));
    ClassPrior pr;
    pr.counts = {5, 0};
    pr.probabilities = {1.0, 0.0};
    Rng r(4);
    auto ms = mixture_sample<double>({&pairs[0], &pairs[1]}, pr, 200, r);
    for (int i : ms.second) CHECK(i == 0);
  });

  std::printf("SUMMARY %d failed\n", g_failures);
  return g_failures;
}
