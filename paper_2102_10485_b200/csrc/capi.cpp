// extern "C" surface: include/pg_kernels.h and include/pg_trainer.h.
#include <cstring>
#include <string>

#include "../../include/pg_trainer.h"
#include "capi_util.hpp"
#include "device_cache.hpp"
#include "gan.hpp"

namespace pg {
std::string& last_error() {
  thread_local std::string e;
  return e;
}
void softmax_rows(const double* logits, long n, long k, double* probs);
void inception_score(const double* probs, long n, long k, int n_splits, double* split_scores, double* mean,
                     double* stddev);
double anova_f(const double* values, const long* sizes, long k);
void anova_per_channel(const float* images, const int* labels, long n, long C, long H, long W, long k, double* f);
}  // namespace pg

namespace {

using pg::guard;

void cuda_ok(cudaError_t e, const char* what) { pg::check_cuda(e, what); }

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

pg::ConvGeo conv_geo(const pg_conv_desc* d) {
  pg::ConvGeo g;
  g.B = d->B;
  g.GH = d->H;
  g.GW = d->W;
  g.CG = static_cast<int>(pg::pad4(d->Cin));
  g.SH = d->OH;
  g.SW = d->OW;
  g.CS = static_cast<int>(pg::pad4(d->Cout));
  g.k = d->k;
  g.s = d->s;
  g.p = d->p;
  return g;
}
pg::ConvGeo convT_geo(const pg_conv_desc* d) {
  pg::ConvGeo g;
  g.B = d->B;
  g.SH = d->H;
  g.SW = d->W;
  g.CS = static_cast<int>(pg::pad4(d->Cin));
  g.GH = d->OH;
  g.GW = d->OW;
  g.CG = static_cast<int>(pg::pad4(d->Cout));
  g.k = d->k;
  g.s = d->s;
  g.p = d->p;
  return g;
}
pg::ConvGeo dense_geo(int B, int in, int out) {
  pg::ConvGeo g;
  g.B = B;
  g.SH = g.SW = g.GH = g.GW = 1;
  g.k = g.s = 1;
  g.p = 0;
  g.CS = static_cast<int>(pg::pad4(out));
  g.CG = static_cast<int>(pg::pad4(in));
  return g;
}

void check_desc(const pg_conv_desc* d, bool transposed) {
  if (!d || d->B < 1 || d->Cin < 1 || d->Cout < 1 || d->k < 1 || d->s < 1 || d->p < 0)
    throw std::invalid_argument("invalid convolution descriptor");
  long oh = transposed ? (d->H - 1L) * d->s - 2L * d->p + d->k : (d->H + 2L * d->p - d->k) / d->s + 1;
  long ow = transposed ? (d->W - 1L) * d->s - 2L * d->p + d->k : (d->W + 2L * d->p - d->k) / d->s + 1;
  if (oh != d->OH || ow != d->OW) throw std::invalid_argument("output extent does not match the geometry");
}

long long small_ls(const pg::ConvGeo& g) { return static_cast<long long>(g.B) * g.SH * g.SW * g.CS; }
long long big_ls(const pg::ConvGeo& g) { return static_cast<long long>(g.B) * g.GH * g.GW * g.CG; }

struct Group {
  int device;
  std::unique_ptr<pg::GanGroup> g;
};

Group* G(pg_group* p) { return reinterpret_cast<Group*>(p); }

}  // namespace

extern "C" {

const char* pg_last_error(void) { return pg::last_error().c_str(); }

int pg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

long long pg_launch_count(void) { return pg::launch_count(); }

int pg_kernel_timing(int on) {
  return guard([&] { pg::gemm_timing_enable(on != 0); });
}

int pg_kernel_timing_read(double* ms) {
  return guard([&] { *ms = pg::gemm_timing_read_ms(); });
}

int pg_tc_tf32_peak(int iters, double* tflops) {
  return guard([&] { pg::check_cuda(pg::tc_tf32_peak(iters, tflops), "tc peak"); });
}

long pg_kernel_timing_report(char* out, long cap) {
  std::string r = pg::gemm_timing_report();
  if (out && cap > 0) {
    long n = std::min<long>(cap - 1, static_cast<long>(r.size()));
    std::memcpy(out, r.data(), static_cast<size_t>(n));
    out[n] = 0;
  }
  return static_cast<long>(r.size());
}

// ---------------- GEMM-shaped operators ----------------
// One argument builder per operator: the operator entry points and
// pg_workspace_size share it, so the size query sees the engine the call takes.
}  // extern "C"
namespace {
struct OpPtrs {
  const float* in = nullptr;   // x (forward), gy (data grad), x (filter grad)
  const float* in2 = nullptr;  // gy of the filter grads
  const float* w = nullptr;
  long long w_ls = 0;
  const float* bias = nullptr;
  long long bias_ls = 0;
  int act = PG_ACT_NONE;
  float slope = 0.f;
  float* out = nullptr;
  long long out_ls = 0;  // filter grads: gw_ls
  int accumulate = 0;
};

pg::GemmArgs op_args(int op, const pg_conv_desc* d, int L, const OpPtrs& p) {
  const bool dense = op >= PG_OP_DENSE_FWD;
  const bool transposed = op >= PG_OP_CONVT2D_FWD && !dense;
  if (op < PG_OP_CONV2D_FWD || op > PG_OP_DENSE_BWD_FILTER) throw std::invalid_argument("unknown operator id");
  if (!d) throw std::invalid_argument("invalid convolution descriptor");
  if (L < 0) throw std::invalid_argument("L must be >= 0");
  if (!dense) check_desc(d, transposed);
  pg::GemmArgs a{};
  a.g = dense ? dense_geo(d->B, d->Cin, d->Cout) : transposed ? convT_geo(d) : conv_geo(d);
  a.L = L;
  a.w = p.w;
  a.w_ls = p.w_ls;
  const int role = (op - PG_OP_CONV2D_FWD) % 3;  // 0 forward, 1 data grad, 2 filter grad
  // forward of Conv2d / Dense = FPROP (big -> small); ConvT forward = DGRAD (small -> big)
  const bool fwd_is_fprop = !transposed;
  if (role == 0) {
    a.kind = fwd_is_fprop ? pg::GEMM_FPROP : pg::GEMM_DGRAD;
    if (fwd_is_fprop) {
      a.big = p.in;
      a.big_ls = big_ls(a.g);
      a.out_ls = small_ls(a.g);
      a.c_valid = d->Cout;
      a.c_pad = a.g.CS;
    } else {
      a.small = p.in;
      a.small_ls = small_ls(a.g);
      a.out_ls = big_ls(a.g);
      a.c_valid = d->Cout;
      a.c_pad = a.g.CG;
    }
    a.out = p.out;
    a.bias = p.bias;
    a.bias_ls = p.bias_ls;
    a.act = p.act;
    a.slope = p.slope;
  } else if (role == 1) {
    a.kind = fwd_is_fprop ? pg::GEMM_DGRAD : pg::GEMM_FPROP;
    if (fwd_is_fprop) {
      a.small = p.in;
      a.small_ls = small_ls(a.g);
      a.out_ls = big_ls(a.g);
      a.c_valid = d->Cin;
      a.c_pad = a.g.CG;
    } else {
      a.big = p.in;
      a.big_ls = big_ls(a.g);
      a.out_ls = small_ls(a.g);
      a.c_valid = d->Cin;
      a.c_pad = a.g.CS;
    }
    a.out = p.out;
  } else {
    a.kind = pg::GEMM_WGRAD;
    // Conv2d / Dense: x is the big map, gy the small one; ConvT: the reverse
    a.small = fwd_is_fprop ? p.in2 : p.in;
    a.big = fwd_is_fprop ? p.in : p.in2;
    a.small_ls = small_ls(a.g);
    a.big_ls = big_ls(a.g);
    a.out = p.out;
    a.out_ls = p.out_ls;
    a.accumulate = p.accumulate;
  }
  return a;
}

int run_op(int op, const pg_conv_desc* d, int L, const OpPtrs& p, int math, void* stream, const char* what) {
  return guard([&] {
    if (math < PG_MATH_FP32_SIMT || math > PG_MATH_BF16) throw std::invalid_argument("unknown math mode");
    const pg::GemmArgs a = op_args(op, d, L, p);
    cuda_ok(pg::launch_gemm(a, math, S(stream)), what);
  });
}

pg_conv_desc dense_desc(int B, int in, int out) { return pg_conv_desc{B, in, 1, 1, out, 1, 1, 1, 1, 0}; }
}  // namespace
extern "C" {

// ---------------- Conv2d ----------------
int pg_conv2d_fwd(const pg_conv_desc* d, int L, const float* x, const float* w, long long w_ls, const float* bias,
                  long long bias_ls, int act, float slope, float* y, int math, void* stream) {
  OpPtrs p;
  p.in = x, p.w = w, p.w_ls = w_ls, p.bias = bias, p.bias_ls = bias_ls, p.act = act, p.slope = slope, p.out = y;
  return run_op(PG_OP_CONV2D_FWD, d, L, p, math, stream, "conv2d_fwd");
}

int pg_conv2d_bwd_data(const pg_conv_desc* d, int L, const float* gy, const float* w, long long w_ls, float* gx,
                       int math, void* stream) {
  OpPtrs p;
  p.in = gy, p.w = w, p.w_ls = w_ls, p.out = gx;
  return run_op(PG_OP_CONV2D_BWD_DATA, d, L, p, math, stream, "conv2d_bwd_data");
}

int pg_conv2d_bwd_filter(const pg_conv_desc* d, int L, const float* x, const float* gy, float* gw, long long gw_ls,
                         int accumulate, int math, void* stream) {
  OpPtrs p;
  p.in = x, p.in2 = gy, p.out = gw, p.out_ls = gw_ls, p.accumulate = accumulate;
  return run_op(PG_OP_CONV2D_BWD_FILTER, d, L, p, math, stream, "conv2d_bwd_filter");
}

// ---------------- ConvTranspose2d ----------------
int pg_convT2d_fwd(const pg_conv_desc* d, int L, const float* x, const float* w, long long w_ls, const float* bias,
                   long long bias_ls, int act, float slope, float* y, int math, void* stream) {
  OpPtrs p;
  p.in = x, p.w = w, p.w_ls = w_ls, p.bias = bias, p.bias_ls = bias_ls, p.act = act, p.slope = slope, p.out = y;
  return run_op(PG_OP_CONVT2D_FWD, d, L, p, math, stream, "convT2d_fwd");
}

int pg_convT2d_bwd_data(const pg_conv_desc* d, int L, const float* gy, const float* w, long long w_ls, float* gx,
                        int math, void* stream) {
  OpPtrs p;
  p.in = gy, p.w = w, p.w_ls = w_ls, p.out = gx;
  return run_op(PG_OP_CONVT2D_BWD_DATA, d, L, p, math, stream, "convT2d_bwd_data");
}

int pg_convT2d_bwd_filter(const pg_conv_desc* d, int L, const float* x, const float* gy, float* gw, long long gw_ls,
                          int accumulate, int math, void* stream) {
  OpPtrs p;
  p.in = x, p.in2 = gy, p.out = gw, p.out_ls = gw_ls, p.accumulate = accumulate;
  return run_op(PG_OP_CONVT2D_BWD_FILTER, d, L, p, math, stream, "convT2d_bwd_filter");
}

// ---------------- Dense ----------------
int pg_dense_fwd(int L, int B, int in, int out, const float* x, const float* w, long long w_ls, const float* bias,
                 long long bias_ls, int act, float slope, float* y, int math, void* stream) {
  const pg_conv_desc d = dense_desc(B, in, out);
  OpPtrs p;
  p.in = x, p.w = w, p.w_ls = w_ls, p.bias = bias, p.bias_ls = bias_ls, p.act = act, p.slope = slope, p.out = y;
  return run_op(PG_OP_DENSE_FWD, &d, L, p, math, stream, "dense_fwd");
}

int pg_dense_bwd_data(int L, int B, int in, int out, const float* gy, const float* w, long long w_ls, float* gx,
                      int math, void* stream) {
  const pg_conv_desc d = dense_desc(B, in, out);
  OpPtrs p;
  p.in = gy, p.w = w, p.w_ls = w_ls, p.out = gx;
  return run_op(PG_OP_DENSE_BWD_DATA, &d, L, p, math, stream, "dense_bwd_data");
}

int pg_dense_bwd_filter(int L, int B, int in, int out, const float* x, const float* gy, float* gw, long long gw_ls,
                        int accumulate, int math, void* stream) {
  const pg_conv_desc d = dense_desc(B, in, out);
  OpPtrs p;
  p.in = x, p.in2 = gy, p.out = gw, p.out_ls = gw_ls, p.accumulate = accumulate;
  return run_op(PG_OP_DENSE_BWD_FILTER, &d, L, p, math, stream, "dense_bwd_filter");
}

// ---------------- Workspace ----------------
size_t pg_workspace_size(int op, const pg_conv_desc* d, int L, int math) {
  size_t bytes = 0;
  const int rc = guard([&] {
    if (math < PG_MATH_FP32_SIMT || math > PG_MATH_BF16) throw std::invalid_argument("unknown math mode");
    OpPtrs p;  // null device pointers pass every alignment test; strides as the arenas would have them
    const pg::GemmArgs probe = op_args(op, d, L, p);
    const pg::ConvGeo& g = probe.g;
    const long long wsz = static_cast<long long>(g.CS) * g.k * g.k * g.CG;
    p.w_ls = wsz;
    p.bias_ls = (op % 3 == 0) ? (g.CS > g.CG ? g.CS : g.CG) : 0;
    p.out_ls = wsz;
    const pg::GemmWorkspace w = pg::gemm_workspace(op_args(op, d, L, p), math);
    auto r = [](size_t f) { return (f * sizeof(float) + 255) / 256 * 256; };
    bytes = r(w.gemm) + r(w.blo);
  });
  return rc == PG_OK ? bytes : static_cast<size_t>(-1);
}

int pg_set_workspace(void* stream, void* workspace, size_t bytes) {
  return guard([&] { pg::set_stream_workspace(S(stream), workspace, bytes); });
}

// ---------------- BatchNorm ----------------
size_t pg_bn_workspace_floats(int L, int R, int Cp) {
  pg::ChannelMap cm{L, R, Cp, Cp, 0};
  return pg::reduce_partial_floats(cm) + static_cast<size_t>(L) * Cp * 3;
}

int pg_bn_fwd(int L, int R, int C, int Cp, const float* x, const float* gamma_beta, long long gb_ls, float* running,
              long long run_ls, float eps, float momentum, int train, int act, float slope, float* mean, float* istd,
              float* y, float* ws, void* stream) {
  return guard([&] {
    if (Cp % 4 || C > Cp || C < 1) throw std::invalid_argument("bn: channel padding must be a multiple of 4");
    pg::ChannelMap cm{L, R, Cp, C, static_cast<long long>(R) * Cp};
    if (train) {
      cuda_ok(pg::launch_channel_reduce(cm, pg::RED_SUM, x, nullptr, nullptr, nullptr, 0, 0.f, ws, S(stream)), "bn");
      cuda_ok(pg::launch_bn_finalize_mean(cm, ws, mean, S(stream)), "bn");
      cuda_ok(pg::launch_channel_reduce(cm, pg::RED_SQDEV, x, nullptr, nullptr, mean, 0, 0.f, ws, S(stream)), "bn");
      cuda_ok(pg::launch_bn_finalize_var(cm, ws, mean, istd, running, run_ls, eps, momentum, running ? 1 : 0, S(stream)),
              "bn");
    } else {
      cuda_ok(pg::launch_bn_eval_stats(cm, running, run_ls, eps, mean, istd, S(stream)), "bn");
    }
    cuda_ok(pg::launch_bn_apply(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y, S(stream)), "bn");
  });
}

int pg_bn_bwd(int L, int R, int C, int Cp, const float* gy, const float* y, const float* x, const float* mean,
              const float* istd, const float* gamma_beta, long long gb_ls, int act, float slope, float* gx,
              float* dgamma_beta, long long dgb_ls, int accumulate, float* ws, void* stream) {
  return guard([&] {
    pg::ChannelMap cm{L, R, Cp, C, static_cast<long long>(R) * Cp};
    float* coef = ws + pg::reduce_partial_floats(cm);
    cuda_ok(pg::launch_channel_reduce(cm, pg::RED_BN_BWD, x, gy, y, mean, act, slope, ws, S(stream)), "bn bwd");
    cuda_ok(pg::launch_bn_bwd_finalize(cm, ws, istd, gamma_beta, gb_ls, dgamma_beta, dgb_ls, nullptr, 0, accumulate, 1,
                                       coef, S(stream)),
            "bn bwd");
    cuda_ok(pg::launch_bn_bwd_apply(cm, gy, y, x, mean, coef, act, slope, gx, S(stream)), "bn bwd");
  });
}

int pg_act_bwd(long long n, const float* gy, const float* y, int act, float slope, float* gx, void* stream) {
  return guard([&] {
    if (n % 4) throw std::invalid_argument("act_bwd: n must be a multiple of 4");
    pg::ChannelMap cm{1, static_cast<int>(n / 4), 4, 4, n};
    cuda_ok(pg::launch_act_bwd(cm, gy, y, act, slope, gx, S(stream)), "act_bwd");
  });
}

int pg_gan_losses(int L, int B, const float* p_real, const float* p_fake, int pstride, double clamp, float* g_real,
                  float* g_fake, double* report, void* stream) {
  return guard([&] {
    if (!(clamp > 0 && clamp < 0.5)) throw std::invalid_argument("probability clamp must lie in (0, 0.5)");
    if (B < 1 || B > 1024) throw std::invalid_argument("gan_losses: batch must be in [1, 1024]");
    cuda_ok(pg::launch_loss_d(L, B, p_real, p_fake, pstride, clamp, g_real, g_fake, report, S(stream)), "loss");
  });
}

int pg_gen_loss(int L, int B, const float* p_fake, int pstride, double clamp, float* g, double* report, void* stream) {
  return guard([&] {
    if (!(clamp > 0 && clamp < 0.5)) throw std::invalid_argument("probability clamp must lie in (0, 0.5)");
    if (B < 1 || B > 1024) throw std::invalid_argument("gen_loss: batch must be in [1, 1024]");
    cuda_ok(pg::launch_loss_g(L, B, p_fake, pstride, clamp, g, report, S(stream)), "loss");
  });
}

int pg_adam_step(int L, long long P, float* params, const float* grads, float* m, float* v, long long* t, int* flags,
                 double lr, double beta1, double beta2, double eps, void* stream) {
  return guard([&] {
    if (P % 4) throw std::invalid_argument("adam_step: arena length must be a multiple of 4");
    cuda_ok(pg::launch_nonfinite_check(L, P, grads, flags, S(stream)), "adam");
    cuda_ok(pg::launch_adam_tick(L, flags, t, S(stream)), "adam");
    cuda_ok(pg::launch_adam(L, P, params, grads, m, v, t, flags, static_cast<float>(lr), beta1, beta2,
                            static_cast<float>(eps), S(stream)),
            "adam");
  });
}

int pg_gather_real(int L, int B, const int* idx, const float* data, long long data_ls, long long sample, int Cp, int C,
                   float* out, void* stream) {
  return guard([&] {
    cuda_ok(pg::launch_gather_real(L, B, idx, data, data_ls, sample, Cp, C, out, S(stream)), "gather");
  });
}

// ---------------- trainer ----------------
int pg_group_create(const pg_group_config* c, pg_group** out) {
  return guard([&] {
    if (!c || !out) throw std::invalid_argument("null argument");
    *out = nullptr;
    cuda_ok(cudaSetDevice(c->device), "cudaSetDevice");
    pg::GroupConfig cfg;
    cfg.gen_spec = c->gen_spec ? c->gen_spec : "";
    cfg.disc_spec = c->disc_spec ? c->disc_spec : "";
    cfg.C = c->C;
    cfg.H = c->H;
    cfg.W = c->W;
    cfg.d_z = c->d_z;
    if (c->n_labels < 1 || !c->class_ids) throw std::invalid_argument("pg_group_create: no labels");
    cfg.class_ids.assign(c->class_ids, c->class_ids + c->n_labels);
    cfg.base_seed = c->base_seed;
    cfg.batch = c->batch;
    cfg.epochs = c->epochs;
    cfg.per_label = c->per_label;
    cfg.lr = c->lr;
    cfg.beta1 = c->beta1;
    cfg.beta2 = c->beta2;
    cfg.eps = c->eps;
    cfg.clamp = c->clamp;
    cfg.init_std = c->init_std;
    if (c->math < PG_MATH_FP32_SIMT || c->math > PG_MATH_BF16) throw std::invalid_argument("unknown math mode");
    cfg.math = c->math;
    cfg.threads = c->threads;
    if (c->seeds) cfg.seeds.assign(c->seeds, c->seeds + c->n_labels);
    auto grp = std::make_unique<Group>();
    grp->device = c->device;
    grp->g = std::make_unique<pg::GanGroup>(cfg);
    *out = reinterpret_cast<pg_group*>(grp.release());
  });
}

void pg_group_destroy(pg_group* g) {
  if (!g) return;
  cudaSetDevice(G(g)->device);
  delete G(g);
}

#define WITH_GROUP(body)                                    \
  guard([&] {                                               \
    if (!g) throw std::invalid_argument("null group");      \
    cuda_ok(cudaSetDevice(G(g)->device), "cudaSetDevice");  \
    pg::GanGroup& grp = *G(g)->g;                           \
    (void)grp;                                              \
    body;                                                   \
  })

int pg_group_set_dataset(pg_group* g, const float* images01) { return WITH_GROUP(grp.set_dataset(images01)); }
int pg_group_generate_dataset(pg_group* g, uint64_t seed) { return WITH_GROUP(grp.generate_dataset(seed)); }
int pg_group_train_steps(pg_group* g, int n) {
  int done = 0;
  int rc = WITH_GROUP(done = grp.train_steps(n));
  return rc == PG_OK ? done : rc;
}
int pg_group_train_step(pg_group* g, const float* real01, int B, double* reports) {
  return WITH_GROUP(grp.train_step_host(real01, B, reports));
}
int pg_group_train_step_inputs(pg_group* g, const float* real01, const float* z1, const float* z2, int B,
                               double* reports) {
  return WITH_GROUP(grp.train_step_inputs(real01, z1, z2, B, reports));
}
long pg_group_get(pg_group* g, int label, int field, double* out, long cap) {
  long n = -1;
  int rc = WITH_GROUP(n = grp.get(label, field, out, cap));
  return rc == PG_OK ? n : rc;
}
int pg_group_set(pg_group* g, int label, int field, const double* in, long n) {
  return WITH_GROUP(grp.set(label, field, in, n));
}
int pg_group_failed(pg_group* g, int* failed) {
  return WITH_GROUP({
    auto f = grp.failed();
    std::memcpy(failed, f.data(), f.size() * sizeof(int));
  });
}
int pg_group_generate(pg_group* g, long n, uint64_t seed, float* out) { return WITH_GROUP(grp.generate(n, seed, out)); }
int pg_group_generate_latents(pg_group* g, const float* z, long n, float* out) {
  return WITH_GROUP(grp.generate_latents(z, n, out));
}
int pg_group_save_checkpoint(pg_group* g, int label_idx, const char* path) {
  return WITH_GROUP(pg::save_checkpoint(grp, label_idx, path));
}
int pg_group_load_checkpoint(pg_group* g, int label_idx, const char* path) {
  return WITH_GROUP(pg::load_checkpoint(grp, label_idx, path));
}
int pg_group_mixture_sample(pg_group* g, const double* priors, long n, uint64_t seed, float* out, int* ids) {
  return WITH_GROUP(grp.mixture_sample(priors, n, seed, out, ids));
}
int pg_group_capture_masks(pg_group* g, int on) { return WITH_GROUP(grp.capture_masks(on != 0)); }
long pg_group_get_masks(pg_group* g, int label_idx, uint8_t* out, long cap) {
  long n = -1;
  int rc = WITH_GROUP(n = grp.get_masks(label_idx, out, cap));
  return rc == PG_OK ? n : rc;
}
float pg_group_last_ms(pg_group* g) { return g ? G(g)->g->last_device_ms() : -1.f; }
int pg_group_sync(pg_group* g) { return WITH_GROUP(grp.sync()); }
int pg_group_sizes(pg_group* g, long long* out) {
  return WITH_GROUP({
    out[0] = grp.gen().ref_params();
    out[1] = grp.disc().ref_params();
    out[2] = grp.gen().P();
    out[3] = grp.disc().P();
  });
}

int pg_softmax_rows(const double* logits, long n, long k, double* probs) {
  return guard([&] { pg::softmax_rows(logits, n, k, probs); });
}
int pg_inception_score(const double* probs, long n, long k, int n_splits, double* split_scores, double* mean,
                       double* stddev) {
  return guard([&] { pg::inception_score(probs, n, k, n_splits, split_scores, mean, stddev); });
}
int pg_anova_f(const double* values, const long* sizes, long k, double* f) {
  return guard([&] { *f = pg::anova_f(values, sizes, k); });
}
int pg_anova_per_channel(const float* images, const int* labels, long n, long C, long H, long W, long k, double* f) {
  return guard([&] { pg::anova_per_channel(images, labels, n, C, H, W, k, f); });
}

uint64_t pg_derive_seed(uint64_t base, uint64_t stream) { return pg::derive_seed(base, stream); }
int pg_shard_begin(int n_labels, int n_gpus, int g) { return pg::shard_begin(n_labels, n_gpus, g); }
int pg_cosine_label(int C, int H, int W, long per_label, uint64_t seed, int label, double* out) {
  return guard([&] { pg::cosine_label(C, H, W, per_label, seed, label, out); });
}

}  // extern "C"
