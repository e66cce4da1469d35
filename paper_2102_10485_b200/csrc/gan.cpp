#include "gan.hpp"

#include "device_cache.hpp"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <optional>

namespace pg {

namespace {
// NVTX range over the host enqueue of one phase of the step: a profiler can
// select a phase's kernels with it (ncu --nvtx --nvtx-include "pg.D_update/"),
// a no-op when no tool is attached
struct Phase {
  explicit Phase(const char* name) { nvtxRangePushA(name); }
  ~Phase() { nvtxRangePop(); }
  Phase(const Phase&) = delete;
  Phase& operator=(const Phase&) = delete;
};
}  // namespace

namespace {
template <class T>
T* pinned(size_t n) {
  void* p = nullptr;
  check_cuda(cudaMallocHost(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMallocHost");
  std::memset(p, 0, std::max<size_t>(n, 1) * sizeof(T));
  return static_cast<T*>(p);
}
template <class T>
T* dev_alloc(size_t n) {
  void* p = nullptr;
  check_cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  check_cuda(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)), "cudaMemset");
  return static_cast<T*>(p);
}
[[maybe_unused]] std::string shape3(long C, long H, long W) {
  return std::to_string(C) + " " + std::to_string(H) + " " + std::to_string(W);
}
}  // namespace

GanGroup::GanGroup(const GroupConfig& cfg) : cfg_(cfg), L_(static_cast<int>(cfg.class_ids.size())) {
  if (L_ < 1) throw std::invalid_argument("GanGroup: no labels");
  if (cfg_.batch < 1) throw std::invalid_argument("GanGroup: batch size must be positive");
  if (cfg_.per_label < 1) throw std::invalid_argument("GanGroup: empty shard");
  if (!(cfg_.clamp > 0.0 && cfg_.clamp < 0.5))
    throw std::invalid_argument("probability clamp must lie in (0, 0.5), got " + std::to_string(cfg_.clamp));
  if (cfg_.d_z < 1) throw std::invalid_argument("latent dimension must be positive");
  const int Bmax = static_cast<int>(std::min<long>(cfg_.batch, cfg_.per_label));
  G_ = std::make_unique<DevNet>(cfg_.gen_spec, std::vector<long>{cfg_.d_z}, L_, Bmax, cfg_.math);
  D_ = std::make_unique<DevNet>(cfg_.disc_spec, std::vector<long>{cfg_.C, cfg_.H, cfg_.W}, L_, Bmax, cfg_.math);
  // make_gan_pair shape checks (gan.cpp:41-48)
  std::vector<long> img{cfg_.C, cfg_.H, cfg_.W};
  auto sstr = [](const std::vector<long>& v) {
    std::string r = "[";
    for (size_t i = 0; i < v.size(); ++i) r += (i ? "x" : "") + std::to_string(v[i]);
    return r + "]";
  };
  if (G_->ref_out_shape() != img)
    throw std::invalid_argument("generator emits " + sstr(G_->ref_out_shape()) + " but images are " + sstr(img));
  long dout = 1;
  for (long d : D_->ref_out_shape()) dout *= d;
  if (dout != 1) throw std::invalid_argument("discriminator must emit a scalar, got " + sstr(D_->ref_out_shape()));

  check_cuda(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
  check_cuda(cudaStreamCreateWithFlags(&cst_, cudaStreamNonBlocking), "copy stream");
  check_cuda(cudaEventCreateWithFlags(&real_ready_, cudaEventDisableTiming), "event");
  tg_ = G_->make_trace(true);
  {
    const char* e = std::getenv("PG_OVERLAP");
    overlap_ = !(e && e[0] == '0');
  }
  if (overlap_) {
    tg2_ = G_->make_trace(true);
    check_cuda(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "stream 2");
    for (cudaEvent_t* ev : {&ev_fork_, &ev_g1_, &ev_g2_})
      check_cuda(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "event");
  }
  tdr_ = D_->make_trace(true);
  tdf_ = D_->make_trace(true);
  zcp_ = pad4(cfg_.d_z);
  const Map& im = D_->in_map();
  data_ = DeviceBuf(static_cast<size_t>(L_) * cfg_.per_label * im.numel());
  real_ = DeviceBuf(static_cast<size_t>(L_) * Bmax * im.numel());
  gimg_ = DeviceBuf(static_cast<size_t>(L_) * Bmax * im.numel());
  const long pout = D_->out_map().Cp;
  gp_real_ = DeviceBuf(static_cast<size_t>(L_) * Bmax * pout);
  gp_fake_ = DeviceBuf(static_cast<size_t>(L_) * Bmax * pout);
  for (int par = 0; par < 2; ++par) {
    for (int k = 0; k < 2; ++k) dz_[par][k] = DeviceBuf(static_cast<size_t>(L_) * Bmax * zcp_);
    d_idx_[par] = dev_alloc<int>(static_cast<size_t>(L_) * Bmax);
    h_idx_[par] = pinned<int>(static_cast<size_t>(L_) * Bmax);
    h_z_[par] = pinned<float>(static_cast<size_t>(2) * L_ * Bmax * zcp_);
    check_cuda(cudaEventCreateWithFlags(&staged_[par], cudaEventDisableTiming), "event");
  }
  check_cuda(cudaEventCreate(&t0_), "event");
  check_cuda(cudaEventCreate(&t1_), "event");
  d_flags_ = dev_alloc<int>(static_cast<size_t>(L_));
  d_t_g_ = dev_alloc<long long>(static_cast<size_t>(L_));
  d_t_d_ = dev_alloc<long long>(static_cast<size_t>(L_));
  rep_cap_ = 256;
  d_rep_ = dev_alloc<double>(static_cast<size_t>(rep_cap_) * L_ * 4);
  d_rep_cur_ = dev_alloc<double>(static_cast<size_t>(L_) * 4);
  {
    const char* e = std::getenv("PG_GRAPH");
    use_graph_ = !(e && e[0] == '0');
  }
  h_rep_ = pinned<double>(static_cast<size_t>(rep_cap_) * L_ * 4);
  pool_ = std::make_unique<ThreadPool>(std::max(1, cfg_.threads));

  // make_gan_pair per label: G from derive_seed(seed, 1), D from derive_seed(seed, 2) (gan.cpp:39-40)
  std::vector<float> gp(static_cast<size_t>(L_) * G_->P()), dp(static_cast<size_t>(L_) * D_->P());
  std::vector<float> gb(static_cast<size_t>(L_) * std::max<long long>(G_->Bf(), 4), 0.f),
      db(static_cast<size_t>(L_) * std::max<long long>(D_->Bf(), 4), 0.f);
  if (!cfg_.seeds.empty() && static_cast<int>(cfg_.seeds.size()) != L_)
    throw std::invalid_argument("GanGroup: " + std::to_string(cfg_.seeds.size()) + " worker seeds for " +
                                std::to_string(L_) + " labels");
  pool_->parallel_for(L_, [&](int l) {
    uint64_t wseed = worker_seed(l);
    auto g = G_->init_ref_params(derive_seed(wseed, 1), cfg_.init_std);
    auto d = D_->init_ref_params(derive_seed(wseed, 2), cfg_.init_std);
    G_->import_params(g.data(), gp.data() + static_cast<size_t>(l) * G_->P());
    D_->import_params(d.data(), dp.data() + static_cast<size_t>(l) * D_->P());
    auto gbuf = G_->init_ref_buffers(), dbuf = D_->init_ref_buffers();
    G_->import_buffers(gbuf.data(), gb.data() + static_cast<size_t>(l) * std::max<long long>(G_->Bf(), 4));
    D_->import_buffers(dbuf.data(), db.data() + static_cast<size_t>(l) * std::max<long long>(D_->Bf(), 4));
  });
  check_cuda(cudaMemcpy(G_->params.p, gp.data(), gp.size() * sizeof(float), cudaMemcpyHostToDevice), "upload G");
  check_cuda(cudaMemcpy(D_->params.p, dp.data(), dp.size() * sizeof(float), cudaMemcpyHostToDevice), "upload D");
  if (G_->Bf()) check_cuda(cudaMemcpy(G_->running.p, gb.data(), gb.size() * sizeof(float), cudaMemcpyHostToDevice), "upload");
  if (D_->Bf()) check_cuda(cudaMemcpy(D_->running.p, db.data(), db.size() * sizeof(float), cudaMemcpyHostToDevice), "upload");

  // run_worker: Rng rng(cfg.seed) per label; order = the label's shard
  rng_.reserve(static_cast<size_t>(L_));
  for (int l = 0; l < L_; ++l) rng_.emplace_back(worker_seed(l));
  order_.assign(static_cast<size_t>(L_), std::vector<int>(static_cast<size_t>(cfg_.per_label)));
  for (auto& o : order_)
    for (long j = 0; j < cfg_.per_label; ++j) o[static_cast<size_t>(j)] = static_cast<int>(j);
  last_batch_.assign(static_cast<size_t>(L_), {});
  reports_.assign(static_cast<size_t>(L_), {});
}

// run_worker: Rng rng(cfg.seed), make_gan_pair(..., cfg.seed) (partition.cpp:85-87) with
// cfg.seed = derive_seed(base_seed, class_id) (run.cpp:376) unless given per label
uint64_t GanGroup::worker_seed(int l) const {
  if (!cfg_.seeds.empty()) return cfg_.seeds[static_cast<size_t>(l)];
  return derive_seed(cfg_.base_seed, static_cast<uint64_t>(cfg_.class_ids[static_cast<size_t>(l)]));
}

GanGroup::~GanGroup() {
  if (st_) cudaStreamSynchronize(st_);
  if (cst_) {
    cudaStreamSynchronize(cst_);
    cudaStreamDestroy(cst_);
  }
  if (real_ready_) cudaEventDestroy(real_ready_);
  for (cudaEvent_t ev : {ev_fork_, ev_g1_, ev_g2_})
    if (ev) cudaEventDestroy(ev);
  if (st2_) {
    cudaStreamSynchronize(st2_);
    release_stream_scratch(st2_);
    cudaStreamDestroy(st2_);
  }
  for (int par = 0; par < 2; ++par) {
    cudaFree(d_idx_[par]);
    cudaFreeHost(h_idx_[par]);
    cudaFreeHost(h_z_[par]);
    if (staged_[par]) cudaEventDestroy(staged_[par]);
  }
  cudaFree(d_flags_);
  if (d_mask_) cudaFree(d_mask_);
  cudaFree(d_t_g_);
  cudaFree(d_t_d_);
  cudaFree(d_rep_);
  cudaFree(d_rep_cur_);
  for (auto& sg : graphs_)
    if (sg.exec) cudaGraphExecDestroy(sg.exec);
  cudaFreeHost(h_rep_);
  if (t0_) cudaEventDestroy(t0_);
  if (t1_) cudaEventDestroy(t1_);
  if (st_) {
    release_stream_scratch(st_);
    cudaStreamDestroy(st_);
  }
}

void GanGroup::set_dataset(const float* images01) {
  const Map& im = D_->in_map();
  const long long n = static_cast<long long>(L_) * cfg_.per_label;
  DeviceBuf tmp(static_cast<size_t>(n) * cfg_.C * cfg_.H * cfg_.W);
  check_cuda(cudaMemcpyAsync(tmp.p, images01, tmp.n * sizeof(float), cudaMemcpyHostToDevice, st_), "dataset H2D");
  // resident copy: NHWC padded, raw [0,1] pixels (the per-step gather applies 2x-1)
  check_cuda(launch_nchw01_to_nhwc(n, static_cast<int>(cfg_.C), static_cast<int>(cfg_.H), static_cast<int>(cfg_.W),
                                   static_cast<int>(im.Cp), tmp.p, data_.p, st_, 0),
             "dataset layout");
  check_cuda(cudaStreamSynchronize(st_), "sync");
}

void GanGroup::generate_dataset(uint64_t data_seed) {
  const Map& im = D_->in_map();
  const long S = cfg_.C * cfg_.H * cfg_.W;
  std::vector<float> h(static_cast<size_t>(L_) * cfg_.per_label * im.numel(), 0.f);
  pool_->parallel_for(L_, [&](int l) {
    std::vector<double> buf(static_cast<size_t>(cfg_.per_label * S));
    cosine_label(cfg_.C, cfg_.H, cfg_.W, cfg_.per_label, data_seed, cfg_.class_ids[static_cast<size_t>(l)], buf.data());
    float* o = h.data() + static_cast<size_t>(l) * cfg_.per_label * im.numel();
    for (long j = 0; j < cfg_.per_label; ++j)
      for (long c = 0; c < cfg_.C; ++c)
        for (long y = 0; y < cfg_.H; ++y)
          for (long x = 0; x < cfg_.W; ++x)
            o[j * im.numel() + (y * cfg_.W + x) * im.Cp + c] =
                static_cast<float>(buf[static_cast<size_t>(((j * cfg_.C + c) * cfg_.H + y) * cfg_.W + x)]);
  });
  check_cuda(cudaMemcpy(data_.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice), "dataset upload");
}

int GanGroup::next_batch_size() const {
  long start = fresh_epoch_ ? 0 : at_;
  return static_cast<int>(std::min<long>(cfg_.batch, cfg_.per_label - start));
}

// Host half of a step for every label (in parallel): the epoch shuffle when
// one starts (std::shuffle on the label's engine, partition.cpp:91), the next
// contiguous batch, then z1 and z2 (gan.cpp:150,161).
void GanGroup::prep_host(int par, int B, bool with_idx) {
  const bool shuffle = fresh_epoch_;
  const long start = shuffle ? 0 : at_;
  int* hidx = h_idx_[par];
  float* hz = h_z_[par];
  const long dz = cfg_.d_z;
  pool_->parallel_for(L_, [&](int l) {
    Rng& r = rng_[static_cast<size_t>(l)];
    auto& ord = order_[static_cast<size_t>(l)];
    if (with_idx) {
      if (shuffle) std::shuffle(ord.begin(), ord.end(), r.engine());
      auto& lb = last_batch_[static_cast<size_t>(l)];
      lb.resize(static_cast<size_t>(B));
      for (int b = 0; b < B; ++b) {
        hidx[l * B + b] = ord[static_cast<size_t>(start + b)];
        lb[static_cast<size_t>(b)] = ord[static_cast<size_t>(start + b)];
      }
    }
    for (int k = 0; k < 2; ++k) {
      float* z = hz + (static_cast<size_t>(k) * L_ + l) * B * zcp_;
      for (int b = 0; b < B; ++b)
        for (long j = 0; j < dz; ++j) z[b * zcp_ + j] = static_cast<float>(r.normal());
    }
  });
  if (with_idx) {
    at_ = start + B;
    fresh_epoch_ = false;
    if (at_ >= cfg_.per_label) {
      epoch_ += 1;
      fresh_epoch_ = true;
      at_ = 0;
    }
  }
}

// The adversarial step (gan.cpp:136-176) for all labels, on st_.
static long long act_mask_bytes(const DevNet& net, int B) {
  long long n = 0;
  for (int i = 0; i < net.blocks(); ++i) {
    const Block& b = net.block(i);
    if (b.act == ACT_RELU || b.act == ACT_LRELU) n += static_cast<long long>(B) * b.out.C * b.out.H * b.out.W;
  }
  return n;
}

void GanGroup::enqueue_step(int B, const float* real_nhwc, int par, cudaEvent_t real_ready) {
  enqueue_step_kernels(B, real_nhwc, par, real_ready, d_rep_ + (steps_ % rep_cap_) * L_ * 4);
  steps_ += 1;
  pending_ += 1;
  if (pending_ >= rep_cap_) drain_reports();
}

// The kernels of one step (gan.cpp:136-176), enqueued on st_; reports to rep.
// With overlap on (PG_OVERLAP, default), both generator forwards -- they depend
// only on G's parameters, which the discriminator half of the step does not
// touch -- run on a second stream (z2 into its own trace): G(z1) beside
// D(real), G(z2) beside the whole discriminator update; st_ joins each before
// the pass that reads it.  The kernels and their order per network are
// unchanged, so results are bit-identical to the serial order.
void GanGroup::enqueue_step_kernels(int B, const float* real_nhwc, int par, cudaEvent_t real_ready, double* rep) {
  const int pstride = static_cast<int>(D_->out_map().Cp);
  const int nbg = G_->blocks(), nbd = D_->blocks();
  // mask capture (parity instrumentation): segment offsets in the order G z1, D real, D fake, G z2, D fake
  const long long gsz = capture_ ? act_mask_bytes(*G_, B) : 0, dsz = capture_ ? act_mask_bytes(*D_, B) : 0;
  // per-launch timing (bench.py's roofline pass) serialises the step: events
  // around a launch would otherwise also time whatever the other stream runs
  const bool ov = overlap_ && !gemm_timing_on();
  const Phase step_range("pg.step");
  cudaStream_t gs = ov ? st2_ : st_;
  Trace& tg2 = ov ? tg2_ : tg_;
  if (ov) {
    check_cuda(cudaEventRecord(ev_fork_, st_), "fork");
    check_cuda(cudaStreamWaitEvent(st2_, ev_fork_, 0), "fork wait");
  }
  // discriminator update on (real, fresh fake); the generator trace is dropped
  std::optional<Phase> phase(std::in_place, "pg.G_forward");
  tg_.act[0] = dz_[par][0].p;
  G_->forward(tg_, B, true, true, gs);
  if (capture_) capture_pass(*G_, tg_, B, 0, gs);
  if (ov) {
    check_cuda(cudaEventRecord(ev_g1_, st2_), "g1");
    // the generator step's forward (z2) right behind it, into its own trace
    tg2.act[0] = dz_[par][1].p;
    G_->forward(tg2, B, true, true, st2_);
    if (capture_) capture_pass(*G_, tg2, B, gsz + 2 * dsz, st2_);
    check_cuda(cudaEventRecord(ev_g2_, st2_), "g2");
  }
  phase.emplace("pg.D_update");
  tdr_.act[0] = const_cast<float*>(real_nhwc);
  if (real_ready) check_cuda(cudaStreamWaitEvent(st_, real_ready, 0), "wait real batch");
  D_->forward(tdr_, B, true, true, st_);
  if (capture_) capture_pass(*D_, tdr_, B, gsz, st_);
  if (ov) check_cuda(cudaStreamWaitEvent(st_, ev_g1_, 0), "join g1");
  tdf_.act[0] = tg_.act[static_cast<size_t>(nbg)];
  D_->forward(tdf_, B, true, true, st_);
  if (capture_) capture_pass(*D_, tdf_, B, gsz + dsz, st_);
  check_cuda(launch_loss_d(L_, B, tdr_.act[static_cast<size_t>(nbd)], tdf_.act[static_cast<size_t>(nbd)], pstride,
                           cfg_.clamp, gp_real_.p, gp_fake_.p, rep, st_),
             "loss_d");
  D_->backward(tdr_, B, gp_real_.p, true, false, nullptr, st_);
  D_->backward(tdf_, B, gp_fake_.p, true, true, nullptr, st_);
  check_cuda(launch_nonfinite_check(L_, D_->P(), D_->grads.p, d_flags_, st_), "nonfinite D");
  check_cuda(launch_adam_tick(L_, d_flags_, d_t_d_, st_), "tick D");
  check_cuda(launch_adam(L_, D_->P(), D_->params.p, D_->grads.p, D_->adam_m.p, D_->adam_v.p, d_t_d_, d_flags_,
                         static_cast<float>(cfg_.lr), cfg_.beta1, cfg_.beta2,
                         static_cast<float>(cfg_.eps), st_),
             "adam D");
  // generator update through the updated discriminator (its grads discarded)
  phase.emplace("pg.G_update");
  if (ov) {
    check_cuda(cudaStreamWaitEvent(st_, ev_g2_, 0), "join g2");
  } else {
    tg_.act[0] = dz_[par][1].p;
    G_->forward(tg_, B, true, true, st_);
    if (capture_) capture_pass(*G_, tg_, B, gsz + 2 * dsz, st_);
  }
  tdf_.act[0] = tg2.act[static_cast<size_t>(nbg)];
  D_->forward(tdf_, B, true, true, st_);
  if (capture_) {
    capture_pass(*D_, tdf_, B, 2 * gsz + 2 * dsz, st_);
    mask_len_ = 2 * gsz + 3 * dsz;
  }
  check_cuda(launch_loss_g(L_, B, tdf_.act[static_cast<size_t>(nbd)], pstride, cfg_.clamp, gp_fake_.p, rep, st_),
             "loss_g");
  D_->backward(tdf_, B, gp_fake_.p, false, false, gimg_.p, st_);
  G_->backward(tg2, B, gimg_.p, true, false, nullptr, st_);
  check_cuda(launch_nonfinite_check(L_, G_->P(), G_->grads.p, d_flags_, st_), "nonfinite G");
  check_cuda(launch_adam_tick(L_, d_flags_, d_t_g_, st_), "tick G");
  check_cuda(launch_adam(L_, G_->P(), G_->params.p, G_->grads.p, G_->adam_m.p, G_->adam_v.p, d_t_g_, d_flags_,
                         static_cast<float>(cfg_.lr), cfg_.beta1, cfg_.beta2,
                         static_cast<float>(cfg_.eps), st_),
             "adam G");
}

// One step of the device-resident worker protocol as a CUDA graph (the real
// batch gather and every kernel of the step), captured per (staging slot,
// batch size) once that batch size has run eagerly (so every grow-only buffer
// has its final size) and replayed afterwards: the c1 / c2 steps are a few
// hundred short kernels, launch-latency bound without it.  PG_GRAPH=0 (read at
// group creation) keeps the eager path.
bool GanGroup::launch_step_graph(int B, int par) {
  if (!use_graph_ || capture_ || B != graph_B_ready_ || gemm_timing_on()) return false;
  StepGraph& sg = graphs_[par];
  if (!sg.exec || sg.B != B) {
    if (sg.exec) {
      cudaGraphExecDestroy(sg.exec);
      sg.exec = nullptr;
    }
    const Map& im = D_->in_map();
    cudaGraph_t graph = nullptr;
    const long long n0 = launch_count();
    check_cuda(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "begin capture");
    check_cuda(launch_gather_real(L_, B, d_idx_[par], data_.p, static_cast<long long>(cfg_.per_label) * im.numel(),
                                  im.numel(), static_cast<int>(im.Cp), static_cast<int>(im.C), real_.p, st_),
               "gather");
    enqueue_step_kernels(B, real_.p, par, nullptr, d_rep_cur_);
    check_cuda(cudaStreamEndCapture(st_, &graph), "end capture");
    const cudaError_t e = cudaGraphInstantiate(&sg.exec, graph, 0);
    cudaGraphDestroy(graph);
    check_cuda(e, "graph instantiate");
    sg.B = B;
    sg.kernels = launch_count() - n0;
  } else {
    add_launches(sg.kernels);  // pg_launch_count counts the replayed kernels (bench.py gpu_launches)
  }
  check_cuda(cudaGraphLaunch(sg.exec, st_), "graph launch");
  check_cuda(cudaMemcpyAsync(d_rep_ + (steps_ % rep_cap_) * L_ * 4, d_rep_cur_, sizeof(double) * L_ * 4,
                             cudaMemcpyDeviceToDevice, st_),
             "reports");
  steps_ += 1;
  pending_ += 1;
  if (pending_ >= rep_cap_) drain_reports();
  return true;
}

void GanGroup::capture_masks(bool on) {
  sync();
  capture_ = on;
  graph_B_ready_ = 0;
  mask_len_ = 0;
  if (on && !d_mask_) {
    const int Bmax = static_cast<int>(std::min<long>(cfg_.batch, cfg_.per_label));
    mask_stride_ = 2 * act_mask_bytes(*G_, Bmax) + 3 * act_mask_bytes(*D_, Bmax);
    d_mask_ = dev_alloc<unsigned char>(static_cast<size_t>(L_) * std::max<long long>(mask_stride_, 1));
  }
}

long long GanGroup::capture_pass(DevNet& net, Trace& t, int B, long long off, cudaStream_t st) {
  for (int i = 0; i < net.blocks(); ++i) {
    const Block& b = net.block(i);
    if (b.act != ACT_RELU && b.act != ACT_LRELU) continue;
    check_cuda(launch_mask_capture(L_, B, static_cast<int>(b.out.H), static_cast<int>(b.out.W),
                                   static_cast<int>(b.out.C), static_cast<int>(b.out.Cp),
                                   static_cast<long long>(B) * b.out.numel(), t.act[static_cast<size_t>(i) + 1], b.act,
                                   d_mask_ + off, mask_stride_, st),
               "mask capture");
    off += static_cast<long long>(B) * b.out.C * b.out.H * b.out.W;
  }
  return off;
}

long GanGroup::get_masks(int label, unsigned char* out, long cap) {
  if (label < 0 || label >= L_) throw std::out_of_range("label index " + std::to_string(label));
  sync();
  if (out && mask_len_ > 0) {
    if (cap < mask_len_) throw std::invalid_argument("output buffer too small");
    check_cuda(cudaMemcpy(out, d_mask_ + static_cast<size_t>(label) * mask_stride_, static_cast<size_t>(mask_len_),
                          cudaMemcpyDeviceToHost),
               "masks D2H");
  }
  return static_cast<long>(mask_len_);
}

void GanGroup::drain_reports() {
  if (pending_ == 0) return;
  check_cuda(cudaStreamSynchronize(st_), "sync");
  check_cuda(cudaMemcpy(h_rep_, d_rep_, static_cast<size_t>(rep_cap_) * L_ * 4 * sizeof(double), cudaMemcpyDeviceToHost),
             "reports D2H");
  for (long s = steps_ - pending_; s < steps_; ++s) {
    const double* r = h_rep_ + (s % rep_cap_) * L_ * 4;
    for (int l = 0; l < L_; ++l)
      reports_[static_cast<size_t>(l)].push_back(StepReport{r[l * 4], r[l * 4 + 1], r[l * 4 + 2], r[l * 4 + 3]});
  }
  pending_ = 0;
}

int GanGroup::train_steps(int n) {
  const Map& im = D_->in_map();
  int done = 0;
  check_cuda(cudaEventRecord(t0_, st_), "event");
  for (int s = 0; s < n; ++s) {
    if (epoch_ >= cfg_.epochs) break;
    const int par = static_cast<int>(steps_ & 1);
    const int B = next_batch_size();
    // the staging slot `par` was last read by the copies of two steps ago
    check_cuda(cudaEventSynchronize(staged_[par]), "staging wait");
    prep_host(par, B, true);
    check_cuda(cudaMemcpyAsync(d_idx_[par], h_idx_[par], sizeof(int) * L_ * B, cudaMemcpyHostToDevice, st_), "idx H2D");
    const size_t zb = sizeof(float) * static_cast<size_t>(L_) * B * zcp_;
    check_cuda(cudaMemcpyAsync(dz_[par][0].p, h_z_[par], zb, cudaMemcpyHostToDevice, st_), "z1 H2D");
    check_cuda(cudaMemcpyAsync(dz_[par][1].p, h_z_[par] + static_cast<size_t>(L_) * B * zcp_, zb,
                               cudaMemcpyHostToDevice, st_),
               "z2 H2D");
    check_cuda(cudaEventRecord(staged_[par], st_), "event");
    if (!launch_step_graph(B, par)) {
      check_cuda(launch_gather_real(L_, B, d_idx_[par], data_.p, static_cast<long long>(cfg_.per_label) * im.numel(),
                                    im.numel(), static_cast<int>(im.Cp), static_cast<int>(im.C), real_.p, st_),
                 "gather");
      enqueue_step(B, real_.p, par);
      if (!capture_) graph_B_ready_ = B;  // buffers now sized for B: later steps of this size may be captured
    }
    ++done;
  }
  check_cuda(cudaEventRecord(t1_, st_), "event");
  check_cuda(cudaEventSynchronize(t1_), "sync");
  check_cuda(cudaEventElapsedTime(&last_ms_, t0_, t1_), "elapsed");
  drain_reports();
  return done;
}

// The host real batch goes up on the copy stream while the generator's forward
// (which only needs z1) runs: H2D into the gradient scratch (same extent, idle
// until the generator step), NCHW -> NHWC with 2x-1, then real_ready_, which
// the discriminator's forward on the real batch waits for.  Callers end every
// step with a stream sync, so both buffers are free here.
void GanGroup::stage_real_async(const float* real01, int B) {
  const Map& im = D_->in_map();
  const size_t rb = sizeof(float) * static_cast<size_t>(L_) * B * cfg_.C * cfg_.H * cfg_.W;
  check_cuda(cudaMemcpyAsync(gimg_.p, real01, rb, cudaMemcpyHostToDevice, cst_), "real H2D");
  check_cuda(launch_nchw01_to_nhwc(static_cast<long long>(L_) * B, static_cast<int>(cfg_.C), static_cast<int>(cfg_.H),
                                   static_cast<int>(cfg_.W), static_cast<int>(im.Cp), gimg_.p, real_.p, cst_),
             "real layout");
  check_cuda(cudaEventRecord(real_ready_, cst_), "event");
}

void GanGroup::train_step_host(const float* real01, int B, double* reports) {
  if (B < 1 || B > std::min<long>(cfg_.batch, cfg_.per_label)) throw std::invalid_argument("train_step: batch size out of range");
  const Map& im = D_->in_map();
  const int par = static_cast<int>(steps_ & 1);
  check_cuda(cudaEventSynchronize(staged_[par]), "staging wait");
  prep_host(par, B, false);
  const size_t zb = sizeof(float) * static_cast<size_t>(L_) * B * zcp_;
  check_cuda(cudaMemcpyAsync(dz_[par][0].p, h_z_[par], zb, cudaMemcpyHostToDevice, st_), "z1 H2D");
  check_cuda(cudaMemcpyAsync(dz_[par][1].p, h_z_[par] + static_cast<size_t>(L_) * B * zcp_, zb, cudaMemcpyHostToDevice,
                             st_),
             "z2 H2D");
  check_cuda(cudaEventRecord(staged_[par], st_), "event");
  stage_real_async(real01, B);
  enqueue_step(B, real_.p, par, real_ready_);
  drain_reports();
  if (reports)
    for (int l = 0; l < L_; ++l) {
      const StepReport& r = reports_[static_cast<size_t>(l)].back();
      reports[l * 4 + 0] = r.j_d;
      reports[l * 4 + 1] = r.j_g;
      reports[l * 4 + 2] = r.d_real_mean;
      reports[l * 4 + 3] = r.d_fake_mean;
    }
}

void GanGroup::train_step_inputs(const float* real01, const float* z1, const float* z2, int B, double* reports) {
  if (B < 1 || B > std::min<long>(cfg_.batch, cfg_.per_label)) throw std::invalid_argument("train_step: batch size out of range");
  const Map& im = D_->in_map();
  const int par = static_cast<int>(steps_ & 1);
  check_cuda(cudaEventSynchronize(staged_[par]), "staging wait");
  float* hz = h_z_[par];
  for (int k = 0; k < 2; ++k) {
    const float* src = k == 0 ? z1 : z2;
    for (long r = 0; r < static_cast<long>(L_) * B; ++r)
      for (long j = 0; j < zcp_; ++j)
        hz[(static_cast<size_t>(k) * L_ * B + r) * zcp_ + j] = j < cfg_.d_z ? src[r * cfg_.d_z + j] : 0.f;
  }
  const size_t zb = sizeof(float) * static_cast<size_t>(L_) * B * zcp_;
  check_cuda(cudaMemcpyAsync(dz_[par][0].p, hz, zb, cudaMemcpyHostToDevice, st_), "z1 H2D");
  check_cuda(cudaMemcpyAsync(dz_[par][1].p, hz + static_cast<size_t>(L_) * B * zcp_, zb, cudaMemcpyHostToDevice, st_),
             "z2 H2D");
  check_cuda(cudaEventRecord(staged_[par], st_), "event");
  stage_real_async(real01, B);
  enqueue_step(B, real_.p, par, real_ready_);
  drain_reports();
  if (reports)
    for (int l = 0; l < L_; ++l) {
      const StepReport& r = reports_[static_cast<size_t>(l)].back();
      reports[l * 4 + 0] = r.j_d;
      reports[l * 4 + 1] = r.j_g;
      reports[l * 4 + 2] = r.d_real_mean;
      reports[l * 4 + 3] = r.d_fake_mean;
    }
}

void GanGroup::sync() {
  check_cuda(cudaStreamSynchronize(st_), "sync");
  drain_reports();
}

std::vector<int> GanGroup::failed() {
  sync();
  std::vector<int> f(static_cast<size_t>(L_));
  check_cuda(cudaMemcpy(f.data(), d_flags_, sizeof(int) * L_, cudaMemcpyDeviceToHost), "flags");
  return f;
}

long GanGroup::get(int label, int what, double* out, long cap) {
  if (label < 0 || label >= L_) throw std::out_of_range("label index " + std::to_string(label));
  sync();
  auto fetch = [&](DevNet& net, const DeviceBuf& arena, bool buffers) -> long {
    long n = buffers ? net.ref_buffers() : net.ref_params();
    if (!out) return n;
    if (cap < n) throw std::invalid_argument("output buffer too small");
    long long per = buffers ? std::max<long long>(net.Bf(), 4) : net.P();
    std::vector<float> h(static_cast<size_t>(per));
    check_cuda(cudaMemcpy(h.data(), arena.p + static_cast<size_t>(label) * per, per * sizeof(float), cudaMemcpyDeviceToHost),
               "readback");
    if (buffers) net.export_buffers(h.data(), out);
    else net.export_params(h.data(), out);
    return n;
  };
  switch (what) {
    case G_PARAMS: return fetch(*G_, G_->params, false);
    case D_PARAMS: return fetch(*D_, D_->params, false);
    case G_BUFFERS: return fetch(*G_, G_->running, true);
    case D_BUFFERS: return fetch(*D_, D_->running, true);
    case G_GRADS: return fetch(*G_, G_->grads, false);
    case D_GRADS: return fetch(*D_, D_->grads, false);
    case G_M: return fetch(*G_, G_->adam_m, false);
    case G_V: return fetch(*G_, G_->adam_v, false);
    case D_M: return fetch(*D_, D_->adam_m, false);
    case D_V: return fetch(*D_, D_->adam_v, false);
    case REPORTS: {
      const auto& r = reports_[static_cast<size_t>(label)];
      long n = static_cast<long>(r.size()) * 4;
      if (out) {
        if (cap < n) throw std::invalid_argument("output buffer too small");
        for (size_t i = 0; i < r.size(); ++i) {
          out[i * 4] = r[i].j_d;
          out[i * 4 + 1] = r[i].j_g;
          out[i * 4 + 2] = r[i].d_real_mean;
          out[i * 4 + 3] = r[i].d_fake_mean;
        }
      }
      return n;
    }
    case LAST_BATCH: {
      const auto& b = last_batch_[static_cast<size_t>(label)];
      if (out) {
        if (cap < static_cast<long>(b.size())) throw std::invalid_argument("output buffer too small");
        for (size_t i = 0; i < b.size(); ++i) out[i] = static_cast<double>(b[i]);
      }
      return static_cast<long>(b.size());
    }
    case COUNTERS: {
      long long tg = 0, td = 0;
      check_cuda(cudaMemcpy(&tg, d_t_g_ + label, sizeof(tg), cudaMemcpyDeviceToHost), "t");
      check_cuda(cudaMemcpy(&td, d_t_d_ + label, sizeof(td), cudaMemcpyDeviceToHost), "t");
      if (out) {
        if (cap < 3) throw std::invalid_argument("output buffer too small");
        out[0] = static_cast<double>(tg);
        out[1] = static_cast<double>(td);
        out[2] = static_cast<double>(steps_);
      }
      return 3;
    }
  }
  throw std::invalid_argument("unknown field code " + std::to_string(what));
}

void GanGroup::set(int label, int what, const double* in, long n) {
  if (label < 0 || label >= L_) throw std::out_of_range("label index " + std::to_string(label));
  sync();
  auto put = [&](DevNet& net, DeviceBuf& arena, bool buffers) {
    long want = buffers ? net.ref_buffers() : net.ref_params();
    if (n != want) throw std::invalid_argument("length mismatch on set");
    long long per = buffers ? std::max<long long>(net.Bf(), 4) : net.P();
    std::vector<float> h(static_cast<size_t>(per));
    if (buffers) net.import_buffers(in, h.data());
    else net.import_params(in, h.data());
    check_cuda(cudaMemcpy(arena.p + static_cast<size_t>(label) * per, h.data(), per * sizeof(float), cudaMemcpyHostToDevice),
               "upload");
  };
  switch (what) {
    case G_PARAMS: put(*G_, G_->params, false); return;
    case D_PARAMS: put(*D_, D_->params, false); return;
    case G_BUFFERS: put(*G_, G_->running, true); return;
    case D_BUFFERS: put(*D_, D_->running, true); return;
    case G_M: put(*G_, G_->adam_m, false); return;
    case G_V: put(*G_, G_->adam_v, false); return;
    case D_M: put(*D_, D_->adam_m, false); return;
    case D_V: put(*D_, D_->adam_v, false); return;
    case COUNTERS: {
      // Adam step counters of this label; the step count is group-wide (labels advance in lockstep)
      if (n != 3) throw std::invalid_argument("length mismatch on set");
      const long long tg = static_cast<long long>(in[0]), td = static_cast<long long>(in[1]);
      check_cuda(cudaMemcpy(d_t_g_ + label, &tg, sizeof(tg), cudaMemcpyHostToDevice), "t");
      check_cuda(cudaMemcpy(d_t_d_ + label, &td, sizeof(td), cudaMemcpyHostToDevice), "t");
      steps_ = static_cast<long>(in[2]);
      return;
    }
  }
  throw std::invalid_argument("field not settable: " + std::to_string(what));
}

// eval-mode generator over all labels in rounds of up to Bmax samples;
// fill_z(l, B, done, z) writes label l's B latents (padded rows of zcp_)
void GanGroup::generate_rounds(long n, const std::function<void(int, int, long, float*)>& fill_z, float* out) {
  sync();
  const int Bmax = static_cast<int>(std::min<long>(cfg_.batch, cfg_.per_label));
  const Map& om = G_->out_map();
  const long S = cfg_.C * cfg_.H * cfg_.W;
  DeviceBuf o(static_cast<size_t>(L_) * Bmax * S);
  std::vector<float> zh(static_cast<size_t>(L_) * Bmax * zcp_, 0.f), oh(o.n);
  for (long done = 0; done < n; done += Bmax) {
    const int B = static_cast<int>(std::min<long>(Bmax, n - done));
    pool_->parallel_for(L_, [&](int l) { fill_z(l, B, done, zh.data() + static_cast<size_t>(l) * B * zcp_); });
    check_cuda(cudaMemcpyAsync(dz_[0][0].p, zh.data(), sizeof(float) * L_ * B * zcp_, cudaMemcpyHostToDevice, st_), "z");
    tg_.act[0] = dz_[0][0].p;
    G_->forward(tg_, B, false, false, st_);
    check_cuda(launch_nhwc_to_nchw01(static_cast<long long>(L_) * B, static_cast<int>(cfg_.C), static_cast<int>(cfg_.H),
                                     static_cast<int>(cfg_.W), static_cast<int>(om.Cp),
                                     tg_.act[static_cast<size_t>(G_->blocks())], o.p, st_),
               "to nchw");
    check_cuda(cudaMemcpyAsync(oh.data(), o.p, sizeof(float) * L_ * B * S, cudaMemcpyDeviceToHost, st_), "samples D2H");
    check_cuda(cudaStreamSynchronize(st_), "sync");
    for (int l = 0; l < L_; ++l)
      std::memcpy(out + (static_cast<size_t>(l) * n + done) * S, oh.data() + static_cast<size_t>(l) * B * S,
                  sizeof(float) * B * S);
  }
}

void GanGroup::generate(long n, uint64_t seed, float* out) {
  std::vector<Rng> rs;
  for (int l = 0; l < L_; ++l) rs.emplace_back(derive_seed(seed, static_cast<uint64_t>(cfg_.class_ids[static_cast<size_t>(l)])));
  generate_rounds(n, [&](int l, int B, long, float* z) {
    for (int b = 0; b < B; ++b)
      for (long j = 0; j < zcp_; ++j) z[b * zcp_ + j] = j < cfg_.d_z ? static_cast<float>(rs[static_cast<size_t>(l)].normal()) : 0.f;
  }, out);
}

void GanGroup::generate_latents(const float* zin, long n, float* out) {
  if (n < 1) throw std::invalid_argument("generate: n must be >= 1");
  generate_rounds(n, [&](int l, int B, long done, float* z) {
    for (int b = 0; b < B; ++b)
      for (long j = 0; j < zcp_; ++j)
        z[b * zcp_ + j] = j < cfg_.d_z ? zin[(static_cast<size_t>(l) * n + done + b) * cfg_.d_z + j] : 0.f;
  }, out);
}

void GanGroup::mixture_sample(const double* priors, long n, uint64_t seed, float* out, int* ids) {
  if (n < 1) throw std::invalid_argument("mixture_sample: n must be >= 1");
  sync();
  const int k = L_;
  Rng rng(seed);
  // 1) class ids from one stream (partition.cpp:192-205); a single pair draws none
  if (k == 1) {
    std::fill(ids, ids + n, 0);
  } else {
    std::vector<double> cdf(static_cast<size_t>(k));
    double acc = 0;
    for (int j = 0; j < k; ++j) cdf[static_cast<size_t>(j)] = (acc += priors[j]);
    for (long i = 0; i < n; ++i) {
      const double u = rng.uniform();
      int j = 0;
      while (j + 1 < k && u >= cdf[static_cast<size_t>(j)]) ++j;
      ids[i] = j;
    }
  }
  // 2) per class, in class order, the latents of its samples from the same
  //    stream (generate -> sample_latent, gan.cpp:54-84,197-201)
  std::vector<std::vector<long>> where(static_cast<size_t>(k));
  for (long i = 0; i < n; ++i) where[static_cast<size_t>(ids[i])].push_back(i);
  std::vector<std::vector<float>> z(static_cast<size_t>(k));
  long most = 0;
  for (int j = 0; j < k; ++j) {
    const long c = static_cast<long>(where[static_cast<size_t>(j)].size());
    most = std::max(most, c);
    z[static_cast<size_t>(j)].resize(static_cast<size_t>(c * cfg_.d_z));
    for (auto& v : z[static_cast<size_t>(j)]) v = static_cast<float>(rng.normal());
  }
  // 3) device: all labels' generators in lockstep rounds of up to Bmax samples
  const int Bmax = static_cast<int>(std::min<long>(cfg_.batch, cfg_.per_label));
  const Map& om = G_->out_map();
  const long S = cfg_.C * cfg_.H * cfg_.W;
  DeviceBuf o(static_cast<size_t>(L_) * Bmax * S);
  std::vector<float> zh(static_cast<size_t>(L_) * Bmax * zcp_), oh(o.n);
  for (long done = 0; done < most; done += Bmax) {
    const int B = static_cast<int>(std::min<long>(Bmax, most - done));
    std::fill(zh.begin(), zh.end(), 0.f);
    for (int l = 0; l < L_; ++l) {
      const long c = static_cast<long>(where[static_cast<size_t>(l)].size());
      for (int b = 0; b < B && done + b < c; ++b)
        std::memcpy(&zh[(static_cast<size_t>(l) * B + b) * zcp_], &z[static_cast<size_t>(l)][(done + b) * cfg_.d_z],
                    sizeof(float) * cfg_.d_z);
    }
    check_cuda(cudaMemcpyAsync(dz_[0][0].p, zh.data(), sizeof(float) * L_ * B * zcp_, cudaMemcpyHostToDevice, st_), "z");
    tg_.act[0] = dz_[0][0].p;
    G_->forward(tg_, B, false, false, st_);
    check_cuda(launch_nhwc_to_nchw01(static_cast<long long>(L_) * B, static_cast<int>(cfg_.C), static_cast<int>(cfg_.H),
                                     static_cast<int>(cfg_.W), static_cast<int>(om.Cp),
                                     tg_.act[static_cast<size_t>(G_->blocks())], o.p, st_),
               "to nchw");
    check_cuda(cudaMemcpyAsync(oh.data(), o.p, sizeof(float) * L_ * B * S, cudaMemcpyDeviceToHost, st_), "samples D2H");
    check_cuda(cudaStreamSynchronize(st_), "sync");
    for (int l = 0; l < L_; ++l) {
      const auto& wl = where[static_cast<size_t>(l)];
      for (int b = 0; b < B && done + b < static_cast<long>(wl.size()); ++b)
        std::memcpy(out + wl[static_cast<size_t>(done + b)] * S, oh.data() + (static_cast<size_t>(l) * B + b) * S,
                    sizeof(float) * S);
    }
  }
}

}  // namespace pg
