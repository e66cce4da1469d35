// Label group trainer: the B200 form of partgan's worker loop and adversarial
// step for all L labels resident on one GPU.
//
//   reference                                   here
//   run_worker (partition.cpp:78-112)           GanGroup: one Rng + shuffle order per label, host side
//   train_step / step_impl (gan.cpp:136-182)    GanGroup::enqueue_step: the same D-then-G sequence, every
//                                               kernel batched over the L labels in lockstep
//   adam_step (optim.cpp:20-34)                 non-finite check + Adam over the [L][P] arenas
//   TrainError (partition.hpp:63-69)            per-label failure flags (a label whose gradients went
//                                               non-finite stops updating, exactly like a failed worker)
//
// Labels never exchange data; grouping changes the launch shape, not the math.
#pragma once

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "host_util.hpp"
#include "net.hpp"
#include "rng.hpp"

namespace pg {

struct GroupConfig {
  std::string gen_spec, disc_spec;
  long C = 1, H = 28, W = 28;
  long d_z = 100;
  std::vector<int> class_ids;  // labels of this group
  uint64_t base_seed = 1;      // worker seed = derive_seed(base_seed, class_id)  (run.cpp:376)
  std::vector<uint64_t> seeds; // explicit per-label worker seeds (WorkerConfig::seed); overrides base_seed
  int batch = 64;
  int epochs = 1;
  long per_label = 64;         // shard size of every label
  double lr = 2e-4, beta1 = 0.5, beta2 = 0.999, eps = 1e-8;
  double clamp = 1e-7, init_std = 0.02;
  int math = MATH_FP32_SIMT;
  int threads = 8;
};

struct StepReport {
  double j_d = 0, j_g = 0, d_real_mean = 0, d_fake_mean = 0;
};

class GanGroup {
 public:
  explicit GanGroup(const GroupConfig& cfg);
  ~GanGroup();

  int L() const { return L_; }
  const GroupConfig& config() const { return cfg_; }
  DevNet& gen() { return *G_; }
  DevNet& disc() { return *D_; }
  cudaStream_t stream() const { return st_; }

  // dataset: [L][per_label][C][H][W] in [0,1] (host, f32) -> device NHWC
  void set_dataset(const float* images01);
  void generate_dataset(uint64_t data_seed);

  // the worker protocol on the device-resident dataset: per label shuffle at
  // each epoch start, contiguous batches (partial tail kept), z1 then z2.
  // Returns the number of steps actually run (stops when every epoch is done).
  int train_steps(int n);
  // steps on host-provided real batches (the reference train_step call):
  // real01 [L][B][C][H][W] in [0,1]; latents from each label's stream.
  void train_step_host(const float* real01, int B, double* reports);
  // fully explicit inputs (no stream use): z1, z2 [L][B][d_z]
  void train_step_inputs(const float* real01, const float* z1, const float* z2, int B, double* reports);

  // reference-layout readback of one label (f64)
  enum Field { G_PARAMS = 0, D_PARAMS, G_BUFFERS, D_BUFFERS, G_GRADS, D_GRADS, G_M, G_V, D_M, D_V, REPORTS, LAST_BATCH, COUNTERS };
  long get(int label, int what, double* out, long cap);
  void set(int label, int what, const double* in, long n);
  std::vector<int> failed();
  // eval-mode samples: n per label with latents from Rng(derive_seed(seed, class_id)),
  // (v+1)/2 mapped, out [L][n][C][H][W]
  void generate(long n, uint64_t seed, float* out);
  // eval-mode samples from given latents z [L][n][d_z] (generate's device half), out [L][n][C][H][W]
  void generate_latents(const float* z, long n, float* out);
  // mixture_sample (partition.cpp:182-227) over the group's labels in order:
  // class ids and latents drawn on the host from Rng(seed) in the reference
  // order, eval-mode generators on the device; out [n][C][H][W] in [0,1]
  void mixture_sample(const double* priors, long n, uint64_t seed, float* out, int* ids);
  void sync();
  long steps_done() const { return steps_; }

  // Parity instrumentation: when on, every step records the ReLU / LeakyReLU
  // masks of its five forward passes (G z1, D real, D fake, G z2, D fake; each
  // activation layer [B][C][H][W] in the reference's order) so a CPU oracle can
  // replay the same activation decisions (oracle MaskTape).  Off by default.
  void capture_masks(bool on);
  // bytes of the last step's masks for one label (out may be null to query)
  long get_masks(int label, unsigned char* out, long cap);

  // time of the last train_steps() call on the device (ms, CUDA events)
  float last_device_ms() const { return last_ms_; }

 private:
  GroupConfig cfg_;
  int L_;
  std::unique_ptr<DevNet> G_, D_;
  Trace tg_, tdr_, tdf_;
  cudaStream_t st_ = nullptr;
  cudaStream_t cst_ = nullptr;      // host batch uploads, overlapped with the generator's forward
  cudaEvent_t real_ready_ = nullptr;
  DeviceBuf data_, dz_[2][2], real_, gp_real_, gp_fake_, gimg_;
  int* d_idx_[2] = {nullptr, nullptr};
  int* d_flags_ = nullptr;
  long long* d_t_g_ = nullptr;
  long long* d_t_d_ = nullptr;
  double* d_rep_ = nullptr;
  // pinned staging
  int* h_idx_[2] = {nullptr, nullptr};
  float* h_z_[2] = {nullptr, nullptr};
  double* h_rep_ = nullptr;
  long rep_cap_ = 0;
  cudaEvent_t staged_[2] = {nullptr, nullptr};
  cudaEvent_t t0_ = nullptr, t1_ = nullptr;
  std::unique_ptr<ThreadPool> pool_;
  // per-label host state (run_worker)
  std::vector<Rng> rng_;
  std::vector<std::vector<int>> order_;
  std::vector<std::vector<long>> last_batch_;
  int epoch_ = 0;
  long at_ = 0;
  bool fresh_epoch_ = true;
  long steps_ = 0, pending_ = 0;
  std::vector<std::vector<StepReport>> reports_;
  float last_ms_ = 0.f;
  long zcp_ = 0;  // padded latent width

  bool capture_ = false;
  unsigned char* d_mask_ = nullptr;
  long long mask_stride_ = 0;  // bytes per label
  long long mask_len_ = 0;     // bytes per label used by the last step
  long long capture_pass(DevNet& net, Trace& t, int B, long long off, cudaStream_t st);
  // generator forwards on a second stream (see enqueue_step_kernels)
  bool overlap_ = true;
  cudaStream_t st2_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_g1_ = nullptr, ev_g2_ = nullptr;
  Trace tg2_;

  uint64_t worker_seed(int l) const;
  void generate_rounds(long n, const std::function<void(int, int, long, float*)>& fill_z, float* out);
  int next_batch_size() const;
  void prep_host(int par, int B, bool with_idx);
  void enqueue_step(int B, const float* real_nhwc, int par, cudaEvent_t real_ready = nullptr);
  void enqueue_step_kernels(int B, const float* real_nhwc, int par, cudaEvent_t real_ready, double* rep);
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    int B = 0;
    long long kernels = 0;
  };
  StepGraph graphs_[2];
  bool use_graph_ = true;
  int graph_B_ready_ = 0;        // batch size whose buffers are grown (eager step done)
  double* d_rep_cur_ = nullptr;  // the graph's report slot (copied into the ring after each replay)
  bool launch_step_graph(int B, int par);
  void stage_real_async(const float* real01, int B);
  void drain_reports();
};

// checkpoint.cpp: one label's pair in the reference file format
// (src/checkpoint.cpp:91-194 save_gan_pair / load_gan_pair)
void save_checkpoint(GanGroup& grp, int label, const std::string& path);
void load_checkpoint(GanGroup& grp, int label, const std::string& path);

}  // namespace pg
