/* pg_trainer.h — trainer-level C-ABI: the B200 drop-in for partgan's
 * make_gan_pair / train_step / run_worker / generate on a group of labels
 * resident on one GPU.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   make_gan_pair            include/partgan/gan.hpp:39-42,  src/gan.cpp:27-52
 *   train_step               include/partgan/gan.hpp:75,     src/gan.cpp:136-182
 *   run_worker protocol      src/partition.cpp:78-112 (per-label Rng, epoch shuffle, batches with tail)
 *   generate                 include/partgan/gan.hpp:83,     src/gan.cpp:197-201
 *   Network::params/buffers  include/partgan/network.hpp:33-38 (reference flat f64 layout on readback)
 *   AdamState m/v/t          include/partgan/optim.hpp:15-23
 *   TrainError               include/partgan/partition.hpp:63-69 (per-label failure flags)
 * train_distributed (partition.hpp:75-76) is composed above this ABI: one
 * group per GPU, labels sharded in balanced contiguous blocks, and a final
 * NCCL gather (paper_2102_10485_b200/distributed.py).
 */
#ifndef PG_TRAINER_H
#define PG_TRAINER_H

#include <stdint.h>

#include "pg_kernels.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pg_group pg_group;

typedef struct {
  const char* gen_spec;   /* layer list text, e.g. "dense 100 8192; reshape 512 4 4; bn 512; relu; ..." */
  const char* disc_spec;
  int C, H, W;            /* image shape */
  int d_z;                /* latent width (LatentSpec::d_z); unconditional (d_y = 0), as in distributed mode */
  int n_labels;
  const int* class_ids;   /* [n_labels] */
  uint64_t base_seed;     /* worker seed = derive_seed(base_seed, class_id)  (run.cpp:376) */
  int batch;              /* WorkerConfig::batch_size */
  int epochs;
  long per_label;         /* shard size (images per label) */
  double lr, beta1, beta2, eps;
  double clamp;           /* GanPair::prob_clamp */
  double init_std;
  int math;               /* PG_MATH_* */
  int threads;            /* host threads for per-label RNG work */
  int device;             /* CUDA device ordinal */
  const uint64_t* seeds;  /* optional [n_labels] worker seeds (WorkerConfig::seed, partition.hpp:34);
                             NULL: derive_seed(base_seed, class_id) */
} pg_group_config;

/* Fields for pg_group_get / pg_group_set (reference layouts, f64). */
enum {
  PG_F_GEN_PARAMS = 0, PG_F_DISC_PARAMS = 1, PG_F_GEN_BUFFERS = 2, PG_F_DISC_BUFFERS = 3,
  PG_F_GEN_GRADS = 4, PG_F_DISC_GRADS = 5, PG_F_GEN_ADAM_M = 6, PG_F_GEN_ADAM_V = 7,
  PG_F_DISC_ADAM_M = 8, PG_F_DISC_ADAM_V = 9, PG_F_REPORTS = 10, PG_F_LAST_BATCH = 11, PG_F_COUNTERS = 12
};

int pg_group_create(const pg_group_config* cfg, pg_group** out);
void pg_group_destroy(pg_group* g);
/* dataset: images01 [n_labels][per_label][C][H][W] host f32 in [0,1], label-blocked in shard order */
int pg_group_set_dataset(pg_group* g, const float* images01);
/* the cosine-field synthetic dataset, generated on host threads */
int pg_group_generate_dataset(pg_group* g, uint64_t data_seed);
/* n steps of the worker protocol over the device-resident dataset; returns steps run (<0 on error) */
int pg_group_train_steps(pg_group* g, int n_steps);
/* one train_step on host batches: real01 [n_labels][B][C][H][W]; latents drawn from each
 * label's stream; reports [n_labels][4] = {j_d, j_g, d_real_mean, d_fake_mean} */
int pg_group_train_step(pg_group* g, const float* real01, int B, double* reports);
/* one step with explicit latents z1, z2 [n_labels][B][d_z] (no stream use) */
int pg_group_train_step_inputs(pg_group* g, const float* real01, const float* z1, const float* z2, int B,
                               double* reports);
/* reference-layout readback; returns element count (out may be NULL to query), <0 on error */
long pg_group_get(pg_group* g, int label_index, int field, double* out, long cap);
int pg_group_set(pg_group* g, int label_index, int field, const double* in, long n);
/* failed[n_labels]: 1 where a non-finite gradient was rejected (TrainError.failed_classes) */
int pg_group_failed(pg_group* g, int* failed);
/* eval-mode samples for every label: latents from Rng(derive_seed(seed, class_id)); out [n_labels][n][C][H][W] in [0,1] */
int pg_group_generate(pg_group* g, long n, uint64_t seed, float* out);
/* generate (gan.cpp:197-201) on caller-drawn latents z [n_labels][n][d_z]: out [n_labels][n][C][H][W] in [0,1] */
int pg_group_generate_latents(pg_group* g, const float* z, long n, float* out);
/* mixture_sample (include/partgan/partition.hpp, src/partition.cpp:182-227) over the
 * group's labels in order: priors[n_labels]; class ids then per-class latents drawn
 * from Rng(seed) exactly as the reference; out [n][C][H][W] in [0,1], ids[n] */
/* one label's (G, D) pair to / from a checkpoint file in the reference format
 * (src/checkpoint.cpp:91-194 save_gan_pair / load_gan_pair: u32 LE header length,
 * JSON header, f64 LE blobs gen_params, gen_buffers, disc_params, disc_buffers,
 * opt_g_m, opt_g_v, opt_d_m, opt_d_v); load requires the group's architecture */
int pg_group_save_checkpoint(pg_group* g, int label_idx, const char* path);
int pg_group_load_checkpoint(pg_group* g, int label_idx, const char* path);
int pg_group_mixture_sample(pg_group* g, const double* priors, long n, uint64_t seed, float* out, int* ids);
/* Parity instrumentation (off by default; costs one small pass per activation
 * layer when on): record the ReLU / LeakyReLU masks of every step's five
 * forward passes (G on z1, D on real, D on fake, G on z2, D on fake), each
 * activation layer as bytes [B][C][H][W] (1 = positive branch, the
 * reference's x > 0 / x >= 0 at network.cpp:384-391).  A CPU oracle replays
 * them to compare gradients without activation-kink discontinuities. */
int pg_group_capture_masks(pg_group* g, int on);
/* the last step's masks of one label; returns the byte count (out may be NULL) */
long pg_group_get_masks(pg_group* g, int label_idx, uint8_t* out, long cap);
/* device time (ms, CUDA events) of the last pg_group_train_steps call */
float pg_group_last_ms(pg_group* g);
int pg_group_sync(pg_group* g);
/* parameter counts: out[4] = {gen ref params, disc ref params, gen device arena, disc device arena} */
int pg_group_sizes(pg_group* g, long long* out);

/* Helpers shared with the reference protocol. */
/* Evaluation of generated samples (host, f64; reference src/eval.cpp):
 * softmax_rows (eval.cpp:18-33), inception_score (43-94: split_scores[n_splits],
 * mean, stddev), anova_f over groups given as concatenated values + sizes[k]
 * (158-186, +inf when the within-group variance is 0), anova_per_channel over
 * images [n][C][H][W] with labels[n] (188-211, f[C]) */
int pg_softmax_rows(const double* logits, long n, long k, double* probs);
int pg_inception_score(const double* probs, long n, long k, int n_splits, double* split_scores, double* mean,
                       double* stddev);
int pg_anova_f(const double* values, const long* sizes, long k, double* f);
int pg_anova_per_channel(const float* images, const int* labels, long n, long C, long H, long W, long k, double* f);
uint64_t pg_derive_seed(uint64_t base, uint64_t stream_id);
/* GPU g of n_gpus owns labels [pg_shard_begin(n, P, g), pg_shard_begin(n, P, g+1)) */
int pg_shard_begin(int n_labels, int n_gpus, int g);
/* one label of the cosine-field dataset, [per_label][C][H][W] f64 in [0,1] */
int pg_cosine_label(int C, int H, int W, long per_label, uint64_t seed, int label, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PG_TRAINER_H */
