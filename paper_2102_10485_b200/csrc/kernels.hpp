// Internal launchers (C++ linkage).  The C-ABI in include/pg_kernels.h wraps
// these; the device network (net.cpp) calls them directly.
#pragma once

#include "common.cuh"

namespace pg {

// MATH_BF16: tensor-core GEMM operands rounded to bfloat16 (nearest even),
// one kind::tf32 MMA pass, fp32 accumulation; the SIMT kernels stay fp32
enum MathMode : int { MATH_FP32_SIMT = 0, MATH_TF32X3 = 1, MATH_TF32 = 2, MATH_BF16 = 3 };

// every launcher ends with `return launched();`: counts the kernel launch
// (bench.py's gpu_launches) and returns the launch status
cudaError_t launched();
long long launch_count();
void add_launches(long long n);  // kernels replayed inside a CUDA graph
bool gemm_timing_on();
// optional per-GEMM timing (CUDA events on the launching stream)
void gemm_timing_enable(bool on);
double gemm_timing_read_ms();
}  // namespace pg
#include <string>
namespace pg {
std::string gemm_timing_report();  // one line per timed GEMM launch: shape tags + ms
// the same per-launch timing for the HBM-bound kernels: tag "hbm <name> bytes=<algorithmic bytes>"
cudaEvent_t timing_start(cudaStream_t st);  // nullptr when timing is off
void timing_stop(cudaEvent_t e0, cudaStream_t st, const std::string& tag);

// measured tcgen05 kind::tf32 dense peak (TFLOP/s), tc_peak.cu
cudaError_t tc_tf32_peak(int iters, double* tflops);
int gemm_max_m(const GemmArgs& a);
int gemm_n(const GemmArgs& a);
cudaError_t launch_gemm_simt(const GemmArgs& a, cudaStream_t st);
cudaError_t launch_gemm_tc(const GemmArgs& a, int math, cudaStream_t st);  // tcgen05 engine
bool gemm_tc_supported(const GemmArgs& a);
cudaError_t launch_gemm_tma(const GemmArgs& a, int math, cudaStream_t st);  // TMA-fed tcgen05 engine
bool gemm_tma_supported(const GemmArgs& a);
cudaError_t launch_gemm_pair(const GemmArgs& a, int math, cudaStream_t st);  // CTA-pair (cta_group::2) engine
bool gemm_pair_supported(const GemmArgs& a);
cudaError_t launch_gemm_lowered(const GemmArgs& a, int math, cudaStream_t st);  // im2col / col2im + pair engine
bool gemm_lowered_supported(const GemmArgs& a);
int gemm_pair_stat_slots(const GemmArgs& a, int* npack = nullptr);
// dense_wide.cu: wide dense FPROP with K <= 256 (the generator's latent projection), fp32 FMA
bool dense_wide_supported(const GemmArgs& a);
int dense_wide_stat_slots(const GemmArgs& a);
cudaError_t launch_dense_wide(const GemmArgs& a, cudaStream_t st);
int gemm_lowered_stat_slots(const GemmArgs& a);
// number of 32-row statistic slots launch_gemm(a, math) writes when a.stat_mode
// is set (0: the engine chosen for this GEMM cannot fuse statistics); *npack =
// GEMM columns per output channel (4 for phase-packed DGRAD: stat rows are
// npack * N_out wide, channel c at columns c + q N_out)
int gemm_stat_slots(const GemmArgs& a, int math, int* npack = nullptr);
// thin.cu; math selects the 4-channel weight gradient's form (TF32 modes: mma.sync tensor cores)
cudaError_t launch_gemm_thin(const GemmArgs& a, cudaStream_t st, int math = MATH_FP32_SIMT);
bool gemm_thin_supported(const GemmArgs& a);
// fprop4.cu: the 4-channel FPROP (CS = 64, k = 4, no fused statistics) on tcgen05, A gathered into TMEM
bool fprop4_supported(const GemmArgs& a, int math);
cudaError_t launch_fprop4(const GemmArgs& a, int math, cudaStream_t st);
// dgrad4.cu: the 4-channel DGRAD (CS = 64, k4 s2 p1, no fused statistics) on tcgen05, phase-packed N = 16
bool dgrad4_supported(const GemmArgs& a, int math);
cudaError_t launch_dgrad4(const GemmArgs& a, int math, cudaStream_t st);
// wgrad4.cu: the 4-channel weight gradient (CS = 64, k = 4) on tcgen05; part = thin.cu's split-K scratch
bool wgrad4_supported(const GemmArgs& a, int math);
cudaError_t launch_wgrad4(const GemmArgs& a, int math, float* part, int nchunk, cudaStream_t st);
float* gemm_scratch(size_t floats, cudaStream_t st);  // grow-only workspace for split-K reductions
// scratch one launch_gemm(a, math) call takes from its stream, per slot
// (SCRATCH_GEMM / SCRATCH_BLO floats); mirrors the engine choice of launch_gemm
struct GemmWorkspace {
  size_t gemm = 0, blo = 0;
};
GemmWorkspace gemm_workspace(const GemmArgs& a, int math);
GemmWorkspace gemm_lowered_workspace(const GemmArgs& a, int math);
size_t gemm_thin_workspace_floats(const GemmArgs& a);
size_t gemm_pair_blo_floats(const GemmArgs& a, int math);
// picks the engine for a math mode and problem shape
cudaError_t launch_gemm(const GemmArgs& a, int math, cudaStream_t st);

// ---- per-channel reductions over [L][R][Cp] maps (deterministic two-level) ----
enum ReduceMode : int {
  RED_SUM = 0,      // s0 = sum x
  RED_SQDEV = 1,    // s0 = sum (x - mean)^2
  RED_BN_BWD = 2,   // g1 = act_bwd(gy, y); s0 = sum g1; s1 = sum g1 (x-mean); s2 = sum (x-mean)
  RED_ACT_G = 3,    // g1 = act_bwd(gy, y); s0 = sum g1
};
struct ChannelMap {
  int L, R, Cp, C;         // rows per label, padded / valid channels
  long long ls;            // label stride of the maps (floats)
  // partials source: 0 = channel_reduce chunks ([L][chunks][3][Cp]); > 0 = that
  // many GEMM-epilogue statistic slots ([L][slots][4][Cp], see StatMode)
  int nslot = 0;
  int npack = 1;  // statistic columns per channel (see gemm_stat_slots)
};
int reduce_chunks(const ChannelMap& cm);
size_t reduce_partial_floats(const ChannelMap& cm);
// partial: [L][chunks][3][Cp]
// RED_ACT_G with g_out: also writes g1 = act_bwd(gy, y) (activation backward + bias sums in one pass)
// BN coefficients of a block (istd [L][Cp], gamma/beta at gb + l gb_ls): given
// to bn_bwd_apply, it recomputes a ReLU / LeakyReLU output from the pre-BN map
// instead of reading the stored y (bit-identical, see bn_pre); channel_reduce
// (RED_BN_BWD) does the same when given them.
struct BnCoef {
  const float* istd = nullptr;
  const float* gb = nullptr;
  long long gb_ls = 0;
};
cudaError_t launch_channel_reduce(const ChannelMap& cm, int mode, const float* x, const float* gy, const float* y,
                                  const float* mean, int act, float slope, float* partial, cudaStream_t st,
                                  float* g_out = nullptr, BnCoef bc = {});

// BN forward finalize: pass 0 -> mean; pass 1 -> var, inv_std, running-stat update.
cudaError_t launch_bn_finalize_mean(const ChannelMap& cm, const float* partial, float* mean, cudaStream_t st);
cudaError_t launch_bn_finalize_var(const ChannelMap& cm, const float* partial, const float* mean, float* istd,
                                   float* running, long long run_ls, float eps, float momentum, int update_running,
                                   cudaStream_t st);
// y = act(gamma (x - mean) istd + beta); eval mode passes running stats as mean/istd source.
cudaError_t launch_bn_apply(const ChannelMap& cm, const float* x, const float* mean, const float* istd,
                            const float* gamma_beta, long long gb_ls, int act, float slope, float* y, cudaStream_t st);
// BN forward statistics from STAT_FWD epilogue slots (cm.nslot > 0): mean,
// istd and the running-stat update in one pass (Chan's parallel merge, f64)
cudaError_t launch_bn_stats_finalize(const ChannelMap& cm, const float* stat, float* mean, float* istd, float* running,
                                     long long run_ls, float eps, float momentum, int update_running, cudaStream_t st);
// [L][nslot][4][Cp] epilogue slot sums -> [L][1][4][Cp]; read it back with cm.nslot = 1
cudaError_t launch_slot_sum(const ChannelMap& cm, const float* stat, float* out, cudaStream_t st);
// eval-mode: istd from running var
cudaError_t launch_bn_eval_stats(const ChannelMap& cm, const float* running, long long run_ls, float eps, float* mean,
                                 float* istd, cudaStream_t st);
// BN backward: from RED_BN_BWD partials build per-channel coefficients and
// write dgamma/dbeta (+ the preceding layer's bias grad) into the grad arena.
cudaError_t launch_bn_bwd_finalize(const ChannelMap& cm, const float* partial, const float* istd,
                                   const float* gamma_beta, long long gb_ls, float* dgamma_beta, long long dgb_ls,
                                   float* dbias, long long dbias_ls, int accumulate, int train, float* coef,
                                   cudaStream_t st);
// gz = act_bwd(gy, y) * gamma istd + dvar 2 (x - mean)/m + dmean/m
cudaError_t launch_bn_bwd_apply(const ChannelMap& cm, const float* gy, const float* y, const float* x,
                                const float* mean, const float* coef, int act, float slope, float* gz,
                                cudaStream_t st, BnCoef bc = {});
// g = act_bwd(gy, y) elementwise (in place allowed)
cudaError_t launch_act_bwd(const ChannelMap& cm, const float* gy, const float* y, int act, float slope, float* g,
                           cudaStream_t st);
// bias grad from RED_SUM / RED_ACT_G partials
cudaError_t launch_bias_finalize(const ChannelMap& cm, const float* partial, float* dbias, long long dbias_ls,
                                 int accumulate, cudaStream_t st);

// ---- GAN losses (gan.cpp:86-132) ----
// p maps are [L][B][pstride] with the probability in channel 0.
cudaError_t launch_loss_d(int L, int B, const float* p_real, const float* p_fake, int pstride, double clamp,
                          float* g_real, float* g_fake, double* report, cudaStream_t st);
cudaError_t launch_loss_g(int L, int B, const float* p_fake, int pstride, double clamp, float* g, double* report,
                          cudaStream_t st);

// ---- Adam over [L][P] arenas (optim.cpp:20-34) ----
cudaError_t launch_nonfinite_check(int L, long long P, const float* grads, int* flags, cudaStream_t st);
cudaError_t launch_adam_tick(int L, const int* flags, long long* t, cudaStream_t st);
cudaError_t launch_adam(int L, long long P, float* params, const float* grads, float* m, float* v,
                        const long long* t, const int* flags, float lr, double b1, double b2, float eps,
                        cudaStream_t st);

// ---- data movement ----
// out[l][b][hw][c] = 2 * data[l][idx[l][b]][hw][c] - 1 (c < C), 0 in pad channels
cudaError_t launch_gather_real(int L, int B, const int* idx, const float* data, long long data_ls, long long sample,
                               int Cp, int C, float* out, cudaStream_t st);
// NCHW [N][C][H][W] (values in [0,1]) -> NHWC padded; map2x1 applies 2x-1
cudaError_t launch_nchw01_to_nhwc(long long N, int C, int H, int W, int Cp, const float* in, float* out,
                                  cudaStream_t st, int map2x1 = 1);
// NHWC padded (tanh range) -> NCHW, mapped (v+1)/2
cudaError_t launch_nhwc_to_nchw01(long long N, int C, int H, int W, int Cp, const float* in, float* out,
                                  cudaStream_t st);
cudaError_t launch_fill(float* p, long long n, float v, cudaStream_t st);
// parity instrumentation: ReLU / LeakyReLU masks of y [L][B][H][W][Cp] as bytes
// out[l * out_ls + ((b C + c) H + h) W + w] (reference NCHW order)
cudaError_t launch_mask_capture(int L, int B, int H, int W, int C, int Cp, long long ls, const float* y, int act,
                                unsigned char* out, long long out_ls, cudaStream_t st);

}  // namespace pg
