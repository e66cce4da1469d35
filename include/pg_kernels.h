/* pg_kernels.h — kernel-level C-ABI of the B200 label-partitioned DC-CGAN step.
 *
 * The reference (/root/reference/proj, CPU C++/Eigen) has no plugin system:
 * its operator boundary is the closed LayerSpec variant dispatched by
 * run_layer / backward (src/network.cpp:357-398, 429-480) into per-layer
 * free functions in an anonymous namespace (src/network.cpp:28-300).  Each
 * entry point below replaces one of those functions; a maintainer binding the
 * reference to this library swaps the function body for the call (see
 * INTEGRATION.md).  Differences from the reference functions, all deliberate:
 *   - every call is batched over L labels with identical shapes ([L][...]
 *     arenas with a per-label stride), because all labels resident on a GPU
 *     step in lockstep;
 *   - device pointers, fp32, NHWC maps with channels padded to a multiple of 4
 *     (pad channels hold zeros), caller-owned memory, stream-ordered, no
 *     allocation inside once a workspace is attached (pg_set_workspace); weights in the device layouts documented per call;
 *   - deterministic: fixed-order reductions, no float atomics.
 * Status: PG_OK or a negative code; pg_last_error() describes the failure.
 */
#ifndef PG_KERNELS_H
#define PG_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PG_OK = 0, PG_EINVAL = -1, PG_ECUDA = -2, PG_ENONFINITE = -3, PG_EUNSUPPORTED = -4 };

/* Math modes for the GEMM-shaped kernels.  FP32_SIMT: exact fp32 FMAs on the
 * CUDA cores.  TF32X3: tcgen05 kind::tf32 with the 3-pass split
 * (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi), fp32-accurate.  TF32: one tcgen05 pass.
 * BF16: the tensor-core GEMMs round both operands to bfloat16 (nearest even)
 * and multiply them in one kind::tf32 pass with fp32 accumulation -- a bf16 x
 * bf16 -> fp32 product (bf16 values are exact in tf32, their products exact in
 * fp32); operands stay fp32 in memory, so it runs at the TF32 rate.  The SIMT
 * dense-head kernels compute in fp32 in every mode. */
enum { PG_MATH_FP32_SIMT = 0, PG_MATH_TF32X3 = 1, PG_MATH_TF32 = 2, PG_MATH_BF16 = 3 };

/* Activations fused into epilogues (network.cpp:384-391). */
enum { PG_ACT_NONE = 0, PG_ACT_RELU = 1, PG_ACT_LRELU = 2, PG_ACT_TANH = 3, PG_ACT_SIGMOID = 4 };

const char* pg_last_error(void);
int pg_device_count(void);
/* number of kernels this library has launched (process-wide counter) */
long long pg_launch_count(void);
/* per-GEMM CUDA-event timing (off by default): enable/disable resets the
 * record; read returns the summed device time of GEMM launches since enable */
int pg_kernel_timing(int on);
int pg_kernel_timing_read(double* gemm_ms);
/* text report, one line per timed GEMM launch ("kind L= M= N= K= ... ms");
 * returns the full length (copies at most cap-1 bytes + NUL) */
long pg_kernel_timing_report(char* out, long cap);
/* measured tcgen05 kind::tf32 dense throughput of the current device (TFLOP/s):
 * back-to-back CTA-pair M=256 N=256 K=8 MMAs from shared memory on every SM
 * pair; the roofline denominator bench.py reports (not a reference interface) */
int pg_tc_tf32_peak(int iters, double* tflops);

/* Convolution geometry of one layer for one label: input map H x W x Cin,
 * output map OH x OW x Cout, square kernel k, stride s, padding p, batch B.
 * Channel counts are the real ones; device maps use padded counts pad4(C). */
typedef struct {
  int B, Cin, H, W, Cout, OH, OW, k, s, p;
} pg_conv_desc;

/* ---- Conv2d (replaces conv_fwd / conv_bwd, network.cpp:86-144) ----
 * x [L][B][H][W][pad4(Cin)], y [L][B][OH][OW][pad4(Cout)],
 * w [L][pad4(Cout)][k][k][pad4(Cin)] (label stride w_ls floats), bias [L][Cout-stride bias_ls].
 * Forward applies bias then `act` in the epilogue. */
int pg_conv2d_fwd(const pg_conv_desc* d, int L, const float* x, const float* w, long long w_ls, const float* bias,
                  long long bias_ls, int act, float slope, float* y, int math, void* stream);
int pg_conv2d_bwd_data(const pg_conv_desc* d, int L, const float* gy, const float* w, long long w_ls, float* gx,
                       int math, void* stream);
/* gw (+)= weight gradient in the device weight layout; accumulate != 0 adds. */
int pg_conv2d_bwd_filter(const pg_conv_desc* d, int L, const float* x, const float* gy, float* gw, long long gw_ls,
                         int accumulate, int math, void* stream);

/* ---- ConvTranspose2d (adjoint of Conv2d) ----
 * x [L][B][H][W][pad4(Cin)] (the small map), y [L][B][OH][OW][pad4(Cout)],
 * OH = (H-1)s - 2p + k; w [L][pad4(Cin)][k][k][pad4(Cout)], bias [Cout]. */
int pg_convT2d_fwd(const pg_conv_desc* d, int L, const float* x, const float* w, long long w_ls, const float* bias,
                   long long bias_ls, int act, float slope, float* y, int math, void* stream);
int pg_convT2d_bwd_data(const pg_conv_desc* d, int L, const float* gy, const float* w, long long w_ls, float* gx,
                        int math, void* stream);
int pg_convT2d_bwd_filter(const pg_conv_desc* d, int L, const float* x, const float* gy, float* gw, long long gw_ls,
                          int accumulate, int math, void* stream);

/* ---- Dense (replaces dense_fwd / dense_bwd, network.cpp:28-45) ----
 * x [L][B][pad4(in)], y [L][B][pad4(out)], w [L][pad4(out)][pad4(in)] row-major. */
int pg_dense_fwd(int L, int B, int in, int out, const float* x, const float* w, long long w_ls, const float* bias,
                 long long bias_ls, int act, float slope, float* y, int math, void* stream);
int pg_dense_bwd_data(int L, int B, int in, int out, const float* gy, const float* w, long long w_ls, float* gx,
                      int math, void* stream);
int pg_dense_bwd_filter(int L, int B, int in, int out, const float* x, const float* gy, float* gw, long long gw_ls,
                        int accumulate, int math, void* stream);

/* ---- Workspace (the C-ABI never allocates) ----
 * Some GEMM shapes need device scratch inside one call: the split-K partials of
 * the 4-channel weight gradient, the column matrix of the lowered
 * 4-channel ConvTranspose2d forward / Conv2d data gradient, and (PG_ATM=0
 * builds of the narrow tiles) the pre-split tf32 lo part of the weights.
 * pg_workspace_size returns the bytes operator `op` with descriptor d (Dense:
 * B, Cin = in, Cout = out, the rest ignored) over L labels in `math` takes
 * (0 for most shapes; (size_t)-1 on an invalid descriptor, see pg_last_error).
 * pg_set_workspace attaches a caller-owned device buffer (256-byte aligned) to
 * a stream on the current device: every later call on that stream carves its
 * scratch from it and never allocates; a call whose need exceeds it fails with
 * PG_EINVAL.  NULL detaches (the library then keeps its own grow-only buffer per
 * stream, as it does when no workspace was ever attached).  The buffer must
 * stay valid until the stream's last call using it has completed. */
enum {
  PG_OP_CONV2D_FWD = 0, PG_OP_CONV2D_BWD_DATA = 1, PG_OP_CONV2D_BWD_FILTER = 2,
  PG_OP_CONVT2D_FWD = 3, PG_OP_CONVT2D_BWD_DATA = 4, PG_OP_CONVT2D_BWD_FILTER = 5,
  PG_OP_DENSE_FWD = 6, PG_OP_DENSE_BWD_DATA = 7, PG_OP_DENSE_BWD_FILTER = 8
};
size_t pg_workspace_size(int op, const pg_conv_desc* d, int L, int math);
int pg_set_workspace(void* stream, void* workspace, size_t bytes);

/* ---- BatchNorm over NHWC maps (replaces bn_fwd / bn_bwd, network.cpp:163-271) ----
 * x, y: [L][R][Cp] with R = B*H*W rows per label; gamma_beta [L][2C] (stride gb_ls);
 * running [L][2C] = {mean[C], var[C]} (stride run_ls); mean/istd [L][Cp] outputs;
 * workspace: pg_bn_workspace_floats(L, R, Cp) floats.
 * Train: batch stats (biased variance), running <- (1-mom) running + mom {mean, var*m/(m-1)};
 * eval (train == 0): running stats.  y = act(gamma (x-mean) istd + beta). */
size_t pg_bn_workspace_floats(int L, int R, int Cp);
int pg_bn_fwd(int L, int R, int C, int Cp, const float* x, const float* gamma_beta, long long gb_ls, float* running,
              long long run_ls, float eps, float momentum, int train, int act, float slope, float* mean, float* istd,
              float* y, float* workspace, void* stream);
/* gy: gradient w.r.t. y (post-activation), y: the forward output (activation
 * derivative is taken from it), x: the BatchNorm input; writes gx and
 * dgamma_beta [L][2C] (accumulate != 0 adds). */
int pg_bn_bwd(int L, int R, int C, int Cp, const float* gy, const float* y, const float* x, const float* mean,
              const float* istd, const float* gamma_beta, long long gb_ls, int act, float slope, float* gx,
              float* dgamma_beta, long long dgb_ls, int accumulate, float* workspace, void* stream);

/* ---- Activation backward from the saved output (network.cpp:463-470) ---- */
int pg_act_bwd(long long n, const float* gy, const float* y, int act, float slope, float* gx, void* stream);

/* ---- GAN losses (gan.cpp:86-132), p maps [L][B][pstride], probability in channel 0 ----
 * report [L][4] doubles = {j_d, j_g, d_real_mean, d_fake_mean}; pg_gan_losses fills
 * j_d and the means, pg_gen_loss fills j_g.  Gradients are zero where the clamp is active. */
int pg_gan_losses(int L, int B, const float* p_real, const float* p_fake, int pstride, double clamp, float* g_real,
                  float* g_fake, double* report, void* stream);
int pg_gen_loss(int L, int B, const float* p_fake, int pstride, double clamp, float* g, double* report, void* stream);

/* ---- Adam over [L][P] arenas (optim.cpp:20-34); P % 4 == 0 ----
 * flags[l] != 0 marks a rejected label: its state is left untouched.
 * pg_adam_step first scans the gradients for non-finite values (setting flags),
 * then advances t[l] and updates every non-flagged label. */
int pg_adam_step(int L, long long P, float* params, const float* grads, float* m, float* v, long long* t, int* flags,
                 double lr, double beta1, double beta2, double eps, void* stream);

/* ---- Real-batch gather (Dataset::gather + 2x-1, data.cpp:13-23, gan.cpp:141) ----
 * data [L][n][sample] (sample = H*W*Cp floats in [0,1]), idx [L][B] row indices,
 * out [L][B][sample] = 2*data-1 in real channels, 0 in pads. */
int pg_gather_real(int L, int B, const int* idx, const float* data, long long data_ls, long long sample, int Cp, int C,
                   float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PG_KERNELS_H */
