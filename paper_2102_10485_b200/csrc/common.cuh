// Shared definitions for the sm_100a kernels of the label-partitioned DC-CGAN
// training step.  Every kernel is batched over the L labels resident on one
// GPU ("label group"): tensors are [L][...] arenas with a per-label stride and
// blockIdx.z (or an explicit label loop) selects the label.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#define PG_DEV __device__ __forceinline__

namespace pg {

// activation fused into an epilogue / elementwise pass
enum Act : int { ACT_NONE = 0, ACT_RELU = 1, ACT_LRELU = 2, ACT_TANH = 3, ACT_SIGMOID = 4 };

#ifdef __CUDACC__

PG_DEV float act_fwd(int act, float x, float slope) {
  switch (act) {
    case ACT_RELU: return x > 0.f ? x : 0.f;
    case ACT_LRELU: return x >= 0.f ? x : x * slope;
    case ACT_TANH: return tanhf(x);
    case ACT_SIGMOID: return 1.f / (expf(-x) + 1.f);
    default: return x;
  }
}

// derivative expressed through the activation OUTPUT y (ReLU: y>0 <=> x>0;
// LeakyReLU with slope>0: y>=0 <=> x>=0; tanh 1-y^2; sigmoid y(1-y)), so the
// pre-activation never has to be kept (reference semantics network.cpp:463-470).
PG_DEV float act_bwd(int act, float g, float y, float slope) {
  switch (act) {
    case ACT_RELU: return y > 0.f ? g : 0.f;
    case ACT_LRELU: return y >= 0.f ? g : g * slope;
    case ACT_TANH: return g * (1.f - y * y);
    case ACT_SIGMOID: return g * y * (1.f - y);
    default: return g;
  }
}
#endif  // __CUDACC__

// Geometry shared by all three implicit-GEMM forms.  The "big" map (GH x GW,
// CG channels) is sampled by the "small" map (SH x SW, CS channels): big pixel
// (y, x) = (i*s - p + ki, j*s - p + kj).  Channel counts are PADDED to a
// multiple of 4 (device layout), all maps are NHWC per sample, [L][B][H][W][C].
//   conv2d   : big = input,  small = output, weight [Cout=CS][k][k][Cin=CG]
//   convT2d  : big = output, small = input,  weight [Cin=CS][k][k][Cout=CG]
//   dense    : k = s = 1, p = 0, spatial 1x1, weight [out=CS][in=CG]
struct ConvGeo {
  int B;
  int SH, SW, CS;
  int GH, GW, CG;
  int k, s, p;
};

// FPROP: C[spix][cs] = sum_{tap,cg} big[gather(spix,tap)][cg] * W[cs][tap][cg]   (conv fwd, convT bwd-data, dense fwd)
// DGRAD: C[bpix][cg] = sum_{tap valid,cs} small[gather(bpix,tap)][cs] * W[cs][tap][cg]  (conv bwd-data, convT fwd, dense bwd-data)
// WGRAD: C[cs][tap][cg] (+)= sum_{spix} smallg[spix][cs] * big[gather(spix,tap)][cg]   (weight gradients)
enum GemmKind : int { GEMM_FPROP = 0, GEMM_DGRAD = 1, GEMM_WGRAD = 2 };

// Per-channel statistics fused into the FPROP / DGRAD epilogue (CTA-pair
// engine; gemm_stat_slots() says whether a GEMM supports it and how many
// 32-row slots it writes).  stat layout: [L][slots][4][N].
//   STAT_FWD     out = z (act must be NONE): {shift, sum(z-shift), sum((z-shift)^2), rows}
//                per slot, shift = the slot's first row (merged with Chan's formula)
//   STAT_BWD_BN  out = g1 = act_bwd(gemm, y) written instead of the raw gradient:
//                {sum g1, sum g1 (z-mu), sum (z-mu), 0}   (BatchNorm backward sums)
//   STAT_BWD_ACT out = g1 = act_bwd(gemm, y): {sum g1, 0, 0, 0}   (bias gradient)
enum StatMode : int { STAT_NONE = 0, STAT_FWD = 1, STAT_BWD_BN = 2, STAT_BWD_ACT = 3 };

struct GemmArgs {
  int kind;
  ConvGeo g;
  int L;
  const float* small;  // FPROP: unused; DGRAD: A source; WGRAD: A source (gradient of small map)
  const float* big;    // FPROP: A source; WGRAD: B source
  const float* w;      // FPROP / DGRAD: weight
  float* out;
  const float* bias;   // FPROP / DGRAD epilogue bias [L][n] (nullable)
  long long small_ls, big_ls, w_ls, out_ls, bias_ls;  // per-label strides (floats)
  int act;
  float slope;
  int accumulate;      // WGRAD: out += result
  int c_valid, c_pad;  // FPROP/DGRAD: output column n is padding (written 0) iff n % c_pad >= c_valid
  int stat_mode;       // StatMode (FPROP / DGRAD on the pair engine only)
  float* stat;
  const float* stat_y;   // BWD: activation output map, same layout and label stride as out
  const float* stat_z;   // BWD_BN: pre-BatchNorm map, same layout and label stride as out
  const float* stat_mu;  // BWD_BN: batch mean [L][N]
  int stat_act;
  float stat_slope;
  // activation backward applied to the small operand as it is loaded (the
  // 4-channel image-side kernels only: wgrad4.cu, dgrad4.cu): the GEMM uses
  // act_bwd(small, in_y) with in_y the layer's activation output (same layout
  // and label stride as small); WGRAD also writes the bias gradient
  // sum_rows act_bwd(...) to in_dbias ([L] x CS, label stride out_ls)
  int in_act;  // ACT_NONE: off
  float in_slope;
  const float* in_y;
  float* in_dbias;
};

// phase decomposition of the big map along one axis for stride s, pad p:
// big coordinate y belongs to phase r = (y + p) mod s; its valid taps are
// ki = r, r+s, ... < k and the small coordinate is (y + p - ki) / s.
#ifdef __CUDACC__
PG_DEV int phase_origin(int r, int s, int p) { return ((r - p) % s + s) % s; }
#endif

}  // namespace pg

#define PG_CUDA_CHECK(x)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      std::fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                    \
  } while (0)
