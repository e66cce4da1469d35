// Image-side convolutions (the 3-channel end of both networks, channels padded
// to 4) lowered onto the CTA-pair tensor-core engine instead of SIMT loops:
//
//   FPROP, CG == 4  (discriminator conv1 forward, generator convT4 data-grad)
//       im2col[pix][tap*4 + c] = big[gather(pix, tap)][c]       (k*k*4 = 64 wide)
//       out = im2col . W^T as a 1x1 FPROP (K = 64): the weight layout
//       [CS][tap][4] already IS the K-major [N][K] operand
//   DGRAD, CG <= 4  (generator convT4 forward, discriminator conv1 data-grad)
//       P[spix][tap*4 + c] = sum_cs small[spix][cs] W[cs][tap][c]  (1x1 FPROP, N = 64)
//       out[bpix][c] = act(bias + sum_{taps reaching bpix} P[spix(bpix, tap)][tap*4 + c])
//   The reference computes the convolution transpose exactly this way: a GEMM
//   into columns followed by col2im scatter-add (network.cpp:123-142); here the
//   scatter is a deterministic gather (each output sums its <= (k/s)^2 taps in
//   a fixed order).
// The im2col / P buffers live in the grow-only GEMM scratch (stream-ordered).
#include "kernels.hpp"

namespace pg {

namespace {

// im2col of a 4-channel NHWC big map for the small-map pixels: one thread per
// (pixel, tap) float4, consecutive threads = consecutive taps of one pixel.
__global__ void im2col4_kernel(ConvGeo g, int L, const float* __restrict__ big, long long big_ls,
                               float* __restrict__ col) {
  const int kk = g.k * g.k;
  const long long per_label = (long long)g.B * g.SH * g.SW * kk;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per_label * L) return;
  const int l = (int)(e / per_label);
  long long r = e % per_label;
  const int tap = (int)(r % kk);
  r /= kk;
  const int j = (int)(r % g.SW);
  r /= g.SW;
  const int i = (int)(r % g.SH);
  const int b = (int)(r / g.SH);
  const int y = i * g.s - g.p + tap / g.k, x = j * g.s - g.p + tap % g.k;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (y >= 0 && y < g.GH && x >= 0 && x < g.GW)
    v = __ldg(reinterpret_cast<const float4*>(big + l * big_ls + (((long long)b * g.GH + y) * g.GW + x) * 4));
  reinterpret_cast<float4*>(col)[e] = v;
}

// wt[l][tap*4 + c][cs] = W[l][cs][tap][c]  (c < CG, zero above)
__global__ void wt_transpose4_kernel(ConvGeo g, int L, const float* __restrict__ w, long long w_ls,
                                     float* __restrict__ wt) {
  const int kk = g.k * g.k;
  const long long per_label = (long long)kk * 4 * g.CS;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per_label * L) return;
  const int l = (int)(e / per_label);
  const long long r = e % per_label;
  const int cs = (int)(r % g.CS);
  const int n = (int)(r / g.CS);
  const int tap = n / 4, c = n % 4;
  wt[e] = c < g.CG ? w[l * w_ls + ((long long)cs * kk + tap) * g.CG + c] : 0.f;
}

// out[l][b][y][x][0:CG] = act(bias + sum_{ki = (y+p) mod s, ...} P[l][b][i][j][(ki k + kj) 4 + 0:4])
__global__ void col2im4_kernel(GemmArgs a, const float* __restrict__ P) {
  const ConvGeo& g = a.g;
  const int kk = g.k * g.k;
  const long long per_label = (long long)g.B * g.GH * g.GW;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per_label * a.L) return;
  const int l = (int)(e / per_label);
  long long r = e % per_label;
  const int x = (int)(r % g.GW);
  r /= g.GW;
  const int y = (int)(r % g.GH);
  const int b = (int)(r / g.GH);
  const float* Pb = P + (long long)l * g.B * g.SH * g.SW * kk * 4 + (long long)b * g.SH * g.SW * kk * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ki = (y + g.p) % g.s; ki < g.k; ki += g.s) {
    const int i = (y + g.p - ki) / g.s;
    if (i < 0 || i >= g.SH) continue;
    for (int kj = (x + g.p) % g.s; kj < g.k; kj += g.s) {
      const int j = (x + g.p - kj) / g.s;
      if (j < 0 || j >= g.SW) continue;
      const float4 v = __ldg(reinterpret_cast<const float4*>(Pb + (((long long)i * g.SW + j) * kk + ki * g.k + kj) * 4));
      acc[0] += v.x;
      acc[1] += v.y;
      acc[2] += v.z;
      acc[3] += v.w;
    }
  }
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
  float* o = a.out + l * a.out_ls + (((long long)b * g.GH + y) * g.GW + x) * g.CG;
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    if (n >= g.CG) break;
    float v = acc[n];
    if (n % a.c_pad >= a.c_valid) {
      v = 0.f;
    } else {
      if (bias) v += bias[n];
      v = act_fwd(a.act, v, a.slope);
    }
    o[n] = v;
  }
}

unsigned blocks_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }

GemmArgs fprop_1x1(const GemmArgs& a, int B, int H, int W, int Cin, int Cout) {
  GemmArgs p{};
  p.kind = GEMM_FPROP;
  p.g = ConvGeo{B, H, W, Cout, H, W, Cin, 1, 1, 0};
  p.L = a.L;
  p.act = ACT_NONE;
  p.c_valid = p.c_pad = Cout;
  return p;
}

}  // namespace

bool gemm_lowered_supported(const GemmArgs& a) {
  const ConvGeo& g = a.g;
  const int kk = g.k * g.k;
  if (g.k == 1 || kk * 4 < 64 || (kk * 4) % 32) return false;
  if (a.kind == GEMM_FPROP && g.CG == 4 && g.CS >= 64 && g.CS % 32 == 0 && a.big_ls % 4 == 0) {
    if (gemm_pair_supported(a)) return false;  // direct 4-channel TMA gather (gemm_pair.cu KIND_F4)
    GemmArgs p = fprop_1x1(a, g.B, g.SH, g.SW, kk * 4, g.CS);
    p.big = p.w = p.out = reinterpret_cast<float*>(256);
    return gemm_pair_supported(p);
  }
  if (a.kind == GEMM_DGRAD && g.CG <= 4 && g.CS % 32 == 0 && g.CS >= 32) {
    GemmArgs p = fprop_1x1(a, g.B, g.SH, g.SW, g.CS, kk * 4);
    p.big = p.w = p.out = reinterpret_cast<float*>(256);
    p.big_ls = a.small_ls;
    return a.small_ls % 4 == 0 && gemm_pair_supported(p);
  }
  return false;
}

int gemm_lowered_stat_slots(const GemmArgs& a) {
  if (a.kind != GEMM_FPROP) return 0;  // the DGRAD output comes out of col2im
  const ConvGeo& g = a.g;
  GemmArgs p = fprop_1x1(a, g.B, g.SH, g.SW, g.k * g.k * 4, g.CS);
  p.big = p.w = p.out = reinterpret_cast<float*>(256);
  return gemm_pair_stat_slots(p);
}

GemmWorkspace gemm_lowered_workspace(const GemmArgs& a, int math) {
  const ConvGeo& g = a.g;
  const long long kk = (long long)g.k * g.k;
  const long long pix = (long long)g.B * g.SH * g.SW;
  GemmWorkspace w;
  GemmArgs p = a.kind == GEMM_FPROP ? fprop_1x1(a, g.B, g.SH, g.SW, (int)kk * 4, g.CS)
                                    : fprop_1x1(a, g.B, g.SH, g.SW, g.CS, (int)kk * 4);
  p.big = p.w = p.out = reinterpret_cast<float*>(256);
  p.big_ls = a.kind == GEMM_FPROP ? pix * kk * 4 : a.small_ls;
  p.w_ls = a.kind == GEMM_FPROP ? a.w_ls : kk * 4 * g.CS;
  p.out_ls = a.kind == GEMM_FPROP ? a.out_ls : pix * kk * 4;
  w.blo = gemm_pair_blo_floats(p, math);  // the inner column GEMM on the pair engine
  w.gemm = a.kind == GEMM_FPROP ? (size_t)(pix * kk * 4 * a.L)
                                : (size_t)(kk * 4 * g.CS * a.L + 63) / 64 * 64 + (size_t)(pix * kk * 4 * a.L);
  return w;
}

cudaError_t launch_gemm_lowered(const GemmArgs& a, int math, cudaStream_t st) {
  const ConvGeo& g = a.g;
  const int kk = g.k * g.k;
  const long long pix = (long long)g.B * g.SH * g.SW;  // small-map pixels per label
  if (a.kind == GEMM_FPROP) {
    const long long col_ls = pix * kk * 4;
    float* col = gemm_scratch((size_t)(col_ls * a.L), st);
    if (!col) return cudaErrorMemoryAllocation;
    im2col4_kernel<<<blocks_for(pix * kk * a.L, 256), 256, 0, st>>>(g, a.L, a.big, a.big_ls, col);
    cudaError_t e = launched();
    if (e != cudaSuccess) return e;
    GemmArgs p = fprop_1x1(a, g.B, g.SH, g.SW, kk * 4, g.CS);
    p.big = col;
    p.big_ls = col_ls;
    p.w = a.w;
    p.w_ls = a.w_ls;
    p.out = a.out;
    p.out_ls = a.out_ls;
    p.bias = a.bias;
    p.bias_ls = a.bias_ls;
    p.act = a.act;
    p.slope = a.slope;
    p.c_valid = a.c_valid;
    p.c_pad = a.c_pad;
    p.stat_mode = a.stat_mode;  // same output map: the fused statistics carry over
    p.stat = a.stat;
    p.stat_y = a.stat_y;
    p.stat_z = a.stat_z;
    p.stat_mu = a.stat_mu;
    p.stat_act = a.stat_act;
    p.stat_slope = a.stat_slope;
    return launch_gemm_pair(p, math, st);
  }
  // DGRAD: columns P = small . Wt, then the col2im gather
  const long long wt_ls = (long long)kk * 4 * g.CS;
  const long long p_ls = pix * kk * 4;
  const size_t wt_floats = (size_t)(wt_ls * a.L + 63) / 64 * 64;
  float* scratch = gemm_scratch(wt_floats + (size_t)(p_ls * a.L), st);
  if (!scratch) return cudaErrorMemoryAllocation;
  float* wt = scratch;
  float* P = scratch + wt_floats;
  wt_transpose4_kernel<<<blocks_for(wt_ls * a.L, 256), 256, 0, st>>>(g, a.L, a.w, a.w_ls, wt);
  cudaError_t e = launched();
  if (e != cudaSuccess) return e;
  GemmArgs p = fprop_1x1(a, g.B, g.SH, g.SW, g.CS, kk * 4);
  p.big = a.small;
  p.big_ls = a.small_ls;
  p.w = wt;
  p.w_ls = wt_ls;
  p.out = P;
  p.out_ls = p_ls;
  e = launch_gemm_pair(p, math, st);
  if (e != cudaSuccess) return e;
  col2im4_kernel<<<blocks_for((long long)g.B * g.GH * g.GW * a.L, 256), 256, 0, st>>>(a, P);
  return launched();
}

}  // namespace pg
