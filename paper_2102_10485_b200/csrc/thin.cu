// Kernels for the "thin" GEMMs of the step, where one GEMM dimension is the
// 3-channel image side (padded to 4) or a dense head of width 1, so a 128-row
// tensor-core tile would be >85% padding and the problem is memory/latency
// bound.  Same semantics as the implicit-GEMM engines (GemmArgs), so the
// dispatcher can route them here:
//   thin_out_dgrad  DGRAD with N = CG <= 4  (generator output ConvT fwd,
//                   discriminator input-gradient): one thread per output pixel
//   thin_in_fprop   FPROP with CG == 4, CS <= 64 (discriminator first conv,
//                   generator output ConvT bwd-data): one thread per output
//                   pixel, all CS channels in registers, weights in smem
//   thin_in_wgrad   WGRAD with CG == 4, CS <= 64, k*k <= 16: split-K SIMT
//                   GEMM over fixed pixel chunks + fixed-order chunk reduce
//   dense_*         the dense heads: FPROP with N <= 4 (warp dot products),
//                   FPROP with small K (weights streamed once), DGRAD with
//                   K <= 4 and WGRAD with M <= 4 (outer products)
#include <algorithm>

#include "device_cache.hpp"
#include "gemm_gather.cuh"
#include "kernels.hpp"

namespace pg {

namespace {

PG_DEV float epi(const GemmArgs& a, const float* bias, int n, float x) {
  if (n % a.c_pad >= a.c_valid) return 0.f;
  if (bias) x += bias[n];
  return act_fwd(a.act, x, a.slope);
}

PG_DEV int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// ---- DGRAD, N = CG <= 4 ---------------------------------------------------
// out[b][y][x][0:4] = sum_{valid taps, cs} small[b][i][j][cs] * W[cs][ki][kj][0:4]
// Block = OD_TY x OD_TX output tile of one image.  The small-map patch every
// tap of the tile reaches is staged in shared memory by coalesced float4
// copies, with a padded pixel stride (CS + 4 floats) so the per-pixel float4
// reads of a warp are bank-conflict free; the label's weights sit beside it
// as one float4 per (cs, tap) (the <= 4 output channels).  Thread = two
// same-phase output pixels (x, x + s) of a row: every weight float4 feeds 8 FMAs.
constexpr int OD_TX = 64, OD_TY = 4, OD_THREADS = OD_TX / 2 * OD_TY;
__host__ __device__ inline int od_patch(int t, int k, int s) { return (t + k - 2) / s + 2; }

__global__ void __launch_bounds__(OD_THREADS) thin_out_dgrad_kernel(GemmArgs a) {
  extern __shared__ float4 sm4[];
  const ConvGeo& g = a.g;
  const int kk = g.k * g.k;
  const int PR = od_patch(OD_TY, g.k, g.s), PC = od_patch(OD_TX, g.k, g.s), PS = g.CS + 4;
  float4* wsm4 = sm4;
  float* patch = reinterpret_cast<float*>(sm4 + g.CS * kk);
  const int ntx = (g.GW + OD_TX - 1) / OD_TX;
  const int x_lo = (blockIdx.x % ntx) * OD_TX, y_lo = (blockIdx.x / ntx) * OD_TY;
  const int b = blockIdx.y, l = blockIdx.z;
  const int i_lo = floordiv(y_lo + g.p - g.k + 1, g.s), j_lo = floordiv(x_lo + g.p - g.k + 1, g.s);
  const float* w = a.w + l * a.w_ls;
  for (int e = threadIdx.x; e < g.CS * kk; e += blockDim.x) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int n = 0; n < g.CG; ++n) v[n] = w[(long long)e * g.CG + n];
    wsm4[e] = make_float4(v[0], v[1], v[2], v[3]);
  }
  const float* small = a.small + l * a.small_ls + (long long)b * g.SH * g.SW * g.CS;
  const int c4n = g.CS / 4;
  for (int e = threadIdx.x; e < PR * PC * c4n; e += blockDim.x) {
    const int c4 = e % c4n, pix = e / c4n;
    const int i = i_lo + pix / PC, j = j_lo + pix % PC;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i >= 0 && i < g.SH && j >= 0 && j < g.SW)
      v = __ldg(reinterpret_cast<const float4*>(small + ((long long)i * g.SW + j) * g.CS) + c4);
    *reinterpret_cast<float4*>(patch + pix * PS + 4 * c4) = v;
  }
  __syncthreads();
  const int q = threadIdx.x % (OD_TX / 2);
  const int y = y_lo + threadIdx.x / (OD_TX / 2);
  const int x0 = x_lo + (q / g.s) * (2 * g.s) + q % g.s;
  if (y >= g.GH) return;
  float acc[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[u][n] = 0.f;
  for (int ki = (y + g.p) % g.s; ki < g.k; ki += g.s) {
    const int i = (y + g.p - ki) / g.s;
    if (i < 0 || i >= g.SH) continue;
    for (int kj = (x0 + g.p) % g.s; kj < g.k; kj += g.s) {
      const int tap = ki * g.k + kj;
      const float* src[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int x = x0 + g.s * u;
        const int j = (x + g.p - kj) / g.s;
        src[u] = (x < g.GW && j >= 0 && j < g.SW) ? patch + ((i - i_lo) * PC + (j - j_lo)) * PS : nullptr;
      }
      for (int c4 = 0; c4 < c4n; ++c4) {
        float4 v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          v[u] = src[u] ? *reinterpret_cast<const float4*>(src[u] + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const float4 wv = wsm4[(c4 * 4 + cc) * kk + tap];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float sv = cc == 0 ? v[u].x : cc == 1 ? v[u].y : cc == 2 ? v[u].z : v[u].w;
            acc[u][0] = fmaf(sv, wv.x, acc[u][0]);
            acc[u][1] = fmaf(sv, wv.y, acc[u][1]);
            acc[u][2] = fmaf(sv, wv.z, acc[u][2]);
            acc[u][3] = fmaf(sv, wv.w, acc[u][3]);
          }
        }
      }
    }
  }
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int x = x0 + g.s * u;
    if (x >= g.GW) continue;
    float* o = a.out + l * a.out_ls + (((long long)b * g.GH + y) * g.GW + x) * g.CG;
#pragma unroll
    for (int n = 0; n < 4; ++n)
      if (n < g.CG) o[n] = epi(a, bias, n, acc[u][n]);
  }
}

// ---- FPROP, CG == 4, CS <= 64 ---------------------------------------------
// out[b][i][j][cs] = sum_{tap} big[b][y][x][0:4] . W[cs][tap][0:4]
// Block = IF_PIX output pixels of one image (TI rows x TJ cols) x all CS
// channels.  The input patch under the tile ((TI-1)s+k rows x (TJ-1)s+k
// columns of 4-channel pixels) and the weights (one float4 per (cs, tap)) are
// staged in shared memory.  Thread = two output pixels x 16 channels (the
// channel group is warp-uniform, so weight reads are broadcasts): each weight
// float4 feeds 8 FMAs, registers stay low enough for full occupancy.
constexpr int IF_PIX = 128, IF_THREADS = 256, IF_CSG = 16;

__global__ void __launch_bounds__(IF_THREADS) thin_in_fprop_kernel(GemmArgs a, int TI, int TJ) {
  extern __shared__ float4 sm4[];
  const ConvGeo& g = a.g;
  const int kk = g.k * g.k;
  const int PR = (TI - 1) * g.s + g.k, PC = (TJ - 1) * g.s + g.k;
  float4* wsm4 = sm4;               // [64][kk], zero beyond CS
  float4* patch = sm4 + 64 * kk;    // [PR][PC]
  const int ntj = (g.SW + TJ - 1) / TJ;
  const int j0 = (blockIdx.x % ntj) * TJ, i0 = (blockIdx.x / ntj) * TI;
  const int b = blockIdx.y, l = blockIdx.z;
  const float4* w = reinterpret_cast<const float4*>(a.w + l * a.w_ls);
  for (int e = threadIdx.x; e < 64 * kk; e += blockDim.x)
    wsm4[e] = e < g.CS * kk ? w[e] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float* big = a.big + l * a.big_ls + (long long)b * g.GH * g.GW * 4;
  const int y_lo = i0 * g.s - g.p, x_lo = j0 * g.s - g.p;
  for (int e = threadIdx.x; e < PR * PC; e += blockDim.x) {
    const int y = y_lo + e / PC, x = x_lo + e % PC;
    patch[e] = (y >= 0 && y < g.GH && x >= 0 && x < g.GW)
                   ? __ldg(reinterpret_cast<const float4*>(big + ((long long)y * g.GW + x) * 4))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const int cs0 = (threadIdx.x / (IF_PIX / 2)) * IF_CSG;
  if (cs0 >= g.CS) return;
  const int pp = threadIdx.x % (IF_PIX / 2);
  int ii[2], jj[2];
  bool ok[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int pix = pp + u * (IF_PIX / 2);
    ii[u] = pix / TJ;
    jj[u] = pix % TJ;
    ok[u] = ii[u] < TI && i0 + ii[u] < g.SH && j0 + jj[u] < g.SW;
  }
  float acc[2][IF_CSG];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int c = 0; c < IF_CSG; ++c) acc[u][c] = 0.f;
  for (int ki = 0; ki < g.k; ++ki) {
    for (int kj = 0; kj < g.k; ++kj) {
      float4 v[2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        v[u] = ok[u] ? patch[(ii[u] * g.s + ki) * PC + jj[u] * g.s + kj] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* wt = wsm4 + cs0 * kk + ki * g.k + kj;
#pragma unroll
      for (int c = 0; c < IF_CSG; ++c) {
        const float4 wv = wt[c * kk];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          acc[u][c] = fmaf(v[u].x, wv.x, fmaf(v[u].y, wv.y, fmaf(v[u].z, wv.z, fmaf(v[u].w, wv.w, acc[u][c]))));
      }
    }
  }
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!ok[u]) continue;
    float* o = a.out + l * a.out_ls + (((long long)b * g.SH + i0 + ii[u]) * g.SW + j0 + jj[u]) * g.CS + cs0;
#pragma unroll
    for (int c = 0; c < IF_CSG; c += 4)
      if (cs0 + c < g.CS)
        *reinterpret_cast<float4*>(o + c) =
            make_float4(epi(a, bias, cs0 + c, acc[u][c]), epi(a, bias, cs0 + c + 1, acc[u][c + 1]),
                        epi(a, bias, cs0 + c + 2, acc[u][c + 2]), epi(a, bias, cs0 + c + 3, acc[u][c + 3]));
  }
}

int pow2ceil_thin(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---- WGRAD, CG == 4, CS <= 64 ---------------------------------------------
// dW[cs][tap][0:4] (+)= sum_{spix} smallg[spix][cs] * big[gather(spix, tap)][0:4]
// A small GEMM (M = CS, N = k*k*4, K = small-map pixels) split over K into
// fixed chunks: block (chunk, label) computes the whole CS x N partial with a
// register-tiled SIMT loop over 32-pixel smem stages (the next stage is
// prefetched into registers while the current one is multiplied); a second
// kernel sums the chunk partials in chunk order (deterministic, no atomics).
constexpr int TW_KC = 32;      // pixels per smem stage
constexpr int TW_SPLIT = 1024; // pixels per chunk
__global__ void __launch_bounds__(256) thin_in_wgrad_partial_kernel(GemmArgs a, float* part, int nchunk) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y, chunk = blockIdx.x;
  const int kk = g.k * g.k;
  const float* sg = a.small + l * a.small_ls;
  const float* big = a.big + l * a.big_ls;
  __shared__ __align__(16) float gs[TW_KC][64];
  __shared__ __align__(16) float xs[TW_KC][64];
  const int tid = threadIdx.x;
  const int tm = tid / 16, tn = tid % 16;  // 4x4 micro tile at (4 tm, 4 tn)
  const int lq = tid / 8, lp = tid % 8;    // loader: pixel lq of the stage, float4 slots lp and lp + 8
  float acc[4][4] = {};
  const long long K = (long long)g.B * g.SH * g.SW;
  const long long k_begin = (long long)chunk * TW_SPLIT;
  const long long k_end = k_begin + TW_SPLIT < K ? k_begin + TW_SPLIT : K;
  float4 ra[2], rb[2];
  auto fetch = [&](long long k0) {
    const long long sp = k0 + lq;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    ra[0] = ra[1] = rb[0] = rb[1] = z;
    if (sp >= k_end) return;
    const int j = (int)(sp % g.SW);
    const long long t = sp / g.SW;
    const int i = (int)(t % g.SH), b = (int)(t / g.SH);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int slot = lp + 8 * h;
      if (slot * 4 < g.CS) ra[h] = __ldg(reinterpret_cast<const float4*>(sg + sp * g.CS) + slot);
      if (slot < kk) {
        const int y = i * g.s - g.p + slot / g.k, x = j * g.s - g.p + slot % g.k;
        if (y >= 0 && y < g.GH && x >= 0 && x < g.GW)
          rb[h] = __ldg(reinterpret_cast<const float4*>(big + (((long long)b * g.GH + y) * g.GW + x) * 4));
      }
    }
  };
  fetch(k_begin);
  for (long long k0 = k_begin; k0 < k_end; k0 += TW_KC) {
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      reinterpret_cast<float4*>(&gs[lq][0])[lp + 8 * h] = ra[h];
      reinterpret_cast<float4*>(&xs[lq][0])[lp + 8 * h] = rb[h];
    }
    __syncthreads();
    if (k0 + TW_KC < k_end) fetch(k0 + TW_KC);
#pragma unroll 8
    for (int q = 0; q < TW_KC; ++q) {
      const float4 av = *reinterpret_cast<const float4*>(&gs[q][tm * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&xs[q][tn * 4]);
      const float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(ar[u], br[v], acc[u][v]);
    }
  }
  float* dst = part + ((long long)l * nchunk + chunk) * 64 * 64;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    *reinterpret_cast<float4*>(dst + (tm * 4 + u) * 64 + tn * 4) =
        make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
}

// Tensor-core form of the same partial GEMM (TF32X3 / TF32 math): the legacy
// warp-level mma.sync m16n8k8 TF32 path -- M = N = 64 is far too narrow for a
// CTA-pair tcgen05 tile, and the SIMT loop above runs at the FP32 FMA roof.
// Block = (chunk, label), 8 warps; warp w owns rows 16 (w / 2) .. + 16 and
// columns 32 (w % 2) .. + 32 of the 64 x 64 partial (four n8 tiles).  The 3xTF32
// split is the tcgen05 path's: hi = the fp32 bits truncated by the tensor core,
// lo = x - trunc(x); products small terms first.
constexpr int TWM_LD = 72;  // smem row pitch (floats): fragment loads conflict-free
PG_DEV void mma_tf32_16x8x8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
PG_DEV uint32_t tf32_lo(float x) { return __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xffffe000u)); }

template <bool X3>
__global__ void __launch_bounds__(256) thin_in_wgrad_mma_kernel(GemmArgs a, float* part, int nchunk) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y, chunk = blockIdx.x;
  const int kk = g.k * g.k;
  const float* sg = a.small + l * a.small_ls;
  const float* big = a.big + l * a.big_ls;
  __shared__ __align__(16) float gs[TW_KC][TWM_LD];
  __shared__ __align__(16) float xs[TW_KC][TWM_LD];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int lq = tid / 8, lp = tid % 8;  // loader: pixel lq of the stage, float4 slots lp and lp + 8
  const int fg = lane >> 2, ft = lane & 3;  // fragment row group / thread in group
  const int m0 = (warp >> 1) * 16, n0 = (warp & 1) * 32;
  float acc[4][4] = {};
  const long long K = (long long)g.B * g.SH * g.SW;
  const long long k_begin = (long long)chunk * TW_SPLIT;
  const long long k_end = k_begin + TW_SPLIT < K ? k_begin + TW_SPLIT : K;
  float4 ra[2], rb[2];
  auto fetch = [&](long long k0) {
    const long long sp = k0 + lq;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    ra[0] = ra[1] = rb[0] = rb[1] = z;
    if (sp >= k_end) return;
    const int j = (int)(sp % g.SW);
    const long long t = sp / g.SW;
    const int i = (int)(t % g.SH), b = (int)(t / g.SH);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int slot = lp + 8 * h;
      if (slot * 4 < g.CS) ra[h] = __ldg(reinterpret_cast<const float4*>(sg + sp * g.CS) + slot);
      if (slot < kk) {
        const int y = i * g.s - g.p + slot / g.k, x = j * g.s - g.p + slot % g.k;
        if (y >= 0 && y < g.GH && x >= 0 && x < g.GW)
          rb[h] = __ldg(reinterpret_cast<const float4*>(big + (((long long)b * g.GH + y) * g.GW + x) * 4));
      }
    }
  };
  fetch(k_begin);
  for (long long k0 = k_begin; k0 < k_end; k0 += TW_KC) {
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      *reinterpret_cast<float4*>(&gs[lq][4 * (lp + 8 * h)]) = ra[h];
      *reinterpret_cast<float4*>(&xs[lq][4 * (lp + 8 * h)]) = rb[h];
    }
    __syncthreads();
    if (k0 + TW_KC < k_end) fetch(k0 + TW_KC);
#pragma unroll
    for (int q = 0; q < TW_KC; q += 8) {
      // A[m][k] = gs[k][m], B[k][n] = xs[k][n]
      const float af[4] = {gs[q + ft][m0 + fg], gs[q + ft][m0 + fg + 8], gs[q + ft + 4][m0 + fg],
                           gs[q + ft + 4][m0 + fg + 8]};
      uint32_t ah[4], al[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ah[u] = __float_as_uint(af[u]);
        al[u] = tf32_lo(af[u]);
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const float b0 = xs[q + ft][n0 + nt * 8 + fg], b1 = xs[q + ft + 4][n0 + nt * 8 + fg];
        if (X3) {
          mma_tf32_16x8x8(acc[nt], al, __float_as_uint(b0), __float_as_uint(b1));
          mma_tf32_16x8x8(acc[nt], ah, tf32_lo(b0), tf32_lo(b1));
        }
        mma_tf32_16x8x8(acc[nt], ah, __float_as_uint(b0), __float_as_uint(b1));
      }
    }
  }
  float* dst = part + ((long long)l * nchunk + chunk) * 64 * 64;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int n = n0 + nt * 8 + 2 * ft;
    *reinterpret_cast<float2*>(dst + (m0 + fg) * 64 + n) = make_float2(acc[nt][0], acc[nt][1]);
    *reinterpret_cast<float2*>(dst + (m0 + fg + 8) * 64 + n) = make_float2(acc[nt][2], acc[nt][3]);
  }
}

__global__ void thin_in_wgrad_reduce_kernel(GemmArgs a, const float* part, int nchunk) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int NN = g.k * g.k * 4;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // over CS x NN
  if (a.in_act != ACT_NONE && e < g.CS && a.in_dbias) {
    // fused activation backward (wgrad4): the bias gradient from the per-chunk,
    // per-group channel sums, added in a fixed order
    const float* bp = part + (size_t)a.L * nchunk * 64 * 64 + (size_t)l * nchunk * 2 * 64 + e;
    float sb = 0.f;
    for (int c = 0; c < nchunk; ++c) sb += bp[c * 128] + bp[c * 128 + 64];
    float* ob = a.in_dbias + l * a.out_ls + e;
    *ob = a.accumulate ? *ob + sb : sb;
  }
  if (e >= g.CS * NN) return;
  const int m = e / NN, n = e % NN;
  float s = 0.f;
  for (int c = 0; c < nchunk; ++c) s += part[(((long long)l * nchunk + c) * 64 + m) * 64 + n];
  float* out = a.out + l * a.out_ls + e;
  *out = a.accumulate ? *out + s : s;
}

// ---- dense heads ----------------------------------------------------------
// FPROP with N = CS <= 4: out[b][0:CS] = x[b] . W[0:CS] (warp per (label, b))
// FPROP with N = CS <= 4 (the discriminator head, K = 6272 / 4096 / 8192):
// block = (row b, label), each thread's float4s of the row loaded at once (a
// warp per row left ~8% of the loads in flight that HBM latency needs), then
// a fixed-order block reduction (lane tree, then the eight warps in order)
constexpr int DN4_NT = 256;
__global__ void __launch_bounds__(DN4_NT) dense_fprop_n4_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y, b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const float* x = a.big + l * a.big_ls + (long long)b * g.CG;
  const float* w = a.w + l * a.w_ls;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int k = tid * 4; k < g.CG; k += DN4_NT * 4) {
    const float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
#pragma unroll
    for (int n = 0; n < 4; ++n)
      if (n < g.CS) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (long long)n * g.CG + k));
        acc[n] = fmaf(xv.x, wv.x, fmaf(xv.y, wv.y, fmaf(xv.z, wv.z, fmaf(xv.w, wv.w, acc[n]))));
      }
  }
  __shared__ float part[DN4_NT / 32][4];
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    for (int o = 16; o > 0; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
    if (lane == 0) part[warp][n] = acc[n];
  }
  __syncthreads();
  if (tid < g.CS) {
    float s = 0.f;
    for (int wi = 0; wi < DN4_NT / 32; ++wi) s += part[wi][tid];
    const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
    a.out[l * a.out_ls + (long long)b * g.CS + tid] = epi(a, bias, tid, s);
  }
}

// FPROP with small K: out[b][n] = x[b] . W[n]; block per (label, 128 rows n);
// the label's inputs x[B][K] in smem, each weight row read once.
constexpr int DS_BMAX = 64;
__global__ void __launch_bounds__(128) dense_fprop_smallk_kernel(GemmArgs a) {
  extern __shared__ float xs[];  // [B][K]
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int K = g.CG, B = g.B;
  const float* x = a.big + l * a.big_ls;
  for (int e = threadIdx.x; e < B * K; e += blockDim.x) xs[e] = x[e];
  __syncthreads();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.CS) return;
  const float* w = a.w + l * a.w_ls + (long long)n * K;
  float acc[DS_BMAX];
#pragma unroll
  for (int b = 0; b < DS_BMAX; ++b) acc[b] = 0.f;
  for (int k = 0; k < K; k += 4) {
    const float4 wv = __ldg(reinterpret_cast<const float4*>(w + k));
#pragma unroll
    for (int b = 0; b < DS_BMAX; ++b)
      if (b < B) {
        const float4 xv = *reinterpret_cast<const float4*>(xs + b * K + k);
        acc[b] = fmaf(xv.x, wv.x, fmaf(xv.y, wv.y, fmaf(xv.z, wv.z, fmaf(xv.w, wv.w, acc[b]))));
      }
  }
  float* out = a.out + l * a.out_ls + n;
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
#pragma unroll
  for (int b = 0; b < DS_BMAX; ++b)
    if (b < B) out[(long long)b * g.CS] = epi(a, bias, n, acc[b]);
}

// DGRAD with K = CS <= 4: gx[b][f] = sum_cs gz[b][cs] W[cs][f]; block =
// (row b, label), every thread's float4s issued together (32-bit indexing: the
// grid-stride form spent its time in 64-bit divisions and one store in flight)
__global__ void __launch_bounds__(DN4_NT) dense_dgrad_k4_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y, b = blockIdx.x;
  const float* w = a.w + l * a.w_ls;
  const float* gz = a.small + l * a.small_ls + (long long)b * g.CS;
  float gv[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) gv[c] = c < g.CS ? __ldg(gz + c) : 0.f;
  float* out = a.out + l * a.out_ls + (long long)b * g.CG;
#pragma unroll 8
  for (int f = threadIdx.x * 4; f < g.CG; f += DN4_NT * 4) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < g.CS) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + c * g.CG + f));
        r.x = fmaf(gv[c], wv.x, r.x);
        r.y = fmaf(gv[c], wv.y, r.y);
        r.z = fmaf(gv[c], wv.z, r.z);
        r.w = fmaf(gv[c], wv.w, r.w);
      }
    float o[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if ((f + u) % a.c_pad >= a.c_valid) o[u] = 0.f;
    *reinterpret_cast<float4*>(out + f) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// WGRAD with M = CS <= 4: dW[cs][f] = sum_b gz[b][cs] x[b][f]
__global__ void dense_wgrad_m4_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (f >= g.CG) return;
  const float* gz = a.small + l * a.small_ls;
  const float* x = a.big + l * a.big_ls;
  float4 acc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b = 0; b < g.B; ++b) {
    const float4 xv = __ldg(reinterpret_cast<const float4*>(x + (long long)b * g.CG + f));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= g.CS) break;
      const float gv = gz[(long long)b * g.CS + c];
      acc[c].x = fmaf(gv, xv.x, acc[c].x);
      acc[c].y = fmaf(gv, xv.y, acc[c].y);
      acc[c].z = fmaf(gv, xv.z, acc[c].z);
      acc[c].w = fmaf(gv, xv.w, acc[c].w);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (c >= g.CS) break;
    float4* out = reinterpret_cast<float4*>(a.out + l * a.out_ls + (long long)c * g.CG + f);
    float4 r = acc[c];
    if (a.accumulate) {
      const float4 o = *out;
      r.x += o.x; r.y += o.y; r.z += o.z; r.w += o.w;
    }
    *out = r;
  }
}

bool is_dense(const ConvGeo& g) { return g.SH == 1 && g.SW == 1 && g.GH == 1 && g.GW == 1 && g.k == 1; }

enum Thin { T_NONE, T_OUT_DGRAD, T_IN_FPROP, T_IN_WGRAD, T_D_FPROP_N4, T_D_FPROP_SK, T_D_DGRAD_K4, T_D_WGRAD_M4 };

Thin classify(const GemmArgs& a) {
  const ConvGeo& g = a.g;
  if (is_dense(g)) {
    if (a.kind == GEMM_FPROP && g.CS <= 4 && g.CG % 4 == 0) return T_D_FPROP_N4;
    if (a.kind == GEMM_FPROP && g.B <= DS_BMAX && g.CG <= 256 && g.CG % 4 == 0) return T_D_FPROP_SK;
    if (a.kind == GEMM_DGRAD && g.CS <= 4 && g.CG % 4 == 0) return T_D_DGRAD_K4;
    if (a.kind == GEMM_WGRAD && g.CS <= 4 && g.CG % 4 == 0) return T_D_WGRAD_M4;
    return T_NONE;
  }
  // shared-memory footprints of the staged kernels (weights + input patch) must fit 200 KB
  const size_t od_smem = sizeof(float4) * g.CS * g.k * g.k +
                         sizeof(float) * od_patch(OD_TY, g.k, g.s) * od_patch(OD_TX, g.k, g.s) * (g.CS + 4);
  const int tj = std::min(pow2ceil_thin(g.SW), IF_PIX), ti = IF_PIX / tj;
  const size_t if_smem = sizeof(float4) * (64 * g.k * g.k + ((ti - 1) * g.s + g.k) * ((tj - 1) * g.s + g.k));
  if (a.kind == GEMM_DGRAD && g.CG <= 4 && g.CS % 4 == 0 && od_smem <= 200 * 1024 && g.B <= 65535) return T_OUT_DGRAD;
  if (a.kind == GEMM_FPROP && g.CG == 4 && g.CS <= 64 && if_smem <= 200 * 1024 && g.B <= 65535) return T_IN_FPROP;
  if (a.kind == GEMM_WGRAD && g.CG == 4 && g.CS <= 64 && g.k * g.k <= 16) return T_IN_WGRAD;
  return T_NONE;
}

}  // namespace

bool gemm_thin_supported(const GemmArgs& a) { return classify(a) != T_NONE; }

size_t gemm_thin_workspace_floats(const GemmArgs& a) {
  if (classify(a) != T_IN_WGRAD) return 0;
  const long long K = (long long)a.g.B * a.g.SH * a.g.SW;
  return (size_t)a.L * ((K + TW_SPLIT - 1) / TW_SPLIT) * 64 * (64 + 2);
}

cudaError_t launch_gemm_thin(const GemmArgs& a, cudaStream_t st, int math) {
  const ConvGeo& g = a.g;
  switch (classify(a)) {
    case T_OUT_DGRAD: {
      const int kk = g.k * g.k;
      const size_t smem = sizeof(float4) * g.CS * kk +
                          sizeof(float) * od_patch(OD_TY, g.k, g.s) * od_patch(OD_TX, g.k, g.s) * (g.CS + 4);
      static PerDeviceMax configured;
      if (smem > 48 * 1024) {
        cudaError_t e = configured.raise(smem, [&] {
          return cudaFuncSetAttribute(thin_out_dgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        if (e != cudaSuccess) return e;
      }
      const unsigned tiles = (unsigned)(((g.GW + OD_TX - 1) / OD_TX) * ((g.GH + OD_TY - 1) / OD_TY));
      thin_out_dgrad_kernel<<<dim3(tiles, g.B, a.L), OD_THREADS, smem, st>>>(a);
      break;
    }
    case T_IN_FPROP: {
      const int TJ = std::min(pow2ceil_thin(g.SW), IF_PIX), TI = IF_PIX / TJ;
      const int kk = g.k * g.k;
      const size_t smem = sizeof(float4) * (64 * kk + ((TI - 1) * g.s + g.k) * ((TJ - 1) * g.s + g.k));
      static PerDeviceMax configured;
      if (smem > 48 * 1024) {
        cudaError_t e = configured.raise(smem, [&] {
          return cudaFuncSetAttribute(thin_in_fprop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        if (e != cudaSuccess) return e;
      }
      const unsigned tiles = (unsigned)(((g.SW + TJ - 1) / TJ) * ((g.SH + TI - 1) / TI));
      thin_in_fprop_kernel<<<dim3(tiles, g.B, a.L), IF_THREADS, smem, st>>>(a, TI, TJ);
      break;
    }
    case T_IN_WGRAD: {
      const long long K = (long long)g.B * g.SH * g.SW;
      const int nchunk = (int)((K + TW_SPLIT - 1) / TW_SPLIT);
      float* part = gemm_scratch((size_t)a.L * nchunk * 64 * (64 + 2), st);  // weight + bias partials
      if (!part) return cudaErrorMemoryAllocation;
      cudaError_t e;
      if (wgrad4_supported(a, math)) {
        e = launch_wgrad4(a, math, part, nchunk, st);  // tcgen05 (wgrad4.cu)
      } else {
        if (math == MATH_TF32X3)
          thin_in_wgrad_mma_kernel<true><<<dim3(nchunk, a.L), 256, 0, st>>>(a, part, nchunk);
        else if (math == MATH_TF32)
          thin_in_wgrad_mma_kernel<false><<<dim3(nchunk, a.L), 256, 0, st>>>(a, part, nchunk);
        else
          thin_in_wgrad_partial_kernel<<<dim3(nchunk, a.L), 256, 0, st>>>(a, part, nchunk);
        e = launched();
      }
      if (e != cudaSuccess) return e;
      const int nout = g.CS * g.k * g.k * 4;
      thin_in_wgrad_reduce_kernel<<<dim3((nout + 255) / 256, a.L), 256, 0, st>>>(a, part, nchunk);
      break;
    }
    case T_D_FPROP_N4:
      dense_fprop_n4_kernel<<<dim3((unsigned)g.B, a.L), DN4_NT, 0, st>>>(a);
      break;
    case T_D_FPROP_SK: {
      const size_t smem = (size_t)g.B * g.CG * sizeof(float);
      dense_fprop_smallk_kernel<<<dim3((unsigned)((g.CS + 127) / 128), a.L), 128, smem, st>>>(a);
      break;
    }
    case T_D_DGRAD_K4:
      dense_dgrad_k4_kernel<<<dim3((unsigned)g.B, a.L), DN4_NT, 0, st>>>(a);
      break;
    case T_D_WGRAD_M4:
      dense_wgrad_m4_kernel<<<dim3((unsigned)((g.CG / 4 + 255) / 256), a.L), 256, 0, st>>>(a);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return launched();
}

}  // namespace pg
