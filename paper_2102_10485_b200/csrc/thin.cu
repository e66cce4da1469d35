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
#include "gemm_gather.cuh"
#include "kernels.hpp"

namespace pg {

namespace {

PG_DEV float epi(const GemmArgs& a, const float* bias, int n, float x) {
  if (n % a.c_pad >= a.c_valid) return 0.f;
  if (bias) x += bias[n];
  return act_fwd(a.act, x, a.slope);
}

// ---- DGRAD, N = CG <= 4 ---------------------------------------------------
// out[b][y][x][0:4] = sum_{valid taps, cs} small[b][i][j][cs] * W[cs][ki][kj][0:4]
__global__ void __launch_bounds__(256) thin_out_dgrad_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const long long npix = (long long)g.B * g.GH * g.GW;
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  const float* small = a.small + l * a.small_ls;
  const float* w = a.w + l * a.w_ls;
  const int x = (int)(pix % g.GW);
  const long long t = pix / g.GW;
  const int y = (int)(t % g.GH), b = (int)(t / g.GH);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int ki = (y + g.p) % g.s; ki < g.k; ki += g.s) {
    const int i = (y + g.p - ki) / g.s;
    if (i < 0 || i >= g.SH) continue;
    for (int kj = (x + g.p) % g.s; kj < g.k; kj += g.s) {
      const int j = (x + g.p - kj) / g.s;
      if (j < 0 || j >= g.SW) continue;
      const float4* src = reinterpret_cast<const float4*>(small + (((long long)b * g.SH + i) * g.SW + j) * g.CS);
      const float* wt = w + (ki * g.k + kj) * g.CG;
      for (int c4 = 0; c4 < g.CS / 4; ++c4) {
        const float4 v = __ldg(src + c4);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* wr = wt + (long long)(c4 * 4 + u) * g.k * g.k * g.CG;
#pragma unroll
          for (int n = 0; n < 4; ++n)
            if (n < g.CG) acc[n] = fmaf(vv[u], __ldg(wr + n), acc[n]);
        }
      }
    }
  }
  float* out = a.out + l * a.out_ls + pix * g.CG;
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
  for (int n = 0; n < g.CG; ++n) out[n] = epi(a, bias, n, acc[n]);
}

// ---- FPROP, CG == 4, CS <= 64 ---------------------------------------------
// out[b][i][j][cs] = sum_{tap} big[b][y][x][0:4] . W[cs][tap][0:4]
template <int CSMAX>
__global__ void __launch_bounds__(128) thin_in_fprop_kernel(GemmArgs a) {
  extern __shared__ float wsm[];  // [CS][k*k][4]
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int kk = g.k * g.k;
  const float* w = a.w + l * a.w_ls;
  for (int e = threadIdx.x; e < g.CS * kk * 4; e += blockDim.x) wsm[e] = w[e];
  __syncthreads();
  const long long npix = (long long)g.B * g.SH * g.SW;
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  const float* big = a.big + l * a.big_ls;
  const int j = (int)(pix % g.SW);
  const long long t = pix / g.SW;
  const int i = (int)(t % g.SH), b = (int)(t / g.SH);
  float acc[CSMAX];
#pragma unroll
  for (int c = 0; c < CSMAX; ++c) acc[c] = 0.f;
  for (int ki = 0; ki < g.k; ++ki) {
    const int y = i * g.s - g.p + ki;
    if (y < 0 || y >= g.GH) continue;
    for (int kj = 0; kj < g.k; ++kj) {
      const int x = j * g.s - g.p + kj;
      if (x < 0 || x >= g.GW) continue;
      const float4 v = __ldg(reinterpret_cast<const float4*>(big + (((long long)b * g.GH + y) * g.GW + x) * 4));
      const float* wt = wsm + (ki * g.k + kj) * 4;
#pragma unroll
      for (int c = 0; c < CSMAX; ++c) {
        if (c >= g.CS) break;
        const float4 wv = *reinterpret_cast<const float4*>(wt + c * kk * 4);
        acc[c] = fmaf(v.x, wv.x, fmaf(v.y, wv.y, fmaf(v.z, wv.z, fmaf(v.w, wv.w, acc[c]))));
      }
    }
  }
  float4* out = reinterpret_cast<float4*>(a.out + l * a.out_ls + pix * g.CS);
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
#pragma unroll
  for (int c = 0; c < CSMAX; c += 4)
    if (c < g.CS)
      out[c / 4] = make_float4(epi(a, bias, c, acc[c]), epi(a, bias, c + 1, acc[c + 1]), epi(a, bias, c + 2, acc[c + 2]),
                               epi(a, bias, c + 3, acc[c + 3]));
}

// ---- WGRAD, CG == 4, CS <= 64 ---------------------------------------------
// dW[cs][tap][0:4] (+)= sum_{spix} smallg[spix][cs] * big[gather(spix, tap)][0:4]
// A small GEMM (M = CS, N = k*k*4, K = small-map pixels) split over K into
// fixed chunks: block (chunk, label) computes the whole CS x N partial with a
// register-tiled SIMT loop over 32-pixel smem stages; a second kernel sums the
// chunk partials in chunk order (deterministic, no atomics).
constexpr int TW_KC = 32;      // pixels per smem stage
constexpr int TW_SPLIT = 1024; // pixels per chunk
__global__ void __launch_bounds__(256) thin_in_wgrad_partial_kernel(GemmArgs a, float* part, int nchunk) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y, chunk = blockIdx.x;
  const int kk = g.k * g.k, NN = kk * 4;  // N <= 64
  const float* sg = a.small + l * a.small_ls;
  const float* big = a.big + l * a.big_ls;
  __shared__ float gs[TW_KC][64];
  __shared__ float xs[TW_KC][64];
  const int tid = threadIdx.x;
  const int tm = tid / 16, tn = tid % 16;  // 4x4 micro tile at (4 tm, 4 tn)
  float acc[4][4] = {};
  const long long K = (long long)g.B * g.SH * g.SW;
  const long long k_begin = (long long)chunk * TW_SPLIT;
  const long long k_end = k_begin + TW_SPLIT < K ? k_begin + TW_SPLIT : K;
  for (long long k0 = k_begin; k0 < k_end; k0 += TW_KC) {
    __syncthreads();
    for (int e = tid; e < TW_KC * 64; e += 256) {
      const int q = e / 64, c = e % 64;
      const long long sp = k0 + q;
      float gv = 0.f, xv = 0.f;
      if (sp < k_end) {
        if (c < g.CS) gv = sg[sp * g.CS + c];
        if (c < NN) {
          const int tap = c / 4, cg = c % 4;
          const int j = (int)(sp % g.SW);
          const long long t = sp / g.SW;
          const int i = (int)(t % g.SH), b = (int)(t / g.SH);
          const int y = i * g.s - g.p + tap / g.k, x = j * g.s - g.p + tap % g.k;
          if (y >= 0 && y < g.GH && x >= 0 && x < g.GW) xv = big[(((long long)b * g.GH + y) * g.GW + x) * 4 + cg];
        }
      }
      gs[q][c] = gv;
      xs[q][c] = xv;
    }
    __syncthreads();
#pragma unroll 4
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

__global__ void thin_in_wgrad_reduce_kernel(GemmArgs a, const float* part, int nchunk) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int NN = g.k * g.k * 4;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // over CS x NN
  if (e >= g.CS * NN) return;
  const int m = e / NN, n = e % NN;
  float s = 0.f;
  for (int c = 0; c < nchunk; ++c) s += part[(((long long)l * nchunk + c) * 64 + m) * 64 + n];
  float* out = a.out + l * a.out_ls + e;
  *out = a.accumulate ? *out + s : s;
}

// ---- dense heads ----------------------------------------------------------
// FPROP with N = CS <= 4: out[b][0:CS] = x[b] . W[0:CS] (warp per (label, b))
__global__ void dense_fprop_n4_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= g.B) return;
  const float* x = a.big + l * a.big_ls + (long long)warp * g.CG;
  const float* w = a.w + l * a.w_ls;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = lane * 4; k < g.CG; k += 128) {
    const float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
#pragma unroll
    for (int n = 0; n < 4; ++n)
      if (n < g.CS) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (long long)n * g.CG + k));
        acc[n] = fmaf(xv.x, wv.x, fmaf(xv.y, wv.y, fmaf(xv.z, wv.z, fmaf(xv.w, wv.w, acc[n]))));
      }
  }
#pragma unroll
  for (int n = 0; n < 4; ++n)
    for (int o = 16; o > 0; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
  if (lane == 0) {
    float* out = a.out + l * a.out_ls + (long long)warp * g.CS;
    const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
    for (int n = 0; n < g.CS; ++n) out[n] = epi(a, bias, n, acc[n]);
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

// DGRAD with K = CS <= 4: gx[b][f] = sum_cs gz[b][cs] W[cs][f]
__global__ void dense_dgrad_k4_kernel(GemmArgs a) {
  const ConvGeo& g = a.g;
  const int l = blockIdx.y;
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // float4 index over [B][CG/4]
  const int f4n = g.CG / 4;
  if (q >= (long long)g.B * f4n) return;
  const int b = (int)(q / f4n), f = (int)(q % f4n) * 4;
  const float* gz = a.small + l * a.small_ls + (long long)b * g.CS;
  const float* w = a.w + l * a.w_ls;
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = 0; c < g.CS; ++c) {
    const float gv = gz[c];
    const float4 wv = __ldg(reinterpret_cast<const float4*>(w + (long long)c * g.CG + f));
    r.x = fmaf(gv, wv.x, r.x);
    r.y = fmaf(gv, wv.y, r.y);
    r.z = fmaf(gv, wv.z, r.z);
    r.w = fmaf(gv, wv.w, r.w);
  }
  float o[4] = {r.x, r.y, r.z, r.w};
  for (int u = 0; u < 4; ++u)
    if ((f + u) % a.c_pad >= a.c_valid) o[u] = 0.f;
  *reinterpret_cast<float4*>(a.out + l * a.out_ls + (long long)b * g.CG + f) = make_float4(o[0], o[1], o[2], o[3]);
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
  for (int c = 0; c < 4; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b = 0; b < g.B; ++b) {
    const float4 xv = __ldg(reinterpret_cast<const float4*>(x + (long long)b * g.CG + f));
    for (int c = 0; c < g.CS; ++c) {
      const float gv = gz[(long long)b * g.CS + c];
      acc[c].x = fmaf(gv, xv.x, acc[c].x);
      acc[c].y = fmaf(gv, xv.y, acc[c].y);
      acc[c].z = fmaf(gv, xv.z, acc[c].z);
      acc[c].w = fmaf(gv, xv.w, acc[c].w);
    }
  }
  for (int c = 0; c < g.CS; ++c) {
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
  if (a.kind == GEMM_DGRAD && g.CG <= 4) return T_OUT_DGRAD;
  if (a.kind == GEMM_FPROP && g.CG == 4 && g.CS <= 64) return T_IN_FPROP;
  if (a.kind == GEMM_WGRAD && g.CG == 4 && g.CS <= 64 && g.k * g.k <= 16) return T_IN_WGRAD;
  return T_NONE;
}

}  // namespace

bool gemm_thin_supported(const GemmArgs& a) { return classify(a) != T_NONE; }

cudaError_t launch_gemm_thin(const GemmArgs& a, cudaStream_t st) {
  const ConvGeo& g = a.g;
  switch (classify(a)) {
    case T_OUT_DGRAD: {
      const long long npix = (long long)g.B * g.GH * g.GW;
      thin_out_dgrad_kernel<<<dim3((unsigned)((npix + 255) / 256), a.L), 256, 0, st>>>(a);
      break;
    }
    case T_IN_FPROP: {
      const long long npix = (long long)g.B * g.SH * g.SW;
      const size_t smem = (size_t)g.CS * g.k * g.k * 4 * sizeof(float);
      dim3 grid((unsigned)((npix + 127) / 128), a.L);
      if (g.CS <= 16) thin_in_fprop_kernel<16><<<grid, 128, smem, st>>>(a);
      else if (g.CS <= 32) thin_in_fprop_kernel<32><<<grid, 128, smem, st>>>(a);
      else thin_in_fprop_kernel<64><<<grid, 128, smem, st>>>(a);
      break;
    }
    case T_IN_WGRAD: {
      const long long K = (long long)g.B * g.SH * g.SW;
      const int nchunk = (int)((K + TW_SPLIT - 1) / TW_SPLIT);
      float* part = gemm_scratch((size_t)a.L * nchunk * 64 * 64, st);
      if (!part) return cudaErrorMemoryAllocation;
      thin_in_wgrad_partial_kernel<<<dim3(nchunk, a.L), 256, 0, st>>>(a, part, nchunk);
      cudaError_t e = launched();
      if (e != cudaSuccess) return e;
      const int nout = g.CS * g.k * g.k * 4;
      thin_in_wgrad_reduce_kernel<<<dim3((nout + 255) / 256, a.L), 256, 0, st>>>(a, part, nchunk);
      break;
    }
    case T_D_FPROP_N4:
      dense_fprop_n4_kernel<<<dim3((unsigned)((g.B * 32 + 255) / 256), a.L), 256, 0, st>>>(a);
      break;
    case T_D_FPROP_SK: {
      const size_t smem = (size_t)g.B * g.CG * sizeof(float);
      dense_fprop_smallk_kernel<<<dim3((unsigned)((g.CS + 127) / 128), a.L), 128, smem, st>>>(a);
      break;
    }
    case T_D_DGRAD_K4: {
      const long long n = (long long)g.B * (g.CG / 4);
      dense_dgrad_k4_kernel<<<dim3((unsigned)((n + 255) / 256), a.L), 256, 0, st>>>(a);
      break;
    }
    case T_D_WGRAD_M4:
      dense_wgrad_m4_kernel<<<dim3((unsigned)((g.CG / 4 + 255) / 256), a.L), 256, 0, st>>>(a);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return launched();
}

}  // namespace pg
