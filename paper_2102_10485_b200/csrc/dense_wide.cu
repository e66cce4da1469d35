// Wide dense FPROP with a small K: the generator's latent projection
// (Dense d_z -> C0*h0*w0, reference dense_fwd / dense_bwd, network.cpp:28-45;
// c4: out[32][8192] = z[32][100] W^T per label, W 3.4 MB per label).
//
// The pair engine ran this GEMM with 32 useful rows in 256-row tiles and four
// k-blocks per tile (12% of the HBM roofline).  The work is
// W-streaming: every weight is used B times, so plain fp32 FMAs on the CUDA
// cores (exact fp32, one fixed summation order) keep up with HBM:
//   FPROP  warp = 32 output features x 32 batch rows (register tile 4 x 8 per
//          lane), the label's latents in shared memory, each weight row
//          streamed from HBM once; epilogue bias + activation, or the
//          BatchNorm statistic slot of the 32 rows (STAT_FWD: shift, sum, sum
//          of squares, count -- the pair engine's format, merged by
//          bn_stats_finalize)
// Measured (c4, 125 labels x 32): 0.27 ms per launch vs 0.69 ms on the pair
// engine; 62% of issued instructions are FFMA, 68% issue-slot utilisation
// (ncu), i.e. ~40% of the CUDA-core FMA roofline (101 us).  The weight gradient
// of the same layer stays on the pair engine (a SIMT version measured 0.26-0.35
// vs 0.27 ms: no gain).
#include "device_cache.hpp"
#include "kernels.hpp"

namespace pg {

namespace {

constexpr int DW_N = 64;     // minimum output width routed here
constexpr int DW_RB = 32;    // batch rows per pass = one statistic slot
constexpr int DW_KMAX = 256;
constexpr int DW_BMAX = 128; // latent rows staged in shared memory

template <int ACT>
PG_DEV float act_dw(float x, float slope) {
  if (ACT == ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == ACT_LRELU) return x >= 0.f ? x : x * slope;
  if (ACT == ACT_TANH) return tanhf(x);
  if (ACT == ACT_SIGMOID) return 1.f / (expf(-x) + 1.f);
  return x;
}

PG_DEV void cp_async16(void* dst, const void* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
PG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
PG_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Warp tile = 32 features x 32 batch rows (one statistic slot); lane = (nq =
// lane % 8, bq = lane / 8) owns features n0 + nq + 8i (i < 4) and rows
// b0 + bq + 4j (j < 8): 128 FMAs per 4-deep k step from four float4 weight
// reads and eight float4 latent reads, all from shared memory.  The weights
// stream from HBM once per pass through a per-warp cp.async ring (lane l
// copies row n0 + l, DW_PF steps ahead; no block-level synchronisation).
constexpr int DW_WN = 32;    // features per warp
constexpr int DW_WARPS = 8;  // warps per block (256 features)
constexpr int DW_PF = 8;     // weight ring depth (k steps of 4)
template <int ACT, bool STATS>
__global__ void __launch_bounds__(DW_WARPS * 32) dense_wide_fprop_kernel(GemmArgs a) {
  extern __shared__ __align__(16) float smem[];
  const ConvGeo& g = a.g;
  const int K = g.CG, N = g.CS, B = g.B;
  const int l = blockIdx.y;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, nq = lane % 8, bq = lane / 8;
  const int nb = (B + DW_RB - 1) / DW_RB;
  float4* ring = reinterpret_cast<float4*>(smem) + warp * DW_PF * 32;  // [DW_PF][32 rows]
  float* zs = smem + DW_WARPS * DW_PF * 32 * 4;                         // [nb * 32][K]
  {
    const float4* x4 = reinterpret_cast<const float4*>(a.big + l * a.big_ls);
    float4* zs4 = reinterpret_cast<float4*>(zs);
    const int nz = nb * DW_RB * (K / 4);
    for (int e = tid; e < nz; e += DW_WARPS * 32) zs4[e] = e < B * (K / 4) ? __ldg(x4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const int n0 = (blockIdx.x * DW_WARPS + warp) * DW_WN;
  if (n0 >= N) return;
  const float* wl = a.w + l * a.w_ls;
  const float4* my_row = reinterpret_cast<const float4*>(wl + (long long)min(n0 + lane, N - 1) * K);  // ring feeder
  const float* bias = a.bias ? a.bias + l * a.bias_ls : nullptr;
  bool nok[4], padc[4];
  float bn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int n = n0 + nq + 8 * i;
    nok[i] = n < N;
    bn[i] = bias && nok[i] ? bias[n] : 0.f;
    padc[i] = nok[i] && (n % a.c_pad >= a.c_valid);
  }
  float* out = a.out + l * a.out_ls;
  const int K4 = K / 4;
  for (int b0 = 0; b0 < B; b0 += DW_RB) {
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const float* zr = zs + (b0 + bq) * K;
#pragma unroll
    for (int s = 0; s < DW_PF - 1; ++s) {
      if (s < K4) cp_async16(ring + s * 32 + lane, my_row + s);
      cp_async_commit();
    }
    for (int k4 = 0; k4 < K4; ++k4) {
      const int kk = k4 + DW_PF - 1;
      if (kk < K4) cp_async16(ring + (kk % DW_PF) * 32 + lane, my_row + kk);
      cp_async_commit();
      cp_async_wait<DW_PF - 1>();
      __syncwarp();
      const float4* rs = ring + (k4 % DW_PF) * 32 + nq;
      float4 w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = rs[8 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 z = *reinterpret_cast<const float4*>(zr + 4 * j * K + 4 * k4);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          acc[i][j] = fmaf(z.w, w[i].w, fmaf(z.z, w[i].z, fmaf(z.y, w[i].y, fmaf(z.x, w[i].x, acc[i][j]))));
      }
      __syncwarp();  // slot k4 % DW_PF is refilled by the next iteration
    }
    cp_async_wait<0>();
    const int rows = min(DW_RB, B - b0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = n0 + nq + 8 * i;
      float s1 = 0.f, s2 = 0.f, sft = 0.f;
      if (STATS) sft = padc[i] ? 0.f : __shfl_sync(0xffffffffu, acc[i][0] + bn[i], nq);  // row b0 (bq = 0, j = 0)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = bq + 4 * j;
        float t = acc[i][j] + bn[i];
        if (!STATS) t = act_dw<ACT>(t, a.slope);
        if (padc[i]) t = 0.f;
        if (nok[i] && b < rows) out[(long long)(b0 + b) * N + n] = t;
        if (STATS && b < rows) {
          const float d = t - sft;
          s1 += d;
          s2 += d * d;
        }
      }
      if (STATS) {
        // rows of the slot are spread over bq = lane / 8: fixed butterfly (deterministic)
        s1 += __shfl_xor_sync(0xffffffffu, s1, 8);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 8);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 16);
        if (bq == 0 && nok[i]) {
          float* st = a.stat + ((long long)l * nb + b0 / DW_RB) * 4 * N + n;
          st[0] = sft;
          st[N] = s1;
          st[2 * N] = s2;
          st[3 * N] = (float)rows;
        }
      }
    }
  }
}

size_t fprop_smem(const ConvGeo& g) {
  return sizeof(float) * ((size_t)DW_WARPS * DW_PF * 32 * 4 + (size_t)((g.B + DW_RB - 1) / DW_RB) * DW_RB * g.CG);
}

template <class Kern>
cudaError_t opt_in(PerDeviceMax& cfg, Kern k, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cfg.raise(smem, [&] { return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
}

template <int ACT, bool STATS>
cudaError_t launch_fprop_t(const GemmArgs& a, size_t smem, cudaStream_t st) {
  static PerDeviceMax cfg;
  cudaError_t e = opt_in(cfg, dense_wide_fprop_kernel<ACT, STATS>, smem);
  if (e != cudaSuccess) return e;
  const int per_block = DW_WARPS * DW_WN;
  dense_wide_fprop_kernel<ACT, STATS>
      <<<dim3((unsigned)((a.g.CS + per_block - 1) / per_block), (unsigned)a.L), DW_WARPS * 32, smem, st>>>(a);
  return launched();
}

}  // namespace

bool dense_wide_supported(const GemmArgs& a) {
  const ConvGeo& g = a.g;
  if (!(g.k == 1 && g.SH == 1 && g.SW == 1 && g.GH == 1 && g.GW == 1)) return false;
  if (g.CS < DW_N || g.CG > DW_KMAX || g.CG % 4 || g.CS % 4 || g.B < 1) return false;
  return a.kind == GEMM_FPROP && g.B <= DW_BMAX && fprop_smem(g) <= 200 * 1024;
}

int dense_wide_stat_slots(const GemmArgs& a) {
  return a.kind == GEMM_FPROP && dense_wide_supported(a) ? (a.g.B + DW_RB - 1) / DW_RB : 0;
}

cudaError_t launch_dense_wide(const GemmArgs& a, cudaStream_t st) {
  const ConvGeo& g = a.g;
  const size_t smem = fprop_smem(g);
  if (a.stat_mode == STAT_FWD) return launch_fprop_t<ACT_NONE, true>(a, smem, st);
  if (a.stat_mode != STAT_NONE) return cudaErrorInvalidValue;
  switch (a.act) {
    case ACT_RELU: return launch_fprop_t<ACT_RELU, false>(a, smem, st);
    case ACT_LRELU: return launch_fprop_t<ACT_LRELU, false>(a, smem, st);
    case ACT_TANH: return launch_fprop_t<ACT_TANH, false>(a, smem, st);
    case ACT_SIGMOID: return launch_fprop_t<ACT_SIGMOID, false>(a, smem, st);
    default: return launch_fprop_t<ACT_NONE, false>(a, smem, st);
  }
}

}  // namespace pg
