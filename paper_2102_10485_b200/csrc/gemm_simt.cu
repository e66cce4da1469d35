// SIMT fp32 implicit-GEMM engine (math mode FP32_SIMT).  Exact-fp32 products
// with a fixed summation order per output element (k ascending), so results
// are deterministic and independent of the launch configuration.  This is the
// strict-fp32 path and the engine for problems too small for a 128-row
// tcgen05 tile; the tensor-core engine lives in gemm_tc.cu.
#include "gemm_gather.cuh"
#include "kernels.hpp"

namespace pg {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <int KIND>
PG_DEV const float* a_ptr(const ConvGeo& g, const GemmView& v, int m, int k) {
  if (KIND == GEMM_FPROP) return fprop_a_ptr(g, v, m, k);
  if (KIND == GEMM_DGRAD) return dgrad_a_ptr(g, v, m, k);
  return wgrad_a_ptr(g, v, m, k);
}
template <int KIND>
PG_DEV const float* b_ptr(const ConvGeo& g, const GemmView& v, int n, int k) {
  if (KIND == GEMM_FPROP) return fprop_b_ptr(g, v, n, k);
  if (KIND == GEMM_DGRAD) return dgrad_b_ptr(g, v, n, k);
  return wgrad_b_ptr(g, v, n, k);
}
template <int KIND>
PG_DEV float* c_ptr(const ConvGeo& g, const GemmView& v, int m, int n) {
  if (KIND == GEMM_FPROP) return fprop_c_ptr(g, v, m, n);
  if (KIND == GEMM_DGRAD) return dgrad_c_ptr(g, v, m, n);
  return wgrad_c_ptr(g, v, m, n);
}

template <int KIND>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs a) {
  const int phases = gemm_phases(a);
  const int label = blockIdx.z / phases, phase = blockIdx.z % phases;
  const GemmView v = make_view(a, label, phase);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= v.M || n0 >= v.N) return;
  const ConvGeo& g = a.g;

  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  // A is K-major for FPROP/DGRAD, MN-major for WGRAD; B is K-major only for FPROP.
  constexpr bool a_kmajor = KIND != GEMM_WGRAD;
  constexpr bool b_kmajor = KIND == GEMM_FPROP;

  for (int k0 = 0; k0 < v.K; k0 += BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + 256 * r;
      int mm = a_kmajor ? e / BK : e % BM;
      int kk = a_kmajor ? e % BK : e / BM;
      int m = m0 + mm, k = k0 + kk;
      float val = 0.f;
      if (m < v.M && k < v.K) {
        const float* p = a_ptr<KIND>(g, v, m, k);
        if (p) val = *p;
      }
      As[kk][mm] = val;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int e = tid + 256 * r;
      int nn = b_kmajor ? e / BK : e % BN;
      int kk = b_kmajor ? e % BK : e / BN;
      int n = n0 + nn, k = k0 + kk;
      float val = 0.f;
      if (n < v.N && k < v.K) {
        const float* p = b_ptr<KIND>(g, v, n, k);
        if (p) val = *p;
      }
      Bs[kk][nn] = val;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tr * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tc * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + tr * 4 + i;
    if (m >= v.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tc * 4 + j;
      if (n >= v.N) continue;
      float* out = c_ptr<KIND>(g, v, m, n);
      float r = acc[i][j];
      if (KIND == GEMM_WGRAD) {
        if (a.accumulate) r += *out;
      } else if (n % a.c_pad < a.c_valid) {
        if (v.bias) r += v.bias[n];
        r = act_fwd(a.act, r, a.slope);
      } else {
        r = 0.f;
      }
      *out = r;
    }
  }
}

}  // namespace

// Grid: x = N tiles, y = M tiles (max over phases), z = labels x phases.
int gemm_max_m(const GemmArgs& a) {
  const ConvGeo& g = a.g;
  if (a.kind == GEMM_FPROP) return g.B * g.SH * g.SW;
  if (a.kind == GEMM_WGRAD) return g.CS;
  int ny = (g.GH + g.s - 1) / g.s, nx = (g.GW + g.s - 1) / g.s;
  return g.B * ny * nx;
}
int gemm_n(const GemmArgs& a) {
  const ConvGeo& g = a.g;
  if (a.kind == GEMM_FPROP) return g.CS;
  if (a.kind == GEMM_DGRAD) return g.CG;
  return g.k * g.k * g.CG;
}

cudaError_t launch_gemm_simt(const GemmArgs& a, cudaStream_t st) {
  dim3 grid((gemm_n(a) + BN - 1) / BN, (gemm_max_m(a) + BM - 1) / BM, a.L * gemm_phases(a));
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return cudaSuccess;
  switch (a.kind) {
    case GEMM_FPROP: gemm_simt_kernel<GEMM_FPROP><<<grid, 256, 0, st>>>(a); break;
    case GEMM_DGRAD: gemm_simt_kernel<GEMM_DGRAD><<<grid, 256, 0, st>>>(a); break;
    default: gemm_simt_kernel<GEMM_WGRAD><<<grid, 256, 0, st>>>(a); break;
  }
  return launched();
}

}  // namespace pg
