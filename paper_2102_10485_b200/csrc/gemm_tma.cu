// TMA-fed tcgen05 implicit-GEMM engine (sm_100a) for the convolution GEMMs of
// the DC-CGAN step: conv k4 s2 p1 forward / data-grad / weight-grad and the
// transposed convolutions, batched over the L labels of a GPU.
//
// Every operand tile is ONE (or a few) TMA boxes straight out of the NHWC maps,
// no im2col buffer and no per-element address math in the kernel:
//   FPROP A   big map  [L][B][GH][GW][CG] as a 5-D tensor (CG, GW, GH, B, L);
//             the k4 s2 gather of one filter tap is a box with traversal
//             stride s along W and H (elementStrides), its top-left corner at
//             (j0 s - p + kj, i0 s - p + ki); padding = TMA out-of-bounds zero
//             fill.  Box rows = output pixels (b, i, j), 32 channels each.
//   DGRAD A   small map (CS, SW, SH, B, L), unit stride: for one output phase
//             (stride-s sub-lattice of the big map) each valid tap is a plain
//             shifted box.
//   WGRAD A/B small-grad map and strided big map with K = output pixels.
//   weights   3-D (K, N, L) K-major or 4-D (CG, k*k, CS, L) N-major boxes.
// K-major tiles use the 128-byte swizzle (32 fp32 per row = one k-block),
// N/M-major tiles the 128B_ATOM_32B swizzle that tcgen05 requires for tf32
// MN-major operands (descriptor layout SWIZZLE_128B_BASE32B).
//
// Warp roles (320 threads, persistent, one CTA per SM):
//   warp 0      one thread issues the TMA boxes of each stage (mbarrier tx)
//   warps 1-4   TF32X3 only: lo = x - trunc_tf32(x) of each landed stage into
//               a separate lo ring (elementwise: same byte offsets, so the
//               swizzle is irrelevant to them)
//   warp 5      TMEM allocation + the single MMA-issuing thread
//   warps 6-9   drain TMEM segments into fp32 registers, epilogue
// Accuracy design (segmented TMEM accumulation, hi = raw fp32) as gemm_tc.cu.
#include <cuda.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "device_cache.hpp"
#include "gemm_gather.cuh"
#include "tma_common.cuh"
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace pg {

namespace {

using namespace tmac;

constexpr int BM = 128;
constexpr int BKT = 32;   // fp32 of K per k-block: one 128-byte row
constexpr int KSEG = 2;   // k-blocks per TMEM accumulation segment (8 K-steps: chain <= 24 MMA adds in TF32X3)
constexpr int NT = 320;
constexpr int SMEM_BUDGET = 200 * 1024;

struct TmaPlan {
  ConvGeo g;
  int L, phases;
  SpatialBox box;  // FPROP / DGRAD: the 128-row M box; WGRAD: the 32-row K box
  int ntn, ntm, nz, nk;
  int N, kcb;      // GEMM N; 32-channel blocks per filter tap (FPROP CG/32, DGRAD CS/32)
  float* out;
  long long out_ls;
  const float* bias;
  long long bias_ls;
  int act;
  float slope;
  int accumulate, c_valid, c_pad;
};

__host__ __device__ constexpr int a_bytes() { return BM * BKT * 4; }
__host__ __device__ constexpr int b_bytes(int bn) { return bn * BKT * 4; }
__host__ __device__ constexpr int hi_bytes(int bn) { return a_bytes() + b_bytes(bn); }
// TF32X3: the lo ring sits between the split warps and the MMA (a slot is
// refilled only after the MMAs that read it retire), so it gets half the
// stages; the hi ring keeps the rest for TMA latency.
__host__ __device__ constexpr int total_stages(int bn) { return SMEM_BUDGET / hi_bytes(bn); }
__host__ __device__ constexpr int lo_stages(int bn, bool split) { return split ? total_stages(bn) / 2 : 0; }
__host__ __device__ constexpr int hi_stages(int bn, bool split) {
  return total_stages(bn) - lo_stages(bn, split) > 8 ? 8 : total_stages(bn) - lo_stages(bn, split);
}
__host__ __device__ constexpr int smem_total(int bn, bool split) {
  return (hi_stages(bn, split) + lo_stages(bn, split)) * hi_bytes(bn) + 1024 + 1024;
}

PG_DEV void tile_decode(const TmaPlan& P, int t, int& label, int& phase, int& mt, int& nt) {
  nt = t % P.ntn;
  const int r = t / P.ntn;
  mt = r % P.ntm;
  const int z = r / P.ntm;
  label = z / P.phases;
  phase = z % P.phases;
}

template <int KIND, int BN, int MODE>
__global__ void __launch_bounds__(NT, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const TmaPlan P) {
  // BF16 runs the three-pass pipeline with hi rounded in place and lo = 0 (this
  // engine only takes the shapes the pair engine does not)
  constexpr bool SPLIT = MODE == MATH_TF32X3 || MODE == MATH_BF16;
  constexpr int SH = hi_stages(BN, SPLIT);
  constexpr int SL = lo_stages(BN, SPLIT);
  constexpr int HI = hi_bytes(BN);
  constexpr int AB = a_bytes();
  constexpr bool A_MN = KIND == GEMM_WGRAD;
  constexpr bool B_MN = KIND != GEMM_FPROP;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // keep the shared-window provenance (LDS/STS, not generic LD/ST) while aligning to 1024
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* lo_base = smem + SH * HI;
  uint64_t* full_h = reinterpret_cast<uint64_t*>(lo_base + SL * HI);
  uint64_t* empty_h = full_h + SH;
  uint64_t* full_l = empty_h + SH;
  uint64_t* empty_l = full_l + (SL ? SL : 1);
  uint64_t* seg_full = empty_l + (SL ? SL : 1);
  uint64_t* seg_empty = seg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const ConvGeo& g = P.g;
  const int ntiles = P.ntn * P.ntm * P.nz;

  if (tid == 0) {
    for (int s = 0; s < SH; ++s) {
      mbar_init(full_h + s, 1);
      mbar_init(empty_h + s, 1);
    }
    for (int s = 0; s < SL; ++s) {
      mbar_init(full_l + s, 128);
      mbar_init(empty_l + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int label, phase, mt, nt;
        tile_decode(P, t, label, phase, mt, nt);
        const int n0 = nt * BN;
        int b0 = 0, i0 = 0, j0 = 0;
        if (KIND != GEMM_WGRAD) box_origin(P.box, mt, b0, i0, j0);
        DgPhase d{};
        if (KIND == GEMM_DGRAD) d = dg_phase(g, phase);
        for (int kb = 0; kb < P.nk; ++kb, ++it) {
          const int s = it % SH;
          mbar_wait(empty_h + s, ((it / SH) & 1) ^ 1);
          mbar_expect_tx(full_h + s, HI);
          const uint32_t a_dst = smem_u32(smem + s * HI);
          const uint32_t b_dst = a_dst + AB;
          if (KIND == GEMM_FPROP) {
            const int tap = kb / P.kcb, c0 = (kb % P.kcb) * BKT;
            const int ki = tap / g.k, kj = tap % g.k;
            tma_load_5d(a_dst, &tmA, full_h + s, c0, j0 * g.s - g.p + kj, i0 * g.s - g.p + ki, b0, label);
            tma_load_3d(b_dst, &tmB, full_h + s, kb * BKT, n0, label);
          } else if (KIND == GEMM_DGRAD) {
            const int tp = kb / P.kcb, c0 = (kb % P.kcb) * BKT;
            const int ty = tp / d.ntx, tx = tp % d.ntx;
            const int ki = d.ry + ty * g.s, kj = d.rx + tx * g.s;
            const int offy = (d.y0 + g.p - d.ry) / g.s - ty;
            const int offx = (d.x0 + g.p - d.rx) / g.s - tx;
            tma_load_5d(a_dst, &tmA, full_h + s, c0, j0 + offx, i0 + offy, b0, label);
#pragma unroll
            for (int q = 0; q < BN / 32; ++q)
              tma_load_4d(b_dst + q * (BKT * 128), &tmB, full_h + s, n0 + 32 * q, ki * g.k + kj, c0, label);
          } else {
            int kb0, ki0, kj0;
            box_origin(P.box, kb, kb0, ki0, kj0);
            const int m0 = mt * BM;
#pragma unroll
            for (int q = 0; q < BM / 32; ++q)
              tma_load_5d(a_dst + q * (BKT * 128), &tmA, full_h + s, m0 + 32 * q, kj0, ki0, kb0, label);
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) {
              const int n = n0 + 32 * q;
              const int tap = n / g.CG, cg0 = n % g.CG;
              const int ki = tap / g.k, kj = tap % g.k;
              tma_load_5d(b_dst + q * (BKT * 128), &tmB, full_h + s, cg0, kj0 * g.s - g.p + kj,
                          ki0 * g.s - g.p + ki, kb0, label);
            }
          }
        }
      }
    }
  } else if (warp <= 4) {
    // ===================== lo split (TF32X3) =====================
    if (SPLIT) {
      const int st = tid - 32;
      uint32_t it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < P.nk; ++kb, ++it) {
          const int s = it % SH, j = it % SL;
          mbar_wait(full_h + s, (it / SH) & 1);
          mbar_wait(empty_l + j, ((it / SL) & 1) ^ 1);
          const float4* src = reinterpret_cast<const float4*>(smem + s * HI);
          float4* dst = reinterpret_cast<float4*>(lo_base + j * HI);
#pragma unroll 4
          for (int i = st; i < HI / 16; i += 128) {
            const float4 v = src[i];
            if (MODE == MATH_BF16) {
              const_cast<float4*>(src)[i] = bf16_rne4(v);
              dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
              dst[i] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                   v.w - tf32_trunc(v.w));
            }
          }
          fence_async_smem();
          mbar_arrive(full_l + j);
        }
      }
    }
  } else if (warp == 5) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      // K-major SW128: 8-row atoms at 1024 B, K-step of 8 fp32 = +32 B inside the row.
      // MN-major SW128_BASE32B: 4-row atoms at 512 B along K, 32-wide MN atoms at 4096 B.
      constexpr uint32_t a_lbo = A_MN ? 4096u : 16u, a_sbo = A_MN ? 512u : 1024u, a_step = A_MN ? 1024u : 32u;
      constexpr uint32_t b_lbo = B_MN ? 4096u : 16u, b_sbo = B_MN ? 512u : 1024u, b_step = B_MN ? 1024u : 32u;
      constexpr uint32_t a_lay = A_MN ? UMMA_SW128_BASE32B : UMMA_SW128;
      constexpr uint32_t b_lay = B_MN ? UMMA_SW128_BASE32B : UMMA_SW128;
      uint32_t it = 0, sc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int k_seg = 0; k_seg < P.nk; k_seg += KSEG, ++sc) {
          const uint32_t buf = sc & 1;
          mbar_wait(seg_empty + buf, ((sc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * BN;
          const int k_end = min(P.nk, k_seg + KSEG);
          for (int kb = k_seg; kb < k_end; ++kb, ++it) {
            const int s = it % SH;
            mbar_wait(full_h + s, (it / SH) & 1);
            const int j = SPLIT ? it % SL : 0;
            if (SPLIT) mbar_wait(full_l + j, (it / SL) & 1);
            tc_fence_after();
            const uint32_t a_hi = smem_u32(smem + s * HI), b_hi = a_hi + AB;
            const uint32_t a_lo = smem_u32(lo_base + j * HI), b_lo = a_lo + AB;
#pragma unroll
            for (int kk = 0; kk < BKT / 8; ++kk) {
              const uint64_t ah = make_desc(a_hi + kk * a_step, a_lbo, a_sbo, a_lay);
              const uint64_t bh = make_desc(b_hi + kk * b_step, b_lbo, b_sbo, b_lay);
              const uint32_t acc = (kb != k_seg || kk) ? 1u : 0u;
              if (SPLIT) {
                const uint64_t al = make_desc(a_lo + kk * a_step, a_lbo, a_sbo, a_lay);
                const uint64_t bl = make_desc(b_lo + kk * b_step, b_lbo, b_sbo, b_lay);
                mma_tf32(d, al, bh, idesc, acc);  // small terms first
                mma_tf32(d, ah, bl, idesc, 1u);
                mma_tf32(d, ah, bh, idesc, 1u);
              } else {
                mma_tf32(d, ah, bh, idesc, acc);
              }
            }
            mma_commit(empty_h + s);
            if (SPLIT) mma_commit(empty_l + j);
          }
          mma_commit(seg_full + buf);
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== drain + epilogue =====================
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t sc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int label, phase, mt, nt;
      tile_decode(P, t, label, phase, mt, nt);
      const int n0 = nt * BN;
      float acc[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0.f;
      for (int k_seg = 0; k_seg < P.nk; k_seg += KSEG, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(seg_full + buf, (sc >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < BN / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(tmem + lane_base + buf * BN + c * 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c * 16 + i] += __uint_as_float(r[i]);
        }
        tc_fence_before();
        mbar_arrive(seg_empty + buf);
      }
      // row of this thread -> output address
      const int r = q * 32 + lane;
      float* crow = nullptr;
      if (KIND == GEMM_WGRAD) {
        const int m = mt * BM + r;
        if (m < g.CS) crow = P.out + (long long)label * P.out_ls + (long long)m * P.N;
      } else {
        int b0, i0, j0;
        box_origin(P.box, mt, b0, i0, j0);
        const int b = b0 + r / (P.box.TH * P.box.TW);
        const int ii = i0 + (r / P.box.TW) % P.box.TH;
        const int jj = j0 + r % P.box.TW;
        if (KIND == GEMM_FPROP) {
          if (b < g.B && ii < g.SH && jj < g.SW)
            crow = P.out + (long long)label * P.out_ls + (((long long)b * g.SH + ii) * g.SW + jj) * g.CS;
        } else {
          const DgPhase d = dg_phase(g, phase);
          if (b < g.B && ii < d.ny && jj < d.nx)
            crow = P.out + (long long)label * P.out_ls +
                   (((long long)b * g.GH + d.y0 + ii * g.s) * g.GW + d.x0 + jj * g.s) * g.CG;
        }
      }
      if (crow) {
        const float* bias = P.bias ? P.bias + (long long)label * P.bias_ls : nullptr;
#pragma unroll
        for (int c4 = 0; c4 < BN; c4 += 4) {
          const int n = n0 + c4;
          if (n < P.N) {
            float o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float x = acc[c4 + u];
              if (KIND != GEMM_WGRAD) {
                const int nn = n + u;
                if (nn % P.c_pad < P.c_valid) {
                  if (bias) x += bias[nn];
                  x = act_fwd(P.act, x, P.slope);
                } else {
                  x = 0.f;
                }
              }
              o[u] = x;
            }
            float4* dst = reinterpret_cast<float4*>(crow + n);
            if (KIND == GEMM_WGRAD && P.accumulate) {
              const float4 old = *dst;
              o[0] += old.x;
              o[1] += old.y;
              o[2] += old.z;
              o[3] += old.w;
            }
            *dst = make_float4(o[0], o[1], o[2], o[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side

template <int KIND, int BN, int MODE>
cudaError_t launch_tma_bn(const CUtensorMap& ta, const CUtensorMap& tb, const TmaPlan& P, cudaStream_t st) {
  constexpr int smem = smem_total(BN, MODE == MATH_TF32X3 || MODE == MATH_BF16);
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([&] {
    return cudaFuncSetAttribute(gemm_tma_kernel<KIND, BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  if (ce != cudaSuccess) return ce;
  const int tiles = P.ntn * P.ntm * P.nz;
  if (tiles == 0 || P.nk == 0) return cudaSuccess;
  const int grid = std::min(tiles, sm_count_tma());
  gemm_tma_kernel<KIND, BN, MODE><<<grid, NT, smem, st>>>(ta, tb, P);
  return launched();
}

template <int KIND, int MODE>
cudaError_t launch_tma_kind(const CUtensorMap& ta, const CUtensorMap& tb, TmaPlan P, int bn, cudaStream_t st) {
  if (bn == 32) return launch_tma_bn<KIND, 32, MODE>(ta, tb, P, st);
  if (bn == 64) return launch_tma_bn<KIND, 64, MODE>(ta, tb, P, st);
  return launch_tma_bn<KIND, 128, MODE>(ta, tb, P, st);
}

}  // namespace

bool gemm_tma_supported(const GemmArgs& a) {
  static const bool disabled = [] {
    const char* e = std::getenv("PG_NO_TMA");
    return e && std::atoi(e) != 0;
  }();
  if (disabled || !encode_fn()) return false;
  const ConvGeo& g = a.g;
  if (g.s < 1 || g.s > 8 || g.k < 1) return false;
  // strided boxes: traversed extent TW * s <= 256 (TW = 128-row M box width, or 32-row K box width)
  if (a.kind == GEMM_FPROP && spatial_box(g.B, g.SH, g.SW, BM).TW * g.s > 256) return false;
  if (a.kind == GEMM_WGRAD && spatial_box(g.B, g.SH, g.SW, BKT).TW * g.s > 256) return false;
  if (a.kind == GEMM_DGRAD && g.k % g.s) return false;  // every phase has the same tap count
  if (!aligned16(a.out) || !aligned16(a.w) || a.out_ls % 4 || a.w_ls % 4) return false;
  switch (a.kind) {
    case GEMM_FPROP:
      return g.CG % 32 == 0 && g.CS >= 32 && aligned16(a.big) && a.big_ls % 4 == 0;
    case GEMM_DGRAD:
      return g.CS % 32 == 0 && g.CG >= 32 && aligned16(a.small) && a.small_ls % 4 == 0;
    default:
      return g.CG % 32 == 0 && g.CS >= 32 && aligned16(a.small) && aligned16(a.big) && a.small_ls % 4 == 0 &&
             a.big_ls % 4 == 0;
  }
}

cudaError_t launch_gemm_tma(const GemmArgs& a, int math, cudaStream_t st) {
  const ConvGeo& g = a.g;
  TmaPlan P{};
  P.g = g;
  P.L = a.L;
  P.phases = a.kind == GEMM_DGRAD ? g.s * g.s : 1;
  P.out = a.out;
  P.out_ls = a.out_ls;
  P.bias = a.bias;
  P.bias_ls = a.bias_ls;
  P.act = a.act;
  P.slope = a.slope;
  P.accumulate = a.accumulate;
  P.c_valid = a.c_valid;
  P.c_pad = a.c_pad;
  P.nz = a.L * P.phases;
  const int kk = g.k * g.k;
  CUtensorMap ta, tb;
  const int one[5] = {1, 1, 1, 1, 1};
  const int sstr[5] = {1, g.s, g.s, 1, 1};
  bool ok = true;
  int bn;
  if (a.kind == GEMM_FPROP) {
    P.N = g.CS;
    P.kcb = g.CG / BKT;
    P.nk = kk * P.kcb;
    P.box = spatial_box(g.B, g.SH, g.SW, BM);
    P.ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = P.N <= 32 ? 32 : P.N <= 64 ? 64 : 128;
    const long long ad[5] = {g.CG, g.GW, g.GH, g.B, a.L};
    const long long as[4] = {g.CG, (long long)g.GW * g.CG, (long long)g.GH * g.GW * g.CG, a.big_ls};
    const int abox[5] = {BKT, P.box.TW * g.s, P.box.TH * g.s, P.box.TB, 1};
    ok = ok && make_map(&ta, a.big, 5, ad, as, abox, sstr, CU_TENSOR_MAP_SWIZZLE_128B);
    const long long K = (long long)kk * g.CG;
    const long long bd[3] = {K, g.CS, a.L};
    const long long bs[2] = {K, a.w_ls};
    const int bbox[3] = {BKT, bn, 1};
    ok = ok && make_map(&tb, a.w, 3, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (a.kind == GEMM_DGRAD) {
    P.N = g.CG;
    P.kcb = g.CS / BKT;
    const int nty = g.k / g.s, ntx = nty;  // taps per phase (k % s == 0, gemm_tma_supported)
    P.nk = nty * ntx * P.kcb;
    const int ny = (g.GH + g.s - 1) / g.s, nx = (g.GW + g.s - 1) / g.s;
    P.box = spatial_box(g.B, ny, nx, BM);
    P.ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = P.N <= 32 ? 32 : P.N <= 64 ? 64 : 128;
    const long long ad[5] = {g.CS, g.SW, g.SH, g.B, a.L};
    const long long as[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
    const int abox[5] = {BKT, P.box.TW, P.box.TH, P.box.TB, 1};
    ok = ok && make_map(&ta, a.small, 5, ad, as, abox, one, CU_TENSOR_MAP_SWIZZLE_128B);
    const long long bd[4] = {g.CG, kk, g.CS, a.L};
    const long long bs[3] = {g.CG, (long long)kk * g.CG, a.w_ls};
    const int bbox[4] = {32, 1, BKT, 1};
    ok = ok && make_map(&tb, a.w, 4, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  } else {
    P.N = kk * g.CG;
    P.kcb = 0;
    P.box = spatial_box(g.B, g.SH, g.SW, BKT);
    P.nk = P.box.nb * P.box.ny * P.box.nx;
    P.ntm = (g.CS + BM - 1) / BM;
    bn = 128;
    const long long ad[5] = {g.CS, g.SW, g.SH, g.B, a.L};
    const long long as[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
    const int abox[5] = {32, P.box.TW, P.box.TH, P.box.TB, 1};
    ok = ok && make_map(&ta, a.small, 5, ad, as, abox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const long long bd[5] = {g.CG, g.GW, g.GH, g.B, a.L};
    const long long bs[4] = {g.CG, (long long)g.GW * g.CG, (long long)g.GH * g.GW * g.CG, a.big_ls};
    const int bbox[5] = {32, P.box.TW * g.s, P.box.TH * g.s, P.box.TB, 1};
    ok = ok && make_map(&tb, a.big, 5, bd, bs, bbox, sstr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  if (!ok) return cudaErrorInvalidValue;
  P.ntn = (P.N + bn - 1) / bn;
#define PG_TMA_MODES(K)                                                         \
  switch (math) {                                                               \
    case MATH_TF32: return launch_tma_kind<K, MATH_TF32>(ta, tb, P, bn, st);    \
    case MATH_BF16: return launch_tma_kind<K, MATH_BF16>(ta, tb, P, bn, st);    \
    default: return launch_tma_kind<K, MATH_TF32X3>(ta, tb, P, bn, st);         \
  }
  switch (a.kind) {
    case GEMM_FPROP: PG_TMA_MODES(GEMM_FPROP)
    case GEMM_DGRAD: PG_TMA_MODES(GEMM_DGRAD)
    default: PG_TMA_MODES(GEMM_WGRAD)
  }
#undef PG_TMA_MODES
}

}  // namespace pg
