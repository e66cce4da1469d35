// Forward convolution from the 4-channel (padded RGB) image map on tcgen05:
// the discriminator's conv1 forward, run three times per step (real batch,
// the discriminator step's fake batch, the generator step's fake batch):
// out[px][co] = act(bias[co] + sum_{tap, c} x[gather(px, tap)][c] W[co][tap][c])
// with k = 4 (16 taps x 4 channels = K = 64) and CS = 64 output channels
// (network.cpp:86-102, conv_fwd's im2col + GEMM).
//
// Round 1 fed these through the CTA-pair engine's KIND_F4 tiles, eight 16-byte
// TMA boxes per k-block (0.52 ms per c4 launch: the TMA moved 16-byte rows,
// the tensor pipe sat at 18%).  Here a tile is 128 consecutive output pixels
// (128 / SW whole output rows of one image): one TMA box brings the input rows
// under them (GW * 16 bytes each), and four gather warps -- one per TMEM lane
// quarter -- read each pixel's 16 taps from that
// patch and write A hi / lo straight into tensor memory (tcgen05.st).  The MMA
// runs in the TS form (A from TMEM, B = the label's weights from shared
// memory, resident while the CTA walks a contiguous range of tiles):
// M = 128, N = 64, K = 64 as 2 x 4 K = 8 steps x 3 (3xTF32: a_lo b_hi +
// a_hi b_lo + a_hi b_hi).  Eight drain warps apply bias + activation into a
// swizzled staging tile that a TMA store writes out (the tile is one contiguous
// 32 KB block of the NHWC output).
//
// Warp roles (448 threads, <= 4 warps per scheduler so 128 registers fit):
// warps 0-3 and 10-13 drain (lane quarter = warp % 4, output channels 0-31 /
// 32-63), warp 4 TMA, warp 5 TMEM allocation + MMA issue, warps 6-9 gather
// (lane quarter = warp % 4, both k-blocks).
// TMEM columns: A stages 0..255 (2 tiles x 2 k-blocks x hi 32 + lo 32),
// accumulators 256..383 (2 tiles x 64).
#include <cuda.h>
#include <stdint.h>

#include <cstdlib>

#include "device_cache.hpp"
#include "kernels.hpp"
#include "tc_ptx.cuh"
#include "tma_common.cuh"

namespace pg {

namespace {

using namespace tmac;

constexpr int F4_TILE = 128;   // output pixels per tile
constexpr int F4_PS = 3;       // patch ring
constexpr int F4_PATCH = 16384;
constexpr int F4_W = 16384;    // weights of one label: 64 co x 64 K fp32 (two SW128 k-blocks)
constexpr int F4_NT = 14 * 32;
constexpr int F4_OUT = F4_TILE * 128;  // output staging of one column half: 128 pixels x 32 channels, SW128
constexpr int F4_SMEM = F4_PS * F4_PATCH + 4 * F4_W + 4 * F4_OUT + 1024 + 1024;  // patch ring | W hi x2 | W lo x2 | out [2 tiles][2 halves]
constexpr uint32_t F4_ACOL = 256;  // first accumulator column

struct F4Plan {
  ConvGeo g;
  int L, tpl;  // labels, tiles per label
  float* out;
  long long out_ls;
  const float* bias;
  long long bias_ls;
  int act;
  float slope;
  int c_valid, c_pad;
  int patch_bytes;
};

// ts-form single-CTA MMA: A (128 rows x K 8) from tensor memory
PG_DEV void mma_tf32_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int ACT>
PG_DEV float f4_act(float x, float slope) {
  if (ACT == ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == ACT_LRELU) return x >= 0.f ? x : x * slope;
  if (ACT == ACT_TANH) return tanhf(x);
  if (ACT == ACT_SIGMOID) return 1.f / (expf(-x) + 1.f);
  return x;
}

// one drain thread: 32 output channels (column half h) of one pixel, into the
// half's 128-byte-swizzled staging rows (16-byte chunk c of row r at c ^ (r & 7):
// consecutive pixels hit distinct banks); a TMA store then writes the tile's
// contiguous 128 x 64 output block (the per-thread 32-byte global stores of the
// first version cost the load/store unit ~4x the wavefronts)
template <int ACT>
PG_DEV void f4_stage(float (&acc)[32], const float (&b)[32], const F4Plan& P, int h, int r, uint8_t* ob) {
  const bool padded = P.c_valid != P.c_pad;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    float x = f4_act<ACT>(acc[c] + b[c], P.slope);
    if (padded && (h * 32 + c) % P.c_pad >= P.c_valid) x = 0.f;
    acc[c] = x;
  }
#pragma unroll
  for (int c4 = 0; c4 < 8; ++c4)
    *reinterpret_cast<float4*>(ob + r * 128 + ((c4 ^ (r & 7)) << 4)) =
        make_float4(acc[4 * c4], acc[4 * c4 + 1], acc[4 * c4 + 2], acc[4 * c4 + 3]);
}

template <int MODE>
__global__ void __launch_bounds__(F4_NT, 1)
    fprop4_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmO, const F4Plan P) {
  constexpr bool X3 = MODE == MATH_TF32X3, RND = MODE == MATH_BF16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* whi = smem + F4_PS * F4_PATCH;  // [2][F4_W]
  uint8_t* wlo = whi + 2 * F4_W;           // [2][F4_W]
  uint8_t* obuf = wlo + 2 * F4_W;           // [2 tiles][2 halves][F4_OUT]
  uint64_t* pfull = reinterpret_cast<uint64_t*>(obuf + 4 * F4_OUT);
  uint64_t* pfree = pfull + F4_PS;
  uint64_t* wfull = pfree + F4_PS;
  uint64_t* wready = wfull + 2;
  uint64_t* wfree = wready + 2;
  uint64_t* aready = wfree + 2;
  uint64_t* afree = aready + 2;
  uint64_t* accfull = afree + 2;
  uint64_t* accfree = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfree + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const ConvGeo& g = P.g;
  // a contiguous range of tiles per CTA: the label (and its weights) rarely changes
  const int ntiles = P.L * P.tpl;
  const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
  const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < F4_PS; ++s) {
      mbar_init(pfull + s, 1);
      mbar_init(pfree + s, 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(wfull + b, 1);
      mbar_init(wready + b, 4);
      mbar_init(wfree + b, 1);
      mbar_init(aready + b, 4);
      mbar_init(afree + b, 1);
      mbar_init(accfull + b, 1);
      mbar_init(accfree + b, 8);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ===================== TMA: weights on a label change, the input patch per tile =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmW);
      tma_prefetch_desc(&tmO);
      int cur = -1, nsw = 0;
      for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int label = t / P.tpl;
        if (label != cur) {
          cur = label;
          const int wb = nsw & 1, u = nsw >> 1;
          ++nsw;
          mbar_wait(wfree + wb, (u & 1) ^ 1);
          mbar_expect_tx(wfull + wb, F4_W);
          tma_load_3d(smem_u32(whi + wb * F4_W), &tmW, wfull + wb, 0, 0, label);
          tma_load_3d(smem_u32(whi + wb * F4_W) + F4_W / 2, &tmW, wfull + wb, 32, 0, label);
        }
        const int ps = i % F4_PS;
        mbar_wait(pfree + ps, ((i / F4_PS) & 1) ^ 1);
        mbar_expect_tx(pfull + ps, P.patch_bytes);
        const int r0 = (t % P.tpl) * (F4_TILE / g.SW);  // first output row (image-major) of the tile
        tma_load_4d(smem_u32(smem + ps * F4_PATCH), &tmX, pfull + ps, 0, (r0 % g.SH) * g.s - g.p, r0 / g.SH, label);
      }
    }
  } else if (warp >= 6 && warp < 10) {
    // ===================== gather: A rows (pixels) -> TMEM hi / lo =====================
    const int gw = warp - 6;
    const int q = warp & 3;
    const int r = q * 32 + lane;  // tile row = pixel
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int orow = r / g.SW, ocol = r % g.SW;
    int cur = -1, nsw = 0;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int label = t / P.tpl;
      if (label != cur) {  // the new weights' lo part (all eight gather warps, elementwise)
        cur = label;
        const int wb = nsw & 1, u = nsw >> 1;
        ++nsw;
        mbar_wait(wfull + wb, u & 1);
        if (X3) {
          const float4* src = reinterpret_cast<const float4*>(whi + wb * F4_W);
          float4* dst = reinterpret_cast<float4*>(wlo + wb * F4_W);
          for (int e = gw * 32 + lane; e < F4_W / 16; e += 128) {
            const float4 v = src[e];
            dst[e] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                 v.w - tf32_trunc(v.w));
          }
          fence_async_smem();
        } else if (RND) {  // bf16 operands: round the landed weights in place
          float4* v4 = reinterpret_cast<float4*>(whi + wb * F4_W);
          for (int e = gw * 32 + lane; e < F4_W / 16; e += 128) v4[e] = bf16_rne4(v4[e]);
          fence_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(wready + wb);
      }
      const int ps = i % F4_PS, ab = i & 1;
      mbar_wait(pfull + ps, (i / F4_PS) & 1);
      mbar_wait(afree + ab, ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const float4* xp = reinterpret_cast<const float4*>(smem + ps * F4_PATCH);
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        const int ki = 2 * kb + (tt >> 2), kj = tt & 3;
        const int pr = orow * g.s + ki, pc = ocol * g.s - g.p + kj;
        const float4 v = (pc >= 0 && pc < g.GW) ? xp[pr * g.GW + pc] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          hi[4 * tt + u] = __float_as_uint(RND ? bf16_rne(e[u]) : e[u]);
          lo[4 * tt + u] = __float_as_uint(e[u] - tf32_trunc(e[u]));
        }
      }
      if (kb == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(pfree + ps);  // patch read
      }
      const uint32_t ta = tmem + lane_off + ab * 128 + kb * 64;
      tmem_st32(ta, hi);
      if (X3) tmem_st32(ta + 32, lo);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(aready + ab);
    }
  } else if (warp == 5) {
    // ===================== MMA issue (TS form) =====================
    constexpr uint32_t idesc = make_idesc(128, 64, false, false);
    const uint64_t bh0 = make_desc(smem_u32(whi), 16u, 1024u, UMMA_SW128);
    const uint64_t bl0 = make_desc(smem_u32(wlo), 16u, 1024u, UMMA_SW128);
    int cur = -1, nsw = 0, wb = 0;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int label = t / P.tpl;
      if (label != cur) {
        if (cur >= 0 && elect_one()) mma_commit(wfree + wb);  // the previous weights are free once these MMAs retire
        __syncwarp();
        cur = label;
        wb = nsw & 1;
        const int u = nsw >> 1;
        ++nsw;
        mbar_wait(wready + wb, u & 1);
      }
      const int ab = i & 1, buf = i & 1;
      mbar_wait(aready + ab, (i >> 1) & 1);
      mbar_wait(accfree + buf, ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + F4_ACOL + buf * 64;
      const uint64_t wofs = (uint64_t)((wb * F4_W) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t a_t = tmem + ab * 128 + kb * 64 + kk * 8;
            const uint64_t bofs = wofs + (uint64_t)((kb * (F4_W / 2) + kk * 32) >> 4);
            const uint32_t acc = (kb || kk) ? 1u : 0u;
            if (X3) {
              mma_tf32_ts(d, a_t + 32, bh0 + bofs, idesc, acc);  // small terms first
              mma_tf32_ts(d, a_t, bl0 + bofs, idesc, 1u);
              mma_tf32_ts(d, a_t, bh0 + bofs, idesc, 1u);
            } else {
              mma_tf32_ts(d, a_t, bh0 + bofs, idesc, acc);
            }
          }
        }
        mma_commit(afree + ab);
        mma_commit(accfull + buf);
      }
      __syncwarp();
    }
  } else {
    // ===================== drain + epilogue (warps 0-3, 14-17) =====================
    const int q = warp & 3, h = warp >= 10 ? 1 : 0;  // lane quarter, column half
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int r = q * 32 + lane;
    float b[32];
    int cur = -1;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int label = t / P.tpl;
      if (label != cur) {
        cur = label;
        const float* bias = P.bias ? P.bias + (long long)label * P.bias_ls + h * 32 : nullptr;
#pragma unroll
        for (int c = 0; c < 32; ++c) b[c] = bias ? __ldg(bias + c) : 0.f;
      }
      const int buf = i & 1;
      mbar_wait(accfull + buf, (i >> 1) & 1);
      tc_fence_after();
      float acc[32];
      {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + F4_ACOL + buf * 64 + h * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) acc[u] = __uint_as_float(v[u]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accfree + buf);
      // staging buffer (tile parity, half): the store issued two tiles ago must
      // have finished reading it
      uint8_t* ob = obuf + ((i & 1) * 2 + h) * F4_OUT;
      const bool issuer = (q == 0) && lane == 0;
      if (issuer) bulk_wait_read<1>();
      named_bar(1 + h, 128);
      switch (P.act) {
        case ACT_RELU: f4_stage<ACT_RELU>(acc, b, P, h, r, ob); break;
        case ACT_LRELU: f4_stage<ACT_LRELU>(acc, b, P, h, r, ob); break;
        case ACT_TANH: f4_stage<ACT_TANH>(acc, b, P, h, r, ob); break;
        case ACT_SIGMOID: f4_stage<ACT_SIGMOID>(acc, b, P, h, r, ob); break;
        default: f4_stage<ACT_NONE>(acc, b, P, h, r, ob); break;
      }
      fence_async_smem();
      named_bar(1 + h, 128);
      if (issuer) {
        tma_store_3d(&tmO, smem_u32(ob), h * 32, (t % P.tpl) * F4_TILE, label);
        bulk_commit();
      }
    }
    if ((q == 0) && lane == 0) bulk_wait<0>();  // stores complete before the CTA's shared memory goes away
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

bool fprop4_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_FPROP4");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bool fprop4_supported(const GemmArgs& a, int math) {
  const ConvGeo& g = a.g;
  if (!fprop4_enabled() || math == MATH_FP32_SIMT || a.kind != GEMM_FPROP || a.stat_mode != STAT_NONE) return false;
  if (g.CG != 4 || g.CS != 64 || g.k != 4 || g.SW < 1 || F4_TILE % g.SW || (g.SH * g.SW) % F4_TILE) return false;
  if (g.GW * 4 > 256 || ((F4_TILE / g.SW - 1) * g.s + g.k) * g.GW * 16 > F4_PATCH) return false;
  if ((long long)g.B * g.SH * g.SW / F4_TILE * a.L >= (1LL << 31)) return false;
  return encode_fn() && aligned16(a.big) && aligned16(a.w) && a.big_ls % 4 == 0 && a.w_ls % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(a.out) & 31) == 0 && a.out_ls % 8 == 0;
}

cudaError_t launch_fprop4(const GemmArgs& a, int math, cudaStream_t st) {
  const ConvGeo& g = a.g;
  F4Plan P{};
  P.g = g;
  P.L = a.L;
  P.tpl = (int)((long long)g.B * g.SH * g.SW / F4_TILE);
  P.out = a.out;
  P.out_ls = a.out_ls;
  P.bias = a.bias;
  P.bias_ls = a.bias_ls;
  P.act = a.act;
  P.slope = a.slope;
  P.c_valid = a.c_valid;
  P.c_pad = a.c_pad;
  const int rows = (F4_TILE / g.SW - 1) * g.s + g.k;
  P.patch_bytes = rows * g.GW * 16;
  CUtensorMap tx, tw;
  const int one[4] = {1, 1, 1, 1};
  const long long xd[4] = {(long long)g.GW * 4, g.GH, g.B, a.L};
  const long long xs[3] = {(long long)g.GW * 4, (long long)g.GH * g.GW * 4, a.big_ls};
  const int xb[4] = {g.GW * 4, rows, 1, 1};
  if (!make_map(&tx, a.big, 4, xd, xs, xb, one, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  const long long wd[3] = {64, g.CS, a.L};
  const long long ws[2] = {64, a.w_ls};
  const int wbx[3] = {32, 64, 1};
  if (!make_map(&tw, a.w, 3, wd, ws, wbx, one, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  CUtensorMap to;
  const long long od[3] = {g.CS, (long long)g.B * g.SH * g.SW, a.L};
  const long long os[2] = {g.CS, a.out_ls};
  const int ob[3] = {32, F4_TILE, 1};
  if (!make_map(&to, a.out, 3, od, os, ob, one, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  static PerDeviceOnce configured;
  cudaError_t e = configured.run([] {
    for (auto f : {fprop4_kernel<MATH_TF32X3>, fprop4_kernel<MATH_TF32>, fprop4_kernel<MATH_BF16>}) {
      cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, F4_SMEM);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  });
  if (e != cudaSuccess) return e;
  const int ntiles = a.L * P.tpl;
  const int grid = std::min(ntiles, sm_count_tma());
  if (ntiles == 0) return cudaSuccess;
  if (math == MATH_TF32X3)
    fprop4_kernel<MATH_TF32X3><<<grid, F4_NT, F4_SMEM, st>>>(tx, tw, to, P);
  else if (math == MATH_BF16)
    fprop4_kernel<MATH_BF16><<<grid, F4_NT, F4_SMEM, st>>>(tx, tw, to, P);
  else
    fprop4_kernel<MATH_TF32><<<grid, F4_NT, F4_SMEM, st>>>(tx, tw, to, P);
  return launched();
}

}  // namespace pg
