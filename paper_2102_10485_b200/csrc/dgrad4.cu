// Data-gradient-shaped GEMM into a 4-channel map on tcgen05: the generator's
// convT4 forward (64 channels at 32 x 32 -> 3 (+1 pad) channels at 64 x 64,
// tanh; run twice per step) and the discriminator's conv1 data gradient (the
// image gradient the generator step needs):
//   big[y][x][c] = act(bias[c] + sum_{taps reaching (y, x)} sum_cs small[i][j][cs] W[cs][tap][c])
// for k = 4, s = 2, p = 1 (network.cpp:123-142: the reference forms it as a
// GEMM into columns plus col2im; round 1 did the same -- a 1 GB column matrix
// written and re-read per c4 launch, 0.74 ms).
//
// Phase-packed form (gemm_pair.cu's KIND_DGP, here with N = 16): a GEMM row is a
// base position (b, i, j) of the (SH + 1) x (SW + 1) grid, its 16 columns are
// the four output pixels (2i - 1 + ry, 2j - 1 + rx) x 4 channels, and its K =
// 256 runs over the 2 x 2 small-map neighbourhood (i - di, j - dj) x 64
// channels (tap (ry + 2 di, rx + 2 dj)).  A tile is 128 consecutive base
// positions of one image; one TMA box per 32-channel half brings the
// small-map rows under them (128-byte swizzle: conflict-free row reads), and
// eight gather warps (two per TMEM lane quarter, thread = base position) write
// A hi / lo k-block by k-block into a tensor-memory ring.  The MMA runs in the
// TS form, M = 128, N = 16, K = 8 (3xTF32: a_lo b_hi + a_hi b_lo + a_hi b_hi);
// B = the label's 16 x 256 packed weights (hi, lo), built in shared memory by
// the gather warps on a label change.  Four drain warps write each base
// position's four output pixels (bias + activation; the two pixels of a row
// as one 32-byte store).
//
// Warp roles (448 threads): warps 0-3 drain, warp 4 TMA, warp 5 TMEM + MMA,
// warps 6-13 gather (two groups of one warp per lane quarter, alternate k-blocks).
// TMEM: A ring 0..255 (4 k-blocks x hi 32 + lo 32), accumulators 256..287
// (2 tiles x 16).
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

constexpr int D4_TILE = 128;
constexpr int D4_PS = 3;             // patch ring (tiles): the TMA latency of a 52 KB patch spans ~2 tiles
constexpr int D4_WB = 1;             // packed-weight buffers (a label change drains the MMAs: <= 3 per CTA)
constexpr int D4_HALF = 26 * 1024;  // one 32-channel half of the patch: prows x (SW + 2) rows of 128 B
constexpr int D4_PATCH = 2 * D4_HALF;
constexpr int D4_B = 16 * 256 * 4;   // packed weights of one label (16 rows x 256 K), hi or lo
constexpr int D4_AS = 4;             // TMEM A ring (k-blocks; 7 measured no faster)
constexpr int D4_NT = 14 * 32;
constexpr int D4_SMEM = D4_PS * D4_PATCH + 2 * D4_WB * D4_B + 1024 + 1024;  // patch ring | B hi | B lo
constexpr uint32_t D4_ACOL = D4_AS * 64;
// partial accumulators per tile (MMA (kb, kk) adds into ((kb & 1) * 4 + kk) % D4_NACC;
// the drain sums them in a fixed order): eight measured slower than one
constexpr int D4_NACC = 1;

struct D4Plan {
  ConvGeo g;
  int L, tpi, tpl;   // tiles per image, per label
  int gw1;           // base grid width SW + 1
  int pcols;         // patch columns SW + 2
  int prows;         // patch rows: base rows a tile spans + 1
  const float* w;
  long long w_ls;
  float* out;
  long long out_ls;
  const float* bias;
  long long bias_ls;
  int act;
  float slope;
  int c_valid, c_pad;
  int box_bytes;     // TMA bytes of one patch half
};

PG_DEV void mma_tf32_ts1(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int ACT>
PG_DEV float d4_act(float x, float slope) {
  if (ACT == ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == ACT_LRELU) return x >= 0.f ? x : x * slope;
  if (ACT == ACT_TANH) return tanhf(x);
  if (ACT == ACT_SIGMOID) return 1.f / (expf(-x) + 1.f);
  return x;
}

// the four output pixels (2 bi - 1 + ry, 2 bj - 1 + rx) of base position (bi, bj):
// bias + activation on the valid channels, zeros in the pad channels
template <int ACT>
PG_DEV void d4_store(const float (&sum)[16], const D4Plan& P, int label, int b, int bi, int bj) {
  const ConvGeo& g = P.g;
  const float* bias = P.bias ? P.bias + (long long)label * P.bias_ls : nullptr;
  float bb[4] = {0.f, 0.f, 0.f, 0.f};
  if (bias)
    for (int c = 0; c < 4 && c < P.c_valid; ++c) bb[c] = __ldg(bias + c);
  float* ob = P.out + (long long)label * P.out_ls + (long long)b * g.GH * g.GW * 4;
#pragma unroll
  for (int ry = 0; ry < 2; ++ry) {
    const int y = 2 * bi - 1 + ry, x0 = 2 * bj - 1;
    if (y < 0 || y >= g.GH) continue;
    float* orow = ob + ((long long)y * g.GW) * 4;
#pragma unroll
    for (int rx = 0; rx < 2; ++rx) {
      const int x = x0 + rx;
      if (x < 0 || x >= g.GW) continue;
      const int n0 = (ry * 2 + rx) * 4;
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c] = c % P.c_pad < P.c_valid ? d4_act<ACT>(sum[n0 + c] + bb[c], P.slope) : 0.f;
      *reinterpret_cast<float4*>(orow + x * 4) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

// first base position and base row of tile t (of its image)
PG_DEV void d4_tile(const D4Plan& P, int t, int& label, int& b, int& p0, int& ib0) {
  label = t / P.tpl;
  const int ti = t % P.tpl;
  b = ti / P.tpi;
  p0 = (ti % P.tpi) * D4_TILE;
  ib0 = p0 / P.gw1;
}

template <int MODE>
__global__ void __launch_bounds__(D4_NT, 1)
    dgrad4_kernel(const __grid_constant__ CUtensorMap tmS, const D4Plan P) {
  constexpr bool X3 = MODE == MATH_TF32X3, RND = MODE == MATH_BF16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* bhi = smem + D4_PS * D4_PATCH;  // [D4_WB][D4_B]
  uint8_t* blo = bhi + D4_WB * D4_B;       // [D4_WB][D4_B]
  uint64_t* pfull = reinterpret_cast<uint64_t*>(blo + D4_WB * D4_B);
  uint64_t* pfree = pfull + D4_PS;
  uint64_t* wready = pfree + D4_PS;
  uint64_t* wfree = wready + 2;
  uint64_t* aready = wfree + 2;
  uint64_t* afree = aready + D4_AS;
  uint64_t* accfull = afree + D4_AS;
  uint64_t* accfree = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfree + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const ConvGeo& g = P.g;
  const int ntiles = P.L * P.tpl;
  const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
  const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
  const int nbase = (g.SH + 1) * P.gw1;  // base positions per image
  if (tid == 0) {
    for (int s = 0; s < D4_PS; ++s) {
      mbar_init(pfull + s, 1);
      mbar_init(pfree + s, 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(wready + b, 8);
      mbar_init(wfree + b, 1);
      mbar_init(accfull + b, 1);
      mbar_init(accfree + b, 4);
    }
    for (int s = 0; s < D4_AS; ++s) {
      mbar_init(aready + s, 4);
      mbar_init(afree + s, 1);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ===================== TMA: small-map rows under each tile (two channel halves) =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmS);
      for (int t = t0, i = 0; t < t1; ++t, ++i) {
        int label, b, p0, ib0;
        d4_tile(P, t, label, b, p0, ib0);
        const int ps = i % D4_PS;
        mbar_wait(pfree + ps, ((i / D4_PS) & 1) ^ 1);
        mbar_expect_tx(pfull + ps, 2 * P.box_bytes);
        const uint32_t dst = smem_u32(smem + ps * D4_PATCH);
        tma_load_5d(dst, &tmS, pfull + ps, 0, -1, ib0 - 1, b, label);  // P.prows x P.pcols pixels
        tma_load_5d(dst + D4_HALF, &tmS, pfull + ps, 32, -1, ib0 - 1, b, label);
      }
    }
  } else if (warp >= 6) {
    // ===================== gather: packed weights on a label change; A rows -> TMEM =====================
    // two groups of four warps (one per lane quarter): group gr takes the
    // k-blocks kb = gr, gr + 2, ... so two k-blocks are in flight
    const int gwp = warp - 6, q = warp & 3, gr = gwp >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int cur = -1, nsw = 0;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      int label, b, p0, ib0;
      d4_tile(P, t, label, b, p0, ib0);
      if (label != cur) {
        // B[n = ph * 4 + c][k = nbr * 64 + cs] = W[cs][tap(ph, nbr)][c], K-major SW128:
        // k-block kb = k / 32 at kb * 2048, row n at n * 128, chunk (k % 32) / 4 ^ (n & 7)
        cur = label;
        const int wb = nsw % D4_WB, u = nsw / D4_WB;
        ++nsw;
        mbar_wait(wfree + wb, (u & 1) ^ 1);
        const float* w = P.w + (long long)label * P.w_ls;
        for (int e = gwp * 32 + lane; e < 16 * 256; e += 256) {
          const int n = e & 15, k = e >> 4;
          const int ph = n >> 2, c = n & 3, nbr = k >> 6, cs = k & 63;
          const int ki = (ph >> 1) + 2 * (nbr >> 1), kj = (ph & 1) + 2 * (nbr & 1);
          const float v = c < g.CG ? __ldg(w + ((long long)cs * 16 + ki * 4 + kj) * g.CG + c) : 0.f;
          const int off = (k >> 5) * 2048 + n * 128 + ((((k & 31) >> 2) ^ (n & 7)) << 4) + (k & 3) * 4;
          *reinterpret_cast<float*>(bhi + wb * D4_B + off) = RND ? bf16_rne(v) : v;
          *reinterpret_cast<float*>(blo + wb * D4_B + off) = v - tf32_trunc(v);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(wready + wb);
      }
      const int ps = i % D4_PS;
      mbar_wait(pfull + ps, (i / D4_PS) & 1);
      const int pos = p0 + r;
      const bool valid = pos < nbase;
      const int bi = valid ? pos / P.gw1 : ib0, bj = valid ? pos % P.gw1 : 0;
#pragma unroll 1
      for (int kb = gr; kb < 8; kb += 2) {
        const uint32_t kit = (uint32_t)i * 8 + kb;  // k-block index of the CTA's sequence
        const int nbr = kb >> 1, h = kb & 1;
        const int di = nbr >> 1, dj = nbr & 1;
        // patch pixel of (bi - di, bj - dj): patch row 0 is small-map row ib0 - 1, column 0 is -1
        const int idx = (bi - di - ib0 + 1) * P.pcols + (bj - dj + 1);
        const uint8_t* row = smem + ps * D4_PATCH + h * D4_HALF + idx * 128;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(row + ((c ^ (idx & 7)) << 4));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int uu = 0; uu < 4; ++uu) {
            hi[4 * c + uu] = __float_as_uint(RND ? bf16_rne(e[uu]) : e[uu]);
            lo[4 * c + uu] = __float_as_uint(e[uu] - tf32_trunc(e[uu]));
          }
        }
        if (kb >= 6) {
          __syncwarp();
          if (lane == 0) mbar_arrive(pfree + ps);  // patch read (both groups)
        }
        const int as = kit % D4_AS;
        mbar_wait(afree + as, ((kit / D4_AS) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ta = tmem + lane_off + as * 64;
        tmem_st32(ta, hi);
        if (X3) tmem_st32(ta + 32, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(aready + as);
      }
    }
  } else if (warp == 5) {
    // ===================== MMA issue (TS form) =====================
    constexpr uint32_t idesc = make_idesc(128, 16, false, false);
    const uint64_t bh0 = make_desc(smem_u32(bhi), 16u, 1024u, UMMA_SW128);
    const uint64_t bl0 = make_desc(smem_u32(blo), 16u, 1024u, UMMA_SW128);
    int cur = -1, nsw = 0, wb = 0;
    uint32_t kit = 0;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int label = t / P.tpl;
      if (label != cur) {
        if (cur >= 0 && elect_one()) mma_commit(wfree + wb);  // the previous weights free once these MMAs retire
        __syncwarp();
        cur = label;
        wb = nsw % D4_WB;
        const int u = nsw / D4_WB;
        ++nsw;
        mbar_wait(wready + wb, u & 1);
      }
      const int buf = i & 1;
      mbar_wait(accfree + buf, ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + D4_ACOL + buf * (16 * D4_NACC);
      const uint64_t wofs = (uint64_t)((wb * D4_B) >> 4);
      for (int kb = 0; kb < 8; ++kb, ++kit) {
        const int as = kit % D4_AS;
        mbar_wait(aready + as, (kit / D4_AS) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t a_t = tmem + as * 64 + kk * 8;
            const uint64_t bofs = wofs + (uint64_t)((kb * 2048 + kk * 32) >> 4);
            const int ai = ((kb & 1) * 4 + kk) % D4_NACC;
            const uint32_t d = d0 + ai * 16;
            const uint32_t acc = (kb * 4 + kk) >= D4_NACC ? 1u : 0u;
            if (X3) {
              mma_tf32_ts1(d, a_t + 32, bh0 + bofs, idesc, acc);  // small terms first
              mma_tf32_ts1(d, a_t, bl0 + bofs, idesc, 1u);
              mma_tf32_ts1(d, a_t, bh0 + bofs, idesc, 1u);
            } else {
              mma_tf32_ts1(d, a_t, bh0 + bofs, idesc, acc);
            }
          }
          mma_commit(afree + as);
          if (kb == 7) mma_commit(accfull + buf);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== drain + epilogue (warps 0-3) =====================
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const int r = warp * 32 + lane;
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      int label, b, p0, ib0;
      d4_tile(P, t, label, b, p0, ib0);
      const int buf = i & 1;
      mbar_wait(accfull + buf, (i >> 1) & 1);
      tc_fence_after();
      float sum[16];
#pragma unroll
      for (int n = 0; n < 16; ++n) sum[n] = 0.f;
#pragma unroll
      for (int a = 0; a < D4_NACC; ++a) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + D4_ACOL + buf * (16 * D4_NACC) + a * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int n = 0; n < 16; ++n) sum[n] += __uint_as_float(v[n]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accfree + buf);
      const int pos = p0 + r;
      if (pos >= nbase) continue;
      const int bi = pos / P.gw1, bj = pos % P.gw1;
      switch (P.act) {  // one specialised epilogue per activation (tanh only on the valid channels)
        case ACT_TANH: d4_store<ACT_TANH>(sum, P, label, b, bi, bj); break;
        case ACT_RELU: d4_store<ACT_RELU>(sum, P, label, b, bi, bj); break;
        case ACT_LRELU: d4_store<ACT_LRELU>(sum, P, label, b, bi, bj); break;
        case ACT_SIGMOID: d4_store<ACT_SIGMOID>(sum, P, label, b, bi, bj); break;
        default: d4_store<ACT_NONE>(sum, P, label, b, bi, bj); break;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

bool dgrad4_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_DGRAD4");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bool dgrad4_supported(const GemmArgs& a, int math) {
  const ConvGeo& g = a.g;
  if (!dgrad4_enabled() || math == MATH_FP32_SIMT || a.kind != GEMM_DGRAD || a.stat_mode != STAT_NONE) return false;
  if (g.CG != 4 || g.CS != 64 || g.k != 4 || g.s != 2 || g.p != 1 || g.GH != 2 * g.SH || g.GW != 2 * g.SW) return false;
  // a tile's 128 base positions span at most 127 / (SW + 1) + 2 base rows; the
  // small-map rows under them (one more) x (SW + 2) columns must fit a patch half
  const int prows = (D4_TILE - 1) / (g.SW + 1) + 3;
  if (g.SW + 2 > 256 || prows > 256 || g.SH < 1 || prows * (g.SW + 2) * 128 > D4_HALF) return false;
  return encode_fn() && aligned16(a.small) && a.small_ls % 4 == 0 && aligned16(a.out) && a.out_ls % 4 == 0;
}

cudaError_t launch_dgrad4(const GemmArgs& a, int math, cudaStream_t st) {
  const ConvGeo& g = a.g;
  D4Plan P{};
  P.g = g;
  P.L = a.L;
  P.gw1 = g.SW + 1;
  P.pcols = g.SW + 2;
  P.tpi = ((g.SH + 1) * P.gw1 + D4_TILE - 1) / D4_TILE;
  P.tpl = P.tpi * g.B;
  P.w = a.w;
  P.w_ls = a.w_ls;
  P.out = a.out;
  P.out_ls = a.out_ls;
  P.bias = a.bias;
  P.bias_ls = a.bias_ls;
  P.act = a.act;
  P.slope = a.slope;
  P.c_valid = a.c_valid;
  P.c_pad = a.c_pad;
  P.prows = (D4_TILE - 1) / P.gw1 + 3;
  P.box_bytes = 32 * 4 * P.pcols * P.prows;
  CUtensorMap ts;
  const long long sd[5] = {g.CS, g.SW, g.SH, g.B, a.L};
  const long long ss[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
  const int sb[5] = {32, P.pcols, P.prows, 1, 1};
  const int one[5] = {1, 1, 1, 1, 1};
  if (!make_map(&ts, a.small, 5, sd, ss, sb, one, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  static PerDeviceOnce configured;
  cudaError_t e = configured.run([] {
    for (auto f : {dgrad4_kernel<MATH_TF32X3>, dgrad4_kernel<MATH_TF32>, dgrad4_kernel<MATH_BF16>}) {
      cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, D4_SMEM);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  });
  if (e != cudaSuccess) return e;
  const int ntiles = a.L * P.tpl;
  if (ntiles == 0) return cudaSuccess;
  const int grid = std::min(ntiles, sm_count_tma());
  if (math == MATH_TF32X3)
    dgrad4_kernel<MATH_TF32X3><<<grid, D4_NT, D4_SMEM, st>>>(ts, P);
  else if (math == MATH_BF16)
    dgrad4_kernel<MATH_BF16><<<grid, D4_NT, D4_SMEM, st>>>(ts, P);
  else
    dgrad4_kernel<MATH_TF32><<<grid, D4_NT, D4_SMEM, st>>>(ts, P);
  return launched();
}

}  // namespace pg
