// CTA-pair tcgen05 implicit-GEMM engine (sm_100a, cluster of 2, cta_group::2)
// for the big convolution GEMMs of the DC-CGAN step.
//
// Why pairs: with fp32 operands a 128 x 128 single-CTA tile needs 32 KB of
// operands per 32-deep k-block, i.e. ~128 B/clk/SM at the tf32 MMA rate —
// three times what L2 can feed 148 SMs (measured: plain TF32 tops out at
// ~28% of the tensor pipe in gemm_tma.cu, TF32X3 at ~50%).  A pair computes a
// 256 x BN tile with `tcgen05.mma.cta_group::2`: each CTA stages its own 128
// rows of A and HALF of the BN columns of B, the two SMs' tensor cores share
// the B halves, so operand bytes per flop halve.
//
//   tile      M = 256 (CTA rank r owns rows 128r..128r+127), N = BN in {64, 128, 256}
//   FPROP     rows = output pixels (M box 2*mtp + r), B = weights [N][K] K-major
//   DGRAD     rows = pixels of one stride phase of the big map, B = weights N-major
//   WGRAD     SWAPPED w.r.t. gemm_tma.cu: rows = (tap, cin) = 16*CG, N = CS (Cout),
//             K = output pixels; A = strided big-map boxes, B = gradient boxes,
//             both MN-major; the epilogue writes W[cs][tap][cg] column-wise
//
// Warp roles (384 threads, persistent, one pair per 2 SMs):
//   warp 0      TMA producer: its CTA's A rows + B half of every stage
//   warps 1-2   TF32X3: lo = x - trunc_tf32(x) of the landed stage into the lo
//               ring; TF32: forward the "landed" event.  Either way they then
//               arrive on the LEADER's `ready` barrier (both CTAs, remote arrive)
//   warp 3      TMEM allocation (cta_group::2, both CTAs); in the leader the
//               single MMA-issuing thread; commits multicast to both CTAs
//   warps 4-11  drain: warp w reads TMEM lane quarter w%4, column half (w-4)/4
//               of its CTA's accumulator rows; fp32 register sums; epilogue
// Accuracy design (segmented TMEM accumulation into IEEE fp32 registers,
// hi = raw fp32, small terms first) as gemm_tc.cu / gemm_tma.cu.
#include <cuda.h>
#include <stdint.h>

#include "device_cache.hpp"
#include "kernels.hpp"
#include "tc_ptx.cuh"
#include "tma_common.cuh"

namespace pg {

namespace {

using namespace tmac;

constexpr int BM = 128;   // rows per CTA
constexpr int BKT = 32;   // fp32 of K per k-block (one 128-byte row)
// split / forward warps: the lo split of a k-block must keep up with its MMAs,
// which take half as long on BN <= 128 tiles (measured: 2 warps paced the
// narrow tiles in TF32X3 once MMA issue was warp-uniform)
// (FPROP / DGRAD in TF32X3; the WGRAD tiles measured slower with 4: 1.45 vs 1.35 ms)
#ifndef PG_NSPLIT_NARROW
#define PG_NSPLIT_NARROW 4
#endif
#ifndef PG_NSPLIT_WG
#define PG_NSPLIT_WG 2
#endif
#ifndef PG_WIDE_REGS
#define PG_WIDE_REGS 1  // setmaxnreg hand-off to the drain warps of the BN = 256 tiles
#endif
#ifndef PG_REGS_LO
#define PG_REGS_LO 56
#endif
#ifndef PG_REGS_HI
#define PG_REGS_HI 224
#endif
__host__ __device__ constexpr int nsplit(int kind, int bn, int mode) {
  return mode != MATH_TF32X3 || bn > 128 ? 2 : kind == GEMM_WGRAD ? PG_NSPLIT_WG : PG_NSPLIT_NARROW;
}
__host__ __device__ constexpr int pair_nt(int kind, int bn, int mode) { return (nsplit(kind, bn, mode) + 2 + 8) * 32; }
constexpr int NDRAIN = 8;
constexpr int W_DRAIN = 4;  // first drain warp of the A-in-TMEM kernel
constexpr int SMEM_BUDGET = 200 * 1024;
constexpr int KIND_DGP = 3;  // phase-packed stride-2 DGRAD (k = 4, s = 2, p = 1), engine-internal
// widest packed N: packing CG = 128 (N = 512) measured 1.36 vs 1.22 ms on the
// 16x16 layer (the 9x9 base grid wastes 27% of the rows), CG = 256: 1.75 vs 0.98
#ifndef PG_DGP_MAXN
#define PG_DGP_MAXN 256
#endif
constexpr int KIND_F4 = 4;   // FPROP from a 4-channel (padded RGB) map: a k-block = 8 taps x 4 channels
#ifndef PG_PAIR_SL
#define PG_PAIR_SL 0
#endif

struct PairPlan {
  ConvGeo g;
  int L, phases;
  SpatialBox box;  // FPROP / DGRAD: the 128-row M box; WGRAD: the 32-row K box
  int ntn, ntmp, nz, nk;
  int N, kcb, mrows;  // GEMM N; 32-channel blocks per tap; WGRAD rows (16 CG)
  int kseg;           // k-blocks per TMEM accumulation segment
  float* out;
  long long out_ls;
  const float* bias;
  long long bias_ls;
  int act;
  float slope;
  int accumulate, c_valid, c_pad;
  int stat_mode, nslot;
  int CGn;  // output channels (stat_mu stride; = N except phase-packed DGRAD)
  int stage_tx;  // TMA bytes per stage (A box rows may be < 128: the rest of the tile is never read back)
  float* stat;
  const float* stat_y;
  const float* stat_z;
  const float* stat_mu;
  int stat_act;
  float stat_slope;
  int blo;  // TF32X3 FPROP: b_lo comes pre-split from global (tmBl) instead of the split warps
};

// Sum of v[0..7] over the 32 lanes of a warp in 9 shuffles (recursive
// halving): afterwards lanes 4c..4c+3 hold the total of column red8_col(lane) = c.
PG_DEV int red8_col(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }
PG_DEV float red8(float (&v)[8], int lane) {
#pragma unroll
  for (int w = 4, m = 16; w >= 1; w >>= 1, m >>= 1) {
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? v[i] : v[i + w];
      const float keep = up ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  float r = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 2);
  return r + __shfl_xor_sync(0xffffffffu, r, 1);
}


// activation derivative through the output for the fused backward modes
// (ReLU / LeakyReLU / none: branch-free selects; see common.cuh act_bwd)
PG_DEV float act_bwd_rl(int act, float g, float y, float slope) {
  const float neg = act == ACT_LRELU ? g * slope : (act == ACT_RELU ? 0.f : g);
  const bool pos = act == ACT_LRELU ? y >= 0.f : y > 0.f;
  return act == ACT_NONE || pos ? g : neg;
}

template <int ACT>
PG_DEV float act_t(float x, float slope) {
  if (ACT == ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == ACT_LRELU) return x >= 0.f ? x : x * slope;
  if (ACT == ACT_TANH) return tanhf(x);
  if (ACT == ACT_SIGMOID) return 1.f / (expf(-x) + 1.f);
  return x;
}

// Where one accumulator row's columns go.  Plain tiles: the row is one output
// pixel, column n = channel n at offset off0 + n.  Phase-packed DGRAD tiles
// (KIND_DGP): the row is a base position (b, i0, j0) of the stride-2 grid and
// column n = (phase, channel) with phase = n / CG, i.e. output pixel
// (2 i0 - 1 + ry, 2 j0 - 1 + rx) -- each 2x2 output block reads the same 2x2
// small-map neighbourhood, so all four phases share one A operand.
struct RowPix {
  long long off0;  // plain: per-label offset of channel 0 (-1: padding row)
  int b, i0, j0;   // packed: base position (b < 0: padding row)
  int packed, CG, GH, GW;
  PG_DEV int chan(int n) const { return packed ? n % CG : n; }
  // per-label offset of column n's element, -1 when it does not exist
  PG_DEV long long addr(int n) const {
    if (!packed) return off0 < 0 ? -1 : off0 + n;
    if (b < 0) return -1;
    const int ph = n / CG;
    const int y = 2 * i0 - 1 + (ph >> 1), x = 2 * j0 - 1 + (ph & 1);
    if (y < 0 || y >= GH || x < 0 || x >= GW) return -1;
    return (((long long)b * GH + y) * GW + x) * CG + n % CG;
  }
};

// bias, padding columns (written 0) and activation of one output row, eight
// columns per 256-bit store (one full 32-byte sector per lane: float4 stores
// left every sector half-written twice); the next group's bias is loaded while
// the current one is computed
template <int ACT, int BH>
PG_DEV void epi_store(const float (&acc)[BH], const RowPix& rp, float* out, int nb, const float* bias,
                      const PairPlan& P) {
  const bool padded = P.c_valid != P.c_pad;
  float4 bn0 = make_float4(0.f, 0.f, 0.f, 0.f), bn1 = bn0;
  if (bias && nb < P.N) {
    bn0 = __ldg(reinterpret_cast<const float4*>(bias + rp.chan(nb)));
    bn1 = __ldg(reinterpret_cast<const float4*>(bias + rp.chan(nb) + 4));
  }
#pragma unroll
  for (int c8 = 0; c8 < BH; c8 += 8) {
    const int n = nb + c8;
    if (n >= P.N) break;
    const float bb[8] = {bn0.x, bn0.y, bn0.z, bn0.w, bn1.x, bn1.y, bn1.z, bn1.w};
    if (bias && c8 + 8 < BH && n + 8 < P.N) {
      bn0 = __ldg(reinterpret_cast<const float4*>(bias + rp.chan(n + 8)));
      bn1 = __ldg(reinterpret_cast<const float4*>(bias + rp.chan(n + 8) + 4));
    }
    const long long a = rp.addr(n);
    if (a < 0) continue;
    const int ch = rp.chan(n);
    float o[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float x = acc[c8 + u] + bb[u];
      x = act_t<ACT>(x, P.slope);
      if (padded && (ch + u) % P.c_pad >= P.c_valid) x = 0.f;
      o[u] = x;
    }
    st_global_v8(out + a, o);
  }
}

// output row + per-channel statistics over the warp's 32 rows (StatMode);
// warp-uniform: every lane runs it, padding rows / missing phase pixels
// contribute nothing.  Statistics are per GEMM column (packed tiles: per
// (phase, channel), folded by the finalize kernels).
template <int MODE, int BH>
PG_DEV void epi_stats(const float (&acc)[BH], const RowPix& rp, float* out, int nb, const float* bias, float* st,
                      int label, int lane, const PairPlan& P) {
  const bool padded = P.c_valid != P.c_pad;
  const int col = red8_col(lane);
#pragma unroll
  for (int c8 = 0; c8 < BH; c8 += 8) {
    const int n0 = nb + c8;
    if (n0 >= P.N) break;
    const long long a = rp.addr(n0);
    const bool valid = a >= 0;
    const long long lo_off = valid ? a : 0;  // per-label offset of this thread's 8 elements
    const int ch = rp.chan(n0);
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    const float rows = (float)__popc(vmask);
    const int src = vmask ? __ffs(vmask) - 1 : 0;  // shift from a real row (never a stale one)
    float v[8], w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float x = acc[c8 + u];
      if (bias) x += bias[ch + u];
      if (padded && (ch + u) % P.c_pad >= P.c_valid) x = 0.f;
      v[u] = x;
    }
    if (MODE != STAT_FWD) {
#pragma unroll
      for (int u4 = 0; u4 < 8; u4 += 4) {
        float4 y4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) y4 = __ldg(reinterpret_cast<const float4*>(P.stat_y + (long long)label * P.out_ls + lo_off + u4));
        v[u4] = act_bwd_rl(P.stat_act, v[u4], y4.x, P.stat_slope);
        v[u4 + 1] = act_bwd_rl(P.stat_act, v[u4 + 1], y4.y, P.stat_slope);
        v[u4 + 2] = act_bwd_rl(P.stat_act, v[u4 + 2], y4.z, P.stat_slope);
        v[u4 + 3] = act_bwd_rl(P.stat_act, v[u4 + 3], y4.w, P.stat_slope);
      }
    }
    if (valid) st_global_v8(out + lo_off, v);
    float* s8 = st + n0;
    if (MODE == STAT_FWD) {
      // shifted sums around the slot's first row (lane 0), merged across slots
      // with Chan's formula by bn_stats_finalize
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float sh = __shfl_sync(0xffffffffu, v[u], src);
        if (lane == src) s8[u] = sh;
        v[u] = valid ? v[u] - sh : 0.f;
        w[u] = v[u] * v[u];
      }
      const float s1 = red8(v, lane);
      const float s2 = red8(w, lane);
      if (!(lane & 3)) {
        s8[P.N + col] = s1;
        s8[2 * P.N + col] = s2;
        s8[3 * P.N + col] = rows;
      }
    } else if (MODE == STAT_BWD_BN) {
      const float* mu = P.stat_mu + (long long)label * P.CGn + ch;
      float t[8];
#pragma unroll
      for (int u4 = 0; u4 < 8; u4 += 4) {
        float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) z4 = __ldg(reinterpret_cast<const float4*>(P.stat_z + (long long)label * P.out_ls + lo_off + u4));
        w[u4] = valid ? z4.x - mu[u4] : 0.f;
        w[u4 + 1] = valid ? z4.y - mu[u4 + 1] : 0.f;
        w[u4 + 2] = valid ? z4.z - mu[u4 + 2] : 0.f;
        w[u4 + 3] = valid ? z4.w - mu[u4 + 3] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (!valid) v[u] = 0.f;
        t[u] = v[u] * w[u];
      }
      const float s1 = red8(v, lane);
      const float s2 = red8(t, lane);
      const float s3 = red8(w, lane);
      if (!(lane & 3)) {
        s8[col] = s1;
        s8[P.N + col] = s2;
        s8[2 * P.N + col] = s3;
        s8[3 * P.N + col] = 0.f;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (!valid) v[u] = 0.f;
      const float s1 = red8(v, lane);
      if (!(lane & 3)) {
        s8[col] = s1;
        s8[P.N + col] = 0.f;
        s8[2 * P.N + col] = 0.f;
        s8[3 * P.N + col] = 0.f;
      }
    }
  }
}

__host__ __device__ constexpr int a_bytes() { return BM * BKT * 4; }
__host__ __device__ constexpr int stage_bytes(int bn) { return a_bytes() + (bn / 2) * BKT * 4; }
__host__ __device__ constexpr int total_stages(int bn) { return SMEM_BUDGET / stage_bytes(bn); }
// Equal hi and lo rings (lo slot j == hi slot s): measured 1.4-1.6x faster on
// the BN = 64 / 128 tiles than one stage more on either side (PG_PAIR_SL = +-1,
// scripts/gemm_sweep.py with tuning-variant builds).
__host__ __device__ constexpr int lo_stages(int bn, bool split) { return split ? (bn >= 256 ? 3 : total_stages(bn) / 2 + PG_PAIR_SL) : 0; }
__host__ __device__ constexpr int hi_stages(int bn, bool split) {
  return total_stages(bn) - lo_stages(bn, split) > 8 ? 8 : total_stages(bn) - lo_stages(bn, split);
}
#ifndef PG_PF_NARROW
#define PG_PF_NARROW 0
#endif
#ifndef PG_PF_WIDE
#define PG_PF_WIDE 0
#endif
// L2 prefetch distance in k-blocks (0 = off).  Measured slower at every
// distance tried (4 / 8 / 16 narrow, 8 wide; up to 1.8x on the conv2 weight
// gradient): the narrow tiles are shared-memory-bandwidth bound, not latency
// bound, and the extra TMA requests only compete.
__host__ __device__ constexpr int pf_dist(int bn, bool split) { return bn >= 256 ? PG_PF_WIDE : PG_PF_NARROW; }
__host__ __device__ constexpr int smem_total(int bn, bool split) {
  return (hi_stages(bn, split) + lo_stages(bn, split)) * stage_bytes(bn) + 1024 + 1024;
}

PG_DEV void pair_tile_decode(const PairPlan& P, int t, int& label, int& phase, int& mtp, int& nt) {
  nt = t % P.ntn;
  const int r = t / P.ntn;
  mtp = r % P.ntmp;
  const int z = r / P.ntmp;
  label = z / P.phases;
  phase = z % P.phases;
}

// TMEM accumulation buffers (segments in flight between the MMA and the drain)
__host__ __device__ constexpr int seg_bufs(int bn) { return 512 / bn > 4 ? 4 : 512 / bn; }

// TMA boxes of k-block kb for this CTA: its 128 A rows and its B half
template <int KIND, int BH, bool PF = false>
PG_DEV void pair_issue(const CUtensorMap& tmA, const CUtensorMap& tmB, const PairPlan& P, uint32_t a_dst,
                       uint32_t b_dst, uint64_t* bar, int kb, int label, int mtp, uint32_t rank, int n0, int b0,
                       int i0, int j0, const DgPhase& d, const CUtensorMap* tmBl = nullptr, uint32_t bl_dst = 0) {
  const ConvGeo& g = P.g;
  if (KIND == KIND_F4) {
    // eight 128-row x 16-byte boxes (one per tap) side by side along K: the
    // no-swizzle K-major layout (core matrix = 8 rows x 4 fp32 = 128 B, +128 B
    // per 8 rows along M, +2048 B per tap along K)
#pragma unroll
    for (int t = 0; t < BKT / 4; ++t) {
      const int tap = kb * (BKT / 4) + t;
      const int ki = tap / g.k, kj = tap % g.k;
      tbox<PF>(a_dst + t * (BM * 16), &tmA, bar, 0, j0 * g.s - g.p + kj, i0 * g.s - g.p + ki, b0, label);
    }
    tbox<PF>(b_dst, &tmB, bar, kb * BKT, n0, label);
  } else if (KIND == GEMM_FPROP) {
    const int tap = kb / P.kcb, c0 = (kb % P.kcb) * BKT;
    const int ki = tap / g.k, kj = tap % g.k;
    tbox<PF>(a_dst, &tmA, bar, c0, j0 * g.s - g.p + kj, i0 * g.s - g.p + ki, b0, label);
    tbox<PF>(b_dst, &tmB, bar, kb * BKT, n0, label);
  } else if (KIND == KIND_DGP) {
    // k-block = (neighbour (di, dj) of the 2x2 small-map block, 32 input channels)
    const int nbr = kb / P.kcb, c0 = (kb % P.kcb) * BKT;
    const int di = nbr >> 1, dj = nbr & 1;
    tbox<PF>(a_dst, &tmA, bar, c0, j0 - dj, i0 - di, b0, label);
#pragma unroll
    for (int q = 0; q < BH / 32; ++q) {
      const int n = n0 + 32 * q, ph = n / g.CG;
      const int ki = (ph >> 1) + 2 * di, kj = (ph & 1) + 2 * dj;
      tbox<PF>(b_dst + q * (BKT * 128), &tmB, bar, n % g.CG, ki * g.k + kj, c0, label);
    }
  } else if (KIND == GEMM_DGRAD) {
    const int tp = kb / P.kcb, c0 = (kb % P.kcb) * BKT;
    const int ty = tp / d.ntx, tx = tp % d.ntx;
    const int ki = d.ry + ty * g.s, kj = d.rx + tx * g.s;
    const int offy = (d.y0 + g.p - d.ry) / g.s - ty;
    const int offx = (d.x0 + g.p - d.rx) / g.s - tx;
    tbox<PF>(a_dst, &tmA, bar, c0, j0 + offx, i0 + offy, b0, label);
#pragma unroll
    for (int q = 0; q < BH / 32; ++q)
      tbox<PF>(b_dst + q * (BKT * 128), &tmB, bar, n0 + 32 * q, ki * g.k + kj, c0, label);
    if (!PF && tmBl != nullptr)  // pre-split b_lo into the lo slot
#pragma unroll
      for (int q = 0; q < BH / 32; ++q)
        tma_load_4d(bl_dst + q * (BKT * 128), tmBl, bar, n0 + 32 * q, ki * g.k + kj, c0, label);
  } else {
    int kb0, ki0, kj0;
    box_origin(P.box, kb, kb0, ki0, kj0);
    const int m0 = mtp * (2 * BM) + (int)rank * BM;
#pragma unroll
    for (int q = 0; q < BM / 32; ++q) {
      const int m = m0 + 32 * q;
      const int tap = m / g.CG, cg0 = m % g.CG;
      const int ki = tap / g.k, kj = tap % g.k;
      tbox<PF>(a_dst + q * (BKT * 128), &tmA, bar, cg0, kj0 * g.s - g.p + kj,
          ki0 * g.s - g.p + ki, kb0, label);
    }
#pragma unroll
    for (int q = 0; q < BH / 32; ++q)
      tbox<PF>(b_dst + q * (BKT * 128), &tmB, bar, n0 + 32 * q, kj0, ki0, kb0, label);
  }
}

// drain + epilogue role: drain warp dw (0..7) reads TMEM lane quarter dw%4 and
// accumulator column half dw/4 of every segment into fp32 registers, then
// writes the tile (epi_store / epi_stats)
template <int KIND, int BN, bool STATS, int NB>
PG_DEV void pair_drain_role(const PairPlan& P, uint32_t tmem, uint64_t* seg_full, uint64_t* seg_empty, int dw,
                            int warp, int lane, uint32_t rank, int cl, int ncl, int ntiles) {
  constexpr int BH = BN / 2;
  const ConvGeo& g = P.g;
    const int q = warp & 3;               // TMEM lane quarter
    const int half = dw >> 2;  // accumulator column half (drain warp index dw = 0..7)
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t seg_empty_leader = mapa_shared(smem_u32(seg_empty), 0);
    uint32_t sc = 0;
    for (int t = cl; t < ntiles; t += ncl) {
      int label, phase, mtp, nt;
      pair_tile_decode(P, t, label, phase, mtp, nt);
      const int row = q * 32 + lane;
      const int nb = nt * BN + half * BH;  // first output column of this thread
      float acc[BH];
#pragma unroll
      for (int i = 0; i < BH; ++i) acc[i] = 0.f;
      for (int k_seg = 0; k_seg < P.nk; k_seg += P.kseg, ++sc) {
        const uint32_t buf = sc % NB;
        mbar_wait_cluster(seg_full + buf, (sc / NB) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < BH / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + buf * BN + half * BH + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[c * 32 + i] += __uint_as_float(r[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(seg_empty_leader + buf * 8);
      }
      RowPix rp{-1, -1, 0, 0, KIND == KIND_DGP, g.CG, g.GH, g.GW};
      if (KIND != GEMM_WGRAD) {
        int b0, i0, j0;
        box_origin(P.box, 2 * mtp + (int)rank, b0, i0, j0);
        const bool in_box = row < P.box.TB * P.box.TH * P.box.TW;  // rows past a short box hold stale data
        const int b = in_box ? b0 + row / (P.box.TH * P.box.TW) : g.B;
        const int ii = i0 + (row / P.box.TW) % P.box.TH;
        const int jj = j0 + row % P.box.TW;
        rp.i0 = ii;
        rp.j0 = jj;
        if (KIND == GEMM_FPROP || KIND == KIND_F4) {
          if (b < g.B && ii < g.SH && jj < g.SW) rp.off0 = (((long long)b * g.SH + ii) * g.SW + jj) * g.CS;
        } else if (KIND == GEMM_DGRAD) {
          const DgPhase d = dg_phase(g, phase);
          if (b < g.B && ii < d.ny && jj < d.nx)
            rp.off0 = (((long long)b * g.GH + d.y0 + ii * g.s) * g.GW + d.x0 + jj * g.s) * g.CG;
        } else {
          if (b < g.B && ii <= g.GH / 2 && jj <= g.GW / 2) rp.b = b;
        }
      }
      if (KIND == GEMM_WGRAD) {
        const int m = mtp * (2 * BM) + (int)rank * BM + row;
        if (m < P.mrows) {
          float* base = P.out + (long long)label * P.out_ls + m;
          if (P.accumulate) {
            // read-modify-write in batches of 32 columns, all loads issued
            // before any store: with load / store interleaved per column (the
            // stores may alias the next load) every column paid a full memory
            // latency -- 3.6x on the second pass of the discriminator weight
            // gradient (real + fake)
#pragma unroll
            for (int c0 = 0; c0 < BH; c0 += 32) {
              float old[32];
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int n = nb + c0 + c;
                old[c] = n < P.N ? base[(long long)n * P.mrows] : 0.f;
              }
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int n = nb + c0 + c;
                if (n < P.N) base[(long long)n * P.mrows] = old[c] + acc[c0 + c];
              }
            }
          } else {
#pragma unroll
            for (int c = 0; c < BH; ++c) {
              const int n = nb + c;
              if (n < P.N) base[(long long)n * P.mrows] = acc[c];
            }
          }
        }
      } else {
        const float* bias = P.bias ? P.bias + (long long)label * P.bias_ls : nullptr;
        float* out = P.out + (long long)label * P.out_ls;
        if (!STATS) {
          // one specialised copy per activation: the executed epilogue stays
          // small (the kernel is instruction-cache sensitive)
          switch (P.act) {
            case ACT_RELU: epi_store<ACT_RELU, BH>(acc, rp, out, nb, bias, P); break;
            case ACT_LRELU: epi_store<ACT_LRELU, BH>(acc, rp, out, nb, bias, P); break;
            case ACT_TANH: epi_store<ACT_TANH, BH>(acc, rp, out, nb, bias, P); break;
            case ACT_SIGMOID: epi_store<ACT_SIGMOID, BH>(acc, rp, out, nb, bias, P); break;
            default: epi_store<ACT_NONE, BH>(acc, rp, out, nb, bias, P); break;
          }
          continue;
        }
        float* st = P.stat + ((long long)label * P.nslot + ((phase * P.ntmp + mtp) * 2 + (int)rank) * 4 + q) * 4 * P.N;
        switch (P.stat_mode) {
          case STAT_FWD: epi_stats<STAT_FWD, BH>(acc, rp, out, nb, bias, st, label, lane, P); break;
          case STAT_BWD_BN: epi_stats<STAT_BWD_BN, BH>(acc, rp, out, nb, bias, st, label, lane, P); break;
          default: epi_stats<STAT_BWD_ACT, BH>(acc, rp, out, nb, bias, st, label, lane, P); break;
        }
      }
    }
  }

template <int KIND, int BN, int MODE, bool STATS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_nt(KIND, BN, MODE), 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmBl, const PairPlan P) {
  constexpr bool SPLIT = MODE == MATH_TF32X3;
  constexpr int SH = hi_stages(BN, SPLIT);
  constexpr int SL = lo_stages(BN, SPLIT);
  constexpr int RS = SPLIT ? SL : SH;  // ready ring (lo ring, or the hi ring itself)
  constexpr int SB = stage_bytes(BN);
  constexpr int AB = a_bytes();
  constexpr int BH = BN / 2;  // B columns staged per CTA; also the drain column half
  constexpr bool A_MN = KIND == GEMM_WGRAD;
  constexpr bool B_MN = KIND != GEMM_FPROP && KIND != KIND_F4;  // DGRAD / KIND_DGP weights, WGRAD gradients: N-major
  constexpr int NB = seg_bufs(BN);
  constexpr uint32_t TMEM_COLS = NB * BN;
  constexpr int NSPLIT = nsplit(KIND, BN, MODE);
  constexpr int W_MMA = NSPLIT + 1, W_DR = NSPLIT + 2;  // warp 0 TMA, 1..NSPLIT split, MMA, 8 drain warps

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* lo_base = smem + SH * SB;
  uint64_t* full_h = reinterpret_cast<uint64_t*>(lo_base + SL * SB);
  uint64_t* empty_h = full_h + SH;
  uint64_t* ready = empty_h + SH;
  uint64_t* empty_l = ready + RS;
  uint64_t* seg_full = empty_l + (SL ? SL : 1);
  uint64_t* seg_empty = seg_full + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + NB);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = cluster_ctarank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const ConvGeo& g = P.g;
  const int ntiles = P.ntn * P.ntmp * P.nz;

  if (tid == 0) {
    for (int s = 0; s < SH; ++s) {
      mbar_init(full_h + s, 1);
      mbar_init(empty_h + s, 1);
    }
    for (int s = 0; s < RS; ++s) mbar_init(ready + s, 2 * NSPLIT);
    for (int s = 0; s < SL; ++s) mbar_init(empty_l + s, 1);
    for (int b = 0; b < NB; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 2 * NDRAIN);
    }
    fence_barrier_init();
  }
  if (warp == W_MMA) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers exist before anyone arrives remotely
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: everything above touches only parameters, shared memory and TMEM, so
  // it overlaps the previous kernel's tail; no global data is read before this
  grid_dep_wait();
  grid_dep_launch();
  // wide tiles: the drain holds 128 fp32 partial sums per thread; at the
  // 168-register cap of 384 threads it spilled (40-104 B/thread).  Warps 0-3
  // (TMA, split, MMA) are one warpgroup and hand registers to the drain; each
  // role calls it inside its own branch so ptxas sees the limit of the region.
  constexpr bool WREGS = BN > 128 && PG_WIDE_REGS;
  static_assert(!WREGS || W_DR == 4, "producer roles must fill warpgroup 0");

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if constexpr (WREGS) regs_dec<PG_REGS_LO>();
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      // opt-in: the boxes of k-block kb + PFD are prefetched into L2 when kb is
      // loaded (pf_dist; off by default, see there)
      struct TileAt {
        int label, mtp, n0, b0, i0, j0;
        DgPhase d;
      };
      auto tile_at = [&](int t) {
        TileAt x{};
        int phase, nt;
        pair_tile_decode(P, t, x.label, phase, x.mtp, nt);
        x.n0 = nt * BN + (int)rank * BH;  // this CTA's B half
        if (KIND != GEMM_WGRAD) box_origin(P.box, 2 * x.mtp + (int)rank, x.b0, x.i0, x.j0);
        if (KIND == GEMM_DGRAD) x.d = dg_phase(g, phase);
        return x;
      };
      constexpr int PFD = pf_dist(BN, SPLIT);
      uint32_t it = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        const TileAt c = tile_at(t);
        TileAt nx{};
        const bool has_next = PFD > 0 && t + ncl < ntiles;
        if (has_next) nx = tile_at(t + ncl);
        for (int kb = 0; kb < P.nk; ++kb, ++it) {
          const int s = it % SH;
          mbar_wait(empty_h + s, ((it / SH) & 1) ^ 1);
          mbar_expect_tx(full_h + s, P.stage_tx);
          const uint32_t a_dst = smem_u32(smem + s * SB);
          const uint32_t b_dst = a_dst + AB;
          pair_issue<KIND, BH>(tmA, tmB, P, a_dst, b_dst, full_h + s, kb, c.label, c.mtp, rank, c.n0, c.b0, c.i0,
                               c.j0, c.d, KIND == GEMM_DGRAD && SPLIT && P.blo ? &tmBl : nullptr,
                               smem_u32(lo_base + (it % (SL ? SL : 1)) * SB) + AB);
          if (KIND == GEMM_FPROP && SPLIT && P.blo)  // lo slot it % SL == s (equal rings), freed with the hi slot
            tma_load_3d(smem_u32(lo_base + (it % SL) * SB) + AB, &tmBl, full_h + s, kb * BKT, c.n0, c.label);
          if (PFD > 0) {
            const int kp = kb + PFD;
            if (kp < P.nk)
              pair_issue<KIND, BH, true>(tmA, tmB, P, 0, 0, nullptr, kp, c.label, c.mtp, rank, c.n0, c.b0, c.i0, c.j0,
                                         c.d);
            else if (has_next && kp - P.nk < P.nk)
              pair_issue<KIND, BH, true>(tmA, tmB, P, 0, 0, nullptr, kp - P.nk, nx.label, nx.mtp, rank, nx.n0, nx.b0,
                                         nx.i0, nx.j0, nx.d);
          }
        }
      }
    }
  } else if (warp <= NSPLIT) {
    // ===================== lo split / landed forward (both CTAs) =====================
    if constexpr (WREGS) regs_dec<PG_REGS_LO>();
    const int st = tid - 32;
    const uint32_t ready_leader = mapa_shared(smem_u32(ready), 0);
    uint32_t it = 0;
    for (int t = cl; t < ntiles; t += ncl) {
      for (int kb = 0; kb < P.nk; ++kb, ++it) {
        const int s = it % SH;
        mbar_wait(full_h + s, (it / SH) & 1);
        int r = s;
        if (SPLIT) {
          const int j = it % SL;
          r = j;
          mbar_wait(empty_l + j, ((it / SL) & 1) ^ 1);
          const float4* src = reinterpret_cast<const float4*>(smem + s * SB);
          float4* dst = reinterpret_cast<float4*>(lo_base + j * SB);
          const int n16 = ((KIND == GEMM_FPROP || KIND == GEMM_DGRAD) && P.blo ? AB : SB) / 16;  // b_lo landed by TMA
#pragma unroll 8
          for (int i = st; i < n16; i += NSPLIT * 32) {
            const float4 v = src[i];
            dst[i] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                 v.w - tf32_trunc(v.w));
          }
          fence_async_smem();
        } else if (MODE == MATH_BF16) {
          // bf16 operands: round the landed A rows and B half in place
          float4* v4 = reinterpret_cast<float4*>(smem + s * SB);
#pragma unroll 8
          for (int i = st; i < SB / 16; i += NSPLIT * 32) v4[i] = bf16_rne4(v4[i]);
          fence_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(ready_leader + r * 8);
      }
    }
  } else if (warp == W_MMA) {
    // ===================== MMA issuer (leader CTA only) =====================
    if constexpr (WREGS) regs_dec<PG_REGS_LO>();
    // The whole warp runs the loop (warp-uniform values stay in uniform
    // registers); one elected lane issues the MMAs and the commits.  With a
    // divergent single-lane loop every MMA paid ~12 instructions of R2UR /
    // ELECT re-materialisation, which paced the narrow (N <= 128) tiles.
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(2 * BM, BN, A_MN, B_MN);
      // K-major SW128: 8-row atoms at 1024 B, K-step of 8 fp32 = +32 B inside the row.
      // MN-major SW128_BASE32B: 4-row atoms at 512 B along K, 32-wide MN atoms at 4096 B.
      constexpr bool F4 = KIND == KIND_F4;
      constexpr uint32_t a_lbo = A_MN ? 4096u : F4 ? 2048u : 16u, a_sbo = A_MN ? 512u : F4 ? 128u : 1024u,
                         a_step = A_MN ? 1024u : F4 ? 4096u : 32u;
      constexpr uint32_t b_lbo = B_MN ? 4096u : 16u, b_sbo = B_MN ? 512u : 1024u, b_step = B_MN ? 1024u : 32u;
      constexpr uint32_t a_lay = A_MN ? UMMA_SW128_BASE32B : F4 ? UMMA_SW_NONE : UMMA_SW128;
      constexpr uint32_t b_lay = B_MN ? UMMA_SW128_BASE32B : UMMA_SW128;
      // descriptors are linear in the start address (bits 0-13 = addr >> 4)
      const uint64_t a_desc0 = make_desc(smem_u32(smem), a_lbo, a_sbo, a_lay);
      const uint64_t b_desc0 = make_desc(smem_u32(smem) + AB, b_lbo, b_sbo, b_lay);
      const uint64_t al_desc0 = make_desc(smem_u32(lo_base), a_lbo, a_sbo, a_lay);
      const uint64_t bl_desc0 = make_desc(smem_u32(lo_base) + AB, b_lbo, b_sbo, b_lay);
      uint32_t it = 0, sc = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        for (int k_seg = 0; k_seg < P.nk; k_seg += P.kseg, ++sc) {
          const uint32_t buf = sc % NB;
          mbar_wait_cluster(seg_empty + buf, ((sc / NB) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * BN;
          const int k_end = min(P.nk, k_seg + P.kseg);
          for (int kb = k_seg; kb < k_end; ++kb, ++it) {
            const int s = it % SH;
            const int j = SPLIT ? it % SL : 0;
            mbar_wait_cluster(ready + (SPLIT ? j : s), (it / RS) & 1);
            tc_fence_after();
            const uint64_t ah0 = a_desc0 + (uint64_t)((s * SB) >> 4), bh0 = b_desc0 + (uint64_t)((s * SB) >> 4);
            const uint64_t al0 = al_desc0 + (uint64_t)((j * SB) >> 4), bl0 = bl_desc0 + (uint64_t)((j * SB) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < BKT / 8; ++kk) {
                const uint64_t ah = ah0 + (kk * a_step >> 4), bh = bh0 + (kk * b_step >> 4);
                const uint32_t acc = (kb != k_seg || kk) ? 1u : 0u;
                if (SPLIT) {
                  mma_tf32_pair(d, al0 + (kk * a_step >> 4), bh, idesc, acc);  // small terms first
                  mma_tf32_pair(d, ah, bl0 + (kk * b_step >> 4), idesc, 1u);
                  mma_tf32_pair(d, ah, bh, idesc, 1u);
                } else {
                  mma_tf32_pair(d, ah, bh, idesc, acc);
                }
              }
              mma_commit_pair(empty_h + s, 3);
              if (SPLIT) mma_commit_pair(empty_l + j, 3);
              if (kb + 1 == k_end) mma_commit_pair(seg_full + buf, 3);
            }
            __syncwarp();
          }
        }
      }
    }
    __syncwarp();
  } else {
    if constexpr (WREGS) regs_inc<PG_REGS_HI>();
    pair_drain_role<KIND, BN, STATS, NB>(P, tmem, seg_full, seg_empty, warp - W_DR, warp, lane, rank, cl, ncl,
                                         ntiles);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no remote arrive / MMA into the peer after this point
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, TMEM_COLS);
  }
}


// ---------------------------------------------------------------------------
// A-in-TMEM variant for the narrow tiles (BN <= 128, TF32X3, FPROP / DGRAD).
// At BN = 64 the single-CTA-equivalent MMA rate needs ~300 B/clk of shared
// memory in the SS form (the tensor core re-reads A for all three products of
// the split) against 128 B/clk available; here the split warps read each A row
// once, write its hi and lo parts to tensor memory (tcgen05.st), and the MMA
// reads A from TMEM ("TS" form), B (hi from the stage, lo from a small ring)
// from shared memory.
//   warps 0-3  split: lane quarter q = warp, thread = A row; B half lo -> smem
//   warps 4-11 drain + epilogue (as pair_drain_role)
//   warp 12    TMA producer;  warp 13  TMEM allocation + MMA issuer (leader)
// TMEM: accumulator buffers in columns [0, 256), A stages (hi 32 + lo 32
// columns each) in [256, 512).
constexpr int ATM_NT = 14 * 32;
constexpr int ATM_SA = 4;
constexpr int ATM_ACOL = 256;
__host__ __device__ constexpr int atm_bufs(int bn) { return 256 / bn; }
__host__ __device__ constexpr int atm_lo_bytes(int bn) { return (bn / 2) * BKT * 4; }
// split slot = a copy of the B half (hi) + its lo part: the MMA reads only
// TMEM (A) and the split slots (B), so a TMA stage is released as soon as the
// split warps have read it, not when the MMAs retire -- the TMA ring stays in
// flight (the single-stage-in-flight ring was the feed limit of these tiles)
__host__ __device__ constexpr int atm_slot_bytes(int bn) { return 2 * atm_lo_bytes(bn); }
__host__ __device__ constexpr int atm_hi_stages(int bn) {
  return (SMEM_BUDGET - ATM_SA * atm_slot_bytes(bn)) / stage_bytes(bn) > 8
             ? 8
             : (SMEM_BUDGET - ATM_SA * atm_slot_bytes(bn)) / stage_bytes(bn);
}
__host__ __device__ constexpr int atm_smem(int bn) {
  return atm_hi_stages(bn) * stage_bytes(bn) + ATM_SA * atm_slot_bytes(bn) + 1024 + 1024;
}

template <int KIND, int BN, bool STATS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ATM_NT, 1)
    gemm_pair_atm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const PairPlan P) {
  static_assert(BN <= 128 && KIND != GEMM_WGRAD, "A-in-TMEM tiles: K-major A, BN <= 128");
  constexpr int SH = atm_hi_stages(BN);
  constexpr int SB = stage_bytes(BN);
  constexpr int AB = a_bytes();
  constexpr int BH = BN / 2;
  constexpr int LB = atm_lo_bytes(BN);
  constexpr bool B_MN = KIND != GEMM_FPROP;
  constexpr int NB = atm_bufs(BN);
  constexpr int W_TMA = 12, W_MMAI = 13;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* lo_base = smem + SH * SB;
  uint64_t* full_h = reinterpret_cast<uint64_t*>(lo_base + ATM_SA * 2 * LB);
  uint64_t* empty_h = full_h + SH;
  uint64_t* ready = empty_h + SH;
  uint64_t* empty_l = ready + ATM_SA;
  uint64_t* seg_full = empty_l + ATM_SA;
  uint64_t* seg_empty = seg_full + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + NB);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = cluster_ctarank();
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntiles = P.ntn * P.ntmp * P.nz;

  if (tid == 0) {
    for (int s = 0; s < SH; ++s) {
      mbar_init(full_h + s, 1);
      mbar_init(empty_h + s, 4);  // released by the four split warps of this CTA
    }
    for (int s = 0; s < ATM_SA; ++s) {
      mbar_init(ready + s, 2 * 4);
      mbar_init(empty_l + s, 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 2 * NDRAIN);
    }
    fence_barrier_init();
  }
  if (warp == W_MMAI) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ===================== split: A rows -> TMEM (hi, lo); B half lo -> smem =====================
    const int r = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t ready_leader = mapa_shared(smem_u32(ready), 0);
    uint32_t it = 0;
    for (int t = cl; t < ntiles; t += ncl) {
      for (int kb = 0; kb < P.nk; ++kb, ++it) {
        const int s = it % SH, j = it % ATM_SA;
        mbar_wait(full_h + s, (it / SH) & 1);
        mbar_wait(empty_l + j, ((it / ATM_SA) & 1) ^ 1);
        // row r of the K-major SW128 A tile: 16-byte chunk c sits at c ^ (r & 7)
        const uint8_t* arow = smem + s * SB + r * 128;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(arow + ((c ^ (r & 7)) << 4));
          const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            hi[4 * c + u] = __float_as_uint(e[u]);
            lo[4 * c + u] = __float_as_uint(e[u] - tf32_trunc(e[u]));
          }
        }
        const uint32_t ta = tmem + lane_off + ATM_ACOL + j * 64;
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        const float4* bsrc = reinterpret_cast<const float4*>(smem + s * SB + AB);
        float4* bhi = reinterpret_cast<float4*>(lo_base + j * 2 * LB);
        float4* blo = reinterpret_cast<float4*>(lo_base + j * 2 * LB + LB);
#pragma unroll
        for (int e = tid; e < LB / 16; e += 128) {
          const float4 v = bsrc[e];
          bhi[e] = v;
          blo[e] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                               v.w - tf32_trunc(v.w));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_h + s);  // the TMA stage is fully read: refill it now
        tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(ready_leader + j * 8);
      }
    }
  } else if (warp < 4 + NDRAIN) {
    pair_drain_role<KIND, BN, STATS, NB>(P, tmem, seg_full, seg_empty, warp - W_DRAIN, warp, lane, rank, cl, ncl,
                                         ntiles);
  } else if (warp == W_TMA) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      uint32_t it = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        int label, phase, mtp, nt;
        pair_tile_decode(P, t, label, phase, mtp, nt);
        const int n0 = nt * BN + (int)rank * BH;
        int b0 = 0, i0 = 0, j0 = 0;
        box_origin(P.box, 2 * mtp + (int)rank, b0, i0, j0);
        DgPhase d{};
        if (KIND == GEMM_DGRAD) d = dg_phase(P.g, phase);
        for (int kb = 0; kb < P.nk; ++kb, ++it) {
          const int s = it % SH;
          mbar_wait(empty_h + s, ((it / SH) & 1) ^ 1);
          mbar_expect_tx(full_h + s, P.stage_tx);
          const uint32_t a_dst = smem_u32(smem + s * SB);
          pair_issue<KIND, BH>(tmA, tmB, P, a_dst, a_dst + AB, full_h + s, kb, label, mtp, rank, n0, b0, i0, j0, d);
        }
      }
    }
  } else {
    // ===================== MMA issuer (leader CTA only): A from TMEM =====================
    // whole warp in the loop (warp-uniform descriptors in uniform registers),
    // one elected lane issues -- the single-lane divergent form paced these
    // tiles on instruction issue (as it did the SS kernel, see there)
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(2 * BM, BN, false, B_MN);
      constexpr uint32_t b_lbo = B_MN ? 4096u : 16u, b_sbo = B_MN ? 512u : 1024u, b_step = B_MN ? 1024u : 32u;
      constexpr uint32_t b_lay = B_MN ? UMMA_SW128_BASE32B : UMMA_SW128;
      const uint64_t bh_desc0 = make_desc(smem_u32(lo_base), b_lbo, b_sbo, b_lay);
      const uint64_t bl_desc0 = make_desc(smem_u32(lo_base) + LB, b_lbo, b_sbo, b_lay);
      uint32_t it = 0, sc = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        for (int k_seg = 0; k_seg < P.nk; k_seg += P.kseg, ++sc) {
          const uint32_t buf = sc % NB;
          mbar_wait_cluster(seg_empty + buf, ((sc / NB) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dacc = tmem + buf * BN;
          const int k_end = min(P.nk, k_seg + P.kseg);
          for (int kb = k_seg; kb < k_end; ++kb, ++it) {
            const int j = it % ATM_SA;
            mbar_wait_cluster(ready + j, (it / ATM_SA) & 1);
            tc_fence_after();
            const uint32_t a_t = tmem + ATM_ACOL + j * 64;
            const uint64_t bh0 = bh_desc0 + (uint64_t)((j * 2 * LB) >> 4), bl0 = bl_desc0 + (uint64_t)((j * 2 * LB) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < BKT / 8; ++kk) {
                const uint64_t bh = bh0 + (kk * b_step >> 4), bl = bl0 + (kk * b_step >> 4);
                const uint32_t acc = (kb != k_seg || kk) ? 1u : 0u;
                mma_tf32_pair_ts(dacc, a_t + 32 + kk * 8, bh, idesc, acc);  // small terms first
                mma_tf32_pair_ts(dacc, a_t + kk * 8, bl, idesc, 1u);
                mma_tf32_pair_ts(dacc, a_t + kk * 8, bh, idesc, 1u);
              }
              mma_commit_pair(empty_l + j, 3);
              if (kb + 1 == k_end) mma_commit_pair(seg_full + buf, 3);
            }
            __syncwarp();
          }
        }
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == W_MMAI) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ---------------------------------------------------------------- host side

template <int KIND, int BN, int MODE, bool STATS>
cudaError_t launch_pair_st(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbl, const PairPlan& P,
                           int grid, cudaStream_t st) {
  constexpr int smem = smem_total(BN, MODE == MATH_TF32X3);
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([&] {
    return cudaFuncSetAttribute(gemm_pair_kernel<KIND, BN, MODE, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem);
  });
  if (ce != cudaSuccess) return ce;
  // programmatic dependent launch (PG_PDL=0 turns it off): the prologue runs
  // while the previous kernel drains (see grid_dep_wait in the kernel)
  static const bool pdl = [] {
    const char* e = std::getenv("PG_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(pair_nt(KIND, BN, MODE));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_pair_kernel<KIND, BN, MODE, STATS>, ta, tb, tbl, P);
  if (e != cudaSuccess) return e;
  return launched();
}

template <int KIND, int BN, bool STATS>
cudaError_t launch_pair_atm(const CUtensorMap& ta, const CUtensorMap& tb, const PairPlan& P, int grid,
                            cudaStream_t st) {
  constexpr int smem = atm_smem(BN);
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([&] {
    return cudaFuncSetAttribute(gemm_pair_atm_kernel<KIND, BN, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem);
  });
  if (ce != cudaSuccess) return ce;
  gemm_pair_atm_kernel<KIND, BN, STATS><<<grid, ATM_NT, smem, st>>>(ta, tb, P);
  return launched();
}

// A-in-TMEM tiles for the narrow FPROP / DGRAD tiles (default; PG_ATM=0 off).
// Round 1 measured them no faster: their MMA issuer was a single divergent
// lane (instruction-issue bound, as the SS kernel had been), and the weight
// lo pre-split added later was never loaded by this producer (a hang).  With
// the warp-uniform issuer: conv2 forward 1.13 -> 1.02 ms, conv3 data gradient
// 1.17 -> 0.98 ms (c4, 125 labels x 32, scripts/gemm_sweep.py).
bool atm_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_ATM");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int KIND, int BN, int MODE>
cudaError_t launch_pair_bn(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbl, const PairPlan& P,
                           cudaStream_t st) {
  const int tiles = P.ntn * P.ntmp * P.nz;
  if (tiles == 0 || P.nk == 0) return cudaSuccess;
  const int pairs = std::min(tiles, sm_count_tma() / 2);
  if constexpr (KIND != GEMM_WGRAD && KIND != KIND_F4 && BN <= 128 && MODE == MATH_TF32X3) {
    if (atm_enabled())
      return P.stat_mode != STAT_NONE ? launch_pair_atm<KIND, BN, true>(ta, tb, P, 2 * pairs, st)
                                      : launch_pair_atm<KIND, BN, false>(ta, tb, P, 2 * pairs, st);
  }
  if (KIND != GEMM_WGRAD && P.stat_mode != STAT_NONE)
    return launch_pair_st<KIND, BN, MODE, KIND != GEMM_WGRAD>(ta, tb, tbl, P, 2 * pairs, st);
  return launch_pair_st<KIND, BN, MODE, false>(ta, tb, tbl, P, 2 * pairs, st);
}

template <int KIND, int MODE>
cudaError_t launch_pair_kind(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbl, const PairPlan& P,
                             int bn, cudaStream_t st) {
  if (bn == 64) return launch_pair_bn<KIND, 64, MODE>(ta, tb, tbl, P, st);
  if (bn == 128) return launch_pair_bn<KIND, 128, MODE>(ta, tb, tbl, P, st);
  return launch_pair_bn<KIND, 256, MODE>(ta, tb, tbl, P, st);
}

int pair_bn(int n) { return n >= 256 ? 256 : n >= 128 ? 128 : 64; }

bool dense_1x1(const ConvGeo& g) {
  return g.k == 1 && g.s == 1 && g.p == 0 && g.SH == 1 && g.SW == 1 && g.GH == 1 && g.GW == 1;
}

// Base grid of the phase-packed DGRAD is (H/2 + 1) x (W/2 + 1) (17 x 17 for a
// 32 x 32 output): a power-of-two box would waste half the rows, so the box
// is W wide (whole rows) and at most 128 rows deep, picking the TH x TB split
// with the least padding; rows past the box are never stored.
SpatialBox packed_box(int B, int H, int W) {
  if ((W & (W - 1)) == 0 || W > BM) return spatial_box(B, H, W, BM);
  SpatialBox best{};
  double best_util = -1.0;
  for (int th = 1; th * W <= BM; ++th) {
    SpatialBox b;
    b.TW = W;
    b.TH = std::min(th, H);
    b.TB = BM / (b.TW * b.TH);
    b.nx = 1;
    b.ny = (H + b.TH - 1) / b.TH;
    b.nb = (B + b.TB - 1) / b.TB;
    const double util = (double)B * H * W / ((double)b.nb * b.ny * BM);
    if (util > best_util) {
      best_util = util;
      best = b;
    }
  }
  return best;
}

// phase-packed DGRAD (KIND_DGP): k4 s2 p1 with 4 CG <= 256, where the per-phase
// form would run BN = 64 tiles re-reading the small map 16 times
bool dgrad_packed(const GemmArgs& a) {
  static const bool disabled = [] {
    const char* e = std::getenv("PG_NO_DGP");
    return e && std::atoi(e) != 0;
  }();
  const ConvGeo& g = a.g;
  return !disabled && a.kind == GEMM_DGRAD && g.k == 4 && g.s == 2 && g.p == 1 && g.GH == 2 * g.SH &&
         g.GW == 2 * g.SW && g.CG % 32 == 0 && 4 * g.CG <= PG_DGP_MAXN && g.CS % 32 == 0;
}

}  // namespace

bool gemm_pair_supported(const GemmArgs& a) {
  static const bool disabled = [] {
    const char* e = std::getenv("PG_NO_PAIR");
    return e && std::atoi(e) != 0;
  }();
  if (disabled || !encode_fn() || sm_count_tma() < 2) return false;
  const ConvGeo& g = a.g;
  static const bool no_f4 = [] {
    const char* e = std::getenv("PG_NO_F4");
    return e && std::atoi(e) != 0;
  }();
  if (a.kind == GEMM_FPROP && g.CG == 4 && no_f4) return false;
  if (g.s < 1 || g.s > 8 || g.k < 1) return false;
  if (a.kind == GEMM_FPROP && spatial_box(g.B, g.SH, g.SW, BM).TW * g.s > 256) return false;
  if (a.kind == GEMM_WGRAD && spatial_box(g.B, g.SH, g.SW, BKT).TW * g.s > 256) return false;
  if (a.kind == GEMM_DGRAD && g.k % g.s) return false;
  if (!aligned16(a.out) || !aligned16(a.w) || a.out_ls % 4 || a.w_ls % 4) return false;
  // FPROP / DGRAD epilogues store 8 columns per 256-bit store
  if (a.kind != GEMM_WGRAD && ((reinterpret_cast<uintptr_t>(a.out) & 31) || a.out_ls % 8)) return false;
  switch (a.kind) {
    case GEMM_FPROP:
      // K tail of a dense layer (e.g. the latent width 100) is zero-filled by TMA out-of-bounds reads
      return (g.CG % 32 == 0 || (g.CG == 4 && (g.k * g.k * 4) % BKT == 0) || (dense_1x1(g) && g.CG % 4 == 0)) &&
             g.CS >= 64 && g.CS % 32 == 0 && aligned16(a.big) && a.big_ls % 4 == 0;
    case GEMM_DGRAD:
      return g.CS % 32 == 0 && g.CG >= 64 && g.CG % 32 == 0 && aligned16(a.small) && a.small_ls % 4 == 0;
    default:
      return g.CG % 32 == 0 && g.CS % 32 == 0 && g.CS >= 64 && aligned16(a.small) && aligned16(a.big) &&
             a.small_ls % 4 == 0 && a.big_ls % 4 == 0;
  }
}

int gemm_pair_stat_slots(const GemmArgs& a, int* npack) {
  const ConvGeo& g = a.g;
  if (npack) *npack = 1;
  if (a.kind == GEMM_WGRAD || !gemm_pair_supported(a)) return 0;
  if (a.kind == GEMM_FPROP) {
    const SpatialBox b = spatial_box(g.B, g.SH, g.SW, BM);
    if (g.CS % 8) return 0;
    return (b.nb * b.ny * b.nx + 1) / 2 * 8;
  }
  if (g.CG % 8) return 0;
  if (dgrad_packed(a)) {
    const SpatialBox b = packed_box(g.B, g.GH / 2 + 1, g.GW / 2 + 1);
    if (npack) *npack = 4;
    return (b.nb * b.ny * b.nx + 1) / 2 * 8;
  }
  const SpatialBox b = spatial_box(g.B, (g.GH + g.s - 1) / g.s, (g.GW + g.s - 1) / g.s, BM);
  return g.s * g.s * ((b.nb * b.ny * b.nx + 1) / 2) * 8;
}

// b_lo of the weights, [L][rows] contiguous (the stride of `w` may be the
// whole parameter arena): lo = x - trunc_tf32(x), the split warps' formula
__global__ void tf32_lo_kernel(const float* __restrict__ w, long long w_ls, long long n, float* __restrict__ out) {
  const int l = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = w[l * w_ls + i];
    out[l * n + i] = v - tf32_trunc(v);
  }
}
cudaError_t launch_tf32_lo(const float* w, long long w_ls, long long n, int L, float* out, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, std::max(1, 148 * 8 / std::max(1, L)));
  tf32_lo_kernel<<<dim3(blocks, L), 256, 0, st>>>(w, w_ls, n, out);
  return launched();
}
// grow-only buffer for b_lo (not gemm_scratch: the lowered paths hand
// gemm_scratch pointers to this engine as operands)
float* blo_buffer(size_t floats, cudaStream_t st) { return stream_scratch(SCRATCH_BLO, floats, st); }
bool blo_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_BLO");
    return !(e && e[0] == '0');
  }();
  return on;
}

// SCRATCH_BLO floats launch_gemm_pair(a, math) takes (the b_lo conditions below)
size_t gemm_pair_blo_floats(const GemmArgs& a, int math) {
  const ConvGeo& g = a.g;
  if (math != MATH_TF32X3 || !blo_enabled() || atm_enabled() || !gemm_pair_supported(a)) return 0;
  const long long kk = (long long)g.k * g.k;
  if (a.kind == GEMM_FPROP && g.CG != 4 && pair_bn(g.CS) <= 128 && (long long)g.B * g.SH * g.SW >= 8LL * g.CS)
    return (size_t)a.L * kk * g.CG * g.CS;
  if (a.kind == GEMM_DGRAD && !dgrad_packed(a) && pair_bn(g.CG) <= 128 && (long long)g.B * g.GH * g.GW >= 8LL * g.CG)
    return (size_t)a.L * g.CS * kk * g.CG;
  return 0;
}

cudaError_t launch_gemm_pair(const GemmArgs& a, int math, cudaStream_t st) {
  const ConvGeo& g = a.g;
  PairPlan P{};
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
  P.stat_mode = a.kind == GEMM_WGRAD ? STAT_NONE : a.stat_mode;
  P.stat = a.stat;
  P.stat_y = a.stat_y;
  P.stat_z = a.stat_z;
  P.stat_mu = a.stat_mu;
  P.stat_act = a.stat_act;
  P.stat_slope = a.stat_slope;
  P.nz = a.L * P.phases;
  // TF32X3 keeps every TMEM accumulation chain short (the tensor core adds with
  // truncation): 8 k-blocks = 96 MMA adds per segment, measured
  // max error 2.9e-6 of f64 over K = 64..16384 -- inside the plain fp32 FMA
  // loop's 0.3e-6..4.4e-6 (scripts/tc_accuracy.py); 16 k-blocks: 5.3e-6.
  // 8 vs 4: -2 ms per c4 step.
  static const int kseg_env = [] {
    const char* e = std::getenv("PG_KSEG");
    return e ? std::atoi(e) : 0;
  }();
  P.kseg = kseg_env > 0 ? kseg_env : 8;
  const int kk = g.k * g.k;
  CUtensorMap ta, tb, tbl{};
  const int one[5] = {1, 1, 1, 1, 1};
  const int sstr[5] = {1, g.s, g.s, 1, 1};
  bool ok = true;
  int bn, ntm = 1;
  const bool f4 = a.kind == GEMM_FPROP && g.CG == 4;
  if (f4) {
    P.N = g.CS;
    P.kcb = 1;
    P.nk = kk * 4 / BKT;
    P.box = spatial_box(g.B, g.SH, g.SW, BM);
    ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = pair_bn(P.N);
    const long long ad[5] = {4, g.GW, g.GH, g.B, a.L};
    const long long as[4] = {4, (long long)g.GW * 4, (long long)g.GH * g.GW * 4, a.big_ls};
    const int abox[5] = {4, P.box.TW * g.s, P.box.TH * g.s, P.box.TB, 1};
    ok = ok && make_map(&ta, a.big, 5, ad, as, abox, sstr, CU_TENSOR_MAP_SWIZZLE_NONE);
    const long long K = (long long)kk * 4;
    const long long bd[3] = {K, g.CS, a.L};
    const long long bs[2] = {K, a.w_ls};
    const int bbox[3] = {BKT, bn / 2, 1};
    ok = ok && make_map(&tb, a.w, 3, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (a.kind == GEMM_FPROP) {
    P.N = g.CS;
    P.kcb = (g.CG + BKT - 1) / BKT;
    P.nk = kk * P.kcb;
    P.box = spatial_box(g.B, g.SH, g.SW, BM);
    ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = pair_bn(P.N);
    const long long ad[5] = {g.CG, g.GW, g.GH, g.B, a.L};
    const long long as[4] = {g.CG, (long long)g.GW * g.CG, (long long)g.GH * g.GW * g.CG, a.big_ls};
    const int abox[5] = {BKT, P.box.TW * g.s, P.box.TH * g.s, P.box.TB, 1};
    ok = ok && make_map(&ta, a.big, 5, ad, as, abox, sstr, CU_TENSOR_MAP_SWIZZLE_128B);
    const long long K = (long long)kk * g.CG;
    const long long bd[3] = {K, g.CS, a.L};
    const long long bs[2] = {K, a.w_ls};
    const int bbox[3] = {BKT, bn / 2, 1};
    ok = ok && make_map(&tb, a.w, 3, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B);
    // b_lo pre-split once per launch for the narrow (shared-memory-bound) tiles
    // when the weights are small against the activations (>= 8 output rows per
    // weight row): the split warps then only touch A (conv2
    // forward 1.21 -> 1.11 ms; the wide tiles lose more to the extra pass)
    if (math == MATH_TF32X3 && bn <= 128 && blo_enabled() && !atm_enabled() && (long long)g.B * g.SH * g.SW >= 8LL * g.CS) {
      float* wl = blo_buffer((size_t)a.L * K * g.CS, st);
      if (!wl) return cudaErrorMemoryAllocation;
      cudaError_t e = launch_tf32_lo(a.w, a.w_ls, K * g.CS, a.L, wl, st);
      if (e != cudaSuccess) return e;
      const long long ls[2] = {K, K * g.CS};
      ok = ok && make_map(&tbl, wl, 3, bd, ls, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B);
      P.blo = 1;
    }
  } else if (dgrad_packed(a)) {
    P.N = 4 * g.CG;
    P.kcb = g.CS / BKT;
    P.nk = 4 * P.kcb;
    P.phases = 1;
    P.nz = a.L;
    P.box = packed_box(g.B, g.GH / 2 + 1, g.GW / 2 + 1);
    ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = pair_bn(P.N);
    const long long ad[5] = {g.CS, g.SW, g.SH, g.B, a.L};
    const long long as[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
    const int abox[5] = {BKT, P.box.TW, P.box.TH, P.box.TB, 1};
    ok = ok && make_map(&ta, a.small, 5, ad, as, abox, one, CU_TENSOR_MAP_SWIZZLE_128B);
    const long long bd[4] = {g.CG, kk, g.CS, a.L};
    const long long bs[3] = {g.CG, (long long)kk * g.CG, a.w_ls};
    const int bbox[4] = {32, 1, BKT, 1};
    ok = ok && make_map(&tb, a.w, 4, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  } else if (a.kind == GEMM_DGRAD) {
    P.N = g.CG;
    P.kcb = g.CS / BKT;
    const int nty = g.k / g.s, ntx = nty;
    P.nk = nty * ntx * P.kcb;
    const int ny = (g.GH + g.s - 1) / g.s, nx = (g.GW + g.s - 1) / g.s;
    P.box = spatial_box(g.B, ny, nx, BM);
    ntm = P.box.nb * P.box.ny * P.box.nx;
    bn = pair_bn(P.N);
    const long long ad[5] = {g.CS, g.SW, g.SH, g.B, a.L};
    const long long as[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
    const int abox[5] = {BKT, P.box.TW, P.box.TH, P.box.TB, 1};
    ok = ok && make_map(&ta, a.small, 5, ad, as, abox, one, CU_TENSOR_MAP_SWIZZLE_128B);
    const long long bd[4] = {g.CG, kk, g.CS, a.L};
    const long long bs[3] = {g.CG, (long long)kk * g.CG, a.w_ls};
    const int bbox[4] = {32, 1, BKT, 1};
    ok = ok && make_map(&tb, a.w, 4, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    // b_lo pre-split for the narrow tiles (as FPROP above)
    if (math == MATH_TF32X3 && bn <= 128 && blo_enabled() && !atm_enabled() && (long long)g.B * g.GH * g.GW >= 8LL * g.CG) {
      const long long nw = (long long)g.CS * kk * g.CG;
      float* wl = blo_buffer((size_t)a.L * nw, st);
      if (!wl) return cudaErrorMemoryAllocation;
      cudaError_t e = launch_tf32_lo(a.w, a.w_ls, nw, a.L, wl, st);
      if (e != cudaSuccess) return e;
      const long long ls[3] = {g.CG, (long long)kk * g.CG, nw};
      ok = ok && make_map(&tbl, wl, 4, bd, ls, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      P.blo = 1;
    }
  } else {
    P.N = g.CS;
    P.mrows = kk * g.CG;
    P.kcb = 0;
    P.box = spatial_box(g.B, g.SH, g.SW, BKT);
    P.nk = P.box.nb * P.box.ny * P.box.nx;
    ntm = (P.mrows + BM - 1) / BM;
    bn = pair_bn(P.N);
    // A: strided big-map boxes (32 channels of one tap), MN-major
    const long long ad[5] = {g.CG, g.GW, g.GH, g.B, a.L};
    const long long as[4] = {g.CG, (long long)g.GW * g.CG, (long long)g.GH * g.GW * g.CG, a.big_ls};
    const int abox[5] = {32, P.box.TW * g.s, P.box.TH * g.s, P.box.TB, 1};
    ok = ok && make_map(&ta, a.big, 5, ad, as, abox, sstr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    // B: gradient of the small map, 32 output channels per box, MN-major
    const long long bd[5] = {g.CS, g.SW, g.SH, g.B, a.L};
    const long long bs[4] = {g.CS, (long long)g.SW * g.CS, (long long)g.SH * g.SW * g.CS, a.small_ls};
    const int bbox[5] = {32, P.box.TW, P.box.TH, P.box.TB, 1};
    ok = ok && make_map(&tb, a.small, 5, bd, bs, bbox, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  if (!ok) return cudaErrorInvalidValue;
  P.ntmp = (ntm + 1) / 2;
  P.ntn = (P.N + bn - 1) / bn;
  P.nslot = P.phases * P.ntmp * 8;
  P.CGn = a.kind == GEMM_FPROP ? g.CS : g.CG;
  P.stage_tx = (a.kind == GEMM_WGRAD ? BM : P.box.TB * P.box.TH * P.box.TW) * BKT * 4 + (bn / 2) * BKT * 4;
  if (P.blo) P.stage_tx += (bn / 2) * BKT * 4;
  // profiling aid: PG_FORCE_STATS=1 runs plain FPROP/DGRAD launches with STAT_FWD into a private buffer
  static const bool force_stats = [] {
    const char* e = std::getenv("PG_FORCE_STATS");
    return e && std::atoi(e) != 0;
  }();
  if (force_stats && a.kind != GEMM_WGRAD && P.stat_mode == STAT_NONE && P.act == ACT_NONE && P.N % 8 == 0) {
    static float* buf = nullptr;
    static size_t cap = 0;
    const size_t need = (size_t)a.L * P.nslot * 4 * P.N;
    if (need > cap) {
      cudaStreamSynchronize(st);
      cudaFree(buf);
      if (cudaMalloc(&buf, need * sizeof(float)) != cudaSuccess) return cudaErrorMemoryAllocation;
      cap = need;
    }
    P.stat_mode = STAT_FWD;
    P.stat = buf;
  }
  if (P.stat_mode != STAT_NONE && (!P.stat || P.N % 8 || P.act != ACT_NONE)) return cudaErrorInvalidValue;
  // one instantiation per math mode (TF32X3 three-pass split, TF32 one pass, BF16 one pass on rounded operands)
#define PG_PAIR_MODES(K)                                                            \
  switch (math) {                                                                   \
    case MATH_TF32: return launch_pair_kind<K, MATH_TF32>(ta, tb, tbl, P, bn, st);  \
    case MATH_BF16: return launch_pair_kind<K, MATH_BF16>(ta, tb, tbl, P, bn, st);  \
    default: return launch_pair_kind<K, MATH_TF32X3>(ta, tb, tbl, P, bn, st);       \
  }
  if (dgrad_packed(a)) PG_PAIR_MODES(KIND_DGP)
  if (f4) PG_PAIR_MODES(KIND_F4)
  switch (a.kind) {
    case GEMM_FPROP: PG_PAIR_MODES(GEMM_FPROP)
    case GEMM_DGRAD: PG_PAIR_MODES(GEMM_DGRAD)
    default: PG_PAIR_MODES(GEMM_WGRAD)
  }
#undef PG_PAIR_MODES
}

}  // namespace pg
