// Weight gradient of the 4-channel image-side convolutions on tcgen05
// (discriminator conv1 weight gradient on the real and fake batches, generator
// convT4 weight gradient): dW[cs][tap][c] = sum_pix gy[pix][cs] x[gather(pix, tap)][c]
// with CS = 64 gradient channels, k = 4 (16 taps x 4 channels = N = 64) and
// K = the B*SH*SW small-map pixels of a label (network.cpp:121, the conv_bwd
// weight-gradient GEMM; ConvT uses the same GEMM with the roles swapped).
//
// Round 1 ran this on warp-level mma.sync (thin.cu, 0.77 ms per c4 launch
// against a 0.20 ms HBM floor).  Here one CTA per SM walks (label, 1024-pixel
// chunk) work items; a chunk's 32 k-blocks of 32 pixels feed
// `tcgen05.mma.cta_group::1.kind::tf32` in the TS form, M = 128, N = 64, K = 8:
//   A = gy^T (M = gradient channel): one TMA box {64 channels, 32 pixels} per
//       k-block (plain 256-byte rows); four "A warps" (lane quarters 0, 1; even
//       and odd k-blocks) read a channel column each and write its hi / lo
//       into a tensor-memory ring.  TMEM lanes 64..127 are never written: the
//       M = 128 MMA's upper half is discarded (tcgen05 costs an M = 64 MMA
//       the same issue slots), which bounds the kernel at ~50% tensor use
//   B = im2col(x) (N = tap x 4 channels, K-major, 128-byte swizzle): the input
//       rows under the k-block arrive as one TMA box next to gy; four groups
//       of two gather warps (one k-block each in flight) read each tap's
//       16-byte pixel from that patch and scatter its channels into the rows
//       n = tap * 4 + c (+ lo parts in TF32X3) of an operand ring
// 3xTF32: a_lo b_hi + a_hi b_lo + a_hi b_hi.  TMEM: the A ring, then two
// 64-column accumulation buffers; a segment of 8 k-blocks (96 MMA adds) is
// drained into fp32 registers (gemm_pair.cu's accuracy design) and a chunk's
// 64 x 64 partial goes to the split-K scratch that thin.cu's fixed-order
// reduce sums (deterministic, no atomics).  Measured steps (c4, per launch):
// SS form with A and A lo in shared memory 0.46 ms (shared-memory bound: the
// M = 128 MMA read 48 KB of A per k-block), this TS form 0.44 ms with the
// tensor pipe 46% busy; two accumulation chains per segment: no change.
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

// Ring depths are multiples of the consumer groups (4 gather groups, 2 A-warp
// groups): every slot is then always filled / read by the same group, in order.
// Otherwise a group running ahead can wait on a slot's mbarrier two phases
// ahead and pass on the older phase of the same parity (a 6-deep operand ring
// with 4 groups corrupted the c4 weight gradient of some labels).
constexpr int W4_T = 4;          // TMA ring: gy tile (+ y tile) + x patch
constexpr int W4_O = 8;          // operand ring: B hi, B lo (gather -> MMA)
constexpr int W4_AS = 4;         // TMEM A ring: gy^T hi / lo (A warps -> MMA)
static_assert(W4_T % 4 == 0 && W4_O % 4 == 0 && W4_AS % 2 == 0, "ring depths vs consumer groups");
constexpr int W4_KB = 32;        // pixels per k-block
constexpr int W4_KSEG = 8;       // k-blocks per TMEM accumulation segment
constexpr int W4_CHUNK = 1024;   // pixels per work item (thin.cu TW_SPLIT: same partial layout)
constexpr int W4_NGRP = 4;       // gather groups of two warps (k-blocks in flight)
constexpr int W4_NT = 16 * 32;
constexpr int W4_A = 64 * 32 * 4;  // gy tile: 32 pixel rows x 64 channels (plain, 256 B rows)
constexpr int W4_B = 16 * 512;     // B operand: 64 rows (tap, channel) x 32 pixels, K-major SW128
constexpr int W4_PATCH = 4096;     // input rows of a k-block (patch mode)
constexpr int W4_TS = 2 * W4_A + W4_PATCH;  // TMA slot: gy tile | y tile (fused activation backward) | x patch
constexpr int W4_OS = 2 * W4_B;         // operand slot: B lo | B hi
constexpr int W4_SMEM = W4_T * W4_TS + W4_O * W4_OS + 1024 + 1024;
constexpr uint32_t W4_ACOL = W4_AS * 64;  // accumulators after the A ring: 2 segments x W4_NACC x 64 columns
#ifndef W4_NACC
#define W4_NACC 1  // (2 measured no faster) independent accumulation chains per segment (MMA kk -> kk % W4_NACC), summed by the drain
#endif

struct W4Plan {
  ConvGeo g;
  int L, nchunk;
  long long K;  // pixels per label
  const float* big;
  long long big_ls;
  float* part;
  int patch_rows, patch_bytes;  // patch mode: input rows per k-block, TMA bytes of the patch box
  // fused activation backward (the small operand is gy of the layer's output,
  // y its activation output: the GEMM uses act_bwd(gy, y), and the A warps
  // sum it per channel into bias partials [L][nchunk][2][64])
  int fuse_act;
  float slope;
  float* bpart;
};

PG_DEV int chunk_kblocks(const W4Plan& P, int chunk) {
  const long long rem = P.K - (long long)chunk * W4_CHUNK;
  const long long px = rem < W4_CHUNK ? rem : W4_CHUNK;
  return (int)((px + W4_KB - 1) / W4_KB);
}

PG_DEV void mma_tf32_ts_w4(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Warp roles (512 threads): 0-1 drain (TMEM lane quarters 0, 1 = gradient
// channels 0..63), 2 TMA, 3 TMEM allocation + MMA issue, 4-5 and 8-9 A warps
// (quarters 0, 1; even / odd k-blocks), 6-7 and 10-15 gather (four groups of
// two warps, k-block it % 4 each).
template <int MODE, bool PATCH>
__global__ void __launch_bounds__(W4_NT, 1) wgrad4_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmY,
                                                         const __grid_constant__ CUtensorMap tmX, const W4Plan P) {
  constexpr bool X3 = MODE == MATH_TF32X3, RND = MODE == MATH_BF16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ops = smem + W4_T * W4_TS;
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + W4_O * W4_OS);
  uint64_t* tfree = full + W4_T;
  uint64_t* ready = tfree + W4_T;
  uint64_t* ofree = ready + W4_O;
  uint64_t* aready = ofree + W4_O;
  uint64_t* afree = aready + W4_AS;
  uint64_t* seg_full = afree + W4_AS;
  uint64_t* seg_empty = seg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const ConvGeo& g = P.g;
  const int nitems = P.L * P.nchunk;
  if (tid == 0) {
    for (int s = 0; s < W4_T; ++s) {
      mbar_init(full + s, 1);
      mbar_init(tfree + s, 4);  // the k-block's two A warps and two gather warps read the slot
    }
    for (int s = 0; s < W4_O; ++s) {
      mbar_init(ready + s, 2);
      mbar_init(ofree + s, 1);
    }
    for (int s = 0; s < W4_AS; ++s) {
      mbar_init(aready + s, 2);
      mbar_init(afree + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 2);
    }
    fence_barrier_init();
  }
  if (warp == 3) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  struct Cur {
    int t, kb, nkb;
  };
  auto start_at = [&](int t) { return Cur{t, 0, t < nitems ? chunk_kblocks(P, t % P.nchunk) : 0}; };
  auto adv = [&](Cur& c) {
    if (++c.kb >= c.nkb) c = start_at(c.t + (int)gridDim.x);
  };

  if (warp == 2) {
    // ===================== TMA: gy tile (+ x patch) per k-block =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      if (P.fuse_act) tma_prefetch_desc(&tmY);
      if (PATCH) tma_prefetch_desc(&tmX);
      uint32_t it = 0;
      for (Cur c = start_at(blockIdx.x); c.t < nitems; adv(c), ++it) {
        const int l = c.t / P.nchunk, chunk = c.t % P.nchunk;
        const int s = it % W4_T;
        mbar_wait(tfree + s, ((it / W4_T) & 1) ^ 1);
        mbar_expect_tx(full + s, W4_A * (P.fuse_act ? 2 : 1) + (PATCH ? P.patch_bytes : 0));
        const int p0 = chunk * W4_CHUNK + c.kb * W4_KB;
        const uint32_t dst = smem_u32(smem + s * W4_TS);
        tma_load_3d(dst, &tmA, full + s, 0, p0, l);
        if (P.fuse_act) tma_load_3d(dst + W4_A, &tmY, full + s, 0, p0, l);
        if (PATCH) {  // the input rows under the k-block's 32 / SW output rows of image b
          const int r = p0 / g.SW;
          tma_load_4d(dst + 2 * W4_A, &tmX, full + s, 0, (r % g.SH) * g.s - g.p, r / g.SH, l);
        }
      }
    }
  } else if (warp == 4 || warp == 5 || warp == 8 || warp == 9) {
    // ===================== A warps: gy^T (row = channel) -> TMEM hi / lo =====================
    const int q = warp & 3, par = warp >= 8 ? 1 : 0;
    const int cs = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    float bsum = 0.f;  // fused mode: this group's sum of act_bwd(gy, y) for channel cs over the chunk
    uint32_t it = 0;
    // each group writes its chunk partial when the loop passes the chunk's last
    // k-block, whichever group owns it (a one-k-block chunk gives the other 0)
    auto flush = [&](const Cur& c) {
      if (P.fuse_act && c.kb + 1 == c.nkb) {
        P.bpart[(((long long)(c.t / P.nchunk) * P.nchunk + c.t % P.nchunk) * 2 + par) * 64 + cs] = bsum;
        bsum = 0.f;
      }
    };
    for (Cur c = start_at(blockIdx.x); c.t < nitems; adv(c), ++it) {
      if ((int)(it & 1) != par) {
        flush(c);
        continue;
      }
      const int s = it % W4_T, as = it % W4_AS;
      mbar_wait(full + s, (it / W4_T) & 1);
      const float* ga = reinterpret_cast<const float*>(smem + s * W4_TS);
      const float* ya = ga + W4_A / 4;
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int px = 0; px < 32; ++px) {
        float v = ga[px * 64 + cs];  // a warp reads one 128-byte run per pixel row
        if (P.fuse_act) {
          v = act_bwd(P.fuse_act, v, ya[px * 64 + cs], P.slope);
          bsum += v;  // pixels past K are zero-filled by TMA
        }
        hi[px] = __float_as_uint(RND ? bf16_rne(v) : v);
        lo[px] = __float_as_uint(v - tf32_trunc(v));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(tfree + s);
      flush(c);
      mbar_wait(afree + as, ((it / W4_AS) & 1) ^ 1);
      tc_fence_after();
      tmem_st32(tmem + lane_off + as * 64, hi);
      if (X3) tmem_st32(tmem + lane_off + as * 64 + 32, lo);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(aready + as);
    }
  } else if (warp >= 6) {
    // ===================== gather: B = im2col(x), K-major SW128 (+ lo) =====================
    // B is K-major (row n = tap * 4 + c holds the k-block's 32 pixels, 128 B,
    // 128-byte swizzle: 16-byte chunk j of row n at chunk j ^ (n % 8)); tcgen05
    // takes tf32 MN-major operands only in the 128B_BASE32B swizzle, which a
    // 16-byte-per-tap gather cannot fill contiguously
    const int gi = warp < 8 ? warp - 6 : warp - 8;  // 0..7 over warps 6, 7, 10..15
    const int grp = gi >> 1;
    const int w2 = gi & 1, odd = lane & 1;
    // element i of this thread (8 per k-block): kernel row ki = 2 w2 + i / 4, pixel
    // px = lane / 2 + 16 (i & 1), kernel column from the lane pair: (1, 2) for
    // i & 2 == 0, (0, 3) otherwise -- a warp's 32 loads then cover ~32 adjacent
    // input columns of one row (contiguous patch reads), and the two rows a
    // store instruction hits (taps kj, kj') sit four swizzle phases apart
    auto elem = [&](int i, int& tap, int& px) {
      const int ki = 2 * w2 + (i >> 2);
      const int kj = (i & 2) ? (odd ? 3 : 0) : 1 + odd;
      tap = ki * 4 + kj;
      px = (lane >> 1) + 16 * (i & 1);
    };
    uint32_t it = 0;
    for (Cur c = start_at(blockIdx.x); c.t < nitems; adv(c), ++it) {
      if ((int)(it & (W4_NGRP - 1)) != grp) continue;
      const int s = it % W4_T, o = it % W4_O;
      float4 cur[8];
      if (!PATCH) {  // direct gather from global memory (geometries the patch box does not cover)
        const int l = c.t / P.nchunk, chunk = c.t % P.nchunk;
        const int p0 = chunk * W4_CHUNK + c.kb * W4_KB;  // K < 2^30 (checked on the host)
        const float* x = P.big + (long long)l * P.big_ls;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int tap, px;
          elem(i, tap, px);
          const int p = p0 + px;
          cur[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p >= P.K) continue;
          const int ow = p % g.SW, r = p / g.SW;
          const int oh = r % g.SH, b = r / g.SH;
          const int iy = oh * g.s - g.p + tap / 4, ix = ow * g.s - g.p + tap % 4;
          if (iy >= 0 && iy < g.GH && ix >= 0 && ix < g.GW)
            cur[i] = __ldg(reinterpret_cast<const float4*>(x + (((long long)b * g.GH + iy) * g.GW + ix) * 4));
        }
      }
      mbar_wait(full + s, (it / W4_T) & 1);          // gy (+ patch) landed
      if (PATCH) {
        const float4* xp = reinterpret_cast<const float4*>(smem + s * W4_TS + 2 * W4_A);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int tap, px;
          elem(i, tap, px);
          const int pr = (px / g.SW) * g.s + tap / 4, pc = (px % g.SW) * g.s - g.p + tap % 4;
          cur[i] = (pc >= 0 && pc < g.GW) ? xp[pr * g.GW + pc] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(tfree + s);  // the slot is read (the A warps release their part)
      mbar_wait(ofree + o, ((it / W4_O) & 1) ^ 1);  // operand slot free (its MMAs retired)
      float* bl = reinterpret_cast<float*>(ops + o * W4_OS);
      float* bh = reinterpret_cast<float*>(ops + o * W4_OS + W4_B);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float e4[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
        int tap, px;
        elem(i, tap, px);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int n = tap * 4 + c4;
          const int off = n * 32 + (((px >> 2) ^ (n & 7)) << 2) + (px & 3);
          bh[off] = RND ? bf16_rne(e4[c4]) : e4[c4];
          if (X3) bl[off] = e4[c4] - tf32_trunc(e4[c4]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(ready + o);
    }
  } else if (warp == 3) {
    // ===================== MMA issue (TS form: A = gy^T from TMEM) =====================
    constexpr uint32_t idesc = make_idesc(128, 64, false, false);
    const uint64_t bl0 = make_desc(smem_u32(ops), 16u, 1024u, UMMA_SW128);
    const uint64_t b0 = make_desc(smem_u32(ops) + W4_B, 16u, 1024u, UMMA_SW128);
    uint32_t it = 0, sc = 0;
    for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
      const int nkb = chunk_kblocks(P, t % P.nchunk);
      for (int k_seg = 0; k_seg < nkb; k_seg += W4_KSEG, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(seg_empty + buf, ((sc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + W4_ACOL + buf * (64 * W4_NACC);
        const int k_end = min(nkb, k_seg + W4_KSEG);
        for (int kb = k_seg; kb < k_end; ++kb, ++it) {
          const int o = it % W4_O, as = it % W4_AS;
          mbar_wait(ready + o, (it / W4_O) & 1);
          mbar_wait(aready + as, (it / W4_AS) & 1);
          tc_fence_after();
          const uint64_t sl = (uint64_t)((o * W4_OS) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < W4_KB / 8; ++kk) {
              const uint32_t a_t = tmem + as * 64 + kk * 8;
              const uint64_t bh = b0 + sl + (kk * 32 >> 4);
              const uint32_t d = d0 + (kk % W4_NACC) * 64;
              const uint32_t acc = (kb != k_seg || kk >= W4_NACC) ? 1u : 0u;
              if (X3) {
                mma_tf32_ts_w4(d, a_t + 32, bh, idesc, acc);  // small terms first
                mma_tf32_ts_w4(d, a_t, bl0 + sl + (kk * 32 >> 4), idesc, 1u);
                mma_tf32_ts_w4(d, a_t, bh, idesc, 1u);
              } else {
                mma_tf32_ts_w4(d, a_t, bh, idesc, acc);
              }
            }
            mma_commit(ofree + o);
            mma_commit(afree + as);
            if (kb + 1 == k_end) mma_commit(seg_full + buf);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ===================== drain: rows 0..63 (cs), 64 columns =====================
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int row = warp * 32 + lane;
    uint32_t sc = 0;
    for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
      const int l = t / P.nchunk, chunk = t % P.nchunk;
      const int nkb = chunk_kblocks(P, chunk);
      float acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.f;
      for (int k_seg = 0; k_seg < nkb; k_seg += W4_KSEG, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(seg_full + buf, (sc >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int a = 0; a < W4_NACC; ++a)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + lane_base + W4_ACOL + buf * (64 * W4_NACC) + a * 64 + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[c * 32 + i] += __uint_as_float(r[i]);
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(seg_empty + buf);
      }
      float4* dst = reinterpret_cast<float4*>(P.part + (((long long)l * P.nchunk + chunk) * 64 + row) * 64);
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool wgrad4_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PG_WGRAD4");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool wgrad4_supported(const GemmArgs& a, int math) {
  const ConvGeo& g = a.g;
  return wgrad4_enabled() && math != MATH_FP32_SIMT && a.kind == GEMM_WGRAD && g.CG == 4 && g.CS == 64 && g.k == 4 &&
         encode_fn() && aligned16(a.small) && aligned16(a.big) && a.small_ls % 4 == 0 && a.big_ls % 4 == 0;
}

// part: [L][nchunk][64][64] chunk partials (nchunk = ceil(K / 1024)), summed by thin.cu's reduce
cudaError_t launch_wgrad4(const GemmArgs& a, int math, float* part, int nchunk, cudaStream_t st) {
  const ConvGeo& g = a.g;
  if ((long long)g.B * g.SH * g.SW > (1LL << 30) || (long long)g.GH * g.GW * 4 > (1LL << 30)) return cudaErrorInvalidValue;
  W4Plan P{};
  P.g = g;
  P.L = a.L;
  P.nchunk = nchunk;
  P.K = (long long)g.B * g.SH * g.SW;
  P.big = a.big;
  P.big_ls = a.big_ls;
  P.part = part;
  // input-side activation backward (GemmArgs::in_act): `small` is the raw output
  // gradient, in_y the activation output; the bias partials follow the weight partials
  P.fuse_act = a.in_act;
  P.slope = a.in_slope;
  P.bpart = part + (size_t)a.L * nchunk * 64 * 64;
  CUtensorMap tm, ty;
  const long long dims[3] = {g.CS, P.K, a.L};
  const long long strides[2] = {g.CS, a.small_ls};
  const int box[3] = {64, W4_KB, 1};
  const int one[3] = {1, 1, 1};
  if (!make_map(&tm, a.small, 3, dims, strides, box, one, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  ty = tm;
  if (P.fuse_act && !make_map(&ty, a.in_y, 3, dims, strides, box, one, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  // patch mode: a k-block = 32 / SW whole output rows of one image, whose input
  // rows (GW * 4 floats each) arrive as one TMA box next to the gy boxes
  const bool patch = W4_KB % g.SW == 0 && (g.SH * g.SW) % W4_KB == 0 && g.GW * 4 <= 256;
  CUtensorMap tx{};
  if (patch) {
    P.patch_rows = (W4_KB / g.SW - 1) * g.s + g.k;
    P.patch_bytes = P.patch_rows * g.GW * 16;
    const long long xd[4] = {(long long)g.GW * 4, g.GH, g.B, a.L};
    const long long xs[3] = {(long long)g.GW * 4, (long long)g.GH * g.GW * 4, a.big_ls};
    const int xb[4] = {g.GW * 4, P.patch_rows, 1, 1};
    const int one4[4] = {1, 1, 1, 1};
    if (P.patch_bytes > W4_PATCH || !make_map(&tx, a.big, 4, xd, xs, xb, one4, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  static PerDeviceOnce configured;
  cudaError_t e = configured.run([] {
    for (auto f : {wgrad4_kernel<MATH_TF32X3, true>, wgrad4_kernel<MATH_TF32X3, false>, wgrad4_kernel<MATH_TF32, true>,
                   wgrad4_kernel<MATH_TF32, false>, wgrad4_kernel<MATH_BF16, true>, wgrad4_kernel<MATH_BF16, false>}) {
      cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, W4_SMEM);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  });
  if (e != cudaSuccess) return e;
  const int items = a.L * nchunk;
  const int grid = std::min(items, sm_count_tma());
#define PG_W4(M)                                                            \
  (patch ? wgrad4_kernel<M, true><<<grid, W4_NT, W4_SMEM, st>>>(tm, ty, tx, P)  \
         : wgrad4_kernel<M, false><<<grid, W4_NT, W4_SMEM, st>>>(tm, ty, tx, P))
  if (math == MATH_TF32X3) PG_W4(MATH_TF32X3);
  else if (math == MATH_BF16) PG_W4(MATH_BF16);
  else PG_W4(MATH_TF32);
#undef PG_W4
  return launched();
}

}  // namespace pg
