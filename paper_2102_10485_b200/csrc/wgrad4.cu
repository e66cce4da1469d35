// Weight gradient of the 4-channel image-side convolutions on tcgen05
// (discriminator conv1 weight gradient on the real and fake batches, generator
// convT4 weight gradient): dW[cs][tap][c] = sum_pix gy[pix][cs] x[gather(pix, tap)][c]
// with CS = 64 gradient channels, k = 4 (16 taps x 4 channels = N = 64) and
// K = the B*SH*SW small-map pixels of a label (network.cpp:121, the conv_bwd
// weight-gradient GEMM; ConvT uses the same GEMM with the roles swapped).
//
// Round 1 ran this on warp-level mma.sync (thin.cu, 0.8 ms per c4 launch
// against a 0.2 ms HBM floor).  Here one CTA per SM walks (label, 1024-pixel
// chunk) work items; a chunk's 32 k-blocks of 32 pixels feed
// `tcgen05.mma.cta_group::1.kind::tf32` with M = 128, N = 64, K = 8:
//   A = gy^T (M = cs, MN-major): two TMA boxes {32 cs, 32 pixels} per k-block
//       in the 128B_ATOM_32B swizzle (the pair engine's MN-major layout); rows
//       64..127 of the M = 128 MMA read the stage's B bytes and land in TMEM
//       lanes no warp reads (tcgen05 has no M = 64 layout that keeps one row per
//       lane in a single lane quarter pair; the half-empty tile costs tensor
//       time the HBM-bound kernel has to spare)
//   B = im2col(x) (N = tap x 4 channels, K-major, 128-byte swizzle): the
//       gather warps read each tap's 16-byte pixel from global memory
//       (L1/L2-resident: a k-block touches ~4 input rows) and scatter its four
//       channels into the rows n = tap * 4 + c -- no 16-byte TMA boxes (512
//       tiny rows per k-block); in TF32X3 they also write lo = x - trunc(x) of
//       A and B into the lo ring (3xTF32: a_lo b_hi + a_hi b_lo + a_hi b_hi)
// TMEM: two 64-column accumulation buffers; a segment of 8 k-blocks (96 MMA
// adds) is drained into fp32 registers (gemm_pair.cu's accuracy design) and a
// chunk's 64 x 64 partial goes to the split-K scratch that thin.cu's fixed-order
// reduce sums (deterministic, no atomics).
//
// Warp roles (384 threads): warps 0-1 drain (TMEM lane quarters 0, 1 = rows
// 0..63), warp 2 TMA, warp 3 TMEM allocation + MMA issue, warps 4-11 gather.
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

constexpr int W4_T = 8;          // TMA ring: gy boxes + x patch (DRAM latency in flight)
constexpr int W4_O = 4;          // operand ring: B hi, A lo, B lo (gather -> MMA)
constexpr int W4_KB = 32;        // pixels per k-block
constexpr int W4_KSEG = 8;       // k-blocks per TMEM accumulation segment
constexpr int W4_CHUNK = 1024;   // pixels per work item (thin.cu TW_SPLIT: same partial layout)
constexpr int W4_NG = 8;         // gather warps
constexpr int W4_NGRP = 4;       // gather groups (k-blocks in flight), W4_NG / W4_NGRP warps each
constexpr int W4_NT = (4 + W4_NG) * 32;
constexpr int W4_A = 2 * 4096;   // A stage: 2 MN atoms of 32 cs x 32 pixels
constexpr int W4_B = 16 * 512;   // B stage: 16 taps x 32 pixels x 16 B
constexpr int W4_PATCH = 4096;  // input rows of a k-block (patch mode)
constexpr int W4_TS = W4_A + W4_PATCH;   // TMA slot: A hi | x patch
constexpr int W4_OS = W4_A + 2 * W4_B;   // operand slot: A lo | B lo | B hi
// the M = 128 MMA reads A rows 64..127 at +8 KB / +12 KB: inside the next
// slot (or the pad after the last one) for A hi, the B lo part for A lo
constexpr int W4_TPAD = 2 * 4096 - W4_PATCH;
constexpr int W4_SMEM = W4_T * W4_TS + W4_TPAD + W4_O * W4_OS + 1024 + 1024;

struct W4Plan {
  ConvGeo g;
  int L, nchunk;
  long long K;  // pixels per label
  const float* big;
  long long big_ls;
  float* part;
  int patch_rows, patch_bytes;  // patch mode: input rows per k-block, TMA bytes of the patch box
};

PG_DEV int chunk_kblocks(const W4Plan& P, int chunk) {
  const long long rem = P.K - (long long)chunk * W4_CHUNK;
  const long long px = rem < W4_CHUNK ? rem : W4_CHUNK;
  return (int)((px + W4_KB - 1) / W4_KB);
}

template <bool X3, bool PATCH>
__global__ void __launch_bounds__(W4_NT, 1) wgrad4_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                                                         const W4Plan P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ops = smem + W4_T * W4_TS + W4_TPAD;
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + W4_O * W4_OS);
  uint64_t* tfree = full + W4_T;
  uint64_t* ready = tfree + W4_T;
  uint64_t* ofree = ready + W4_O;
  uint64_t* seg_full = ofree + W4_O;
  uint64_t* seg_empty = seg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const ConvGeo& g = P.g;
  const int nitems = P.L * P.nchunk;
  if (tid == 0) {
    for (int s = 0; s < W4_T; ++s) {
      mbar_init(full + s, 1);
      mbar_init(tfree + s, 1);
    }
    for (int s = 0; s < W4_O; ++s) {
      mbar_init(ready + s, W4_NG / W4_NGRP);
      mbar_init(ofree + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, 2);
    }
    fence_barrier_init();
  }
  if (warp == 3) tmem_alloc(tmem_slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 2) {
    // ===================== TMA: gy boxes =====================
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      if (PATCH) tma_prefetch_desc(&tmX);
      uint32_t it = 0;
      for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
        const int l = t / P.nchunk, chunk = t % P.nchunk;
        const int nkb = chunk_kblocks(P, chunk);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % W4_T;
          mbar_wait(tfree + s, ((it / W4_T) & 1) ^ 1);
          mbar_expect_tx(full + s, W4_A + (PATCH ? P.patch_bytes : 0));
          const int p0 = chunk * W4_CHUNK + kb * W4_KB;
          const uint32_t dst = smem_u32(smem + s * W4_TS);
          tma_load_3d(dst, &tmA, full + s, 0, p0, l);
          tma_load_3d(dst + 4096, &tmA, full + s, 32, p0, l);
          if (PATCH) {  // the input rows under the k-block's 32 / SW output rows of image b
            const int r = p0 / g.SW;
            tma_load_4d(dst + W4_A, &tmX, full + s, 0, (r % g.SH) * g.s - g.p, r / g.SH, l);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== gather: B = im2col(x) (+ lo parts) =====================
    // B is K-major (row n = tap * 4 + c holds the k-block's 32 pixels, 128 B,
    // 128-byte swizzle: 16-byte chunk j of row n at chunk j ^ (n % 8)); tcgen05
    // takes tf32 MN-major operands only in the 128B_BASE32B swizzle, which a
    // 16-byte-per-tap gather cannot fill contiguously.  Loads run three
    // k-blocks ahead of the stores (L2 latency >> one k-block of MMAs).
    // four groups of two warps take every fourth k-block: a group's body is a
    // dependency chain (barrier, loads, splits, stores, proxy fence, arrive), so
    // k-blocks in flight, not warps per k-block, set the gather throughput
    const int grp = (warp - 4) >> 1;
    const int gt = (tid - 128) & 63;
    // element i of this thread (8 per k-block): kernel row ki = 2 w + i / 4, pixel
    // px = lane / 2 + 16 (i & 1), kernel column from the lane pair: (1, 2) for
    // i & 2 == 0, (0, 3) otherwise -- a warp's 32 loads then cover ~32 adjacent
    // input columns of one row (contiguous patch reads), and the two rows a
    // store instruction hits (taps kj, kj') sit four swizzle phases apart
    const int w2 = gt >> 5, odd = lane & 1;
    auto elem = [&](int i, int& tap, int& px) {
      const int ki = 2 * w2 + (i >> 2);
      const int kj = (i & 2) ? (odd ? 3 : 0) : 1 + odd;
      tap = ki * 4 + kj;
      px = (lane >> 1) + 16 * (i & 1);
    };
    struct Cur {
      int t, kb, nkb;
    };
    auto start_at = [&](int t) { return Cur{t, 0, t < nitems ? chunk_kblocks(P, t % P.nchunk) : 0}; };
    auto adv = [&](Cur& c) {
      if (++c.kb >= c.nkb) c = start_at(c.t + (int)gridDim.x);
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
      mbar_wait(full + s, (it / W4_T) & 1);          // A (+ patch) landed
      mbar_wait(ofree + o, ((it / W4_O) & 1) ^ 1);  // operand slot free (its MMAs retired)
      float* bh = reinterpret_cast<float*>(ops + o * W4_OS + W4_A + W4_B);
      float* bl = reinterpret_cast<float*>(ops + o * W4_OS + W4_A);
      const float4* ah = reinterpret_cast<const float4*>(smem + s * W4_TS);
      float4 a4[W4_A / 16 / 64];
      if (X3) {
#pragma unroll
        for (int i = 0; i < W4_A / 16 / 64; ++i) a4[i] = ah[gt + 64 * i];
      }
      if (PATCH) {
        const float4* xp = reinterpret_cast<const float4*>(smem + s * W4_TS + W4_A);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          int tap, px;
          elem(i, tap, px);
          const int pr = (px / g.SW) * g.s + tap / 4, pc = (px % g.SW) * g.s - g.p + tap % 4;
          cur[i] = (pc >= 0 && pc < g.GW) ? xp[pr * g.GW + pc] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float e4[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
        int tap, px;
        elem(i, tap, px);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int n = tap * 4 + c4;
          const int off = n * 32 + (((px >> 2) ^ (n & 7)) << 2) + (px & 3);
          bh[off] = e4[c4];
          if (X3) bl[off] = e4[c4] - tf32_trunc(e4[c4]);
        }
      }
      if (X3) {
        float4* al = reinterpret_cast<float4*>(ops + o * W4_OS);
#pragma unroll
        for (int i = 0; i < W4_A / 16 / 64; ++i) {
          const float4 a = a4[i];
          al[gt + 64 * i] =
              make_float4(a.x - tf32_trunc(a.x), a.y - tf32_trunc(a.y), a.z - tf32_trunc(a.z), a.w - tf32_trunc(a.w));
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(ready + o);
    }
  } else if (warp == 3) {
    // ===================== MMA issue =====================
    constexpr uint32_t idesc = make_idesc(128, 64, true, false);
    const uint64_t a0 = make_desc(smem_u32(smem), 4096u, 512u, UMMA_SW128_BASE32B);
    const uint64_t al0 = make_desc(smem_u32(ops), 4096u, 512u, UMMA_SW128_BASE32B);
    const uint64_t bl0 = make_desc(smem_u32(ops) + W4_A, 16u, 1024u, UMMA_SW128);
    const uint64_t b0 = make_desc(smem_u32(ops) + W4_A + W4_B, 16u, 1024u, UMMA_SW128);
    uint32_t it = 0, sc = 0;
    for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
      const int nkb = chunk_kblocks(P, t % P.nchunk);
      for (int k_seg = 0; k_seg < nkb; k_seg += W4_KSEG, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(seg_empty + buf, ((sc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * 64;
        const int k_end = min(nkb, k_seg + W4_KSEG);
        for (int kb = k_seg; kb < k_end; ++kb, ++it) {
          const int s = it % W4_T, o = it % W4_O;
          mbar_wait(ready + o, (it / W4_O) & 1);  // the gather saw slot s land before it arrived
          tc_fence_after();
          const uint64_t so = (uint64_t)((s * W4_TS) >> 4), sl = (uint64_t)((o * W4_OS) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < W4_KB / 8; ++kk) {
              const uint64_t ah = a0 + so + (kk * 1024 >> 4), bh = b0 + sl + (kk * 32 >> 4);
              const uint32_t acc = (kb != k_seg || kk) ? 1u : 0u;
              if (X3) {
                mma_tf32(d, al0 + sl + (kk * 1024 >> 4), bh, idesc, acc);  // small terms first
                mma_tf32(d, ah, bl0 + sl + (kk * 32 >> 4), idesc, 1u);
                mma_tf32(d, ah, bh, idesc, 1u);
              } else {
                mma_tf32(d, ah, bh, idesc, acc);
              }
            }
            mma_commit(tfree + s);
            mma_commit(ofree + o);
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
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + buf * 64 + c * 32, r);
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
    tmem_dealloc(tmem, 128);
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
  CUtensorMap tm;
  const long long dims[3] = {g.CS, P.K, a.L};
  const long long strides[2] = {g.CS, a.small_ls};
  const int box[3] = {32, W4_KB, 1};
  const int one[3] = {1, 1, 1};
  if (!make_map(&tm, a.small, 3, dims, strides, box, one, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
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
    for (auto f : {wgrad4_kernel<true, true>, wgrad4_kernel<true, false>, wgrad4_kernel<false, true>,
                   wgrad4_kernel<false, false>}) {
      cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, W4_SMEM);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  });
  if (e != cudaSuccess) return e;
  const int items = a.L * nchunk;
  const int grid = std::min(items, sm_count_tma());
  const bool x3 = math == MATH_TF32X3;
  if (x3 && patch) wgrad4_kernel<true, true><<<grid, W4_NT, W4_SMEM, st>>>(tm, tx, P);
  else if (x3) wgrad4_kernel<true, false><<<grid, W4_NT, W4_SMEM, st>>>(tm, tx, P);
  else if (patch) wgrad4_kernel<false, true><<<grid, W4_NT, W4_SMEM, st>>>(tm, tx, P);
  else wgrad4_kernel<false, false><<<grid, W4_NT, W4_SMEM, st>>>(tm, tx, P);
  return launched();
}

}  // namespace pg
