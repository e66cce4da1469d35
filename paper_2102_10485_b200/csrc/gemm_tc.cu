// tcgen05 implicit-GEMM engine (sm_100a): math modes TF32 (one kind::tf32
// MMA per K-step) and TF32X3 (split a = a_hi + a_lo, b = b_hi + b_lo in
// shared memory; D += a_lo b_hi + a_hi b_lo + a_hi b_hi, fp32-accurate).
//
// Persistent, warp-specialized; each CTA walks 128 x BN output tiles of the
// (label, phase) problems in a static round-robin:
//   warps 0-3  producers: cp.async-gather the A / B tiles straight from the
//              NHWC maps into the UMMA canonical layouts (implicit-GEMM index
//              maps of gemm_gather.cuh, per-row state hoisted out of the K
//              loop, zero-fill for padding), STAGES-2 k-blocks in flight; in
//              TF32X3 write lo = x - trunc_tf32(x) beside the raw tile (the
//              raw fp32 tile is the hi operand: tcgen05 truncates to tf32).
//   warp 4     the single MMA-issuing thread (and TMEM allocation): K is cut
//              into segments of KSEG k-blocks; each segment accumulates into
//              one of two TMEM buffers (ping-pong) and is committed to
//              seg_full[buf].
//   warps 5-8  drain + epilogue: each segment is pulled out of TMEM
//              (tcgen05.ld) and added into an IEEE fp32 running sum in
//              registers, then the buffer is released (seg_empty[buf]).
//              After the last segment of a tile: bias + activation, store.
// Why drain: the tensor core accumulates with truncation, so one TMEM
// accumulator over K = 16384 loses ~1e-4 relative; segments of 2 k-blocks
// keep every accumulation chain at <= 24 MMA adds, which brings 3xTF32 to
// the accuracy of a plain fp32 FMA loop (scripts/tc_accuracy.py).
//
// Shared-memory operand layouts:
//   K-major  (contiguous K in global), SWIZZLE_NONE: 16-byte chunk c of row r
//            at c*(R*16) + (r/8)*128 + (r%8)*16; LBO = R*16, SBO = 128.
//   MN-major (contiguous M/N in global): tcgen05 accepts tf32 MN-major
//            operands only in SWIZZLE_128B_BASE32B (see mn_offset).
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "device_cache.hpp"
#include "gemm_gather.cuh"
#include "tc_ptx.cuh"
#include "kernels.hpp"

namespace pg {

namespace {

constexpr int BM = 128;
constexpr int BK = 16;          // fp32 elements of K per stage
constexpr int NPROD = 128;      // warps 0-3
constexpr int NDRAIN = 128;     // warps 5-8
constexpr int NTHREADS = NPROD + 32 + NDRAIN;
constexpr int KSEG = 4;         // k-blocks per TMEM accumulation segment (chain <= 24 MMA adds)
__constant__ int c_dbg = 0;     // PG_TC_DEBUG bits: 1 no loads, 2 no split, 4 no MMA, 8 no drain loads

// MN-major atom: 32 MN elements (128 B) x 4 K rows (128 B apart); the 16-byte
// chunk bits [5,7) are XORed with the row bits [7,9).  Atoms MN-adjacent at
// 512 B (LBO), K-adjacent at (R/32)*512 B (SBO).
PG_DEV int mn_offset(int R, int col4, int kr) {
  const int row = kr & 3;
  return (kr >> 2) * ((R / 32) * 512) + (col4 >> 3) * 512 + row * 128 + (((col4 & 7) * 16) ^ (row << 5));
}

// ---- tile geometry ------------------------------------------------------
__host__ __device__ constexpr int tile_bytes(int rows) { return rows * BK * 4; }
__host__ __device__ constexpr bool a_is_mn(int kind) { return kind == GEMM_WGRAD; }
__host__ __device__ constexpr bool b_is_mn(int kind) { return kind != GEMM_FPROP; }
__host__ __device__ constexpr int stage_bytes(int bn, bool split) {
  return (tile_bytes(BM) + tile_bytes(bn)) * (split ? 2 : 1);
}
__host__ __device__ constexpr int num_stages(int bn, bool split) {
  return 192 * 1024 / stage_bytes(bn, split) > 8 ? 8 : 192 * 1024 / stage_bytes(bn, split);
}
// k-blocks the producers run ahead; a stage is re-filled only after the MMA
// released it two k-blocks earlier, so producers never wait on the MMA that
// is currently running
__host__ __device__ constexpr int lookahead(int stages) { return stages - 2 < 1 ? 1 : stages - 2; }
__host__ __device__ constexpr int smem_bytes(int bn, bool split) {
  return num_stages(bn, split) * stage_bytes(bn, split) + 1024 /* barriers */ + 1024 /* alignment */;
}
__host__ __device__ constexpr uint32_t tmem_cols(int bn) { return 2 * bn <= 32 ? 32 : 2 * bn; }

PG_DEV float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

PG_DEV float4 ld4(const float* p) { return p ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0, 0, 0, 0); }

PG_DEV void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
PG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
PG_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// lo = x - trunc_tf32(x) for one 16-byte chunk (the raw chunk stays as "hi")
PG_DEV void store_lo(uint8_t* dst, float4 v) {
  *reinterpret_cast<float4*>(dst) =
      make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
}

// ---- per-row producer state for the K-major A operand (FPROP / DGRAD) ----
struct RowState {
  bool valid;
  int b, y0, x0;  // FPROP: top-left of the receptive field; DGRAD: big pixel (y0, x0)
};

template <int KIND>
PG_DEV RowState row_state(const ConvGeo& g, const GemmView& v, int m) {
  RowState r;
  r.valid = m < v.M;
  r.b = r.y0 = r.x0 = 0;
  if (!r.valid) return r;
  if (KIND == GEMM_FPROP) {
    int j = m % g.SW, t = m / g.SW;
    int i = t % g.SH;
    r.b = t / g.SH;
    r.y0 = i * g.s - g.p;
    r.x0 = j * g.s - g.p;
  } else {
    int xi = m % v.nx, t = m / v.nx;
    int yi = t % v.ny;
    r.b = t / v.ny;
    r.y0 = v.y0 + yi * g.s;
    r.x0 = v.x0 + xi * g.s;
  }
  return r;
}

// address of A[m][kk .. kk+3] given the row state (nullptr = zero padding)
template <int KIND>
PG_DEV const float* a_row_ptr(const ConvGeo& g, const GemmView& v, const RowState& r, int kk) {
  if (!r.valid || kk >= v.K) return nullptr;
  if (KIND == GEMM_FPROP) {
    int tap = kk / g.CG, cg = kk - tap * g.CG;
    int ki = tap / g.k, kj = tap - ki * g.k;
    int y = r.y0 + ki, x = r.x0 + kj;
    if (y < 0 || y >= g.GH || x < 0 || x >= g.GW) return nullptr;
    return v.A + (((long long)r.b * g.GH + y) * g.GW + x) * g.CG + cg;
  } else {
    int t = kk / g.CS, cs = kk - t * g.CS;
    int ty = t / v.ntx, tx = t - ty * v.ntx;
    int ki = v.ry + ty * g.s, kj = v.rx + tx * g.s;
    int i = (r.y0 + g.p - ki) / g.s, j = (r.x0 + g.p - kj) / g.s;
    if (i < 0 || i >= g.SH || j < 0 || j >= g.SW) return nullptr;
    return v.A + (((long long)r.b * g.SH + i) * g.SW + j) * g.CS + cs;
  }
}

struct TileGrid {
  int ntn, ntm, nz;  // n tiles, m tiles (max over phases), labels x phases
  __host__ __device__ int total() const { return ntn * ntm * nz; }
};

PG_DEV void tile_coords(const TileGrid& tg, int t, int& z, int& mt, int& nt) {
  nt = t % tg.ntn;
  const int r = t / tg.ntn;
  mt = r % tg.ntm;
  z = r / tg.ntm;
}

template <int KIND, int BN, int MODE>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_tc_kernel(GemmArgs a, TileGrid tg) {
  constexpr bool SPLIT = MODE == MATH_TF32X3;
  constexpr int STAGES = num_stages(BN, SPLIT);
  constexpr int A_BYTES = tile_bytes(BM);
  constexpr int B_BYTES = tile_bytes(BN);
  constexpr int STAGE = stage_bytes(BN, SPLIT);
  constexpr bool A_MN = a_is_mn(KIND), B_MN = b_is_mn(KIND);
  constexpr uint32_t TMEM_COLS = tmem_cols(BN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* seg_full = empty + STAGES;
  uint64_t* seg_empty = seg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(seg_empty + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int phases = gemm_phases(a);
  const ConvGeo& g = a.g;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, NPROD);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(seg_full + b, 1);
      mbar_init(seg_empty + b, NDRAIN);
    }
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  uint32_t kc = 0;  // k-blocks consumed / produced so far (stage ring)
  uint32_t sc = 0;  // segments so far (TMEM ping-pong)
  const int ntiles = tg.total();

  if (warp < 4) {
    // ===================== producers =====================
    // cp.async straight into the canonical layouts (zero-fill for padding),
    // lookahead(STAGES) k-blocks in flight per thread; the raw fp32 tile is the "hi"
    // operand as-is (the tensor core reads the top 19 bits of each fp32, i.e.
    // truncates to tf32), and in TF32X3 each thread then writes lo = x -
    // trunc_tf32(x) for exactly the chunks it copied.
    const int mn4 = tid % 32, krow0 = tid / 32;
    const bool one_tap = (KIND == GEMM_FPROP ? g.CG : g.CS) % BK == 0;
    // issue cursor: (tile, k-block) of the next k-block to fetch
    int it_t = 0, it_kb = 0, it_nk = 0, im0 = 0, in0 = 0;
    GemmView iv = make_view(a, 0, 0);
    RowState irs = row_state<KIND>(g, iv, 0);
    auto load_tile = [&](int t) -> bool {
      int z, mt, nt;
      tile_coords(tg, t, z, mt, nt);
      iv = make_view(a, z / phases, z % phases);
      im0 = mt * BM;
      in0 = nt * BN;
      if (im0 >= iv.M || in0 >= iv.N) return false;
      it_nk = (iv.K + BK - 1) / BK;
      if (it_nk == 0) return false;
      irs = row_state<KIND>(g, iv, im0 + tid);
      return true;
    };
    auto seek = [&](int t) -> bool {
      for (; t < ntiles; t += gridDim.x)
        if (load_tile(t)) {
          it_t = t;
          it_kb = 0;
          return true;
        }
      return false;
    };
    bool ivalid = seek(blockIdx.x);
    uint32_t issued = 0, done = 0;

    auto issue = [&]() {
      const int s = issued % STAGES;
      mbar_wait(empty + s, ((issued / STAGES) & 1) ^ 1);
      const uint32_t a_hi = smem_u32(smem + s * STAGE);
      const uint32_t b_hi = a_hi + A_BYTES;
      const int k0 = it_kb * BK;
      const GemmView& v = iv;
      if (c_dbg & 1) goto issued_done;
      // ---------------- A ----------------
      if (!A_MN) {
        // 128 rows x 8 chunks; this thread owns row tid
        const uint32_t row_off = (tid / 8) * 128 + (tid % 8) * 16;
        if (one_tap) {
          const float* base = a_row_ptr<KIND>(g, v, irs, k0);
#pragma unroll
          for (int c = 0; c < BK / 4; ++c) {
            const bool ok = base && k0 + 4 * c < v.K;
            cp_async16(a_hi + c * (BM * 16) + row_off, ok ? base + 4 * c : v.A, ok);
          }
        } else {
#pragma unroll 2
          for (int c = 0; c < BK / 4; ++c) {
            const float* p = a_row_ptr<KIND>(g, v, irs, k0 + 4 * c);
            cp_async16(a_hi + c * (BM * 16) + row_off, p ? p : v.A, p != nullptr);
          }
        }
      } else {
        // WGRAD A[m = cs][k = spix] = smallg[spix][cs]: 32 float4 columns x 32 k rows
#pragma unroll
        for (int j = 0; j < BK / 4; ++j) {
          const int kr = krow0 + 4 * j, k = k0 + kr, m = im0 + 4 * mn4;
          const bool ok = k < v.K && m < v.M;
          cp_async16(a_hi + mn_offset(BM, mn4, kr), ok ? v.A + (long long)k * g.CS + m : v.A, ok);
        }
      }
      // ---------------- B ----------------
      if (!B_MN) {
        // FPROP: B[n][k] = W[n][k], rows contiguous over K; BN rows x 8 chunks
#pragma unroll
        for (int it = 0; it < (BN * (BK / 4) + NPROD - 1) / NPROD; ++it) {
          const int item = tid + it * NPROD;
          if (item < BN * (BK / 4)) {
            const int c = item / BN, r = item % BN;
            const int n = in0 + r, k = k0 + 4 * c;
            const bool ok = n < v.N && k < v.K;
            cp_async16(b_hi + c * (BN * 16) + (r / 8) * 128 + (r % 8) * 16, ok ? v.Bw + (long long)n * v.K + k : v.Bw,
                       ok);
          }
        }
      } else {
        // MN-major B: (BN/4) float4 columns x 32 k rows
        constexpr int COLS = BN / 4;
        constexpr int ITEMS = COLS * BK;
#pragma unroll
        for (int it = 0; it < (ITEMS + NPROD - 1) / NPROD; ++it) {
          const int item = tid + it * NPROD;
          if (item < ITEMS) {
            const int col = item % COLS, kr = item / COLS;
            const int n = in0 + 4 * col, k = k0 + kr;
            const float* p = nullptr;
            if (n < v.N && k < v.K) {
              if (KIND == GEMM_DGRAD) p = dgrad_b_ptr(g, v, n, k);
              else p = wgrad_b_ptr(g, v, n, k);
            }
            cp_async16(b_hi + mn_offset(BN, col, kr), p ? p : v.Bw, p != nullptr);
          }
        }
      }
    issued_done:
      ++issued;
      if (++it_kb >= it_nk) ivalid = seek(it_t + gridDim.x);
    };

    // chunk offsets this thread owns in every stage (identical for issue and split)
    constexpr int NA = BK / 4;
    constexpr int NB_ITEMS = BN * (BK / 4);  // same count for both B layouts
    constexpr int NB = (NB_ITEMS + NPROD - 1) / NPROD;
    int a_off[NA], b_off[NB];
#pragma unroll
    for (int c = 0; c < NA; ++c)
      a_off[c] = A_MN ? mn_offset(BM, mn4, krow0 + 4 * c) : c * (BM * 16) + (tid / 8) * 128 + (tid % 8) * 16;
#pragma unroll
    for (int it = 0; it < NB; ++it) {
      const int item = tid + it * NPROD;
      if (B_MN) b_off[it] = mn_offset(BN, item % (BN / 4), item / (BN / 4));
      else b_off[it] = (item / BN) * (BN * 16) + ((item % BN) / 8) * 128 + (item % 8) * 16;
      if (item >= NB_ITEMS) b_off[it] = -1;
    }

    auto finalize = [&]() {
      const int s = done % STAGES;
      if (SPLIT && !(c_dbg & 2)) {
        uint8_t* a_hi = smem + s * STAGE;
        uint8_t* b_hi = a_hi + A_BYTES;
        uint8_t* a_lo = b_hi + B_BYTES;
        uint8_t* b_lo = a_lo + A_BYTES;
        // all loads first (independent), then the splits and stores
        float4 va[NA], vb[NB];
#pragma unroll
        for (int c = 0; c < NA; ++c) va[c] = *reinterpret_cast<const float4*>(a_hi + a_off[c]);
#pragma unroll
        for (int it = 0; it < NB; ++it)
          if (b_off[it] >= 0) vb[it] = *reinterpret_cast<const float4*>(b_hi + b_off[it]);
#pragma unroll
        for (int c = 0; c < NA; ++c) store_lo(a_lo + a_off[c], va[c]);
#pragma unroll
        for (int it = 0; it < NB; ++it)
          if (b_off[it] >= 0) store_lo(b_lo + b_off[it], vb[it]);
      }
      if (MODE == MATH_BF16) {  // bf16 operands: round this thread's chunks in place
        uint8_t* a_hi = smem + s * STAGE;
        uint8_t* b_hi = a_hi + A_BYTES;
#pragma unroll
        for (int c = 0; c < NA; ++c) {
          float4* p = reinterpret_cast<float4*>(a_hi + a_off[c]);
          *p = bf16_rne4(*p);
        }
#pragma unroll
        for (int it = 0; it < NB; ++it)
          if (b_off[it] >= 0) {
            float4* p = reinterpret_cast<float4*>(b_hi + b_off[it]);
            *p = bf16_rne4(*p);
          }
      }
      fence_async_smem();
      mbar_arrive(full + s);
      ++done;
    };

    constexpr int D = lookahead(STAGES);
    for (int d = 0; d < D; ++d) {
      if (ivalid) issue();
      cp_async_commit();
    }
    while (done < issued) {
      if (ivalid) issue();
      cp_async_commit();
      cp_async_wait<D>();
      finalize();
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      // one K=8 MMA spans two K-chunks (K-major) or two 4-row K atoms (MN-major)
      constexpr uint32_t alb = A_MN ? 512u : BM * 16u, asb = A_MN ? (BM / 32) * 512u : 128u;
      constexpr uint32_t blb = B_MN ? 512u : BN * 16u, bsb = B_MN ? (BN / 32) * 512u : 128u;
      constexpr uint32_t astep = A_MN ? 2 * asb : 2 * alb, bstep = B_MN ? 2 * bsb : 2 * blb;
      constexpr uint32_t alay = A_MN ? 1u : 0u, blay = B_MN ? 1u : 0u;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int z, mt, nt;
        tile_coords(tg, t, z, mt, nt);
        const GemmView v = make_view(a, z / phases, z % phases);
        if (mt * BM >= v.M || nt * BN >= v.N) continue;
        const int nk = (v.K + BK - 1) / BK;
        for (int k_seg = 0; k_seg < nk; k_seg += KSEG, ++sc) {
          const uint32_t buf = sc & 1;
          mbar_wait(seg_empty + buf, ((sc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * BN;
          const int k_end = min(nk, k_seg + KSEG);
          for (int kb = k_seg; kb < k_end; ++kb, ++kc) {
            const int s = kc % STAGES;
            mbar_wait(full + s, (kc / STAGES) & 1);
            tc_fence_after();
            const uint32_t a_hi = smem_u32(smem + s * STAGE);
            const uint32_t b_hi = a_hi + A_BYTES;
            const uint32_t a_lo = b_hi + B_BYTES;
            const uint32_t b_lo = a_lo + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t ah = make_desc(a_hi + kk * astep, alb, asb, alay);
              const uint64_t bh = make_desc(b_hi + kk * bstep, blb, bsb, blay);
              const uint32_t acc = (kb != k_seg || kk) ? 1u : 0u;
              if (c_dbg & 4) {
              } else if (SPLIT) {
                const uint64_t al = make_desc(a_lo + kk * astep, alb, asb, alay);
                const uint64_t bl = make_desc(b_lo + kk * bstep, blb, bsb, blay);
                mma_tf32(d, al, bh, idesc, acc);  // small terms first
                mma_tf32(d, ah, bl, idesc, 1u);
                mma_tf32(d, ah, bh, idesc, 1u);
              } else {
                mma_tf32(d, ah, bh, idesc, acc);
              }
            }
            mma_commit(empty + s);  // frees the stage when these MMAs retire
          }
          mma_commit(seg_full + buf);  // segment accumulated
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== drain + epilogue =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int z, mt, nt;
      tile_coords(tg, t, z, mt, nt);
      const GemmView v = make_view(a, z / phases, z % phases);
      const int m0 = mt * BM, n0 = nt * BN;
      if (m0 >= v.M || n0 >= v.N) continue;
      const int nk = (v.K + BK - 1) / BK;
      float acc[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) acc[i] = 0.f;
      for (int k_seg = 0; k_seg < nk; k_seg += KSEG, ++sc) {
        const uint32_t buf = sc & 1;
        mbar_wait(seg_full + buf, (sc >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < BN / 16; ++c) {
          uint32_t r[16];
          if (c_dbg & 8) continue;
          tmem_ld16(tmem + lane_base + buf * BN + c * 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c * 16 + i] += __uint_as_float(r[i]);
        }
        tc_fence_before();
        mbar_arrive(seg_empty + buf);
      }
      // epilogue for row m0 + 32 q + lane
      const int row = m0 + q * 32 + lane;
      if (row < v.M) {
        float* crow;
        if (KIND == GEMM_FPROP) crow = fprop_c_ptr(g, v, row, 0);
        else if (KIND == GEMM_DGRAD) crow = dgrad_c_ptr(g, v, row, 0);
        else crow = wgrad_c_ptr(g, v, row, 0);
#pragma unroll
        for (int c4 = 0; c4 < BN; c4 += 4) {
          const int n = n0 + c4;
          if (n < v.N) {
            float o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float x = acc[c4 + u];
              if (KIND != GEMM_WGRAD) {
                const int nn = n + u;
                if (nn % a.c_pad < a.c_valid) {
                  if (v.bias) x += v.bias[nn];
                  x = act_fwd(a.act, x, a.slope);
                } else {
                  x = 0.f;
                }
              }
              o[u] = x;
            }
            float4* dst = reinterpret_cast<float4*>(crow + n);
            if (KIND == GEMM_WGRAD && a.accumulate) {
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
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  }
  return n;
}

template <int KIND, int BN, int MODE>
cudaError_t launch_bn(const GemmArgs& a, cudaStream_t st) {
  constexpr int smem = smem_bytes(BN, MODE == MATH_TF32X3);
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([&] {
    return cudaFuncSetAttribute(gemm_tc_kernel<KIND, BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  if (ce != cudaSuccess) return ce;
  TileGrid tg{(gemm_n(a) + BN - 1) / BN, (gemm_max_m(a) + BM - 1) / BM, a.L * gemm_phases(a)};
  if (tg.total() == 0) return cudaSuccess;
  const int grid = std::min(tg.total(), sm_count());
  gemm_tc_kernel<KIND, BN, MODE><<<grid, NTHREADS, smem, st>>>(a, tg);
  return launched();
}

template <int KIND, int MODE>
cudaError_t launch_kind(const GemmArgs& a, cudaStream_t st) {
  const int n = gemm_n(a);
  // MN-major B tiles (DGRAD / WGRAD) are built from 32-element swizzle atoms
  if (KIND == GEMM_FPROP && n <= 16) return launch_bn<KIND, 16, MODE>(a, st);
  if (n <= 32) return launch_bn<KIND, 32, MODE>(a, st);
  if (n <= 64) return launch_bn<KIND, 64, MODE>(a, st);
  return launch_bn<KIND, 128, MODE>(a, st);
}

template <int MODE>
cudaError_t launch_mode(const GemmArgs& a, cudaStream_t st) {
  switch (a.kind) {
    case GEMM_FPROP: return launch_kind<GEMM_FPROP, MODE>(a, st);
    case GEMM_DGRAD: return launch_kind<GEMM_DGRAD, MODE>(a, st);
    default: return launch_kind<GEMM_WGRAD, MODE>(a, st);
  }
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& a) {
  // every problem maps onto 128-row tiles; float4 operand chunks need the
  // padded channel counts (multiples of 4), which the device layout guarantees
  return a.g.CS % 4 == 0 && a.g.CG % 4 == 0;
}

cudaError_t launch_gemm_tc(const GemmArgs& a, int math, cudaStream_t st) {
  static PerDeviceOnce dbg_set;  // __constant__ memory is per device
  dbg_set.run([] {
    const char* e = std::getenv("PG_TC_DEBUG");
    int v = e ? std::atoi(e) : 0;
    return cudaMemcpyToSymbol(c_dbg, &v, sizeof(int));
  });
  if (math == MATH_TF32) return launch_mode<MATH_TF32>(a, st);
  if (math == MATH_BF16) return launch_mode<MATH_BF16>(a, st);
  return launch_mode<MATH_TF32X3>(a, st);
}

}  // namespace pg
