// Shared pieces of the TMA-fed tcgen05 engines (gemm_tma.cu: one CTA per
// tile, gemm_pair.cu: CTA pairs with cta_group::2): spatial boxes over NHWC
// maps, the stride-phase decomposition of DGRAD, fp32 tensor maps.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace pg {
namespace tmac {

struct SpatialBox {
  int TB, TH, TW;  // box extent in samples / rows / columns (product = rows of the box)
  int nb, ny, nx;  // number of boxes along each
};

struct DgPhase {
  int ry, rx, y0, x0, ny, nx, ntx;
};

PG_DEV DgPhase dg_phase(const ConvGeo& g, int phase) {
  DgPhase d;
  d.ry = phase / g.s;
  d.rx = phase % g.s;
  d.y0 = phase_origin(d.ry, g.s, g.p);
  d.x0 = phase_origin(d.rx, g.s, g.p);
  d.ny = d.y0 < g.GH ? (g.GH - d.y0 + g.s - 1) / g.s : 0;
  d.nx = d.x0 < g.GW ? (g.GW - d.x0 + g.s - 1) / g.s : 0;
  d.ntx = d.rx < g.k ? (g.k - d.rx + g.s - 1) / g.s : 0;
  return d;
}

PG_DEV float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

PG_DEV void box_origin(const SpatialBox& b, int idx, int& b0, int& i0, int& j0) {
  const int xt = idx % b.nx;
  const int r = idx / b.nx;
  const int yt = r % b.ny;
  const int bt = r / b.ny;
  b0 = bt * b.TB;
  i0 = yt * b.TH;
  j0 = xt * b.TW;
}

// ---------------------------------------------------------------- host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// fp32 tensor map over `rank` dims (innermost first); strides in floats for dims 1..rank-1
inline bool make_map(CUtensorMap* m, const float* base, int rank, const long long* dims, const long long* strides,
              const int* box, const int* estr, CUtensorMapSwizzle swz) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bd[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = static_cast<cuuint64_t>(dims[i]);
    bd[i] = static_cast<cuuint32_t>(box[i]);
    es[i] = static_cast<cuuint32_t>(estr[i]);
  }
  for (int i = 0; i + 1 < rank; ++i) gs[i] = static_cast<cuuint64_t>(strides[i]) * 4;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), gd, gs, bd, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

inline SpatialBox spatial_box(int B, int H, int W, int rows) {
  SpatialBox b;
  b.TW = std::min(pow2ceil(W), rows);
  b.TH = std::min(pow2ceil(H), rows / b.TW);
  b.TB = rows / (b.TW * b.TH);
  b.nx = (W + b.TW - 1) / b.TW;
  b.ny = (H + b.TH - 1) / b.TH;
  b.nb = (B + b.TB - 1) / b.TB;
  return b;
}

inline int sm_count_tma() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  }
  return n;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace tmac
}  // namespace pg
