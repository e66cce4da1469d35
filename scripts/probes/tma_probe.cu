// TMA feed probe: every CTA streams boxes into a 6-stage ring, consumer = a
// single thread that waits for full and re-arms empty (no compute).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "/root/repo/paper_2102_10485_b200/csrc/tc_ptx.cuh"
using namespace pg;
constexpr int ST = 6;
template <int MODE>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, int iters, int box_bytes, int nbox) {
  extern __shared__ __align__(1024) uint8_t sraw[];
  uint8_t* smem = sraw + ((1024u - (smem_u32(sraw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * 32768);
  uint64_t* empty = full + ST;
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); } fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      int s = it % ST;
      mbar_wait(empty + s, ((it / ST) & 1) ^ 1);
      mbar_expect_tx(full + s, box_bytes * nbox);
      uint32_t dst = smem_u32(smem + s * 32768);
      int c = (blockIdx.x * 37 + it) % 64;
      for (int q = 0; q < nbox; ++q) {
        if (MODE == 0) tma_load_5d(dst + q * box_bytes, &tm, full + s, 0, (c % 4) * 2 + q, c / 4, blockIdx.x % 32, blockIdx.x % 100);
        else tma_load_3d(dst + q * box_bytes, &tm, full + s, 0, ((c + q) * 128) % 8192, blockIdx.x % 100);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) { int s = it % ST; mbar_wait(full + s, (it / ST) & 1); mbar_arrive(empty + s); }
  }
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fp; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  // strided conv input: [L=100][B=32][H=32][W=32][C=64] fp32
  size_t n = 100ull * 32 * 32 * 32 * 64; float* buf; cudaMalloc(&buf, n * 4); cudaMemset(buf, 0, n * 4);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * 32768 + 2048);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * 32768 + 2048);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  for (int mode = 0; mode < 2; ++mode) for (int nbox = 1; nbox <= 2; ++nbox) {
    CUtensorMap tm;
    if (mode == 0) {
      cuuint64_t gd[5] = {64, 32, 32, 32, 100}, gs[4] = {64 * 4, 32 * 64 * 4, 32 * 32 * 64 * 4, 32ull * 32 * 32 * 64 * 4};
      cuuint32_t bd[5] = {32, 32, 8, 1, 1}, es[5] = {1, 2, 2, 1, 1};  // 16 x 4 strided = 64 rows? -> 32 wide/2 * 8/2 = 64 rows
      bd[1] = 32; bd[2] = 16; // 16 x 8 = 128 rows after stride 2
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t gd[3] = {32, 8192, 100}, gs[2] = {32 * 4, 8192ull * 32 * 4};
      cuuint32_t bd[3] = {32, 128, 1}, es[3] = {1, 1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) probe<0><<<148, 64, ST * 32768 + 2048>>>(tm, iters, 16384, nbox); else probe<1><<<148, 64, ST * 32768 + 2048>>>(tm, iters, 16384, nbox);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double bytes = 148.0 * iters * 16384 * nbox;
      printf("mode %s nbox %d: %.3f ms  %.2f TB/s  (%.1f B/clk/SM at 1.9GHz) err=%s\n", mode ? "contig2D" : "strided5D", nbox, ms, bytes / ms / 1e9, bytes / ms / 1e-3 / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
