// Measured tcgen05 kind::tf32 peak of this GPU (the roofline denominator for
// the implicit-GEMM engines): every SM pair issues back-to-back
// cta_group::2 M = 256, N = 256, K = 8 MMAs on operands resident in shared
// memory (no loads, no epilogue), one commit at the end.  The same
// instruction shape and issue path as gemm_pair.cu, so the figure is the
// ceiling that engine can approach.
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace pg {

namespace {

constexpr int PEAK_SMEM = 2 * 16384 + 1024 + 64;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) tc_peak_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + 2 * 16384);
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  float* f = reinterpret_cast<float*>(smem);
  for (int i = tid; i < 2 * 4096; i += blockDim.x) f[i] = 1.0f / (1 + (i & 15));
  fence_async_smem();
  if (tid == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (tid / 32 == 0) tmem_alloc_pair(slot, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (rank == 0 && tid == 0) {
    constexpr uint32_t idesc = make_idesc(256, 256, false, false);
    const uint32_t a = smem_u32(smem), b = a + 16384;
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      mma_tf32_pair(tmem, make_desc(a + kk * 32, 16, 1024, UMMA_SW128), make_desc(b + kk * 32, 16, 1024, UMMA_SW128),
                    idesc, i > 0 ? 1u : 0u);
    }
    mma_commit_pair(done, 3);
  }
  mbar_wait(done, 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (tid / 32 == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 256);
  }
}

}  // namespace

cudaError_t tc_tf32_peak(int iters, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pairs = sms / 2;
  cudaError_t e = cudaFuncSetAttribute(tc_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PEAK_SMEM);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tc_peak_kernel<<<2 * pairs, 128, PEAK_SMEM>>>(iters / 8);  // warm-up
  cudaEventRecord(e0);
  tc_peak_kernel<<<2 * pairs, 128, PEAK_SMEM>>>(iters);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) return e;
  *tflops = (double)pairs * iters * 2.0 * 256 * 256 * 8 / (ms * 1e-3) / 1e12;
  return launched();
}

}  // namespace pg
