// Per-device / per-stream host-side caches.
//
// The reference runs one worker thread per label pair (partition.cpp:116-180)
// and the B200 design one host thread per GPU, each with its own stream; so
// nothing the launchers cache may be process-global:
//   - cudaFuncSetAttribute applies to the *current device* only -> a per-device
//     "configured" bit (PerDeviceOnce / PerDeviceMax);
//   - grow-only scratch buffers are owned per (device, stream) -> two label
//     groups stepping concurrently (same or different GPUs) never share one.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>

namespace pg {

inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// f() once per device (retried on failure); cheap lock-free check on the hot path
struct PerDeviceOnce {
  std::atomic<unsigned long long> mask{0};
  template <class F>
  cudaError_t run(F f) {
    const unsigned long long bit = 1ull << (cur_device() & 63);
    if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    const cudaError_t e = f();
    if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
};

// largest value configured so far, per device (dynamic shared-memory opt-ins of varying size)
struct PerDeviceMax {
  std::atomic<size_t> v[64] = {};
  template <class F>
  cudaError_t raise(size_t want, F f) {
    std::atomic<size_t>& cur = v[cur_device() & 63];
    if (want <= cur.load(std::memory_order_acquire)) return cudaSuccess;
    const cudaError_t e = f();
    if (e != cudaSuccess) return e;
    size_t old = cur.load();
    while (old < want && !cur.compare_exchange_weak(old, want)) {
    }
    return cudaSuccess;
  }
};

// grow-only device scratch of the current device for stream st (slot selects
// one of several independent buffers); stream-ordered users only
enum ScratchSlot : int { SCRATCH_GEMM = 0, SCRATCH_BLO = 1, SCRATCH_SLOTS = 2 };
float* stream_scratch(int slot, size_t floats, cudaStream_t st);
// frees every scratch buffer of stream st (call before destroying the stream)
void release_stream_scratch(cudaStream_t st);
// caller-owned workspace for stream st (pg_set_workspace; nullptr detaches):
// stream_scratch then carves its slots from it and never allocates
void set_stream_workspace(cudaStream_t st, void* p, size_t bytes);
// start of one GEMM call on st: resets the per-slot usage of a caller workspace
void scratch_call_begin(cudaStream_t st);

}  // namespace pg
