// Shared device helpers for the stbta sm_100a kernels.
//
// Everything here is FP64: the BTA solver path computes in IEEE double exactly
// like the reference's numpy/LAPACK calls (SURVEY.md §8 "All arithmetic is
// IEEE FP64").  The tensor-core path on sm_100a for f64 is the warp-level
// `mma.sync ... f64` (SASS DMMA.8x8x4); tcgen05 has no f64 kind.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define STBTA_DEV __device__ __forceinline__

// Device bounds checks of the checked build (make check -> libstbta_check.so,
// -DSTBTA_CHECKS; loaded with STBTA_LIB=...): a violated invariant prints and
// traps, so an out-of-region tile address fails loudly instead of reading or
// writing a neighbour's storage.  Compiled out of the product library.
#ifdef STBTA_CHECKS
#include <cstdio>
#define STBTA_CHECK(cond)                                                              \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("stbta check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);            \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define STBTA_CHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace stbta {

// Kernel attributes (max dynamic shared memory) are per device: track, per
// call site, the devices on which they have been set.
inline int current_device_bit(unsigned long long* bit) {
  int dev = 0;
  cudaGetDevice(&dev);
  *bit = 1ull << (dev & 63);
  return dev;
}
inline bool attr_pending(const std::atomic<unsigned long long>& mask) {
  unsigned long long bit;
  current_device_bit(&bit);
  return (mask.load(std::memory_order_relaxed) & bit) == 0;
}
inline void attr_mark(std::atomic<unsigned long long>& mask) {
  unsigned long long bit;
  current_device_bit(&bit);
  mask.fetch_or(bit, std::memory_order_relaxed);
}

// Host-side count of kernel launches issued by the library (bench.py's
// gpu_launches; read with stbta_launch_count()).
void count_launch();
// Stream-ordered zero fill by an SM kernel.  cudaMemsetAsync may be carried
// out by a copy engine and then queues behind unrelated bulk host<->device
// copies of other streams (the pipelined uploads), stalling the compute
// stream; a kernel does not.
int zero_async(void* p, size_t bytes, cudaStream_t st);
// Debug profile buffer set by stbta_debug_set_profile (nullptr: disabled).
unsigned long long* debug_profile();

// ---------------------------------------------------------------- cp.async
// 8-byte element copy global->shared with zero fill when !valid.
STBTA_DEV void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
// 16-byte copy (both addresses 16-byte aligned); src_bytes in {0, 8, 16}.
STBTA_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
STBTA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
STBTA_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------- DMMA
// D(8x8) += A(8x4, row) * B(4x8, col), f64.  Fragment ownership for lane l,
// g = l>>2, t = l&3:  a = A[g][t];  b = B[t][g];  c0,c1 = C[g][2t], C[g][2t+1].
STBTA_DEV void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Deterministic warp sum (fixed butterfly order).
STBTA_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace stbta
