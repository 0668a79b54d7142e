// Debug micro-probes for tools/ (libstbta_tools.so, not the product
// library): DFMA peak, dependent-chain DMMA / DFMA latency, %globaltimer.
#include "../../../include/stbta_tools.h"
#include "../common.cuh"

namespace stbta {

__global__ void __launch_bounds__(256) dfma_probe_kernel(int iters, double* out) {
  constexpr int ACC = 8;
  double c[ACC];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// Dependent-chain latency probes: one warp, `iters` dependent DMMA / DFMA.
__global__ void dmma_latency_kernel(int iters, double* out, long long* cycles) {
  double c0 = 0.0, c1 = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) dmma884(c0, c1, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  if (c0 + c1 == 12345.678) out[0] = c0;
}
__global__ void dfma_latency_kernel(int iters, double* out, long long* cycles) {
  double c = threadIdx.x;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) c = fma(c, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  if (c == 12345.678) out[0] = c;
}

}  // namespace stbta

extern "C" {
int stbta_debug_latency(int which, int iters, double* scratch, long long* cycles, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (which == 0) stbta::dmma_latency_kernel<<<1, 32, 0, st>>>(iters, scratch, cycles);
  else stbta::dfma_latency_kernel<<<1, 32, 0, st>>>(iters, scratch, cycles);
  return (int)cudaGetLastError();
}

// blocks x 256 threads, each thread iters*8 DFMA.  FLOPs = blocks*256*iters*16.
int stbta_probe_dfma(int blocks, int iters, double* scratch, void* stream) {
  stbta::dfma_probe_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters,
                                                                                        scratch);
  return (int)cudaGetLastError();
}
}

namespace stbta {
__global__ void globaltimer_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace stbta

extern "C" int stbta_debug_globaltimer(unsigned long long* out, void* stream) {
  stbta::globaltimer_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out);
  return (int)cudaGetLastError();
}
