// Library runtime: the launch counter (bench.py's gpu_launches), the
// optional POBTAF profile hook, the stream-ordered zero fill, and the FP64
// tensor-pipe peak probe -- a register-resident DMMA.8x8x4 loop with enough
// independent accumulators to saturate the pipe, bench.py's roofline
// denominator (MEASURED_PEAKS.json has no FP64 entry).
#include "../../include/stbta.h"
#include "common.cuh"

#include <atomic>

namespace stbta {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static unsigned long long* g_prof = nullptr;
unsigned long long* debug_profile() { return g_prof; }

__global__ void __launch_bounds__(256) dmma_probe_kernel(int iters, double* out) {
  constexpr int ACC = 16;
  double c0[ACC], c1[ACC];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < ACC; ++i) c0[i] = c1[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma884(c0[i], c1[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c0[i] + c1[i];
  if (s == 12345.678) out[0] = s;  // keep the loop alive
}

}  // namespace stbta

extern "C" {
long long stbta_launch_count(void) { return stbta::g_launches.load(); }
// Debug hook: see include/stbta.h.
void stbta_debug_set_profile(unsigned long long* buf) { stbta::g_prof = buf; }
// Launch blocks x 256 threads, each warp issuing iters*16 DMMA.8x8x4
// (256 FMA each).  FLOPs = blocks * 8 * iters * 16 * 512.
int stbta_probe_dmma(int blocks, int iters, double* scratch, void* stream) {
  stbta::dmma_probe_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters,
                                                                                        scratch);
  return (int)cudaGetLastError();
}
}

namespace stbta {

__global__ void zero_words_kernel(unsigned long long* p, size_t nwords, unsigned char* tail,
                                  int ntail) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) p[i] = 0ull;
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) tail[threadIdx.x] = 0;
}

int zero_async(void* p, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return 0;
  const uintptr_t u = reinterpret_cast<uintptr_t>(p);
  if (u % 8 != 0) {  // unaligned: byte kernel path through the tail (small buffers only)
    if (bytes > 256) return (int)cudaMemsetAsync(p, 0, bytes, st);
    zero_words_kernel<<<1, 256, 0, st>>>(nullptr, 0, reinterpret_cast<unsigned char*>(p), (int)bytes);
  } else {
    const size_t nw = bytes / 8;
    const int ntail = (int)(bytes % 8);
    int grid = (int)((nw + 255) / 256);
    if (grid > 1184) grid = 1184;
    if (grid < 1) grid = 1;
    zero_words_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(p), nw,
                                            reinterpret_cast<unsigned char*>(p) + nw * 8, ntail);
  }
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace stbta

