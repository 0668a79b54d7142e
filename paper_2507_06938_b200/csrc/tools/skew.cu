// Cross-SM hand-off latency and %globaltimer offset probe (tools only).
// CTA 0 ping-pongs a flag with every other CTA k in turn (one co-resident CTA
// per SM): CTA 0 writes ping, k sees it and writes pong, CTA 0 sees pong.
// out[k*4 + {0,1,2,3}] = {ping written (CTA 0 clock), ping seen (k clock),
// pong seen (CTA 0 clock), smid of k}; round trip = [2]-[0] (one clock),
// offset of k's clock = [1] - ([0]+[2])/2.
#include <cuda_runtime.h>

#include "../../../include/stbta_tools.h"

namespace {

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__global__ void skew_kernel(int* flags, long long* out, int reps) {
  if (threadIdx.x != 0) return;
  const int k = blockIdx.x, G = gridDim.x;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (k == 0) {
    for (int j = 1; j < G; ++j)
      for (int r = 0; r < reps; ++r) {
        const int tag = j * 1000 + r + 1;
        const unsigned long long t0 = gt();
        st_rel(flags + 32 * j, tag);
        while (ld_acq(flags + 32 * j + 1) != tag) {}
        const unsigned long long t2 = gt();
        if (r == reps - 1) { out[4LL * j] = (long long)t0; out[4LL * j + 2] = (long long)t2; }
      }
    out[3] = smid;
  } else {
    for (int r = 0; r < reps; ++r) {
      const int tag = k * 1000 + r + 1;
      while (ld_acq(flags + 32 * k) != tag) {}
      const unsigned long long t1 = gt();
      st_rel(flags + 32 * k + 1, tag);
      if (r == reps - 1) { out[4LL * k + 1] = (long long)t1; out[4LL * k + 3] = smid; }
    }
  }
}

}  // namespace

extern "C" int stbta_debug_timer_skew(int reps, int* flags, long long* out, void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* args[] = {&flags, &out, &reps};
  return (int)cudaLaunchCooperativeKernel((const void*)skew_kernel, dim3(sms), dim3(32), args, 0,
                                          reinterpret_cast<cudaStream_t>(stream));
}
