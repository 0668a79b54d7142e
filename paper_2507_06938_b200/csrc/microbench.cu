// Micro-benchmarks of the task-graph building blocks (debug exports, not part
// of the solver path): the UPDATE tile product in isolation, per CTA shape.
#include "../../include/stbta.h"
#include "potrf_tile.cuh"
#include "tile_mma.cuh"

namespace stbta {

// Each CTA repeatedly computes C_t -= A_t B_t^T for 128x128 tiles t with K=128,
// tiles taken round-robin from `ntile` operand tiles (ld 128*ntile... packed).
template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1) mb_tile_kernel(const double* A, const double* B,
                                                            double* C, int ntile, int reps) {
  extern __shared__ __align__(16) double smem[];
  for (int r = 0; r < reps; ++r) {
    const int t = (blockIdx.x + r * gridDim.x) % ntile;
    const double* a = A + (long long)t * 128 * 128;
    const double* b = B + (long long)t * 128 * 128;
    double* c = C + (long long)t * 128 * 128;
    double acc[Cfg::MF][Cfg::NF][2];
    acc_load<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0);
    tile_mma<Cfg, true>(acc, Opnd{a, 128, Cfg::BM, 1}, Opnd{b, 128, Cfg::BN, 1}, 128, Cfg::BN, smem);
    acc_store<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0, 0, 1.0);
    __syncthreads();
  }
}

template <class Cfg>
static int mb_launch(const double* A, const double* B, double* C, int ntile, int reps, int grid,
                     cudaStream_t st) {
  const size_t smem = Cfg::SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_tile_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_tile_kernel<Cfg><<<grid, Cfg::NT, smem, st>>>(A, B, C, ntile, reps);
  return (int)cudaGetLastError();
}

// Each CTA factorizes + inverts the SPD tile A (128x128, row-major) `reps`
// times; ph[0..4] accumulate phase ns of CTA 0, ph[5] the total.
__global__ void __launch_bounds__(256, 1) mb_potrf_kernel(const double* A, double* out, int reps,
                                                         unsigned long long* ph) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_fail;
  __shared__ double s_ld;
  double* T = smem;
  double* WT = T + 128 * PT_LD;
  double* scratch = WT + 4 * 32 * PT_WLD;
  unsigned long long loc[4] = {0, 0, 0, 0};
  (void)WT;
  const unsigned long long t0 = pt_timer();
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < 128 * 128; e += 256) T[(e >> 7) * PT_LD + (e & 127)] = A[e];
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    potrf_tile_smem<256>(T, WT, scratch, &s_ld, &s_fail, blockIdx.x == 0 ? loc : nullptr);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) ph[k] = loc[k];
    ph[5] = pt_timer() - t0;
    out[0] = s_ld;
    out[1] = T[127 * PT_LD + 0];
  }
}

}  // namespace stbta

extern "C" int stbta_debug_potrf_bench(const double* A, double* out, int reps, int grid,
                                       unsigned long long* ph, void* stream) {
  using namespace stbta;
  const size_t smem = PT_SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_potrf_kernel<<<grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(A, out, reps, ph);
  return (int)cudaGetLastError();
}

extern "C" int stbta_debug_tile_bench(int variant, const double* A, const double* B, double* C,
                                      int ntile, int reps, int grid, void* stream) {
  using namespace stbta;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (variant) {
    case 0: return mb_launch<MmaCfg<128, 128, 64, 32, 256>>(A, B, C, ntile, reps, grid, st);
    case 1: return mb_launch<MmaCfg<128, 128, 32, 32, 512>>(A, B, C, ntile, reps, grid, st);
    case 2: return mb_launch<MmaCfg<128, 128, 64, 64, 128>>(A, B, C, ntile, reps, grid, st);
    case 3: return mb_launch<MmaCfg<128, 128, 32, 64, 256>>(A, B, C, ntile, reps, grid, st);
    default: return -1;
  }
}
