// Micro-benchmarks of the task-graph building blocks (debug exports, not part
// of the solver path): the UPDATE tile product in isolation, per CTA shape.
#include "../../../include/stbta_tools.h"
#include "../potrf_tile.cuh"
#include "mma_variants.cuh"

namespace stbta {

// Each CTA repeatedly computes C_t -= A_t B_t^T for 128x128 tiles t with K=128,
// tiles taken round-robin from `ntile` operand tiles (ld 128*ntile... packed).
template <class Cfg, int DBG = 0>
__global__ void __launch_bounds__(Cfg::NT, 1) mb_tile_kernel(const double* A, const double* B,
                                                            double* C, int ntile, int reps, int K) {
  extern __shared__ __align__(16) double smem[];
  for (int r = 0; r < reps; ++r) {
    const int t = (blockIdx.x + r * gridDim.x) % ntile;
    const double* a = A + (long long)t * 128 * K;
    const double* b = B + (long long)t * 128 * K;
    double* c = C + (long long)t * 128 * 128;
    double acc[Cfg::MF][Cfg::NF][2];
    acc_load<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0);
    tile_mma<Cfg, true, DBG>(acc, Opnd{a, K, Cfg::BM, 1}, Opnd{b, K, Cfg::BN, 1}, K, Cfg::BN, smem);
    acc_store<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0, 0, 1.0);
    __syncthreads();
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1) mb_bulk_kernel(const double* A, const double* B,
                                                            double* C, int ntile, int reps, int K) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long bars[2 * Cfg::STAGES];
  bulk_bars_init<Cfg>(bars);
  unsigned slab = 0;
  for (int r = 0; r < reps; ++r) {
    const int t = (blockIdx.x + r * gridDim.x) % ntile;
    const double* a = A + (long long)t * 128 * K;
    const double* b = B + (long long)t * 128 * K;
    double* c = C + (long long)t * 128 * 128;
    double acc[Cfg::MF][Cfg::NF][2];
    acc_load<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0);
    tile_mma_bulk<Cfg, true>(acc, a, K, b, K, K, smem, bars, slab);
    acc_store<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0, 0, 1.0);
  }
}

template <class Cfg>
static int mb_launch_bulk(const double* A, const double* B, double* C, int ntile, int reps,
                          int grid, cudaStream_t st, int K) {
  const size_t smem = Cfg::SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_bulk_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_bulk_kernel<Cfg><<<grid, Cfg::NT, smem, st>>>(A, B, C, ntile, reps, K);
  return (int)cudaGetLastError();
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT + 32, 1) mb_ws_kernel(const double* A, const double* B,
                                                               double* C, int ntile, int reps,
                                                               int K) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) unsigned long long bars[2 * Cfg::STAGES];
  ws_bars_init<Cfg>(bars);
  unsigned slab = 0;
  const bool consumer = threadIdx.x < Cfg::NT;
  for (int r = 0; r < reps; ++r) {
    const int t = (blockIdx.x + r * gridDim.x) % ntile;
    const double* a = A + (long long)t * 128 * K;
    const double* b = B + (long long)t * 128 * K;
    double* c = C + (long long)t * 128 * 128;
    double acc[Cfg::MF][Cfg::NF][2];
    if (consumer) acc_load<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0);
    tile_mma_ws<Cfg, true>(acc, a, K, b, K, K, smem, bars, slab);
    if (consumer) acc_store<Cfg>(acc, c, 128, Cfg::BM, Cfg::BN, 0, 0, 0, 1.0);
  }
}

template <class Cfg>
static int mb_launch_ws(const double* A, const double* B, double* C, int ntile, int reps, int grid,
                        cudaStream_t st, int K) {
  const size_t smem = Cfg::SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_ws_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_ws_kernel<Cfg><<<grid, Cfg::NT + 32, smem, st>>>(A, B, C, ntile, reps, K);
  return (int)cudaGetLastError();
}

template <class Cfg, int DBG = 0>
static int mb_launch(const double* A, const double* B, double* C, int ntile, int reps, int grid,
                     cudaStream_t st, int K) {
  const size_t smem = Cfg::SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_tile_kernel<Cfg, DBG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_tile_kernel<Cfg, DBG><<<grid, Cfg::NT, smem, st>>>(A, B, C, ntile, reps, K);
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

// DMMA throughput with fragment loads from shared memory (no global traffic):
// mode 0: LDS.64 per fragment (as tile_mma), 1: LDS.128 (two k-steps per
// load), 2: no loads (fragments reused).  64x32 warp tiles, 8 warps.
template <int MODE>
__global__ void __launch_bounds__(256, 1) mb_lds_kernel(int iters, double* out) {
  extern __shared__ __align__(16) double sm[];
  for (int e = threadIdx.x; e < 256 * 36; e += 256) sm[e] = 1.0 + e * 1e-9;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % 2) * 64, wn0 = (warp / 2) * 32;
  const double* as = sm;
  const double* bs = sm + 128 * 36;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double af[8], bf[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) af[i] = as[(wm0 + i * 8 + g) * 36 + t];
#pragma unroll
  for (int j = 0; j < 4; ++j) bf[j] = bs[(wn0 + j * 8 + g) * 36 + t];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 8; ks += 2) {
      double af2[8], bf2[4];
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { af[i] = as[(wm0 + i * 8 + g) * 36 + ks * 4 + t]; af2[i] = as[(wm0 + i * 8 + g) * 36 + ks * 4 + 4 + t]; }
#pragma unroll
        for (int j = 0; j < 4; ++j) { bf[j] = bs[(wn0 + j * 8 + g) * 36 + ks * 4 + t]; bf2[j] = bs[(wn0 + j * 8 + g) * 36 + ks * 4 + 4 + t]; }
      } else if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(as + (wm0 + i * 8 + g) * 36 + ks * 4 + 2 * t);
          af[i] = v.x; af2[i] = v.y;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(bs + (wn0 + j * 8 + g) * 36 + ks * 4 + 2 * t);
          bf[j] = v.x; bf2[j] = v.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) af2[i] = af[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf2[j] = bf[j];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af2[i], bf2[j]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace stbta

extern "C" int stbta_debug_lds_bench(int mode, int iters, int grid, double* out, void* stream) {
  using namespace stbta;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int smem = 256 * 36 * 8;
  cudaFuncSetAttribute(mb_lds_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mb_lds_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mb_lds_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (mode == 0) mb_lds_kernel<0><<<grid, 256, smem, st>>>(iters, out);
  else if (mode == 1) mb_lds_kernel<1><<<grid, 256, smem, st>>>(iters, out);
  else mb_lds_kernel<2><<<grid, 256, smem, st>>>(iters, out);
  return (int)cudaGetLastError();
}

extern "C" int stbta_debug_potrf_bench(const double* A, double* out, int reps, int grid,
                                       unsigned long long* ph, void* stream) {
  using namespace stbta;
  const size_t smem = PT_SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(mb_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mb_potrf_kernel<<<grid, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(A, out, reps, ph);
  return (int)cudaGetLastError();
}

extern "C" int stbta_debug_tile_bench(int variant, const double* A, const double* B, double* C,
                                      int ntile, int reps, int grid, int K, void* stream) {
  using namespace stbta;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (variant) {
    case 0: return mb_launch<MmaCfg<128, 128, 64, 32, 256>>(A, B, C, ntile, reps, grid, st, K);
    case 1: return mb_launch<MmaCfg<128, 128, 32, 32, 512>>(A, B, C, ntile, reps, grid, st, K);
    case 2: return mb_launch<MmaCfg<128, 128, 64, 32, 256, 32, 3>>(A, B, C, ntile, reps, grid, st, K);
    case 3: return mb_launch<MmaCfg<128, 128, 64, 32, 256, 32, 2>>(A, B, C, ntile, reps, grid, st, K);
    case 4: return mb_launch<MmaCfg<128, 128, 64, 32, 256, 16, 3>>(A, B, C, ntile, reps, grid, st, K);
    case 5: return mb_launch<MmaCfg<128, 128, 32, 32, 512, 32, 3>>(A, B, C, ntile, reps, grid, st, K);
    case 6: return mb_launch_bulk<MmaCfg<128, 128, 64, 32, 256, 16, 4>>(A, B, C, ntile, reps, grid, st, K);
    case 7: return mb_launch_bulk<MmaCfg<128, 128, 64, 32, 256, 32, 3>>(A, B, C, ntile, reps, grid, st, K);
    case 8: return mb_launch<MmaCfg<128, 128, 64, 32, 256, 32, 2>, 1>(A, B, C, ntile, reps, grid, st, K);
    case 9: return mb_launch<MmaCfg<128, 128, 64, 32, 256, 32, 2>, 2>(A, B, C, ntile, reps, grid, st, K);
    case 10: return mb_launch_ws<MmaCfg<128, 128, 64, 32, 256, 16, 4>>(A, B, C, ntile, reps, grid, st, K);
    case 11: return mb_launch_ws<MmaCfg<128, 128, 64, 32, 256, 32, 3>>(A, B, C, ntile, reps, grid, st, K);
    case 12: return mb_launch_ws<MmaCfg<128, 128, 64, 32, 256, 16, 6>>(A, B, C, ntile, reps, grid, st, K);
    default: return -1;
  }
}
