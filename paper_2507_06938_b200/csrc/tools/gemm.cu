// FP64 DMMA GEMM engine for sm_100a (see gemm.cuh for the contract).
//
// CTA tile BM x BN, K staged through a STAGES-deep cp.async ring in shared
// memory (8-byte element copies so any leading dimension / offset works, 16-byte
// copies when both the base and the leading dimension are 16-byte aligned).
// Each warp owns a WM x WN sub-tile held as (WM/8) x (WN/8) DMMA.8x8x4
// accumulators.  Shared tiles keep the operand's storage orientation with a
// 4-double row pad, which makes every fragment load conflict-free (two
// wavefronts per 256-byte warp load).
#include <cstdio>

#include "../../../include/stbta_tools.h"
#include "gemm.cuh"

namespace stbta {

STBTA_DEV const double* seg_row(const SegMat& s, int r, int z) {
  if (r < s.r0) return s.p0 + (long long)z * s.bs0 + (long long)r * s.ld0;
  return s.p1 + (long long)z * s.bs1 + (long long)(r - s.r0) * s.ld1;
}

STBTA_DEV double* seg_elem(const SegMat& s, int r, int c, int z) {
  if (r < s.r0) return s.p0 + (long long)z * s.bs0 + (long long)r * s.ld0 + c;
  r -= s.r0;
  if (c < s.c0) return s.p1 + (long long)z * s.bs1 + (long long)r * s.ld1 + c;
  return s.p2 + (long long)z * s.bs2 + (long long)r * s.ld2 + (c - s.c0);
}

// Copy a ROWS x COLS tile (storage orientation) starting at (row0, col0) into
// shared memory with row stride LDS.  Out-of-range elements become zero.
template <int ROWS, int COLS, int LDS, int THREADS>
STBTA_DEV void load_tile(double* sm, const SegMat& s, int row0, int col0, int nrows, int ncols,
                         int z, bool vec) {
  const int tid = threadIdx.x;
  if (vec) {
    constexpr int PAIRS = ROWS * COLS / 2;
#pragma unroll
    for (int e = tid; e < PAIRS; e += THREADS) {
      const int r = e / (COLS / 2);
      const int c = 2 * (e % (COLS / 2));
      const int gr = row0 + r, gc = col0 + c;
      int bytes = 0;
      const double* src = s.p0;
      if (gr < nrows && gc < ncols) {
        bytes = (gc + 1 < ncols) ? 16 : 8;
        src = seg_row(s, gr, z) + gc;
      }
      cp_async16(sm + r * LDS + c, src, bytes);
    }
  } else {
    constexpr int ELEMS = ROWS * COLS;
#pragma unroll
    for (int e = tid; e < ELEMS; e += THREADS) {
      const int r = e / COLS;
      const int c = e % COLS;
      const int gr = row0 + r, gc = col0 + c;
      const bool ok = gr < nrows && gc < ncols;
      const double* src = ok ? seg_row(s, gr, z) + gc : s.p0;
      cp_async8(sm + r * LDS + c, src, ok);
    }
  }
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN, int BK, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int A_ROWS = TA ? BK : BM, A_COLS = TA ? BM : BK, A_LDS = A_COLS + 4;
  static constexpr int B_ROWS = TB ? BN : BK, B_COLS = TB ? BK : BN, B_LDS = B_COLS + 4;
  static constexpr int A_STAGE = A_ROWS * A_LDS, B_STAGE = B_ROWS * B_LDS;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
};

template <bool TA, bool TB, int BM, int BN, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(GemmCfg<TA, TB, BM, BN, WM, WN, BK, STAGES>::THREADS, 1)
    dgemm_kernel(const GemmArgs g, const int tiles_m, const int tiles_n, const int vec_a,
                 const int vec_b) {
  using Cfg = GemmCfg<TA, TB, BM, BN, WM, WN, BK, STAGES>;
  constexpr int THREADS = Cfg::THREADS, MF = Cfg::MF, NF = Cfg::NF;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;

  if (g.info != nullptr && *g.info != 0) return;

  // grouped tile order (GROUP rows of tiles share their B panels in L2)
  constexpr int GROUP = 8;
  const int tile = blockIdx.x;
  const int group_tiles = GROUP * tiles_n;
  const int first_m = (tile / group_tiles) * GROUP;
  const int gm = min(tiles_m - first_m, GROUP);
  const int bm = first_m + (tile % group_tiles) % gm;
  const int bn = (tile % group_tiles) / gm;
  const int m0 = bm * BM, n0 = bn * BN;
  const int z = blockIdx.y;
  if (g.c_lower && n0 > m0 + BM - 1) return;

  int kbeg = 0, kend = g.K;
  if (g.a_tri == TRI_LOWER) kend = min(kend, m0 + BM);
  if (g.a_tri == TRI_UPPER) kbeg = max(kbeg, m0);
  if (g.b_tri == TRI_LOWER) kbeg = max(kbeg, n0);
  if (g.b_tri == TRI_UPPER) kend = min(kend, n0 + BN);
  kbeg = (kbeg / BK) * BK;
  const int ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * WM;
  const int wn0 = (warp / Cfg::WARPS_M) * WN;

  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int slot, int k) {
    double* as = As + slot * Cfg::A_STAGE;
    double* bs = Bs + slot * Cfg::B_STAGE;
    if (TA)
      load_tile<BK, BM, Cfg::A_LDS, THREADS>(as, g.A, k, m0, g.K, g.M, z, vec_a);
    else
      load_tile<BM, BK, Cfg::A_LDS, THREADS>(as, g.A, m0, k, g.M, g.K, z, vec_a);
    if (TB)
      load_tile<BN, BK, Cfg::B_LDS, THREADS>(bs, g.B, n0, k, g.N, g.K, z, vec_b);
    else
      load_tile<BK, BN, Cfg::B_LDS, THREADS>(bs, g.B, k, n0, g.K, g.N, z, vec_b);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, kbeg + s * BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nt = kt + STAGES - 1;
    if (nt < ktiles) load_stage(nt % STAGES, kbeg + nt * BK);
    cp_async_commit();

    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + tq;
      double af[MF], bf[NF];
#pragma unroll
      for (int i = 0; i < MF; ++i) {
        const int m = wm0 + i * 8 + gq;
        af[i] = TA ? as[k * Cfg::A_LDS + m] : as[m * Cfg::A_LDS + k];
      }
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int n = wn0 + j * 8 + gq;
        bf[j] = TB ? bs[n * Cfg::B_LDS + k] : bs[k * Cfg::B_LDS + n];
      }
#pragma unroll
      for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha * acc + beta * C, lower-only filter, segment routing
#pragma unroll
  for (int i = 0; i < MF; ++i) {
    const int m = m0 + wm0 + i * 8 + gq;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn0 + j * 8 + 2 * tq + e;
        if (n >= g.N || (g.c_lower && n > m)) continue;
        double* p = seg_elem(g.C, m, n, z);
        double v = g.alpha * acc[i][j][e];
        if (g.beta != 0.0) v += g.beta * *p;
        *p = v;
      }
    }
  }
}

static bool aligned16(const SegMat& s, bool two) {
  auto ok = [](const double* p, long long ld) {
    return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0);
  };
  return ok(s.p0, s.ld0) && (!two || ok(s.p1, s.ld1));
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN, int BK, int STAGES>
static int launch_cfg(const GemmArgs& g, cudaStream_t stream) {
  using Cfg = GemmCfg<TA, TB, BM, BN, WM, WN, BK, STAGES>;
  auto kern = dgemm_kernel<TA, TB, BM, BN, WM, WN, BK, STAGES>;
  static std::atomic<unsigned long long> attr_mask{0};  // per device
  if (attr_pending(attr_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return (int)e;
    attr_mark(attr_mask);
  }
  const int tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
  const bool two_a = g.A.r0 < (TA ? g.K : g.M);
  const bool two_b = g.B.r0 < (TB ? g.N : g.K);
  const int vec_a = aligned16(g.A, two_a);
  const int vec_b = aligned16(g.B, two_b);
  dim3 grid(tiles_m * tiles_n, g.batch > 0 ? g.batch : 1);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, stream>>>(g, tiles_m, tiles_n, vec_a, vec_b);
  count_launch();
  return (int)cudaGetLastError();
}

template <bool TA, bool TB>
static int launch_ops(const GemmArgs& g, cudaStream_t stream) {
  const long long big_tiles = (long long)((g.M + 127) / 128) * ((g.N + 127) / 128);
  if (big_tiles >= 120 || (g.M >= 512 && g.N >= 512))
    return launch_cfg<TA, TB, 128, 128, 64, 32, 16, 3>(g, stream);
  return launch_cfg<TA, TB, 64, 64, 32, 32, 16, 3>(g, stream);
}

int gemm_launch(const GemmArgs& g, bool ta, bool tb, cudaStream_t stream) {
  if (g.M <= 0 || g.N <= 0) return 0;
  if (ta && tb) return launch_ops<true, true>(g, stream);
  if (ta) return launch_ops<true, false>(g, stream);
  if (tb) return launch_ops<false, true>(g, stream);
  return launch_ops<false, false>(g, stream);
}

}  // namespace stbta

extern "C" int stbta_dgemm(int ta, int tb, int M, int N, int K, double alpha, const double* A,
                           long long lda, const double* B, long long ldb, double beta, double* C,
                           long long ldc, void* stream) {
  using namespace stbta;
  if (M < 0 || N < 0 || K < 0) return STBTA_EARG;
  GemmArgs gm{};
  gm.A = seg1(const_cast<double*>(A), lda);
  gm.B = seg1(const_cast<double*>(B), ldb);
  gm.C = seg1(C, ldc);
  gm.M = M; gm.N = N; gm.K = K;
  gm.alpha = alpha; gm.beta = beta;
  gm.batch = 1;
  return gemm_launch(gm, ta != 0, tb != 0, reinterpret_cast<cudaStream_t>(stream));
}
