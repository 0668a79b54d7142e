// CTA-level FP64 DMMA tile product for the persistent task-graph kernels:
//
//   acc(BM x BN) = A(BM x K) * B(BN x K)^T        ("NT": both operands K-contiguous)
//
// Operands are row sets of BTA storage (row r at p + r*ld).  K is staged
// through a STAGES-deep cp.async ring of BK-wide slabs in shared memory
// (16-byte copies when rows are 16-byte aligned, 8-byte otherwise; rows >=
// `rows` and columns >= K are zero-filled), and every warp accumulates its
// WM x WN sub-tile as (WM/8) x (WN/8) DMMA.8x8x4 fragments.  A 4-double row
// pad makes every fragment load conflict-free (two wavefronts per 256 B).
#pragma once

#include "common.cuh"

namespace stbta {

struct Opnd {
  const double* p;
  long long ld;
  int rows;  // valid rows (rest read as zero)
  int vec;   // 16-byte copies allowed
};

template <int BM_, int BN_, int WM_, int WN_, int NT_>
struct MmaCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, NT = NT_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static_assert(WARPS_M * WARPS_N * 32 == NT, "warp layout must cover the CTA");
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int BK = 16, STAGES = 4, LDS = BK + 4;
  static constexpr int A_STAGE = BM * LDS, B_STAGE = BN * LDS;
  static constexpr int SMEM_DOUBLES = STAGES * (A_STAGE + B_STAGE);
};

template <int ROWS, int NT>
STBTA_DEV void load_slab(double* sm, const Opnd& o, int k0, int K) {
  constexpr int LDS = 16 + 4;
  const int tid = threadIdx.x;
  if (o.vec) {
    constexpr int PAIRS = ROWS * 8;
#pragma unroll
    for (int e = tid; e < PAIRS; e += NT) {
      const int r = e >> 3, c = (e & 7) * 2;
      const int gc = k0 + c;
      int bytes = 0;
      const double* src = o.p;
      if (r < o.rows && gc < K) {
        bytes = (gc + 1 < K) ? 16 : 8;
        src = o.p + (long long)r * o.ld + gc;
      }
      cp_async16(sm + r * LDS + c, src, bytes);
    }
  } else {
    constexpr int ELEMS = ROWS * 16;
#pragma unroll
    for (int e = tid; e < ELEMS; e += NT) {
      const int r = e >> 4, c = e & 15;
      const int gc = k0 + c;
      const bool ok = r < o.rows && gc < K;
      cp_async8(sm + r * LDS + c, ok ? o.p + (long long)r * o.ld + gc : o.p, ok);
    }
  }
}

// acc += A * B^T over k in [0, K).  `n_active`: warps whose first output
// column is >= n_active skip the arithmetic (triangular strips).  All threads
// of the CTA must call; smem holds Cfg::SMEM_DOUBLES doubles.  Ends with a
// __syncthreads so the caller may reuse shared memory.
template <class Cfg, bool NEG = false>
STBTA_DEV void tile_mma(double (&acc)[Cfg::MF][Cfg::NF][2], const Opnd& A, const Opnd& B, int K,
                        int n_active, double* smem) {
  constexpr int MF = Cfg::MF, NF = Cfg::NF, BK = Cfg::BK, ST = Cfg::STAGES, LDS = Cfg::LDS;
  double* As = smem;
  double* Bs = smem + ST * Cfg::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const bool active = wn0 < n_active;
  const int ktiles = (K + BK - 1) / BK;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < ktiles) {
      load_slab<Cfg::BM, Cfg::NT>(As + s * Cfg::A_STAGE, A, s * BK, K);
      load_slab<Cfg::BN, Cfg::NT>(Bs + s * Cfg::B_STAGE, B, s * BK, K);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    const int nt = kt + ST - 1;
    if (nt < ktiles) {
      load_slab<Cfg::BM, Cfg::NT>(As + (nt % ST) * Cfg::A_STAGE, A, nt * BK, K);
      load_slab<Cfg::BN, Cfg::NT>(Bs + (nt % ST) * Cfg::B_STAGE, B, nt * BK, K);
    }
    cp_async_commit();
    if (active) {
      const double* as = As + (kt % ST) * Cfg::A_STAGE;
      const double* bs = Bs + (kt % ST) * Cfg::B_STAGE;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int k = ks * 4 + tq;
        double af[MF], bf[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) af[i] = as[(wm0 + i * 8 + gq) * LDS + k];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[j] = NEG ? -bs[(wn0 + j * 8 + gq) * LDS + k] : bs[(wn0 + j * 8 + gq) * LDS + k];
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
          for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

template <class Cfg>
STBTA_DEV void acc_zero(double (&acc)[Cfg::MF][Cfg::NF][2]) {
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// acc = C[m][n] for m < rows, n < cols (and n <= m + diag when lower), else 0.
// All loads are issued before any use, so their latency overlaps.
template <class Cfg>
STBTA_DEV void acc_load(double (&acc)[Cfg::MF][Cfg::NF][2], const double* C, long long ldc,
                        int rows, int cols, int lower, int diag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i) {
    const int m = wm0 + i * 8 + gq;
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nn = wn0 + j * 8 + 2 * tq + e;
        const bool ok = m < rows && nn < cols && !(lower && nn > m + diag);
        acc[i][j][e] = ok ? __ldcg(C + (long long)m * ldc + nn) : 0.0;
      }
    }
  }
}

// Epilogue: C[m][n] (op)= acc for m < rows, n < cols, and n <= m + diag when
// lower != 0.  op: 0 -> C = alpha*acc ; 1 -> C += alpha*acc.
template <class Cfg>
STBTA_DEV void acc_store(const double (&acc)[Cfg::MF][Cfg::NF][2], double* C, long long ldc,
                         int rows, int cols, int lower, int diag, int op, double alpha) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i) {
    const int m = wm0 + i * 8 + gq;
    if (m >= rows) continue;
    double* crow = C + (long long)m * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nn = wn0 + j * 8 + 2 * tq + e;
        if (nn >= cols || (lower && nn > m + diag)) continue;
        double v = alpha * acc[i][j][e];
        if (op) v += __ldcg(crow + nn);
        crow[nn] = v;
      }
    }
  }
}

}  // namespace stbta
