// In-CTA Cholesky factorization of one 128 x 128 diagonal tile (the panel
// task of the POBTAF task graph) and the blocked TRSM that applies it.
//
// Reference: np.linalg.cholesky of the pivot (bta.py:206, 230) restricted to
// one tile, its log-det contribution (bta.py:238-246), and the TRSM
// X := X L^-T (bta.py:213-219, scipy solve_triangular).
//
// Factorization: blocked right-looking on 32-wide sub-blocks in shared memory
// with a one-block look-ahead (see potrf_tile_smem).  Output: L (tile), the
// four W_kk^T blocks (the TRSM tasks' diagonal inverses) and sum log diag L.
#pragma once

#include "common.cuh"

namespace stbta {

constexpr int PT_LD = 129;   // row stride of the tile in shared memory
constexpr int PT_WLD = 33;   // row stride of 32x32 blocks in shared memory
constexpr int PT_SMEM_DOUBLES = 128 * PT_LD + 4 * 32 * PT_WLD + 128 + 144;

// 8x8 DMMA fragments of up to U independent output tiles, interleaved so the
// accumulator chains overlap: c[u] += sum_k A(m_u + g, k) * B(k, n_u + g').
// A(m,k) = a[m * lda + k];  B(k, n) = bt ? b[n * ldb + k] : b[k * ldb + n].
template <int U>
STBTA_DEV void frags_mma(double (&c0)[U], double (&c1)[U], const double* a, int lda,
                         const double* b, int ldb, bool bt, const int (&mt)[U], const int (&nt)[U],
                         int cnt, int K) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll 2
  for (int k = 0; k < K; k += 4) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < cnt) {
        const double av = a[(mt[u] + g) * lda + k + t];
        const double bv = bt ? b[(nt[u] + g) * ldb + k + t] : b[(k + t) * ldb + nt[u] + g];
        dmma884(c0[u], c1[u], av, bv);
      }
    }
  }
}

// SIMT 4x4 register micro-tile: acc[i][j] += sum_{k<K} A[i][k] * B(k, j) with
// A[i][k] = a[i * lda + k] and B(k, j) = BT ? b[j * ldb + k] : b[k * ldb + j].
// (FP64 FMA and DMMA throughput are within 10% of each other on B200; for
// the tiny in-tile products plain FMAs avoid the DMMA fragment latency chains.)
template <int K, bool BT>
STBTA_DEV void mma4x4(double (&acc)[4][4], const double* a, int lda, const double* b, int ldb) {
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) av[i] = a[i * lda + k];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = BT ? b[j * ldb + k] : b[k * ldb + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
  }
}

// Conflict-free SIMT product on a 32x32 output block by 64 threads: thread
// (tr, tc) = (id & 7, id >> 3) owns rows tr + 8i and cols tc + 8j, i, j < 4,
// so a warp's A loads touch 8 consecutive rows (odd row stride: distinct
// banks) and its B loads 4 distinct rows (broadcast).
// acc[i][j] = sum_k A[tr+8i][k] * B(k, tc+8j), A row-major (lda), B(k, n) =
// b[n * ldb + k] (BT) or b[k * ldb + n].
template <int K, bool BT>
STBTA_DEV void mma32_blk(double (&acc)[4][4], const double* a, int lda, const double* b, int ldb,
                         int id) {
  const int tr = id & 7, tc = id >> 3;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) av[i] = a[(tr + 8 * i) * lda + k];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = BT ? b[(tc + 8 * j) * ldb + k] : b[k * ldb + tc + 8 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
  }
}

STBTA_DEV void zero4x4(double (&acc)[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
}

// lower-triangular index -> (row, col), col <= row
STBTA_DEV void tri_decode(int t, int* r, int* c) {
  int tr = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  if ((tr + 1) * (tr + 2) / 2 <= t) ++tr;
  if (tr * (tr + 1) / 2 > t) --tr;
  *r = tr;
  *c = t - tr * (tr + 1) / 2;
}

STBTA_DEV unsigned long long pt_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Warp-level pieces of the tile Cholesky (one warp each; lane = row or column).

// 1/sqrt(d) for d > 0: hardware approximation + two Newton steps (about 1 ulp;
// avoids the library rsqrt's special-case paths, which are unrolled 32x in
// factor32 and would blow up its instruction footprint).
STBTA_DEV double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

STBTA_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// One warp's share of the tall factorization of column block kb (rows
// [k0, 128) of the 32 columns [k0, k0+32)), right-looking column by column:
//   role 0: the diagonal block, lane = row (factor; 1/L_jj to dinv, log-det)
//   role 1: a 32-row block below it, lane = row (X := X L_kk^-T, i.e. the TRSM)
//   role 2: identity rows, lane = row: the result is e_lane L_kk^-T, which is
//           row `lane` of W_kk^T -- the diagonal-block inverse for the TRSM
//           tasks, at no extra latency.
// Two pivot columns per step.  With column j (cb0) and column j+1 (cb1, not
// yet updated by j) of the diagonal block:
//   rs0 = 1/sqrt(d0), l1 = L[j+1][j] = cb0[j+1] rs0, d1 = cb1[j+1] - l1^2,
//   rs1 = 1/sqrt(d1), L[i][j] = r_i[j] rs0, L[i][j+1] = (r_i[j+1] - L[i][j] l1) rs1,
//   and the rank-2 trailing update of row i is, per column c,
//   r_i[c] -= A_i cb0[c] + B_i cb1[c],  A_i = L[i][j] rs0 - B_i l1 rs0,  B_i = L[i][j+1] rs1.
// Producer / consumer: only the diagonal warp (role 0) runs the pivot chain,
// from its own registers (shuffles), and publishes each step -- cb0, cb1 and
// the scalars rs0, rs1, l1 -- into one of two smem buffers (colbuf + 72 k,
// k = step & 1) with bar.arrive on FULL[k] (named barrier 1 + k); the other
// factor warps wait there, apply the step to their rows and release the buffer
// with bar.arrive on EMPTY[k] (3 + k), which the producer waits on before it
// refills it two steps later.  The pivot chain no longer waits for every
// warp's 30-column update; the arithmetic (and so every bit) is unchanged.
// `nthr` = 32 x factor warps.  Returns false on a non-positive pivot.
STBTA_DEV void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

STBTA_DEV bool factor_col32(double* T, int k0, int row0, int role, double* WTb, double* colbuf,
                            double* dinv, double* ld_acc, int nthr) {
  const int lane = threadIdx.x & 31;
  double r[32];
  if (role == 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = (c == lane) ? 1.0 : 0.0;
  } else {
    const double* src = T + (row0 + lane) * PT_LD + k0;
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = (role == 1 || c <= lane) ? src[c] : 0.0;
  }
  bool ok = true;
  double mydiag = 1.0;
  if (role == 0) {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const int k = (j >> 1) & 1;
      double* buf = colbuf + 72 * k;
      const double d0 = __shfl_sync(0xffffffffu, r[j], j);
      const double c01 = __shfl_sync(0xffffffffu, r[j], j + 1);
      const double d1r = __shfl_sync(0xffffffffu, r[j + 1], j + 1);
      const double rs0 = rsqrt_nr(d0);
      const double l1 = c01 * rs0;
      const double d1 = fma(-l1, l1, d1r);
      const double rs1 = rsqrt_nr(d1);
      const double lj0 = r[j] * rs0;
      const double lj1 = fma(-lj0, l1, r[j + 1]) * rs1;
      ok = ok && (d0 > 0.0) && (d1 > 0.0);
      if (lane == j) {
        dinv[j] = rs0;
        mydiag = lj0;
      }
      if (lane == j + 1) {
        dinv[j + 1] = rs1;
        mydiag = lj1;
      }
      if (j >= 4) named_bar_sync(3 + k, nthr);  // consumers are done with this buffer
      buf[lane] = r[j];
      buf[32 + lane] = r[j + 1];
      if (lane == 0) {
        buf[64] = rs0;
        buf[65] = rs1;
        buf[66] = l1;
      }
      named_bar_arrive(1 + k, nthr);
      __syncwarp();
      r[j] = lj0;
      r[j + 1] = lj1;
      const double B = lj1 * rs1;
      const double A = fma(-B, l1, lj0) * rs0;
#pragma unroll
      for (int c = j + 2; c < 32; ++c) r[c] = fma(-A, buf[c], fma(-B, buf[32 + c], r[c]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const int k = (j >> 1) & 1;
      const double* buf = colbuf + 72 * k;
      named_bar_sync(1 + k, nthr);
      const double rs0 = buf[64], rs1 = buf[65], l1 = buf[66];
      const double lj0 = r[j] * rs0;
      const double lj1 = fma(-lj0, l1, r[j + 1]) * rs1;
      r[j] = lj0;
      r[j + 1] = lj1;
      const double B = lj1 * rs1;
      const double A = fma(-B, l1, lj0) * rs0;
#pragma unroll
      for (int c = j + 2; c < 32; ++c) r[c] = fma(-A, buf[c], fma(-B, buf[32 + c], r[c]));
      if (j < 28) named_bar_arrive(3 + k, nthr);
    }
  }
  if (role == 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) WTb[lane * PT_WLD + c] = r[c];
  } else {
    double* dst = T + (row0 + lane) * PT_LD + k0;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (role == 1 || c <= lane) dst[c] = r[c];
  }
  if (role == 0) *ld_acc += log(mydiag);
  return role != 0 || __all_sync(0xffffffffu, ok);
}

// 32x32 block (br, bc) -= L_{br,kc} L_{bc,kc}^T over the 32 columns at kc, by
// two whole warps (id in [0, 64)) on the DMMA pipe: warp w owns the output
// fragments of rows 16w..16w+15 (2 x 4 fragments of 8x8), 8 k-steps of 4.
// (The SIMT form took 1.7 us per block on the panel chain.)
STBTA_DEV void upd_blk32(double* T, int br, int bc, int kc, int id) {
  const int w = id >> 5, lane = id & 31, g = lane >> 2, t = lane & 3;
  const double* A = T + (br * 32 + 16 * w) * PT_LD + kc;
  const double* B = T + bc * 32 * PT_LD + kc;
  double c0[2][4], c1[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c0[i][j] = c1[i][j] = 0.0;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) af[i] = A[(8 * i + g) * PT_LD + k + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = B[(8 * j + g) * PT_LD + k + t];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(c0[i][j], c1[i][j], af[i], bf[j]);
  }
  // the operands (column block kc) and the output (column block bc) are
  // disjoint, so the two warps need no barrier between reads and writes
  double* d = T + (br * 32 + 16 * w) * PT_LD + bc * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      d[(8 * i + g) * PT_LD + 8 * j + 2 * t] -= c0[i][j];
      d[(8 * i + g) * PT_LD + 8 * j + 2 * t + 1] -= c1[i][j];
    }
}

// Returns 0 on success, 1 when a pivot is not positive (or NaN).
// T: tile in shared memory (ld PT_LD), lower part valid on entry.
// On exit: T lower = L; WT[kb] (32 x 32, ld PT_WLD) = (W_kk)^T, i.e.
// WT[kb][c][i] = W_kk[i][c]; *logdet = sum log diag(L) (fixed order).
//
// Blocked right-looking Cholesky on 32-wide column blocks with a one-block
// look-ahead, so only the pivot chain is serial:
//   phase A (kb): warps 0..4-kb factor column block kb as one tall panel
//                 (diagonal block, the blocks below = TRSM, identity rows =
//                 W_kk^T); the other warps, in pairs, apply column block kb-1
//                 to the trailing blocks right of column block kb+1.
//   phase C (kb): column block kb+1 -= L_{.,kb} L_{kb+1,kb}^T (64 threads per
//                 32x32 block), which the next tall panel needs.
// ph (optional, thread 0): ns of {A, C}.  NT must be 256.
template <int NT>
STBTA_DEV int potrf_tile_smem(double* T, double* WT, double* scratch, double* logdet_out,
                              int* s_fail, unsigned long long* ph = nullptr) {
  static_assert(NT == 256, "potrf_tile_smem is laid out for 8 warps");
  const int tid = threadIdx.x, warp = tid >> 5;
  double* dinv = scratch;          // 128: 1 / L_ii
  double* colbuf = scratch + 128;  // 2 x 72: pivot column pair + scalars, double-buffered
  double ld_acc = 0.0;
  unsigned long long tp = (ph && tid == 0) ? pt_timer() : 0;
  auto stamp = [&](int k) {
    if (ph && tid == 0) {
      const unsigned long long tn = pt_timer();
      ph[k] += tn - tp;
      tp = tn;
    }
  };

#pragma unroll 1
  for (int kb = 0; kb < 4; ++kb) {
    const int k0 = kb * 32;
    const int nfw = 5 - kb;  // factor warps: diagonal, 3-kb row blocks, identity
    // ---- phase A
    if (warp < nfw) {
      const int role = warp == 0 ? 0 : (warp == nfw - 1 ? 2 : 1);
      if (!factor_col32(T, k0, k0 + 32 * warp, role, WT + kb * 32 * PT_WLD, colbuf, dinv + k0,
                        &ld_acc, 32 * nfw) &&
          tid == 0)
        *s_fail = 1;
    } else if (kb > 0) {
      // blocks (br, bc), kb+1 <= bc <= br < 4, -= L_{br,kb-1} L_{bc,kb-1}^T
      const int grp = (warp - nfw) >> 1, ngrp = (8 - nfw) >> 1;
      const int id = tid - 32 * nfw - 64 * grp;
      if (grp < ngrp) {
        int idx = 0;
#pragma unroll 1
        for (int bc = kb + 1; bc < 4; ++bc)
#pragma unroll 1
          for (int br = bc; br < 4; ++br)
            if (idx++ % ngrp == grp) upd_blk32(T, br, bc, k0 - 32, id);
      }
    }
    __syncthreads();
    stamp(0);
    if (*s_fail) return 1;
    if (kb == 3) break;
    // ---- phase C: blocks (br, kb+1), br = kb+1..3, from column block kb
    {
      const int blk = tid >> 6, id = tid & 63;
      if (blk < 3 - kb) upd_blk32(T, kb + 1 + blk, kb + 1, k0, id);
    }
    __syncthreads();
    stamp(1);
  }
  if (warp == 0) {
    const double s = warp_sum(ld_acc);
    if ((tid & 31) == 0) *logdet_out = s;
  }
  __syncthreads();
  return 0;
}

// Blocked TRSM of one row strip against a factored diagonal tile:
//   X (32 x w, in shared memory, ld XLD) := X L^-T
// with L's strictly-lower 32-blocks in Ls (ld PT_LD) and the diagonal block
// inverses as WT[kb][c][i] = W_kk[i][c] (ld PT_WLD).  Right-looking over the
// 32-column blocks; zero rows stay zero.
template <int NT, int XLD, int LLD = PT_LD>
STBTA_DEV void trsm_strip_smem(double* X, const double* Ls, const double* WT, int w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int NW = NT / 32;
  const int nkb = (w + 31) / 32;
#pragma unroll 1
  for (int kb = 0; kb < nkb; ++kb) {
    // Z_kb = X_kb W_kk^T : 16 output fragments (32 x 32)
    {
      constexpr int U = 16 / NW;
      int mt[U], nt[U];
      double c0[U], c1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tix = warp + u * NW;
        mt[u] = (tix >> 2) * 8;
        nt[u] = (tix & 3) * 8;
        c0[u] = c1[u] = 0.0;
      }
      frags_mma<U>(c0, c1, X + kb * 32, XLD, WT + kb * 32 * PT_WLD, PT_WLD, false, mt, nt, U, 32);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double* d = X + (mt[u] + g) * XLD + kb * 32 + nt[u] + 2 * t;
        d[0] = c0[u];
        d[1] = c1[u];
      }
    }
    __syncthreads();
    // X_jb -= Z_kb L_{jb,kb}^T for jb > kb
    const int njb = nkb - 1 - kb;
    if (njb > 0) {
      constexpr int U = 48 / NW;
      int mt[U], nt[U];
      double c0[U], c1[U];
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tix = warp + u * NW;  // tix = (jb-kb-1)*16 + (m*4 + n)
        mt[u] = ((tix & 15) >> 2) * 8;
        nt[u] = (kb + 1 + (tix >> 4)) * 32 + (tix & 3) * 8;  // output column in the tile
        c0[u] = c1[u] = 0.0;
        if (tix < njb * 16) cnt = u + 1;
      }
      // B(k, n) = L[n][kb*32 + k]
      frags_mma<U>(c0, c1, X + kb * 32, XLD, Ls + kb * 32, LLD, true, mt, nt, cnt, 32);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < cnt) {
          double* d = X + (mt[u] + g) * XLD + nt[u] + 2 * t;
          d[0] -= c0[u];
          d[1] -= c1[u];
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// In-CTA inversion of a factored lower 128x128 tile (identity-padded) held in
// smem[0 .. 128*INV_LD): W = L^-1.  Warp kb inverts the 32x32 diagonal block
// kb (one column per lane); the off-diagonal blocks follow by diagonals,
// W_ij = -W_ii sum_{k=j}^{i-1} L_ik W_kj (SIMT 32x32 block products).
// Layout after return: L lower unchanged, W_ij^T (i > j) in the upper block
// (j, i), W_kk row-major in the Wd area.  Read with inv_tile_at().
constexpr int INV_LD = 129, BLD = 33;
constexpr int INV_SMEM_DOUBLES = 128 * INV_LD + 11 * 32 * BLD;

template <int NT>
STBTA_DEV void invert_tile_smem(double* sm) {
  double* T = sm;
  double* WT = T + 128 * INV_LD;   // W_kk^T: WT[kb][c][i] = W_kk[i][c]
  double* Wd = WT + 4 * 32 * BLD;  // W_kk row-major
  double* TS = Wd + 4 * 32 * BLD;  // scratch products, 3 blocks
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    const int k0 = warp * 32;
    double* dinv = TS + warp * 32;
    dinv[lane] = 1.0 / T[(k0 + lane) * INV_LD + k0 + lane];
    __syncwarp();
    double w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll 32
    for (int k = 0; k < 32; ++k) {
      w[k] *= dinv[k];
#pragma unroll 32
      for (int i = k + 1; i < 32; ++i) w[i] = fma(-T[(k0 + i) * INV_LD + k0 + k], w[k], w[i]);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      WT[warp * 32 * BLD + lane * BLD + i] = w[i];
      Wd[warp * 32 * BLD + i * BLD + lane] = w[i];
    }
  }
  __syncthreads();
  for (int d = 1; d < 4; ++d) {
    const int nb = 4 - d, blk = tid >> 6, id = tid & 63, tr = id & 7, tc = id >> 3;
    if (blk < nb) {  // T_j = sum_k L_ik W_kj  (i = j + d)
      const int j = blk, i = j + d;
      double acc[4][4];
      zero4x4(acc);
      for (int k = j; k < i; ++k) {
        const double* b = (k == j) ? WT + j * 32 * BLD : T + (32 * j) * INV_LD + 32 * k;
        const int ldb = (k == j) ? BLD : INV_LD;
        mma32_blk<32, true>(acc, T + (32 * i) * INV_LD + 32 * k, INV_LD, b, ldb, id);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) TS[j * 32 * BLD + (tr + 8 * a) * BLD + tc + 8 * c] = acc[a][c];
    }
    __syncthreads();
    if (blk < nb) {  // W_ij = -W_ii T_j, stored transposed into T's upper block (j, i)
      const int j = blk, i = j + d;
      double acc[4][4];
      zero4x4(acc);
      mma32_blk<32, false>(acc, Wd + i * 32 * BLD, BLD, TS + j * 32 * BLD, BLD, id);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          T[(32 * j + tc + 8 * c) * INV_LD + 32 * i + tr + 8 * a] = -acc[a][c];
    }
    __syncthreads();
  }
}

STBTA_DEV double inv_tile_at(const double* sm, int r, int c) {
  if (c > r) return 0.0;
  const double* Wd = sm + 128 * INV_LD + 4 * 32 * BLD;
  if ((r >> 5) == (c >> 5)) return Wd[(r >> 5) * 32 * BLD + (r & 31) * BLD + (c & 31)];
  return sm[c * INV_LD + r];
}

}  // namespace stbta
