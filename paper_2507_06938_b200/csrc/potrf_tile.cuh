// In-CTA Cholesky factorization of one 128 x 128 diagonal tile (the panel
// task of the POBTAF task graph) and the blocked TRSM that applies it.
//
// Reference: np.linalg.cholesky of the pivot (bta.py:206, 230) restricted to
// one tile, its log-det contribution (bta.py:238-246), and the TRSM
// X := X L^-T (bta.py:213-219, scipy solve_triangular).
//
// Factorization: blocked right-looking on 32-wide sub-blocks in shared memory.
//   kb = 0..3:  warp 0 factors L_kk in registers (one row per lane) and
//               inverts it (one column per lane, loop form) -> W_kk;
//               all warps: L_ik = A_ik W_kk^T (i > kb), then the trailing
//               update A_ij -= L_ik L_jk^T, as interleaved 8x8 DMMA fragments.
// Output: L (tile), the four W_kk^T blocks (the TRSM tasks' diagonal
// inverses) and sum log diag L.  The code is kept compact (loops, not full
// unrolling) because the persistent kernel's instruction footprint matters.
#pragma once

#include "common.cuh"

namespace stbta {

constexpr int PT_LD = 129;   // row stride of the tile in shared memory
constexpr int PT_WLD = 33;   // row stride of 32x32 blocks in shared memory
constexpr int PT_SMEM_DOUBLES = 128 * PT_LD + 4 * 32 * PT_WLD + 128;

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

// Returns 0 on success, 1 when a pivot is not positive (or NaN).
// T: tile in shared memory (ld PT_LD), lower part valid on entry.
// On exit: T lower = L; WT[kb] (32 x 32, ld PT_WLD) = (W_kk)^T, i.e.
// WT[kb][c][i] = W_kk[i][c]; *logdet = sum log diag(L) (fixed order).
// ph (optional, thread 0): ns of {factor+inverse, trsm, update}.
template <int NT>
STBTA_DEV int potrf_tile_smem(double* T, double* WT, double* scratch, double* logdet_out,
                              int* s_fail, unsigned long long* ph = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
    if (warp == 0) {
      // ---- factor the 32x32 diagonal block, lane = row (registers)
      double r[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = (c <= lane) ? T[(k0 + lane) * PT_LD + k0 + c] : 0.0;
      bool ok = true;
      double* colbuf = scratch + 32;  // 2 x 32, double-buffered column of the pivot step
#pragma unroll 32
      for (int j = 0; j < 32; ++j) {
        double* cb = colbuf + (j & 1) * 32;
        cb[lane] = r[j];  // unscaled column j (this lane's row)
        __syncwarp();
        const double d = cb[j];
        ok = ok && (d > 0.0);
        const double rs = rsqrt(d);
        const double lj = (lane == j) ? d * rs : r[j] * rs;  // L[lane][j]
        r[j] = lj;
        const double t = lj * rs;
        // entries above this lane's diagonal are never read: update them freely
#pragma unroll 32
        for (int c = j + 1; c < 32; ++c) r[c] = fma(-t, cb[c], r[c]);  // L[c][j] = cb[c] * rs
      }
      if (!ok && lane == 0) *s_fail = 1;
      stamp(3);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c <= lane) T[(k0 + lane) * PT_LD + k0 + c] = r[c];
      __syncwarp();
      const double dl = T[(k0 + lane) * PT_LD + k0 + lane];
      ld_acc += log(dl);
      scratch[lane] = 1.0 / dl;
      __syncwarp();
      // ---- W_kk = L_kk^-1, lane = column c: w[i] for i >= c (registers)
      double w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll 32
      for (int k = 0; k < 32; ++k) {
        w[k] *= scratch[k];
#pragma unroll 32
        for (int i = k + 1; i < 32; ++i) w[i] = fma(-T[(k0 + i) * PT_LD + k0 + k], w[k], w[i]);
      }
      double* wc = WT + kb * 32 * PT_WLD + lane * PT_WLD;  // WT[kb][c][i] = W[i][c]
#pragma unroll
      for (int i = 0; i < 32; ++i) wc[i] = w[i];
    }
    __syncthreads();
    stamp(0);
    if (*s_fail) return 1;
    const int rem = 96 - k0;  // rows below the diagonal block
    if (rem == 0) break;
    // ---- TRSM: L_ik = A_ik W_kk^T for rows [k0+32, 128) (32x32 blocks, 64 threads each)
    {
      const int nblk = rem / 32;
      const int blk = tid >> 6, id = tid & 63;
      double acc[4][4];
      zero4x4(acc);
      if (blk < nblk)
        mma32_blk<32, false>(acc, T + (k0 + 32 + blk * 32) * PT_LD + k0, PT_LD,
                             WT + kb * 32 * PT_WLD, PT_WLD, id);
      __syncthreads();
      if (blk < nblk) {
        const int tr = id & 7, tc = id >> 3;
        double* d = T + (k0 + 32 + blk * 32) * PT_LD + k0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) d[(tr + 8 * i) * PT_LD + tc + 8 * j] = acc[i][j];
      }
    }
    __syncthreads();
    stamp(1);
    // ---- trailing update: A_rc -= L_r L_c^T on lower 32x32 blocks (64 threads each)
    {
      const int nb = rem / 32;
      const int nblk = nb * (nb + 1) / 2;
      const double* base = T + (k0 + 32) * PT_LD + k0;
#pragma unroll 1
      for (int blk = tid >> 6; blk < nblk; blk += NT / 64) {
        int br, bc;
        tri_decode(blk, &br, &bc);
        const int id = tid & 63, tr = id & 7, tc = id >> 3;
        double acc[4][4];
        zero4x4(acc);
        mma32_blk<32, true>(acc, base + br * 32 * PT_LD, PT_LD, base + bc * 32 * PT_LD, PT_LD, id);
        double* d = T + (k0 + 32 + br * 32) * PT_LD + k0 + 32 + bc * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) d[(tr + 8 * i) * PT_LD + tc + 8 * j] -= acc[i][j];
      }
    }
    __syncthreads();
    stamp(2);
  }
  if (warp == 0) {
    const double s = warp_sum(ld_acc);
    if (lane == 0) *logdet_out = s;
  }
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
