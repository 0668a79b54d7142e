// POBTASI: selected inversion of a factored BTA matrix (C ABI).
//
// Reference: bta.selected_invert (pkg/src/stinla/bta.py:310-359):
//   X_tip = L_tip^-T L_tip^-1;  for i = n-1 .. 0, W = L_ii^-1:
//   X_{i+1,i} = -(X_{i+1,i+1} L_{i+1,i} + X_{a,i+1}^T L_{a,i}) W
//   X_{a,i}   = -(X_tip L_{a,i} + X_{a,i+1} L_{i+1,i}) W
//   X_{i,i}   = (W^T - X_{i+1,i}^T L_{i+1,i} - X_{a,i}^T L_{a,i}) W
//
// B200 mapping.
//  1. Every inverse W_i = L_ii^-1 (and the tip's) is computed up front, all
//     blocks at once, since they do not depend on the recursion: the 128x128
//     diagonal tiles are inverted in-CTA (potrf_tile.cuh), then the
//     off-diagonal tiles diagonal by diagonal, W_rc = -W_rr sum_k L_rk W_kc,
//     one launch per tile diagonal covering all blocks.
//  2. The recursion is then a chain of full-size FP64 DMMA tile GEMMs (one CTA
//     per 128x128 output tile, K streamed through a cp.async ring, operands in
//     either storage orientation so no transposes are materialised), with the
//     triangular structure of W used to skip the zero K-range and X_ii formed
//     on its lower tiles and mirrored.
#include <cstdlib>
#include <cstring>

#include "../../include/stbta.h"
#include "band.cuh"
#include "potrf_tile.cuh"
#include "tile_mma.cuh"
#include "tma_mma.cuh"
#include "memops.cuh"

namespace stbta {

constexpr int SI_NT = 256;
using SiCfg = MmaCfg<128, 128, 64, 32, SI_NT, 32, 2>;
constexpr int SI_SMEM_DOUBLES =
    SiCfg::SMEM_DOUBLES > INV_SMEM_DOUBLES ? SiCfg::SMEM_DOUBLES : INV_SMEM_DOUBLES;

// one product of a tile job: acc += sgn * sum_k A(m, k) B(n, k) for k in
// [kbeg, K), A(m,k) = akm ? A[k*lda + m] : A[m*lda + k] (B likewise); ktri:
// kbeg = first column of the output tile (B is lower-triangular W^T-like).
struct Prod {
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  int K, akm, bkm, ktri, arows_all;
  double sgn;
  int amap, bmap;  // tensor-map index of the operand region (-1: none)
  int ablk, bblk;  // block of the region holding the operand
};

// Tensor maps of the recursion's operand regions (persistent kernel only).
enum { SM_XD = 0, SM_LL, SM_W, SM_T1, SM_T3, SM_XL, SM_NMAP };
struct SiMaps {
  CUtensorMap m[SM_NMAP];
  int ok[SM_NMAP];
};
struct TmaCtx {
  const SiMaps* maps;
  unsigned long long* bars;
  unsigned* phase;
};

struct TileJob {
  double* C;
  long long ldc;
  int M, N;
  int init;        // 0: zero, 1: acc = C, 2: acc[m][n] = ci[n][m] (transposed init)
  const double* ci;
  long long ldci;
  double alpha;    // C = alpha * acc
  int lower;       // only tiles with tr >= tc
  int mirror;      // also write the transposed tile to (tc, tr)
  int nprod;
  Prod p[2];
};

template <class Cfg, bool AKM, bool BKM>
STBTA_DEV void run_prod(double (&acc)[Cfg::MF][Cfg::NF][2], const Prod& p, int tr, int tc,
                        int mrows, int ncols, double* smem, const TmaCtx* tc_) {
  if constexpr (Cfg::BM == 128) {
    if (tc_ != nullptr && p.amap >= 0 && p.bmap >= 0 && tc_->maps->ok[p.amap] &&
        tc_->maps->ok[p.bmap]) {
      const int kb = p.ktri ? tc * 128 : 0;
      if (kb >= p.K) return;
      if ((p.K - kb) % 32 == 0) {
        const TmaOpnd3 ta{&tc_->maps->m[p.amap], tr * 128, p.ablk};
        const TmaOpnd3 tb{&tc_->maps->m[p.bmap], tc * 128, p.bblk};
        tile_mma_tma3<Cfg, AKM, BKM>(acc, ta, tb, kb, p.K, smem, tc_->bars, *tc_->phase, mrows,
                                     ncols);
        return;
      }
    }
  }
  Opnd a{AKM ? p.A + tr * Cfg::BM : p.A + (long long)tr * Cfg::BM * p.lda, p.lda, mrows, 0};
  Opnd b{BKM ? p.B + tc * 128 : p.B + (long long)tc * 128 * p.ldb, p.ldb, ncols, 0};
  a.vec = ((uintptr_t)a.p % 16 == 0) && (a.ld % 2 == 0);
  b.vec = ((uintptr_t)b.p % 16 == 0) && (b.ld % 2 == 0);
  const int kbeg = p.ktri ? tc * 128 : 0;
  if (kbeg >= p.K) return;
  tile_mma<Cfg, false, 0, AKM, BKM>(acc, a, b, p.K, 128, smem, kbeg);
}

template <class Cfg>
STBTA_DEV void acc_neg(double (&acc)[Cfg::MF][Cfg::NF][2]) {
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = -acc[i][j][0], acc[i][j][1] = -acc[i][j][1];
}

// One output tile (BM x 128) of a job: init, signed products, store (+ mirror).
template <class Cfg>
STBTA_DEV void tile_job_body(const TileJob& j, int tr, int tc, double* smem,
                             const TmaCtx* tx = nullptr) {
  const int mrows = min(Cfg::BM, j.M - tr * Cfg::BM), ncols = min(128, j.N - tc * 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM, wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int r0 = tr * Cfg::BM, c0 = tc * 128;
  double acc[Cfg::MF][Cfg::NF][2];
  if (j.init == 1) {
    acc_load<Cfg>(acc, j.C + (long long)r0 * j.ldc + c0, j.ldc, mrows, ncols, 0, 0);
  } else if (j.init == 2) {  // acc[m][n] = ci[c0+n][r0+m]; ci lower triangular
#pragma unroll
    for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
      for (int jj = 0; jj < Cfg::NF; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = wm0 + i * 8 + gq, n = wn0 + jj * 8 + 2 * tq + e;
          acc[i][jj][e] = (m < mrows && n < ncols && c0 + n >= r0 + m)
                              ? __ldcg(j.ci + (long long)(c0 + n) * j.ldci + r0 + m)
                              : 0.0;
        }
  } else {
    acc_zero<Cfg>(acc);
  }
  for (int q = 0; q < j.nprod; ++q) {
    const Prod& p = j.p[q];
    if (p.sgn < 0) acc_neg<Cfg>(acc);
    if (p.akm && p.bkm) run_prod<Cfg, true, true>(acc, p, tr, tc, mrows, ncols, smem, tx);
    else if (p.akm) run_prod<Cfg, true, false>(acc, p, tr, tc, mrows, ncols, smem, tx);
    else if (p.bkm) run_prod<Cfg, false, true>(acc, p, tr, tc, mrows, ncols, smem, tx);
    else run_prod<Cfg, false, false>(acc, p, tr, tc, mrows, ncols, smem, tx);
    if (p.sgn < 0) acc_neg<Cfg>(acc);
  }
  acc_store<Cfg>(acc, j.C + (long long)r0 * j.ldc + c0, j.ldc, mrows, ncols, 0, 0, 0, j.alpha);
  if (j.mirror && tr != tc) {  // transposed copy to tile (tc, tr)
    double* Ct = j.C + (long long)c0 * j.ldc + r0;
#pragma unroll
    for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
      for (int jj = 0; jj < Cfg::NF; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = wm0 + i * 8 + gq, n = wn0 + jj * 8 + 2 * tq + e;
          if (m < mrows && n < ncols) Ct[(long long)n * j.ldc + m] = j.alpha * acc[i][jj][e];
        }
  }
}

// Tile order: when a product's K range depends on the output column (W's
// triangle), columns are issued heaviest first (tc = 0 has the full K), which
// packs the second wave with the light tiles (longest-processing-time order).
template <class Cfg>
__global__ void __launch_bounds__(SI_NT, 1) tile_job_kernel(TileJob j, int tiles_m, int tiles_n,
                                                           int colmajor) {
  extern __shared__ __align__(16) double smem[];
  const int t = blockIdx.x;
  int tr, tc;
  if (j.lower) {  // lower tiles, column by column: column c holds tiles_m - c tiles
    int c = 0, rem = t;
    while (rem >= tiles_m - c) {
      rem -= tiles_m - c;
      ++c;
    }
    tc = c;
    tr = c + rem;
  } else if (colmajor) {
    tc = t / tiles_m;
    tr = t % tiles_m;
  } else {
    tr = t / tiles_n;
    tc = t % tiles_n;
  }
  tile_job_body<Cfg>(j, tr, tc, smem);
}

using SiCfg32 = MmaCfg<32, 128, 32, 16, SI_NT, 16, 4>;

// ------------------------------------------------------- inverses W_i, W_tip
// Matrix z < nm: lower-triangular L at Lp(z) (ld, size), inverse written to
// Wp(z) (same ld).  z < n: diagonal block i of the factor; z == n: the tip.
struct InvSet {
  const double* L;  // factor base (diag blocks)
  double* W;        // W_all: n blocks of b x b
  const double* Lt; // tip factor (a x a)
  double* Wt;       // tip inverse (a x a)
  int n, b, a;
  double* tmp;      // per (matrix, column tile) scratch tile, 128 x 128
  int ntb;          // tiles per block dim = ceil(b / 128)
};

STBTA_DEV void inv_mat(const InvSet& s, int z, const double** L, double** W, int* ld, int* size) {
  if (z < s.n) {
    *L = s.L + (long long)z * s.b * s.b;
    *W = s.W + (long long)z * s.b * s.b;
    *ld = s.b;
    *size = s.b;
  } else {
    *L = s.Lt;
    *W = s.Wt;
    *ld = s.a;
    *size = s.a;
  }
}

// diagonal tiles: grid (ntb, nm)
__global__ void __launch_bounds__(SI_NT, 1) inv_diag_tiles_kernel(InvSet s) {
  extern __shared__ __align__(16) double sm[];
  const double* L;
  double* W;
  int ld, size;
  inv_mat(s, blockIdx.y, &L, &W, &ld, &size);
  const int t = blockIdx.x;
  if (t * 128 >= size) return;
  const int ext = min(128, size - t * 128);
  const double* Lp = L + (long long)t * 128 * ld + t * 128;
  double* Wp = W + (long long)t * 128 * ld + t * 128;
  for (int e = threadIdx.x; e < 128 * 128; e += SI_NT) {
    const int r = e >> 7, c = e & 127;
    double v;
    if (r < ext && c < ext) v = (c <= r) ? __ldg(Lp + (long long)r * ld + c) : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    sm[r * INV_LD + c] = v;
  }
  __syncthreads();
  invert_tile_smem<SI_NT>(sm);
  for (int e = threadIdx.x; e < ext * ext; e += SI_NT) {
    const int r = e / ext, c = e % ext;
    Wp[(long long)r * ld + c] = inv_tile_at(sm, r, c);
  }
}

// tile diagonal d >= 1: CTA (c, z) forms T = sum_{k=c}^{r-1} L_rk W_kc (r = c+d)
// into its scratch tile, then W_rc = -W_rr T.
__global__ void __launch_bounds__(SI_NT, 1) inv_offdiag_kernel(InvSet s, int d) {
  extern __shared__ __align__(16) double smem[];
  const double* L;
  double* W;
  int ld, size;
  const int z = blockIdx.y;
  inv_mat(s, z, &L, &W, &ld, &size);
  const int ntiles = (size + 127) / 128;
  const int c = blockIdx.x, r = c + d;
  if (r >= ntiles) return;
  const int er = min(128, size - r * 128), ec = min(128, size - c * 128);
  double* T = s.tmp + ((long long)z * s.ntb + c) * 128 * 128;
  double acc[SiCfg::MF][SiCfg::NF][2];
  acc_zero<SiCfg>(acc);
  {
    // A(m, k) = L[r*128 + m][k], k in [c*128, r*128);  B(n, k) = W[k][c*128 + n]
    Opnd A{L + (long long)r * 128 * ld, ld, er, 0};
    Opnd B{W + c * 128, ld, ec, 0};
    A.vec = ((uintptr_t)A.p % 16 == 0) && (ld % 2 == 0);
    B.vec = ((uintptr_t)B.p % 16 == 0) && (ld % 2 == 0);
    tile_mma<SiCfg, false, 0, false, true>(acc, A, B, r * 128, 128, smem, c * 128);
  }
  acc_store<SiCfg>(acc, T, 128, 128, 128, 0, 0, 0, 1.0);
  __syncthreads();
  acc_zero<SiCfg>(acc);
  {
    // A = W_rr (er x er), B(n, k) = T[k][n]
    Opnd A{W + (long long)r * 128 * ld + r * 128, ld, er, 0};
    Opnd B{T, 128, ec, 1};
    A.vec = ((uintptr_t)A.p % 16 == 0) && (ld % 2 == 0);
    tile_mma<SiCfg, false, 0, false, true>(acc, A, B, er, 128, smem, 0);
  }
  acc_store<SiCfg>(acc, W + (long long)r * 128 * ld + c * 128, ld, er, ec, 0, 0, 0, -1.0);
}

// ------------------------------------------------- persistent recursion kernel
// The whole recursion as one persistent kernel (one CTA per SM): output tiles
// of all jobs are claimed from an atomic ticket in the recursion's order, and
// each tile waits (acquire) only on the row / column stripes of earlier jobs
// it reads, so there are no launch gaps and no half-empty last waves:
//   per block i, tickets  Ta_i | T1_i | Xa_i | Xl_i | T3_i | Xii_i
//   Ta_i  = X_tip L_a,i + X_a,i+1 L_i+1,i        waits X_a,i+1 (all), X_tip (all)
//   T1_i  = X_i+1,i+1 L_i+1,i + X_a,i+1^T L_a,i  waits row+col tr of Xii_i+1, col tr of X_a,i+1
//   X_a,i = -Ta_i W_i                            waits Ta_i (all)
//   X_l,i = -T1_i W_i                            waits row tr of T1_i
//   T3_i  = W_i^T - X_l,i^T L_i+1,i - X_a,i^T L_a,i   waits col tr of X_l,i and X_a,i
//   Xii_i = T3_i W_i (lower, mirrored)           waits row tr of T3_i
// Every wait targets a strictly earlier ticket, so the schedule cannot
// deadlock.  T1/T3/Ta alternate between two buffers by block parity; the
// transitive waits above guarantee a buffer's readers have finished before
// it is rewritten two blocks later.  Rows are issued last-first so the
// (row, column) crosses of Xii that T1 of the next block needs complete early.
enum { K_TA = 0, K_T1 = 1, K_XA = 2, K_XL = 3, K_T3 = 4, K_XII = 5, K_NKIND = 6 };

struct SiParams {
  const double *Ld, *Ll, *La, *Lt;
  double *Xd, *Xl, *Xa, *Xt;
  const double *W, *Wt;
  double *T1[2], *T3[2], *Ta[2];
  int n, b, a, arrow, nstart, tip;
  int ntb;       // 128-tiles per block dimension
  int tma;       // row tiles of the a-row jobs (1 when a <= 32: 32-row tiles)
  int tnt;       // column tiles of the tip job
  int cs, cm;    // counter slot stride, column offset inside a slot
  int p0;        // tickets of the tip job
  int c_last;    // tickets of block n-1 (no sub-diagonal)
  int c_full;    // tickets of every other block
  long long total;
  int* ctr;
  unsigned long long* ticket;
  int* abortw;  // stays zero (no failure mode in the recursion)
};

struct Shape {
  int tm, tn, lower, small;
};

__host__ __device__ inline Shape kind_shape(const SiParams& P, int kind, int has_sub) {
  switch (kind) {
    case K_TA:
    case K_XA: return {P.arrow ? P.tma : 0, P.ntb, 0, P.a <= 32};
    case K_T1:
    case K_XL: return {has_sub ? P.ntb : 0, P.ntb, 0, 0};
    case K_T3: return {P.ntb, P.ntb, 0, 0};
    default: return {P.ntb, P.ntb, 1, 0};
  }
}
__host__ __device__ inline int shape_tiles(const Shape& s) {
  return s.lower ? s.tm * (s.tm + 1) / 2 : s.tm * s.tn;
}

STBTA_DEV int* ctr_slot(const SiParams& P, int i, int kind) {  // i < 0: tip job
  if (i < 0) return P.ctr;
  return P.ctr + (long long)(1 + (long long)(P.nstart - 1 - i) * K_NKIND + kind) * P.cs;
}

// Builds the job (kind, i) exactly as the per-launch recursion would.
STBTA_DEV void make_job(const SiParams& P, int kind, int i, TileJob& j) {
  const long long bb = (long long)P.b * P.b;
  const int b = P.b, a = P.a;
  const double* W = P.W + i * bb;
  const double* sub = (i < P.n - 1) ? P.Ll + i * bb : nullptr;
  const double* arr = P.arrow ? P.La + (long long)i * a * b : nullptr;
  const int par = i & 1;
  j = TileJob{};
  j.alpha = 1.0;
  auto pr = [](const double* A, long long lda, int akm, const double* B, long long ldb, int bkm,
               int K, double sgn, int ktri, int am = -1, int ab = 0, int bm = -1, int bblk = 0) {
    Prod p{};
    p.A = A; p.lda = lda; p.akm = akm; p.B = B; p.ldb = ldb; p.bkm = bkm;
    p.K = K; p.sgn = sgn; p.ktri = ktri;
    p.amap = am; p.ablk = ab; p.bmap = bm; p.bblk = bblk;
    return p;
  };
  switch (kind) {
    case K_TA:
      j.C = P.Ta[par]; j.ldc = b; j.M = a; j.N = b;
      j.p[j.nprod++] = pr(P.Xt, a, 0, arr, b, 1, a, 1.0, 0);
      if (sub) j.p[j.nprod++] = pr(P.Xa + (long long)(i + 1) * a * b, b, 0, sub, b, 1, b, 1.0, 0);
      break;
    case K_T1:
      j.C = P.T1[par]; j.ldc = b; j.M = b; j.N = b;
      j.p[j.nprod++] = pr(P.Xd + (i + 1) * bb, b, 0, sub, b, 1, b, 1.0, 0, SM_XD, i + 1, SM_LL, i);
      if (arr) j.p[j.nprod++] = pr(P.Xa + (long long)(i + 1) * a * b, b, 1, arr, b, 1, a, 1.0, 0);
      break;
    case K_XA:
      j.C = P.Xa + (long long)i * a * b; j.ldc = b; j.M = a; j.N = b; j.alpha = -1.0;
      j.p[j.nprod++] = pr(P.Ta[par], b, 0, W, b, 1, b, 1.0, 1);
      break;
    case K_XL:
      j.C = P.Xl + i * bb; j.ldc = b; j.M = b; j.N = b; j.alpha = -1.0;
      j.p[j.nprod++] = pr(P.T1[par], b, 0, W, b, 1, b, 1.0, 1, SM_T1, par, SM_W, i);
      break;
    case K_T3:
      j.C = P.T3[par]; j.ldc = b; j.M = b; j.N = b;
      j.init = 2; j.ci = W; j.ldci = b;
      if (sub) j.p[j.nprod++] = pr(P.Xl + i * bb, b, 1, sub, b, 1, b, -1.0, 0, SM_XL, i, SM_LL, i);
      if (arr) j.p[j.nprod++] = pr(P.Xa + (long long)i * a * b, b, 1, arr, b, 1, a, -1.0, 0);
      break;
    default:  // K_XII
      j.C = P.Xd + i * bb; j.ldc = b; j.M = b; j.N = b;
      j.lower = 1; j.mirror = 1;
      j.p[j.nprod++] = pr(P.T3[par], b, 0, W, b, 1, b, 1.0, 1, SM_T3, par, SM_W, i);
      break;
  }
}

// (tr, tc) of the t-th tile of a job: rows last-first, columns first-first
// (the heaviest K of a W-triangular product first within a row).
STBTA_DEV void tile_of(const Shape& s, int t, int& tr, int& tc) {
  if (s.lower) {
    int r = s.tm - 1;
    while (t > r) {
      t -= r + 1;
      --r;
    }
    tr = r;
    tc = t;
  } else {
    tr = s.tm - 1 - t / s.tn;
    tc = t % s.tn;
  }
}

STBTA_DEV void wait_all(const SiParams& P, int kind, int i, int tr) {
  // thread 0 only
  const bool sub = i < P.n - 1;
  const bool prev = i + 1 < P.nstart;  // block i+1 computed in this call
  switch (kind) {
    case K_TA:
      if (P.tip) spin_geq(ctr_slot(P, -1, 0) + 2 * P.cm, P.p0, P.abortw);
      if (sub && prev)
        spin_geq(ctr_slot(P, i + 1, K_XA) + 2 * P.cm, P.tma * P.ntb, P.abortw);
      break;
    case K_T1:
      if (prev) {
        const int* x = ctr_slot(P, i + 1, K_XII);
        spin_geq(x + tr, tr + 1, P.abortw);
        spin_geq(x + P.cm + tr, P.ntb - tr, P.abortw);
        if (P.arrow) spin_geq(ctr_slot(P, i + 1, K_XA) + P.cm + tr, P.tma, P.abortw);
      }
      break;
    case K_XA: spin_geq(ctr_slot(P, i, K_TA) + 2 * P.cm, P.tma * P.ntb, P.abortw); break;
    case K_XL: spin_geq(ctr_slot(P, i, K_T1) + tr, P.ntb, P.abortw); break;
    case K_T3:
      if (sub) spin_geq(ctr_slot(P, i, K_XL) + P.cm + tr, P.ntb, P.abortw);
      if (P.arrow) {
        spin_geq(ctr_slot(P, i, K_XA) + P.cm + tr, P.tma, P.abortw);
      }
      break;
    default: spin_geq(ctr_slot(P, i, K_T3) + tr, P.ntb, P.abortw); break;
  }
}

constexpr int SIP_SMEM_DOUBLES =
    SiCfg::SMEM_DOUBLES > TMA_SMEM_DOUBLES ? SiCfg::SMEM_DOUBLES : TMA_SMEM_DOUBLES;

__global__ void __launch_bounds__(SI_NT, 1) sinv_persistent_kernel(SiParams P,
                                                                   const __grid_constant__ SiMaps maps) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long s_tbars[TMA_NBARS];
  tma_bars_init(s_tbars);
  unsigned tphase = 0;
  const TmaCtx tx{&maps, s_tbars, &tphase};
  __shared__ TileJob s_job;
  __shared__ int s_info[4];  // kind, i, tr, tc (+ small flag in kind's high bit)
  for (;;) {
    if (threadIdx.x == 0) {
      long long t = (long long)atomicAdd(P.ticket, 1ull);
      int kind = -1, i = -1, tr = 0, tc = 0;
      Shape sh{0, 0, 0, 0};
      if (t < P.p0) {  // X_tip = W_t^T W_t
        kind = 0;
        sh = {P.tma, P.tnt, 0, P.a <= 32};
        tile_of(sh, (int)t, tr, tc);
        TileJob j{};
        j.C = P.Xt; j.ldc = P.a; j.M = P.a; j.N = P.a; j.alpha = 1.0; j.nprod = 1;
        j.p[0].A = P.Wt; j.p[0].lda = P.a; j.p[0].akm = 1;
        j.p[0].B = P.Wt; j.p[0].ldb = P.a; j.p[0].bkm = 1;
        j.p[0].K = P.a; j.p[0].sgn = 1.0;
        s_job = j;
      } else if (t < P.total) {
        t -= P.p0;
        int step;
        if (P.nstart == P.n) {
          if (t < P.c_last) step = 0;
          else { t -= P.c_last; step = 1 + (int)(t / P.c_full); t %= P.c_full; }
        } else {
          step = (int)(t / P.c_full);
          t %= P.c_full;
        }
        i = P.nstart - 1 - step;
        const int has_sub = i < P.n - 1;
        for (kind = 0; kind < K_NKIND; ++kind) {
          sh = kind_shape(P, kind, has_sub);
          const int nt = shape_tiles(sh);
          if (t < nt) break;
          t -= nt;
        }
        tile_of(sh, (int)t, tr, tc);
        wait_all(P, kind, i, tr);
        TileJob j;
        make_job(P, kind, i, j);
        s_job = j;
      } else {
        kind = -2;
      }
      s_info[0] = kind | (sh.small ? 0x100 : 0);
      s_info[1] = i;
      s_info[2] = tr;
      s_info[3] = tc;
    }
    __syncthreads();
    const int kinfo = s_info[0], i = s_info[1], tr = s_info[2], tc = s_info[3];
    if (kinfo == -2) return;
    if (kinfo & 0x100) tile_job_body<SiCfg32>(s_job, tr, tc, smem);
    else tile_job_body<SiCfg>(s_job, tr, tc, smem, &tx);
    __syncthreads();
    if (threadIdx.x == 0) {
      int* c = ctr_slot(P, i, kinfo & 0xff);
      // finished X blocks may be read by a copy engine (stbta_pobtasi_stream_out)
      if (i < 0 || (kinfo & 0xff) == K_XII) __threadfence_system();
      else __threadfence();
      atomicAdd(c + tr, 1);
      atomicAdd(c + P.cm + tc, 1);
      atomicAdd(c + 2 * P.cm, 1);
    }
  }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct PobtasiWs {
  double *Wall, *Wt, *T1[2], *T3[2], *Ta[2], *tmp;
  int* ctr;  // ticket (8 bytes) | abort word | pad | tile counters
  size_t ctr_bytes;
};

static int si_cm(int b, int a) {
  const int ntb = (b + 127) / 128;
  const int tma = a <= 32 ? 1 : (a + 127) / 128;
  const int tnt = (a + 127) / 128;
  int cm = ntb > tma ? ntb : tma;
  return cm > tnt ? cm : tnt;
}

static size_t pobtasi_ws(int n, int b, int a, char* base, PobtasiWs* o) {
  const int ntb = (b + 127) / 128;
  const int nta = a > 0 ? (a + 127) / 128 : 0;
  const int ntm = ntb > nta ? ntb : nta;
  const size_t wall = align_up((size_t)n * b * b * sizeof(double));
  const size_t wt = align_up((size_t)(a > 0 ? a * a : 1) * sizeof(double));
  const size_t bb = align_up((size_t)b * b * sizeof(double));
  const size_t ta = align_up((size_t)(a > 0 ? a : 1) * b * sizeof(double));
  const size_t tmp = align_up((size_t)(n + 1) * ntm * 128 * 128 * sizeof(double));
  const size_t ctr = align_up(16 + (size_t)(1 + 6LL * n) * (2 * si_cm(b, a) + 1) * sizeof(int));
  if (o) {
    char* p = base;
    o->Wall = reinterpret_cast<double*>(p); p += wall;
    o->Wt = reinterpret_cast<double*>(p); p += wt;
    for (int q = 0; q < 2; ++q) { o->T1[q] = reinterpret_cast<double*>(p); p += bb; }
    for (int q = 0; q < 2; ++q) { o->T3[q] = reinterpret_cast<double*>(p); p += bb; }
    for (int q = 0; q < 2; ++q) { o->Ta[q] = reinterpret_cast<double*>(p); p += ta; }
    o->tmp = reinterpret_cast<double*>(p); p += tmp;
    o->ctr = reinterpret_cast<int*>(p);
    o->ctr_bytes = ctr;
  }
  return wall + wt + 4 * bb + 2 * ta + tmp + ctr;
}

// 3D tensor maps {b columns, b rows, blocks} (row stride b doubles) of the
// recursion's b x b operand regions: row-major operands with 16 x 128 boxes,
// k-major ones with 16 x 32 boxes (tma_mma.cuh).  None when b is odd (rows not
// 16-byte aligned), the driver entry point is missing or STBTA_NO_TMA=1.
static void make_si_maps(const SiParams& P, const PobtasiWs& ws, SiMaps* mp) {
  memset(mp, 0, sizeof(*mp));
  static const bool off = [] {
    const char* v = getenv("STBTA_NO_TMA");
    return v && v[0] == '1';
  }();
  TensorMapEncodeFn enc = tensor_map_encode();
  const int b = P.b;
  if (off || enc == nullptr || (b % 2) != 0) return;
  const unsigned long long bbytes = (unsigned long long)b * b * sizeof(double);
  struct R {
    const double* base;
    int blocks;
    unsigned long long bstride;
    int kmajor;
  } reg[SM_NMAP] = {
      {P.Xd, P.n, bbytes, 0},
      {P.Ll, P.n - 1, bbytes, 1},
      {P.W, P.nstart, bbytes, 1},
      {P.T1[0], 2, (unsigned long long)((const char*)P.T1[1] - (const char*)P.T1[0]), 0},
      {P.T3[0], 2, (unsigned long long)((const char*)P.T3[1] - (const char*)P.T3[0]), 0},
      {P.Xl, P.n - 1, bbytes, 1},
  };
  for (int r = 0; r < SM_NMAP; ++r) {
    if (reg[r].base == nullptr || reg[r].blocks < 1 || ((uintptr_t)reg[r].base % 16) != 0 ||
        (reg[r].bstride % 16) != 0)
      continue;
    const cuuint64_t dims[3] = {(cuuint64_t)b, (cuuint64_t)b, (cuuint64_t)reg[r].blocks};
    const cuuint64_t strides[2] = {(cuuint64_t)b * sizeof(double), (cuuint64_t)reg[r].bstride};
    const cuuint32_t box[3] = {16, reg[r].kmajor ? 32u : 128u, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult e = enc(&mp->m[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                           const_cast<double*>(reg[r].base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    mp->ok[r] = (e == CUDA_SUCCESS) ? 1 : 0;
  }
}

static int sm_count() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

static int launch_job(const TileJob& j, cudaStream_t st) {
  const bool small = j.M <= 32 && !j.lower && !j.mirror;
  const int bm = small ? 32 : 128;
  const int tm = (j.M + bm - 1) / bm, tn = (j.N + 127) / 128;
  const int tiles = j.lower ? tm * (tm + 1) / 2 : tm * tn;
  if (tiles <= 0) return 0;
  int colmajor = 0;
  for (int q = 0; q < j.nprod; ++q) colmajor |= j.p[q].ktri;
  if (small) {
    tile_job_kernel<SiCfg32><<<tiles, SI_NT, SiCfg32::SMEM_DOUBLES * sizeof(double), st>>>(
        j, tm, tn, colmajor);
  } else {
    tile_job_kernel<SiCfg><<<tiles, SI_NT, SiCfg::SMEM_DOUBLES * sizeof(double), st>>>(
        j, tm, tn, colmajor);
  }
  count_launch();
  return (int)cudaGetLastError();
}

static Prod prod(const double* A, long long lda, int akm, const double* B, long long ldb, int bkm,
                 int K, double sgn, int ktri = 0) {
  Prod p{};
  p.A = A; p.lda = lda; p.akm = akm;
  p.B = B; p.ldb = ldb; p.bkm = bkm;
  p.K = K; p.sgn = sgn; p.ktri = ktri;
  p.arows_all = 0;
  return p;
}

static TileJob job(double* C, long long ldc, int M, int N, double alpha) {
  TileJob j{};
  j.C = C; j.ldc = ldc; j.M = M; j.N = N; j.alpha = alpha;
  return j;
}

// ------------------------------------------------ W-based solve (POBTAS)
// With the block inverses W_t = L_tt^-1 at hand (the selected inversion's
// pre-pass), the block triangular solves need no tile chain:
//   forward   y_t = W_t (r_t - L_{t,t-1} y_{t-1})            t = 0 .. n-1
//             y_tip = W_tip (r_tip - sum_t A_t y_t)
//   backward  x_tip = W_tip^T y_tip
//             x_t = W_t^T (y_t - L_{t+1,t}^T x_{t+1} - A_t^T x_tip)   t = n-1 .. 0
// One persistent kernel (one CTA per SM, grid-wide barriers between the
// phases) streams every block GEMV at HBM rate across all SMs: rows -> warps
// for L y / W z (coalesced rows, warp sum), columns -> threads with row
// chunks for the transposed products (coalesced, partial sums reduced in
// chunk order).  Deterministic: every sum has a fixed order.
constexpr int WS_NT = 512;
constexpr int WS_NR = 8;          // right-hand sides per launch
constexpr int WS_CHUNK = 64;      // rows per partial sum of a transposed product (default)
constexpr int WS_CHUNK_MIN = 32;  // smallest chunk the workspace is sized for

struct WsArgs {
  const double *dg, *lw, *ar, *tp;  // factor regions (row stride b)
  const double *W, *Wt;             // block inverses (lower), tip inverse
  double* x;                        // rhs / solution (dim x nrhs, row-major)
  double* z;                        // WS_NR x zld scratch (one contiguous vector per rhs)
  double* part;                     // WS_NR x pld partial sums (chunk-major per rhs)
  unsigned* bar;                    // grid barrier counter (zeroed)
  long long zld, pld;
  int n, b, a, arrow, mode, nrhs, ncols;
  int chunk, colmap;                // transposed products: rows per partial; 1 = round robin
  unsigned long long* prof;         // debug: per-phase ns (CTA 0) at prof[40 + phase]
};

STBTA_DEV unsigned long long ws_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

STBTA_DEV unsigned ld_acquire_u(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all CTAs of the (co-resident, one per SM: cooperative launch) grid
STBTA_DEV void grid_sync(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire_u(bar) < target) __nanosleep(20);
  }
  __syncthreads();
}

// s[c] += sum_{j < len} row[j] * v[j * sj + c * sc], lane-strided, U row loads
// in flight per lane (factor / W rows are read-only for the whole launch).
template <int NRC, int U>
STBTA_DEV void row_dot(const double* __restrict__ row, int len, const double* v, long long sj,
                       long long sc, int nc, int lane, double (&s)[NRC]) {
  for (int j0 = lane; j0 < len; j0 += 32 * U) {
    double m[U];
#pragma unroll
    for (int u = 0; u < U; ++u) m[u] = (j0 + 32 * u < len) ? __ldg(row + j0 + 32 * u) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + 32 * u;
      if (j < len) {
#pragma unroll
        for (int c = 0; c < NRC; ++c)
          if (c < nc) s[c] = fma(m[u], v[j * sj + c * sc], s[c]);
      }
    }
  }
}

// s[c] += sum_{i0 <= i < i1} M[i * ld + j] * v[i * sj + c * sc]: one column, U loads in flight
template <int NRC, int U>
STBTA_DEV void col_dot(const double* __restrict__ M, long long ld, int j, int i0, int i1,
                       const double* v, long long sj, long long sc, int nc, double (&s)[NRC]) {
  for (int i = i0; i < i1; i += U) {
    double m[U];
#pragma unroll
    for (int u = 0; u < U; ++u) m[u] = (i + u < i1) ? __ldg(M + (long long)(i + u) * ld + j) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u < i1) {
#pragma unroll
        for (int c = 0; c < NRC; ++c)
          if (c < nc) s[c] = fma(m[u], v[(i + u) * sj + c * sc], s[c]);
      }
    }
  }
}

// sum_{ch0 <= ch < ch1} pc[ch * b + j] in chunk order, 16 loads in flight
STBTA_DEV double sum_chunks(const double* pc, long long b, int j, int ch0, int ch1) {
  double acc = 0.0;
  for (int ch = ch0; ch < ch1; ch += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = (ch + u < ch1) ? pc[(long long)(ch + u) * b + j] : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += v[u];
  }
  return acc;
}

template <int NRC, int U, int UC>
__global__ void __launch_bounds__(WS_NT, 1) wsolve_kernel(WsArgs p) {
  const int tid = threadIdx.x, lane = tid & 31;
  // warp-level work items (a row, or 32 columns of one row chunk) go round
  // robin over the CTAs (item = blockIdx + grid * k), so triangular row
  // lengths and the W^T chunks' triangle spread evenly over the SMs
  const int nwarp = gridDim.x * (WS_NT / 32);
  const int gw = blockIdx.x + gridDim.x * (tid >> 5);
  const long long b = p.b, bb = b * b;
  const int a = p.a, n = p.n, ldx = p.nrhs, nc = p.ncols;
  const long long tipr = (long long)n * b;  // first tip row of x
  const long long zld = p.zld, pld = p.pld;
  const int njb = (p.b + 31) / 32;
  unsigned target = 0;
  const int CH = p.chunk;
  const int nch = (p.b + CH - 1) / CH;
  // column work item k -> (chunk, column j) of this lane, or j = b when idle
  const int ncw = p.colmap ? nch * njb : (nch * (int)b + WS_NT - 1) / WS_NT * (WS_NT / 32);
  double* const z = p.z;
  double* const part = p.part;
  int nwt = 0;  // W^T items on / below the diagonal
  for (int ch = 0; ch < nch; ++ch) nwt += min(njb, (ch * CH + CH + 31) / 32);
  unsigned long long tl = (p.prof && blockIdx.x == 0 && tid == 0) ? ws_timer() : 0;
#define WS_SYNC(k)                                                \
  do {                                                            \
    grid_sync(p.bar, target);                                     \
    if (p.prof && blockIdx.x == 0 && tid == 0) {                  \
      const unsigned long long now_ = ws_timer();                 \
      p.prof[40 + (k)] += now_ - tl;                              \
      tl = now_;                                                  \
    }                                                             \
  } while (0)

  if (p.mode != 2) {  // ------------------------------------------ forward
    for (int t = 0; t < n; ++t) {
      // z = r_t - L_{t,t-1} y_{t-1}
      for (int i = gw; i < b; i += nwarp) {
        double s[NRC];
#pragma unroll
        for (int c = 0; c < NRC; ++c) s[c] = 0.0;
        if (t > 0)
          row_dot<NRC, U>(p.lw + (long long)(t - 1) * bb + (long long)i * b, (int)b,
                          p.x + (long long)(t - 1) * b * ldx, ldx, 1, nc, lane, s);
#pragma unroll
        for (int c = 0; c < NRC; ++c) {
          const double v = warp_sum(s[c]);
          if (lane == 0 && c < nc) z[c * zld + i] = p.x[((long long)t * b + i) * ldx + c] - v;
        }
      }
      WS_SYNC(0);
      // y_t = W_t z (lower triangle of W_t)
      for (int i = gw; i < b; i += nwarp) {
        double s[NRC];
#pragma unroll
        for (int c = 0; c < NRC; ++c) s[c] = 0.0;
        row_dot<NRC, U>(p.W + (long long)t * bb + (long long)i * b, i + 1, z, 1, zld, nc, lane, s);
#pragma unroll
        for (int c = 0; c < NRC; ++c) {
          const double v = warp_sum(s[c]);
          if (lane == 0 && c < nc) p.x[((long long)t * b + i) * ldx + c] = v;
        }
      }
      WS_SYNC(1);
    }
    if (a > 0) {
      // arrow partials part[c][t * a + r] = A_t[r] . y_t (warp per (t, r)), then the tip on CTA 0
      if (p.arrow) {
        for (int w = gw; w < n * a; w += nwarp) {
          const int t = w / a, r = w % a;
          double s[NRC];
#pragma unroll
          for (int c = 0; c < NRC; ++c) s[c] = 0.0;
          row_dot<NRC, U>(p.ar + (long long)t * a * b + (long long)r * b, (int)b,
                          p.x + (long long)t * b * ldx, ldx, 1, nc, lane, s);
#pragma unroll
          for (int c = 0; c < NRC; ++c) {
            const double v = warp_sum(s[c]);
            if (lane == 0 && c < nc) part[c * pld + w] = v;
          }
        }
        WS_SYNC(2);
      }
      if (blockIdx.x == 0) {  // y_tip = W_tip (r_tip - sum_t part[t]): CTA 0, warp per tip row
        const int wc = tid >> 5;
        for (int r = wc; r < a; r += WS_NT / 32)
          for (int c = 0; c < nc; ++c) {
            double acc = 0.0;
            if (p.arrow)
              for (int t = lane; t < n; t += 32) acc += part[c * pld + (long long)t * a + r];
            acc = warp_sum(acc);
            if (lane == 0) z[c * zld + r] = p.x[(tipr + r) * ldx + c] - acc;
          }
        __syncthreads();
        for (int r = wc; r < a; r += WS_NT / 32)
          for (int c = 0; c < nc; ++c) {
            double acc = 0.0;
            for (int q = lane; q <= r; q += 32) acc = fma(p.Wt[(long long)r * a + q], z[c * zld + q], acc);
            acc = warp_sum(acc);
            if (lane == 0) p.x[(tipr + r) * ldx + c] = acc;
          }
      }
      WS_SYNC(3);
    }
  }
  if (p.mode == 1) return;
  // -------------------------------------------------------------- backward
  if (a > 0) {  // x_tip = W_tip^T y_tip: CTA 0, warp per tip row
    if (blockIdx.x == 0) {
      const int wc = tid >> 5;
      for (int q = tid; q < a; q += WS_NT)
        for (int c = 0; c < nc; ++c) z[c * zld + q] = p.x[(tipr + q) * ldx + c];
      __syncthreads();
      for (int r = wc; r < a; r += WS_NT / 32)
        for (int c = 0; c < nc; ++c) {
          double acc = 0.0;
          for (int q = r + lane; q < a; q += 32) acc = fma(p.Wt[(long long)q * a + r], z[c * zld + q], acc);
          acc = warp_sum(acc);
          if (lane == 0) p.x[(tipr + r) * ldx + c] = acc;
        }
    }
    WS_SYNC(4);
  }
  const int gt = blockIdx.x * WS_NT + tid;
  for (int t = n - 1; t >= 0; --t) {
    // partials of L_{t+1,t}^T x_{t+1}: item (row chunk, 32 columns)
    if (t < n - 1) {
      const double* L = p.lw + (long long)t * bb;  // block (t+1, t): rows of t+1, cols of t
      const double* xn = p.x + (long long)(t + 1) * b * ldx;
      for (int k = p.colmap ? gw : gt / 32; k < ncw; k += nwarp) {
        int ch, j;
        if (p.colmap) {
          ch = k / njb;
          j = (k % njb) * 32 + lane;
        } else {
          const int job = k * 32 + lane;
          ch = job / (int)b;
          j = job % (int)b;
          if (ch >= nch) continue;
        }
        if (j >= b) continue;
        double s[NRC];
#pragma unroll
        for (int c = 0; c < NRC; ++c) s[c] = 0.0;
        col_dot<NRC, UC>(L, b, j, ch * CH, min((int)b, ch * CH + CH), xn, ldx, 1, nc, s);
#pragma unroll
        for (int c = 0; c < NRC; ++c)
          if (c < nc) part[c * pld + (long long)ch * b + j] = s[c];
      }
      WS_SYNC(5);
    }
    // z = y_t - sum_chunks part - A_t^T x_tip (32-column items round robin over the CTAs)
    for (int k = gw; k < njb; k += nwarp) {
      const int j = k * 32 + lane;
      if (j >= b) continue;
      double s[NRC];
#pragma unroll
      for (int c = 0; c < NRC; ++c) s[c] = (c < nc) ? p.x[((long long)t * b + j) * ldx + c] : 0.0;
      if (t < n - 1)
#pragma unroll
        for (int c = 0; c < NRC; ++c)
          if (c < nc) s[c] -= sum_chunks(part + c * pld, b, j, 0, nch);
      if (p.arrow)
        for (int r = 0; r < a; ++r) {
          const double m = p.ar[(long long)t * a * b + (long long)r * b + j];
#pragma unroll
          for (int c = 0; c < NRC; ++c)
            if (c < nc) s[c] = fma(-m, p.x[(tipr + r) * ldx + c], s[c]);
        }
#pragma unroll
      for (int c = 0; c < NRC; ++c)
        if (c < nc) z[c * zld + j] = s[c];
    }
    WS_SYNC(6);
    // partials of W_t^T z: x_t[j] = sum_{i >= j} W_t[i][j] z[i]
    {
      // only the items on / below the diagonal (chunk ch: column blocks
      // jb < nact(ch)), enumerated densely so they spread evenly
      const double* Wb = p.W + (long long)t * bb;
      for (int k = gw; k < nwt; k += nwarp) {
        int ch = 0, r = k;
        while (r >= min(njb, (ch * CH + CH + 31) / 32)) r -= min(njb, (ch * CH + CH + 31) / 32), ++ch;
        const int j = r * 32 + lane;
        if (j >= b || ch * CH + CH <= j) continue;  // above the diagonal: no partial
        double s[NRC];
#pragma unroll
        for (int c = 0; c < NRC; ++c) s[c] = 0.0;
        col_dot<NRC, UC>(Wb, b, j, max(ch * CH, j), min((int)b, ch * CH + CH), z, 1, zld, nc, s);
#pragma unroll
        for (int c = 0; c < NRC; ++c)
          if (c < nc) part[c * pld + (long long)ch * b + j] = s[c];
      }
    }
    WS_SYNC(7);
    for (int k = gw; k < njb; k += nwarp) {
      const int j = k * 32 + lane;
      if (j >= b) continue;
      double s[NRC];
#pragma unroll
      for (int c = 0; c < NRC; ++c) s[c] = 0.0;
#pragma unroll
      for (int c = 0; c < NRC; ++c)  // chunks above j's own hold no partial
        if (c < nc) s[c] = sum_chunks(part + c * pld, b, j, j / CH, nch);
#pragma unroll
      for (int c = 0; c < NRC; ++c)
        if (c < nc) p.x[((long long)t * b + j) * ldx + c] = s[c];
    }
    WS_SYNC(8);
  }
}
#undef WS_SYNC

// workspace: barrier | z (WS_NR x zld) | part (WS_NR x pld)
static void wsolve_ld(int n, int b, int a, long long* zld, long long* pld) {
  const long long nch = (b + WS_CHUNK_MIN - 1) / WS_CHUNK_MIN;
  const long long rows = nch * b > (long long)n * a ? nch * b : (long long)n * a;
  *zld = ((b > a ? b : a) + 31) / 32 * 32;
  *pld = (rows + 31) / 32 * 32;
}

static size_t wsolve_ws_bytes(int n, int b, int a) {
  long long zld, pld;
  wsolve_ld(n, b, a, &zld, &pld);
  return 256 + (size_t)(zld + pld) * WS_NR * sizeof(double);
}

}  // namespace stbta

using namespace stbta;

extern "C" {

size_t stbta_pobtasi_workspace_bytes(int n, int b, int a) {
  if (n < 1 || b < 1 || a < 0) return 0;
  return pobtasi_ws(n, b, a, nullptr, nullptr);
}

int stbta_pobtasi(const double* factor, double* inv, int n, int b, int a, int has_arrow,
                  void* workspace, size_t workspace_bytes, void* stream) {
  if (factor == nullptr || inv == nullptr) return STBTA_EARG;
  const long long bb = (long long)b * b;
  const double* L[4] = {factor, factor + n * bb, factor + (2LL * n - 1) * bb,
                        factor + (2LL * n - 1) * bb + (long long)n * a * b};
  double* X[4] = {inv, inv + n * bb, inv + (2LL * n - 1) * bb,
                  inv + (2LL * n - 1) * bb + (long long)n * a * b};
  return stbta_pobtasi_ex(L[0], L[1], L[2], L[3], X[0], X[1], X[2], X[3], n, b, a, has_arrow, -1,
                          workspace, workspace_bytes, stream);
}

static int pobtasi_impl(const double* Ld, const double* Ll, const double* La, const double* Lt,
                        double* Xd, double* Xl, double* Xa, double* Xt, int n, int b, int a,
                        int has_arrow, int nstart, void* workspace, size_t workspace_bytes,
                        void* stream, cudaEvent_t ctr_ready, int* persistent, int w_ready = 0);

int stbta_pobtasi_ex(const double* Ld, const double* Ll, const double* La, const double* Lt,
                     double* Xd, double* Xl, double* Xa, double* Xt, int n, int b, int a,
                     int has_arrow, int nstart, void* workspace, size_t workspace_bytes,
                     void* stream) {
  return pobtasi_impl(Ld, Ll, La, Lt, Xd, Xl, Xa, Xt, n, b, a, has_arrow, nstart, workspace,
                      workspace_bytes, stream, nullptr, nullptr);
}

static int stream_out_impl(const double* factor, double* inv, double* host_out, int n, int b,
                           int a, int has_arrow, void* workspace, size_t workspace_bytes,
                           void* stream, void* copy_stream, int w_ready);

int stbta_pobtasi_stream_out(const double* factor, double* inv, double* host_out, int n, int b,
                             int a, int has_arrow, void* workspace, size_t workspace_bytes,
                             void* stream, void* copy_stream) {
  return stream_out_impl(factor, inv, host_out, n, b, a, has_arrow, workspace, workspace_bytes,
                         stream, copy_stream, 0);
}

static int stream_out_impl(const double* factor, double* inv, double* host_out, int n, int b,
                           int a, int has_arrow, void* workspace, size_t workspace_bytes,
                           void* stream, void* copy_stream, int w_ready) {
  if (factor == nullptr || inv == nullptr || host_out == nullptr || n < 1 || b < 1 || a < 0)
    return STBTA_EARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(copy_stream);
  const long long bb = (long long)b * b;
  const long long o_low = (long long)n * bb, o_arr = o_low + (long long)(n - 1) * bb;
  const long long o_tip = o_arr + (long long)n * a * b;
  cudaEvent_t ev;
  int e = (int)cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e) return e;
  int persistent = 0;
  e = pobtasi_impl(factor, factor + o_low, factor + o_arr, factor + o_tip, inv, inv + o_low,
                   inv + o_arr, inv + o_tip, n, b, a, has_arrow, -1, workspace, workspace_bytes,
                   stream, memops().ok ? ev : nullptr, &persistent, w_ready);
  if (e) {
    cudaEventDestroy(ev);
    return e;
  }
  auto d2h = [&](long long off, long long elems) {
    return (int)cudaMemcpyAsync(host_out + off, inv + off, elems * sizeof(double),
                                cudaMemcpyDeviceToHost, cs);
  };
  if (!persistent || !memops().ok) {  // whole buffer once the recursion is done
    if (!(e = (int)cudaEventRecord(ev, st)) && !(e = (int)cudaStreamWaitEvent(cs, ev, 0)))
      e = d2h(0, o_tip + (long long)a * a);
    cudaEventDestroy(ev);
    return e;
  }
  // counters of the persistent kernel (same layout as SiParams / ctr_slot)
  PobtasiWs ws;
  pobtasi_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  const int ntb = (b + 127) / 128, tma = a <= 32 ? 1 : (a + 127) / 128, tnt = (a + 127) / 128;
  const int cm = si_cm(b, a), cslot = 2 * cm + 1;
  const int* ctr = ws.ctr + 4;
  if ((e = (int)cudaStreamWaitEvent(cs, ev, 0))) return cudaEventDestroy(ev), e;
  cudaEventDestroy(ev);
  if (a > 0) {
    if ((e = memops_wait_geq(cs, ctr + 2 * cm, (unsigned)(tma * tnt)))) return e;
    if ((e = d2h(o_tip, (long long)a * a))) return e;
  }
  for (int i = n - 1; i >= 0; --i) {
    const int* c = ctr + (long long)(1 + (long long)(n - 1 - i) * K_NKIND + K_XII) * cslot;
    if ((e = memops_wait_geq(cs, c + 2 * cm, (unsigned)(ntb * (ntb + 1) / 2)))) return e;
    if ((e = d2h((long long)i * bb, bb))) return e;
    if (i < n - 1 && (e = d2h(o_low + (long long)i * bb, bb))) return e;
    if (a > 0 && (e = d2h(o_arr + (long long)i * a * b, (long long)a * b))) return e;
  }
  return 0;
}


static int prepare_w(const double* Ld, const double* Lt, int nw, int b, int a, bool tip,
                     const PobtasiWs& ws, cudaStream_t st);

int stbta_pobtasi_prepare(const double* factor, int n, int b, int a, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (factor == nullptr || workspace == nullptr || n < 1 || b < 1 || a < 0) return STBTA_EARG;
  if (workspace_bytes < stbta_pobtasi_workspace_bytes(n, b, a)) return STBTA_EWORKSPACE;
  PobtasiWs ws;
  pobtasi_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  const long long bb = (long long)b * b;
  const double* tip = factor + (2LL * n - 1) * bb + (long long)n * a * b;
  return prepare_w(factor, tip, n, b, a, true, ws, reinterpret_cast<cudaStream_t>(stream));
}

int stbta_pobtasi_prepared(const double* factor, double* inv, double* host_out, int n, int b,
                           int a, int has_arrow, void* workspace, size_t workspace_bytes,
                           void* stream, void* copy_stream) {
  if (factor == nullptr || inv == nullptr) return STBTA_EARG;
  if (host_out != nullptr)
    return stream_out_impl(factor, inv, host_out, n, b, a, has_arrow, workspace, workspace_bytes,
                           stream, copy_stream, 1);
  const long long bb = (long long)b * b;
  const long long o_low = (long long)n * bb, o_arr = o_low + (long long)(n - 1) * bb;
  const long long o_tip = o_arr + (long long)n * a * b;
  return pobtasi_impl(factor, factor + o_low, factor + o_arr, factor + o_tip, inv, inv + o_low,
                      inv + o_arr, inv + o_tip, n, b, a, has_arrow, -1, workspace,
                      workspace_bytes, stream, nullptr, nullptr, 1);
}

size_t stbta_pobtas_w_workspace_bytes(int n, int b, int a) {
  if (n < 1 || b < 1 || a < 0) return 0;
  return wsolve_ws_bytes(n, b, a);
}

int stbta_pobtas_w(const double* factor, int n, int b, int a, int has_arrow, double* rhs,
                   int nrhs, int mode, const void* si_workspace, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (factor == nullptr || rhs == nullptr || si_workspace == nullptr || workspace == nullptr ||
      n < 1 || b < 1 || a < 0 || nrhs < 1 || mode < 0 || mode > 2)
    return STBTA_EARG;
  if (workspace_bytes < wsolve_ws_bytes(n, b, a)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtasiWs si;
  pobtasi_ws(n, b, a, reinterpret_cast<char*>(const_cast<void*>(si_workspace)), &si);
  const long long bb = (long long)b * b;
  char* base = reinterpret_cast<char*>(workspace);
  WsArgs p{};
  p.dg = factor;
  p.lw = factor + (long long)n * bb;
  p.ar = p.lw + (long long)(n - 1) * bb;
  p.tp = p.ar + (long long)n * a * b;
  p.W = si.Wall;
  p.Wt = si.Wt;
  p.bar = reinterpret_cast<unsigned*>(base);
  wsolve_ld(n, b, a, &p.zld, &p.pld);
  p.z = reinterpret_cast<double*>(base + 256);
  p.part = p.z + (size_t)p.zld * WS_NR;
  p.n = n; p.b = b; p.a = a;
  p.arrow = (has_arrow && a > 0) ? 1 : 0;
  p.mode = mode;
  p.nrhs = nrhs;
  p.chunk = b <= 3072 ? WS_CHUNK_MIN : WS_CHUNK;  // measured: C2 (b 2048) 32, C3 (b 5025) 64
  p.colmap = 1;
  p.prof = debug_profile();
  int uw = 32;  // loads in flight per lane (single right-hand side)
  if (const char* v = getenv("STBTA_WS_U")) uw = atoi(v);
  if (const char* v = getenv("STBTA_WS_CHUNK")) p.chunk = atoi(v) >= WS_CHUNK_MIN ? atoi(v) : p.chunk;
  if (const char* v = getenv("STBTA_WS_COLMAP")) p.colmap = atoi(v) ? 1 : 0;
  const int grid = sm_count();
  for (int c0 = 0; c0 < nrhs; c0 += WS_NR) {
    p.x = rhs + c0;
    p.ncols = nrhs - c0 < WS_NR ? nrhs - c0 : WS_NR;
    int e = zero_async(p.bar, sizeof(unsigned), st);
    if (e) return e;
    void* args[] = {&p};
    const void* fn = (const void*)wsolve_kernel<WS_NR, 4, 4>;
    if (p.ncols == 1)
      fn = uw >= 32 ? (const void*)wsolve_kernel<1, 16, 32> : (const void*)wsolve_kernel<1, 16, 16>;
    e = (int)cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(WS_NT), args, 0, st);
    count_launch();
    if (e) return e;
  }
  return 0;
}

}  // extern "C"

// W_i = L_ii^-1 for blocks i < nw (and W_tip when `tip`) into the workspace
// (diagonal tiles in-CTA, then the off-diagonal tile diagonals).
static int prepare_w(const double* Ld, const double* Lt, int nw, int b, int a, bool tip,
                     const PobtasiWs& ws, cudaStream_t st) {
  static std::atomic<unsigned long long> attr_mask{0};  // per device
  const size_t smem = SI_SMEM_DOUBLES * sizeof(double);
  int e;
  if (attr_pending(attr_mask)) {
    if ((e = (int)cudaFuncSetAttribute(inv_diag_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = (int)cudaFuncSetAttribute(inv_offdiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    attr_mark(attr_mask);
  }
  InvSet s{};
  s.L = Ld; s.W = ws.Wall; s.Lt = Lt; s.Wt = ws.Wt;
  s.n = nw; s.b = b; s.a = a; s.tmp = ws.tmp;
  s.ntb = (b + 127) / 128;
  const int nta = (a > 0 && tip) ? (a + 127) / 128 : 0;
  const int nm = nw + ((a > 0 && tip) ? 1 : 0);
  const int ntm = s.ntb > nta ? s.ntb : nta;
  if (a > 0 && tip && (e = zero_async(ws.Wt, (size_t)a * a * sizeof(double), st))) return e;
  inv_diag_tiles_kernel<<<dim3(ntm, nm), SI_NT, smem, st>>>(s);
  count_launch();
  if ((e = (int)cudaGetLastError())) return e;
  for (int d = 1; d < ntm; ++d) {
    inv_offdiag_kernel<<<dim3(ntm - d, nm), SI_NT, smem, st>>>(s, d);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
  }
  return 0;
}

static int pobtasi_impl(const double* Ld, const double* Ll, const double* La, const double* Lt,
                        double* Xd, double* Xl, double* Xa, double* Xt, int n, int b, int a,
                        int has_arrow, int nstart, void* workspace, size_t workspace_bytes,
                        void* stream, cudaEvent_t ctr_ready, int* persistent, int w_ready) {
  if (Ld == nullptr || Xd == nullptr || n < 1 || b < 1 || a < 0 || nstart > n) return STBTA_EARG;
  if ((n > 1 && (Ll == nullptr || Xl == nullptr)) ||
      (a > 0 && (La == nullptr || Lt == nullptr || Xa == nullptr || Xt == nullptr)))
    return STBTA_EARG;
  if (workspace_bytes < stbta_pobtasi_workspace_bytes(n, b, a)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtasiWs ws;
  pobtasi_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  const long long bb = (long long)b * b;
  const bool arrow = has_arrow && a > 0;
  const bool full = nstart < 0;  // otherwise X_tip, X_{nstart..} and X_a,{nstart..} are inputs
  if (full) nstart = n;
  const size_t smem = SI_SMEM_DOUBLES * sizeof(double);
  static std::atomic<unsigned long long> attr_mask{0};  // per device
  int e;
  if (attr_pending(attr_mask)) {
    if ((e = (int)cudaFuncSetAttribute(tile_job_kernel<SiCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SiCfg::SMEM_DOUBLES * sizeof(double))))) return e;
    if ((e = (int)cudaFuncSetAttribute(tile_job_kernel<SiCfg32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SiCfg32::SMEM_DOUBLES * sizeof(double))))) return e;
    if ((e = (int)cudaFuncSetAttribute(inv_diag_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    if ((e = (int)cudaFuncSetAttribute(inv_offdiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
    attr_mark(attr_mask);
  }
  if (nstart == 0) return 0;

  // ---- 1. all inverses W_i (and W_tip) up front (already in the workspace
  // when a W-based solve of the same factor prepared them)
  if (!(w_ready && full) && (e = prepare_w(Ld, Lt, nstart, b, a, full, ws, st))) return e;

  if (a > 0 && !arrow && (e = zero_async(Xa, (size_t)nstart * a * b * sizeof(double), st)))
    return e;

  static const bool use_launches = [] {
    const char* v = getenv("STBTA_SINV_LAUNCHES");
    return v && v[0] == '1';
  }();
  if (!use_launches) {
    // ---- 2+3. X_tip and the whole recursion in one persistent kernel
    SiParams P{};
    P.Ld = Ld; P.Ll = Ll; P.La = La; P.Lt = Lt;
    P.Xd = Xd; P.Xl = Xl; P.Xa = Xa; P.Xt = Xt;
    P.W = ws.Wall; P.Wt = ws.Wt;
    for (int q = 0; q < 2; ++q) { P.T1[q] = ws.T1[q]; P.T3[q] = ws.T3[q]; P.Ta[q] = ws.Ta[q]; }
    P.n = n; P.b = b; P.a = a; P.arrow = arrow; P.nstart = nstart; P.tip = a > 0 && full;
    P.ntb = (b + 127) / 128;
    P.tma = a <= 32 ? 1 : (a + 127) / 128;
    P.tnt = (a + 127) / 128;
    P.cm = si_cm(b, a);
    P.cs = 2 * P.cm + 1;
    P.p0 = P.tip ? P.tma * P.tnt : 0;
    P.c_last = P.c_full = 0;
    for (int k = 0; k < K_NKIND; ++k) {
      P.c_last += shape_tiles(kind_shape(P, k, 0));
      P.c_full += shape_tiles(kind_shape(P, k, 1));
    }
    P.total = P.p0 + (nstart == n ? P.c_last + (long long)(nstart - 1) * P.c_full
                                   : (long long)nstart * P.c_full);
    P.ticket = reinterpret_cast<unsigned long long*>(ws.ctr);
    P.abortw = ws.ctr + 2;
    P.ctr = ws.ctr + 4;
    if ((e = zero_async(ws.ctr, ws.ctr_bytes, st))) return e;
    if (ctr_ready && (e = (int)cudaEventRecord(ctr_ready, st))) return e;
    if (persistent) *persistent = 1;
    static std::atomic<unsigned long long> pmask{0};
    const size_t psmem = SIP_SMEM_DOUBLES * sizeof(double);
    if (attr_pending(pmask)) {
      if ((e = (int)cudaFuncSetAttribute(sinv_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem))) return e;
      attr_mark(pmask);
    }
    SiMaps maps;
    make_si_maps(P, ws, &maps);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sinv_persistent_kernel, SI_NT, psmem);
    if (occ < 1) return STBTA_EARG;
    long long grid = (long long)sm_count() * occ;
    if (grid > P.total) grid = P.total;
    if (grid < 1) return 0;
    sinv_persistent_kernel<<<(int)grid, SI_NT, psmem, st>>>(P, maps);
    count_launch();
    return (int)cudaGetLastError();
  }

  // ---- per-launch variant (STBTA_SINV_LAUNCHES=1; A/B reference for the persistent kernel)
  if (a > 0 && full) {
    TileJob j = job(Xt, a, a, a, 1.0);
    j.nprod = 1;
    j.p[0] = prod(ws.Wt, a, 1, ws.Wt, a, 1, a, 1.0);
    if ((e = launch_job(j, st))) return e;
  }

  // ---- 3. the recursion, i = nstart-1 .. 0
  for (int i = nstart - 1; i >= 0; --i) {
    const double* W = ws.Wall + i * bb;
    const double* sub = (i < n - 1) ? Ll + i * bb : nullptr;
    const double* arr = arrow ? La + (long long)i * a * b : nullptr;
    if (sub) {
      // T1 = X_{i+1,i+1} L_{i+1,i} (+ X_{a,i+1}^T L_{a,i})
      TileJob j = job(ws.T1[0], b, b, b, 1.0);
      j.p[j.nprod++] = prod(Xd + (i + 1) * bb, b, 0, sub, b, 1, b, 1.0);
      if (arr) j.p[j.nprod++] = prod(Xa + (long long)(i + 1) * a * b, b, 1, arr, b, 1, a, 1.0);
      if ((e = launch_job(j, st))) return e;
      // X_{i+1,i} = -T1 W
      TileJob j2 = job(Xl + i * bb, b, b, b, -1.0);
      j2.p[j2.nprod++] = prod(ws.T1[0], b, 0, W, b, 1, b, 1.0, 1);
      if ((e = launch_job(j2, st))) return e;
    }
    if (arr) {
      // Ta = X_tip L_{a,i} (+ X_{a,i+1} L_{i+1,i});  X_{a,i} = -Ta W
      TileJob j = job(ws.Ta[0], b, a, b, 1.0);
      j.p[j.nprod++] = prod(Xt, a, 0, arr, b, 1, a, 1.0);
      if (sub) j.p[j.nprod++] = prod(Xa + (long long)(i + 1) * a * b, b, 0, sub, b, 1, b, 1.0);
      if ((e = launch_job(j, st))) return e;
      TileJob j2 = job(Xa + (long long)i * a * b, b, a, b, -1.0);
      j2.p[j2.nprod++] = prod(ws.Ta[0], b, 0, W, b, 1, b, 1.0, 1);
      if ((e = launch_job(j2, st))) return e;
    }
    // T3 = W^T - X_{i+1,i}^T L_{i+1,i} - X_{a,i}^T L_{a,i}
    {
      TileJob j = job(ws.T3[0], b, b, b, 1.0);
      j.init = 2;
      j.ci = W;
      j.ldci = b;
      if (sub) j.p[j.nprod++] = prod(Xl + i * bb, b, 1, sub, b, 1, b, -1.0);
      if (arr) j.p[j.nprod++] = prod(Xa + (long long)i * a * b, b, 1, arr, b, 1, a, -1.0);
      if ((e = launch_job(j, st))) return e;
    }
    // X_ii = T3 W  (lower tiles, mirrored)
    {
      TileJob j = job(Xd + i * bb, b, b, b, 1.0);
      j.lower = 1;
      j.mirror = 1;
      j.p[j.nprod++] = prod(ws.T3[0], b, 0, W, b, 1, b, 1.0, 1);
      if ((e = launch_job(j, st))) return e;
    }
  }
  return 0;
}
