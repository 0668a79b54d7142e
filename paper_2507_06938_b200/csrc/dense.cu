// Recursive dense FP64 block kernels built on the DMMA engine.
//
// potrf_rec     np.linalg.cholesky of one b x b pivot      (bta.py:206, 230)
// trsm_rlt_rec  X := X L^-T  == solve_triangular(L, X^T).T (bta.py:213-219,
//               bta_dist.py:171)
// trtri_rec     L^-1 == solve_triangular(L, I)             (bta.py:327, 330)
//
// The recursion halves the matrix on 64-row leaf boundaries, so all flops
// except the 64x64 diagonal tiles run as large-K DMMA GEMMs, and the leaf
// inverses produced by the diagonal-tile kernel turn each TRSM leaf into a GEMM.
#include "stbta_internal.cuh"

namespace stbta {

static int gemm_nt(DenseCtx& c, SegMat C, SegMat A, SegMat B, int M, int N, int K, double alpha,
                   double beta, int c_lower) {
  GemmArgs g{};
  g.A = A; g.B = B; g.C = C;
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha; g.beta = beta;
  g.a_tri = TRI_NONE; g.b_tri = TRI_NONE;
  g.c_lower = c_lower;
  g.info = c.info;
  g.batch = 1;
  return gemm_launch(g, false, true, c.st);
}

int potrf_rec(DenseCtx& c, double* A, long long lda, int n, int leaf0, int slot0, int code) {
  if (n <= 0) return 0;
  if (n <= LEAF)
    return launch_leaf(A, lda, n, c.winv ? c.winv + (long long)leaf0 * LEAF * LEAF : nullptr,
                       c.ldslots ? c.ldslots + slot0 + leaf0 : nullptr, c.info, code, LEAF_FACTOR,
                       c.st);
  const int n1 = rec_split(n), n2 = n - n1;
  int e = potrf_rec(c, A, lda, n1, leaf0, slot0, code);
  if (e) return e;
  double* A21 = A + (long long)n1 * lda;
  double* A22 = A21 + n1;
  e = trsm_rlt_rec(c, seg1(A21, lda), n2, A, lda, n1, leaf0);
  if (e) return e;
  // A22 -= A21 A21^T (lower triangle only)
  e = gemm_nt(c, seg1(A22, lda), seg1(A21, lda), seg1(A21, lda), n2, n2, n1, -1.0, 1.0, 1);
  if (e) return e;
  return potrf_rec(c, A22, lda, n2, leaf0 + n1 / LEAF, slot0, code);
}

int trsm_rlt_rec(DenseCtx& c, SegMat X, int m, const double* L, long long ldl, int n, int leaf0) {
  if (m <= 0 || n <= 0) return 0;
  if (n <= LEAF) {
    // X := X W^T with W = L^-1 of this leaf; in place is safe because one CTA
    // owns complete rows (N = n <= BN) and reads them before its epilogue.
    double* W = c.winv + (long long)leaf0 * LEAF * LEAF;
    return gemm_nt(c, X, X, seg1(W, LEAF), m, n, n, 1.0, 0.0, 0);
  }
  const int n1 = rec_split(n), n2 = n - n1;
  int e = trsm_rlt_rec(c, X, m, L, ldl, n1, leaf0);
  if (e) return e;
  // X2 -= X1 L21^T
  SegMat X2 = shift_cols(X, n1);
  e = gemm_nt(c, X2, X, seg1(const_cast<double*>(L) + (long long)n1 * ldl, ldl), m, n2, n1, -1.0,
              1.0, 0);
  if (e) return e;
  return trsm_rlt_rec(c, X2, m, L + (long long)n1 * ldl + n1, ldl, n2, leaf0 + n1 / LEAF);
}

// W = L^-1.  [[L11, 0], [L21, L22]]^-1 = [[W11, 0], [-W22 L21 W11, W22]].
int trtri_rec(DenseCtx& c, const double* L, long long ldl, double* W, long long ldw, int n,
              double* tmp, int leaf0) {
  if (n <= 0) return 0;
  if (n <= LEAF) {
    double* wl = c.winv + (long long)leaf0 * LEAF * LEAF;
    int e = launch_leaf(const_cast<double*>(L), ldl, n, wl, nullptr, c.info, 0, LEAF_INVERT, c.st);
    if (e) return e;
    // copy the leaf inverse into W (n x n, upper part zero)
    return (int)cudaMemcpy2DAsync(W, ldw * sizeof(double), wl, LEAF * sizeof(double),
                                  n * sizeof(double), n, cudaMemcpyDeviceToDevice, c.st);
  }
  const int n1 = rec_split(n), n2 = n - n1;
  int e = trtri_rec(c, L, ldl, W, ldw, n1, tmp, leaf0);
  if (e) return e;
  e = trtri_rec(c, L + (long long)n1 * ldl + n1, ldl, W + (long long)n1 * ldw + n1, ldw, n2, tmp,
                leaf0 + n1 / LEAF);
  if (e) return e;
  // T = L21 W11   (n2 x n1; W11 lower => op(B) lower: zero for k < n)
  {
    GemmArgs g{};
    g.A = seg1(const_cast<double*>(L) + (long long)n1 * ldl, ldl);
    g.B = seg1(W, ldw);
    g.C = seg1(tmp, n1);
    g.M = n2; g.N = n1; g.K = n1;
    g.alpha = 1.0; g.beta = 0.0;
    g.b_tri = TRI_LOWER;
    g.info = c.info; g.batch = 1;
    e = gemm_launch(g, false, false, c.st);
    if (e) return e;
  }
  // W21 = -W22 T   (W22 lower => op(A) lower: zero for k > m)
  {
    GemmArgs g{};
    g.A = seg1(W + (long long)n1 * ldw + n1, ldw);
    g.B = seg1(tmp, n1);
    g.C = seg1(W + (long long)n1 * ldw, ldw);
    g.M = n2; g.N = n1; g.K = n2;
    g.alpha = -1.0; g.beta = 0.0;
    g.a_tri = TRI_LOWER;
    g.info = c.info; g.batch = 1;
    e = gemm_launch(g, false, false, c.st);
    if (e) return e;
  }
  // W12 = 0
  return (int)cudaMemset2DAsync(W + n1, ldw * sizeof(double), 0, n2 * sizeof(double), n1, c.st);
}

}  // namespace stbta
