// FP64 DMMA tile engine: C = alpha * op(A) * op(B) + beta * C.
//
// One engine serves every dense block operation of the BTA solver
// (reference call sites: bta.py:206-230 factorize, bta.py:326-354
// selected_invert, bta_dist.py:171-253 partition elimination):
//   * SYRK / Schur updates   diag[i+1] -= lower[i] lower[i]^T   (lower-only C)
//   * TRSM panels            X := X L^-T  through 64x64 leaf inverses
//   * TRMM / GEMM chains     selected inversion recursion
//
// Operands are row-major sub-matrices of the flat BTA buffer.  A "segmented"
// operand stacks two storage regions vertically (e.g. lower[i] on top of
// arrow[i], both with leading dimension b) so one launch covers the block
// and its arrowhead rows; C may have a third region for the tip.
#pragma once

#include "../common.cuh"

namespace stbta {

struct SegMat {
  double* p0;
  long long ld0, bs0;  // storage rows [0, r0)
  double* p1;
  long long ld1, bs1;  // storage rows >= r0 (cols < c0 when p2 is used)
  double* p2;
  long long ld2, bs2;  // storage rows >= r0, cols >= c0 (C only)
  int r0, c0;
};

enum { TRI_NONE = 0, TRI_LOWER = 1, TRI_UPPER = 2 };

struct GemmArgs {
  SegMat A, B, C;
  int M, N, K;
  double alpha, beta;
  int a_tri;    // structure of op(A) (M x K): LOWER => zero for k > m
  int b_tri;    // structure of op(B) (K x N): LOWER => zero for k < n, UPPER => zero for k > n
  int c_lower;  // only produce / write entries with col <= row
  const int* info;  // skip all work when *info != 0 (failed factorization)
  int batch;
};

// Single-region view helper.
inline SegMat seg1(double* p, long long ld, long long bstride = 0) {
  SegMat s;
  s.p0 = p; s.ld0 = ld; s.bs0 = bstride;
  s.p1 = p; s.ld1 = ld; s.bs1 = bstride;
  s.p2 = p; s.ld2 = ld; s.bs2 = bstride;
  s.r0 = 0x7fffffff; s.c0 = 0x7fffffff;
  return s;
}
// Two stacked regions: rows [0, r0) at p0, rows [r0, ...) at p1.
inline SegMat seg2(double* p0, long long ld0, int r0, double* p1, long long ld1) {
  SegMat s = seg1(p0, ld0);
  s.p1 = p1; s.ld1 = ld1; s.r0 = r0;
  s.p2 = p1; s.ld2 = ld1;
  return s;
}
// Column sub-range view: every region shifted right by `col` columns.
inline SegMat shift_cols(SegMat s, int col) {
  s.p0 += col; s.p1 += col; s.p2 += col;
  return s;
}

// Launch C = alpha op(A) op(B) + beta C on `stream`.  Returns cudaError_t.
int gemm_launch(const GemmArgs& g, bool ta, bool tb, cudaStream_t stream);

}  // namespace stbta
