// Internal (C++) interfaces shared by the stbta translation units.
#pragma once

#include <cuda_runtime.h>

#include "gemm.cuh"

namespace stbta {

constexpr int LEAF = 64;  // diagonal-tile size of the recursive factorization
enum { LEAF_FACTOR = 0, LEAF_INVERT = 1 };

int launch_leaf(double* A, long long lda, int n, double* winv, double* ldslot, int* info, int code,
                int mode, cudaStream_t st);
int launch_zero_upper(double* A, long long lda, int n, const int* info, cudaStream_t st);
int launch_logdet_reduce(const double* slots, int count, double* out, cudaStream_t st);

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
inline int leaves_of(int n) { return ceil_div(n, LEAF); }
// split point of the recursion: half of the leaves, rounded up, in elements
inline int rec_split(int n) { return LEAF * ((leaves_of(n) + 1) / 2); }

// Recursive dense kernels on the current stream.
struct DenseCtx {
  cudaStream_t st;
  int* info;        // device failure word (0 = ok)
  double* winv;     // LEAF*LEAF doubles per leaf of the current diagonal block
  double* ldslots;  // per-leaf log-det partials (may be null)
};

// Cholesky of the n x n lower block A in place; leaves [leaf0, ...) of ctx.
int potrf_rec(DenseCtx& c, double* A, long long lda, int n, int leaf0, int slot0, int code);
// X (m x n, segmented rows) := X L^-T, L = n x n lower with leaf inverses in ctx.winv.
int trsm_rlt_rec(DenseCtx& c, SegMat X, int m, const double* L, long long ldl, int n, int leaf0);
// W := L^-1 (n x n lower) out of place; tmp needs n*n doubles.
int trtri_rec(DenseCtx& c, const double* L, long long ldl, double* W, long long ldw, int n,
              double* tmp, int leaf0);

}  // namespace stbta
