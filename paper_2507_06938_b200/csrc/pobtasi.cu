// POBTASI: selected inversion of a factored BTA matrix (C ABI).
//
// Reference: bta.selected_invert (pkg/src/stinla/bta.py:310-359):
//   X_tip = L_tip^-T L_tip^-1;  for i = n-1 .. 0, W = L_ii^-1:
//   X_{i+1,i} = -(X_{i+1,i+1} L_{i+1,i} + X_{a,i+1}^T L_{a,i}) W
//   X_{a,i}   = -(X_tip L_{a,i} + X_{a,i+1} L_{i+1,i}) W
//   X_{i,i}   = (W^T - X_{i+1,i}^T L_{i+1,i} - X_{a,i}^T L_{a,i}) W
// Every product is one DMMA engine launch (NN / TN, with W's triangle used to
// bound the K range), W comes from the recursive TRTRI (dense.cu).
#include "../../include/stbta.h"
#include "stbta_internal.cuh"

namespace stbta {

// out (n x n, ld_out) = in^T (n x n, ld_in)
__global__ void transpose_kernel(const double* __restrict__ in, long long ld_in, double* out,
                                 long long ld_out, int n, const int* info) {
  __shared__ double t[32][33];
  if (info != nullptr && *info != 0) return;
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int gr = by + r, gc = bx + threadIdx.x;
    if (gr < n && gc < n) t[r][threadIdx.x] = in[(long long)gr * ld_in + gc];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int gr = bx + r, gc = by + threadIdx.x;
    if (gr < n && gc < n) out[(long long)gr * ld_out + gc] = t[threadIdx.x][r];
  }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct PobtasiWs {
  double *W, *T1, *tmp, *T2, *winv, *Wt;
};

static size_t pobtasi_ws(int n, int b, int a, char* base, PobtasiWs* o) {
  (void)n;
  const size_t bb = align_up((size_t)b * b * sizeof(double));
  const size_t ab = align_up((size_t)(a > 0 ? a : 1) * b * sizeof(double));
  const int m = b > a ? b : a;
  const size_t wl = align_up((size_t)leaves_of(m) * LEAF * LEAF * sizeof(double));
  const size_t aa = align_up((size_t)(a > 0 ? a * a : 1) * sizeof(double) * 2);
  if (o) {
    o->W = reinterpret_cast<double*>(base);
    o->T1 = reinterpret_cast<double*>(base + bb);
    o->tmp = reinterpret_cast<double*>(base + 2 * bb);
    o->T2 = reinterpret_cast<double*>(base + 3 * bb);
    o->winv = reinterpret_cast<double*>(base + 3 * bb + ab);
    o->Wt = reinterpret_cast<double*>(base + 3 * bb + ab + wl);
  }
  return 3 * bb + ab + wl + aa;
}

static int gemm(cudaStream_t st, bool ta, bool tb, double* C, long long ldc, const double* A,
                long long lda, const double* B, long long ldb, int M, int N, int K, double alpha,
                double beta, int a_tri, int b_tri) {
  GemmArgs g{};
  g.A = seg1(const_cast<double*>(A), lda);
  g.B = seg1(const_cast<double*>(B), ldb);
  g.C = seg1(C, ldc);
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha; g.beta = beta;
  g.a_tri = a_tri; g.b_tri = b_tri;
  g.batch = 1;
  return gemm_launch(g, ta, tb, st);
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
  if (factor == nullptr || inv == nullptr || n < 1 || b < 1 || a < 0) return STBTA_EARG;
  if (workspace_bytes < stbta_pobtasi_workspace_bytes(n, b, a)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtasiWs ws;
  pobtasi_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  const long long bb = (long long)b * b;
  const double* Ld = factor;
  const double* Ll = Ld + n * bb;
  const double* La = Ll + (n - 1) * bb;
  const double* Lt = La + (long long)n * a * b;
  double* Xd = inv;
  double* Xl = Xd + n * bb;
  double* Xa = Xl + (n - 1) * bb;
  double* Xt = Xa + (long long)n * a * b;
  const bool arrow = has_arrow && a > 0;
  DenseCtx c{st, nullptr, ws.winv, nullptr};
  int e = (int)cudaMemsetAsync(inv, 0, stbta_storage_elems(n, b, a) * sizeof(double), st);
  if (e) return e;

  if (a > 0) {  // X_tip = W_t^T W_t
    double* Wt = ws.Wt;
    if ((e = trtri_rec(c, Lt, a, Wt, a, a, ws.tmp, 0))) return e;
    if ((e = gemm(st, true, false, Xt, a, Wt, a, Wt, a, a, a, a, 1.0, 0.0, TRI_UPPER, TRI_LOWER)))
      return e;
  }
  const dim3 tgrid(ceil_div(b, 32), ceil_div(b, 32)), tblk(32, 8);
  for (int i = n - 1; i >= 0; --i) {
    const double* Lii = Ld + i * bb;
    const double* sub = (i < n - 1) ? Ll + i * bb : nullptr;
    const double* arr = arrow ? La + (long long)i * a * b : nullptr;
    if ((e = trtri_rec(c, Lii, b, ws.W, b, b, ws.tmp, 0))) return e;
    if (sub) {
      // T1 = X_{i+1,i+1} L_{i+1,i} (+ X_{a,i+1}^T L_{a,i});  X_{i+1,i} = -T1 W
      if ((e = gemm(st, false, false, ws.T1, b, Xd + (i + 1) * bb, b, sub, b, b, b, b, 1.0, 0.0,
                    TRI_NONE, TRI_NONE)))
        return e;
      if (arr && (e = gemm(st, true, false, ws.T1, b, Xa + (long long)(i + 1) * a * b, b, arr, b,
                           b, b, a, 1.0, 1.0, TRI_NONE, TRI_NONE)))
        return e;
      if ((e = gemm(st, false, false, Xl + i * bb, b, ws.T1, b, ws.W, b, b, b, b, -1.0, 0.0,
                    TRI_NONE, TRI_LOWER)))
        return e;
    }
    if (arr) {
      // T2 = X_tip L_{a,i} (+ X_{a,i+1} L_{i+1,i});  X_{a,i} = -T2 W
      if ((e = gemm(st, false, false, ws.T2, b, Xt, a, arr, b, a, b, a, 1.0, 0.0, TRI_NONE,
                    TRI_NONE)))
        return e;
      if (sub && (e = gemm(st, false, false, ws.T2, b, Xa + (long long)(i + 1) * a * b, b, sub, b,
                           a, b, b, 1.0, 1.0, TRI_NONE, TRI_NONE)))
        return e;
      if ((e = gemm(st, false, false, Xa + (long long)i * a * b, b, ws.T2, b, ws.W, b, a, b, b,
                    -1.0, 0.0, TRI_NONE, TRI_LOWER)))
        return e;
    }
    // T1 = W^T - X_{i+1,i}^T L_{i+1,i} - X_{a,i}^T L_{a,i};  X_ii = T1 W
    transpose_kernel<<<tgrid, tblk, 0, st>>>(ws.W, b, ws.T1, b, b, nullptr);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
    if (sub && (e = gemm(st, true, false, ws.T1, b, Xl + i * bb, b, sub, b, b, b, b, -1.0, 1.0,
                         TRI_NONE, TRI_NONE)))
      return e;
    if (arr && (e = gemm(st, true, false, ws.T1, b, Xa + (long long)i * a * b, b, arr, b, b, b, a,
                         -1.0, 1.0, TRI_NONE, TRI_NONE)))
      return e;
    if ((e = gemm(st, false, false, Xd + i * bb, b, ws.T1, b, ws.W, b, b, b, b, 1.0, 0.0, TRI_NONE,
                  TRI_LOWER)))
      return e;
  }
  return 0;
}

}  // extern "C"
