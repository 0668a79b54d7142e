// Coupling products of the time-partitioned solver (S3; reference
// bta_dist.py:370-458 d_solve and the reduced-system assembly around it).
//
// A partition's interior solve z = A_int^-1 x_int is joined to the reduced
// separator system by a handful of thin products, all HBM-bound:
//
//   left separator   r_left  -= L(lo,lo-1)^T z_lo          (b x b)^T  (b x k)
//   right separator  r_right -= L(hi,hi-1)   z_{hi-1}      (b x b)    (b x k)
//   arrow rows       r_tip   -= sum_j A_arrow[j] z_j       (a x b)    (b x k), j over the interior
//   back-substitution w_lo = L(lo,lo-1) x_left, w_{hi-1} = L(hi,hi-1)^T x_right,
//                     w_j += A_arrow[j]^T x_tip
//
// One entry point covers them: Y (+)= alpha * op(A_j) X_j for a batch of
// row-major A_j (m x n, row stride lda, batch stride strideA), with the
// batch either kept apart (Y_j) or reduced into one Y in batch order.
// X_j / Y_j rows are k wide (row strides ldx / ldy).  Every reduction runs in
// a fixed order (warp butterfly, then slices / batches in index order), so
// the results are bitwise reproducible.
//
//   trans = 0: one warp per output row (j, i), lanes stride the contiguous
//              row of A_j -> coalesced; partial rows to the workspace when
//              reduced over the batch.
//   trans = 1: one thread per output column (j, c, slice s of 128 rows of
//              A_j): consecutive threads read consecutive columns of a row
//              -> coalesced; the slices (and the batch) are summed after.
#include "../../include/stbta.h"
#include "common.cuh"

namespace stbta {

constexpr int CPL_K = 16;      // right-hand sides per pass (host splits wider X)
constexpr int CPL_ROWS = 128;  // rows of A_j per slice (trans = 1)

struct CoupleArgs {
  int trans, nbatch, m, n, k;
  double alpha;
  const double* A;
  long long lda, strideA;
  const double* X;
  long long ldx, strideX;
  double* Y;
  long long ldy, strideY;
  int reduce;
};

// trans = 0: out(j, i, :) = A_j[i, :] . X_j[:, :]
__global__ void __launch_bounds__(256) couple_n_kernel(CoupleArgs p, double* partial) {
  const int lane = threadIdx.x & 31;
  const long long warp = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (warp >= (long long)p.nbatch * p.m) return;
  const int j = (int)(warp / p.m), i = (int)(warp % p.m);
  const double* a = p.A + j * p.strideA + (long long)i * p.lda;
  const double* x = p.X + j * p.strideX;
  double acc[CPL_K];
#pragma unroll
  for (int q = 0; q < CPL_K; ++q) acc[q] = 0.0;
  for (int c = lane; c < p.n; c += 32) {
    const double av = a[c];
    const double* xr = x + (long long)c * p.ldx;
#pragma unroll
    for (int q = 0; q < CPL_K; ++q)
      if (q < p.k) acc[q] = fma(av, xr[q], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < CPL_K; ++q) {
    if (q >= p.k) break;
    const double s = warp_sum(acc[q]);
    if (lane == 0) {
      if (p.reduce)
        partial[((long long)j * p.m + i) * CPL_K + q] = s;
      else
        p.Y[j * p.strideY + (long long)i * p.ldy + q] += p.alpha * s;
    }
  }
}

// reduce over the batch: Y[i, q] += alpha * sum_j partial(j, i, q), j ascending
__global__ void couple_n_reduce(CoupleArgs p, const double* partial) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)p.m * p.k) return;
  const int i = (int)(t / p.k), q = (int)(t % p.k);
  double s = 0.0;
  for (int j = 0; j < p.nbatch; ++j) s += partial[((long long)j * p.m + i) * CPL_K + q];
  p.Y[(long long)i * p.ldy + q] += p.alpha * s;
}

// trans = 1: out(j, s, c, :) = sum_{r in slice s} A_j[r, c] X_j[r, :]
__global__ void __launch_bounds__(256) couple_t_kernel(CoupleArgs p, double* partial, int S) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)p.nbatch * S * p.n;
  if (t >= total) return;
  const int c = (int)(t % p.n);
  const long long js = t / p.n;
  const int s = (int)(js % S), j = (int)(js / S);
  const int r0 = s * (S > 1 ? CPL_ROWS : p.m);
  const int r1 = min(p.m, r0 + (S > 1 ? CPL_ROWS : p.m));
  const double* a = p.A + j * p.strideA + c;
  const double* x = p.X + j * p.strideX;
  double acc[CPL_K];
#pragma unroll
  for (int q = 0; q < CPL_K; ++q) acc[q] = 0.0;
  for (int r = r0; r < r1; ++r) {
    const double av = a[(long long)r * p.lda];
    const double* xr = x + (long long)r * p.ldx;
#pragma unroll
    for (int q = 0; q < CPL_K; ++q)
      if (q < p.k) acc[q] = fma(av, xr[q], acc[q]);
  }
  if (S == 1 && !p.reduce) {
    double* y = p.Y + j * p.strideY + (long long)c * p.ldy;
#pragma unroll
    for (int q = 0; q < CPL_K; ++q)
      if (q < p.k) y[q] += p.alpha * acc[q];
    return;
  }
  double* out = partial + (((long long)j * S + s) * p.n + c) * CPL_K;
#pragma unroll
  for (int q = 0; q < CPL_K; ++q)
    if (q < p.k) out[q] = acc[q];
}

// Y_j[c, q] (or Y[c, q] when reduced) += alpha * sum over (j,) s ascending
__global__ void couple_t_reduce(CoupleArgs p, const double* partial, int S) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = p.reduce ? 1 : p.nbatch;
  if (t >= (long long)nb * p.n * p.k) return;
  const int q = (int)(t % p.k);
  const int c = (int)((t / p.k) % p.n);
  const int jo = (int)(t / ((long long)p.k * p.n));
  const int j0 = p.reduce ? 0 : jo, j1 = p.reduce ? p.nbatch : jo + 1;
  double sum = 0.0;
  for (int j = j0; j < j1; ++j)
    for (int s = 0; s < S; ++s) sum += partial[(((long long)j * S + s) * p.n + c) * CPL_K + q];
  p.Y[jo * p.strideY + (long long)c * p.ldy + q] += p.alpha * sum;
}

static int couple_slices_host(int trans, int m) {
  return trans ? (m > 2 * CPL_ROWS ? (m + CPL_ROWS - 1) / CPL_ROWS : 1) : 1;
}

}  // namespace stbta

using namespace stbta;

extern "C" size_t stbta_couple_workspace_bytes(int trans, int nbatch, int m, int n, int reduce) {
  if (nbatch <= 0 || m <= 0 || n <= 0) return 0;
  if (!trans) return reduce ? (size_t)nbatch * m * CPL_K * sizeof(double) : 0;
  const int S = couple_slices_host(1, m);
  if (S == 1 && !reduce) return 0;
  return (size_t)nbatch * S * n * CPL_K * sizeof(double);
}

extern "C" int stbta_couple(int trans, int nbatch, int m, int n, int k, double alpha,
                            const double* A, long long lda, long long strideA, const double* X,
                            long long ldx, long long strideX, double* Y, long long ldy,
                            long long strideY, int reduce, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (nbatch < 0 || m < 0 || n < 0 || k < 0 || lda < n || ldx < k || ldy < k) return STBTA_EARG;
  if (nbatch == 0 || m == 0 || n == 0 || k == 0) return 0;
  if (!A || !X || !Y) return STBTA_EARG;
  if (workspace_bytes < stbta_couple_workspace_bytes(trans, nbatch, m, n, reduce))
    return STBTA_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)workspace;
  for (int q0 = 0; q0 < k; q0 += CPL_K) {  // right-hand-side chunks
    CoupleArgs p{trans, nbatch, m, n, min(CPL_K, k - q0), alpha, A, lda, strideA,
                 X + q0, ldx, strideX, Y + q0, ldy, strideY, reduce};
    if (!trans) {
      const long long warps = (long long)nbatch * m;
      couple_n_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(p, part);
      count_launch();
      if (reduce) {
        const long long t = (long long)m * p.k;
        couple_n_reduce<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(p, part);
        count_launch();
      }
    } else {
      const int S = couple_slices_host(1, m);
      const long long t = (long long)nbatch * S * n;
      couple_t_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(p, part, S);
      count_launch();
      if (S > 1 || reduce) {
        const long long tr = (long long)(reduce ? 1 : nbatch) * n * p.k;
        couple_t_reduce<<<(unsigned)((tr + 255) / 256), 256, 0, st>>>(p, part, S);
        count_launch();
      }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}
