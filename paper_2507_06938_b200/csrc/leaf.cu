// Diagonal-tile kernels on 64x64 leaves of the recursive block Cholesky.
//
//   leaf_kernel(mode=FACTOR): Cholesky of one <=64x64 diagonal tile in place
//       (the unblocked part of np.linalg.cholesky at bta.py:206 / 230 and
//       bta_dist.py:215), the tile's log-det contribution sum(log diag L)
//       (bta.py:238-246), and W = L^-1 of the tile, which turns every TRSM leaf
//       of the recursion into a DMMA GEMM (X := X W^T).
//   leaf_kernel(mode=INVERT): W = L^-1 only, for TRTRI leaves (bta.py:327, 330).
//
// Non-positive (or NaN) pivots raise the reference's FactorizationError: the
// first failure records `code` (= 1 + time-block index) in *info and every
// later kernel of the factorization exits immediately.
#include "common.cuh"
#include "stbta_internal.cuh"

namespace stbta {

__global__ void __launch_bounds__(256) leaf_kernel(double* __restrict__ A, long long lda, int n,
                                                   double* __restrict__ winv,
                                                   double* __restrict__ ldslot, int* info,
                                                   int code, int mode) {
  __shared__ double s[LEAF][LEAF + 1];
  if (info != nullptr && *info != 0) return;
  const int tid = threadIdx.x;

  for (int idx = tid; idx < LEAF * LEAF; idx += 256) {
    const int r = idx / LEAF, c = idx % LEAF;
    double v;
    if (r < n && c < n)
      v = (c <= r) ? A[(long long)r * lda + c] : 0.0;
    else
      v = (r == c) ? 1.0 : 0.0;
    s[r][c] = v;
  }
  __syncthreads();

  if (mode == LEAF_FACTOR) {
    // right-looking rank-1 updates on the unscaled tile; column j of L is
    // s[:, j] / sqrt(p_j) and is applied lazily, so one barrier per step.
    const int c = tid % LEAF, r0 = tid / LEAF;
    for (int j = 0; j < n; ++j) {
      const double p = s[j][j];
      if (!(p > 0.0)) {  // uniform: every thread read the same pivot
        if (tid == 0 && info != nullptr) atomicCAS(info, 0, code);
        return;
      }
      if (c > j) {
        const double lcj = s[c][j] / p;
        for (int r = r0; r < LEAF; r += 4)
          if (r >= c) s[r][c] -= s[r][j] * lcj;
      }
      __syncthreads();
    }
    double vals[LEAF / 4];
#pragma unroll
    for (int q = 0; q < LEAF / 4; ++q) {
      const int r = r0 + 4 * q;
      double v = 0.0;
      if (c < r)
        v = s[r][c] / sqrt(s[c][c]);
      else if (c == r)
        v = sqrt(s[r][r]);
      vals[q] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LEAF / 4; ++q) s[r0 + 4 * q][c] = vals[q];
    __syncthreads();

    if (tid < 32) {  // fixed-order log-det partial of this tile
      double acc = 0.0;
      for (int j = tid; j < n; j += 32) acc += log(s[j][j]);
      acc = warp_sum(acc);
      if (tid == 0 && ldslot != nullptr) *ldslot = acc;
    }
    // write L back (strict upper of the tile cleared, as np.linalg.cholesky)
#pragma unroll
    for (int q = 0; q < LEAF / 4; ++q) {
      const int r = r0 + 4 * q;
      if (r < n && c < n) A[(long long)r * lda + c] = vals[q];
    }
  }

  if (winv == nullptr) return;
  // W = L^-1 by row-oriented forward elimination.  Warp w owns columns
  // 8w..8w+7; lane (h, cc) holds rows h, h+4, ..., h+60 of column 8w+cc, so
  // row j of W is a warp-local shuffle and no barrier is needed.
  const int warp = tid >> 5, lane = tid & 31;
  const int h = lane >> 3, cc = lane & 7;
  const int col = warp * 8 + cc;
  double w[LEAF / 4];
#pragma unroll
  for (int q = 0; q < LEAF / 4; ++q) w[q] = (h + 4 * q == col) ? 1.0 : 0.0;
#pragma unroll
  for (int qj = 0; qj < LEAF / 4; ++qj) {
#pragma unroll
    for (int hj = 0; hj < 4; ++hj) {
      const int j = 4 * qj + hj;
      if (h == hj) w[qj] /= s[j][j];
      const double wj = __shfl_sync(0xffffffffu, w[qj], hj * 8 + cc);
#pragma unroll
      for (int q = 0; q < LEAF / 4; ++q) {
        const int i = h + 4 * q;
        if (i > j) w[q] -= s[i][j] * wj;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < LEAF / 4; ++q) winv[(h + 4 * q) * LEAF + col] = w[q];
}

// Clear the strict upper triangle of an n x n row-major block.
__global__ void zero_upper_kernel(double* A, long long lda, int n, const int* info) {
  if (info != nullptr && *info != 0) return;
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / n), c = (int)(idx % n);
    if (c > r) A[(long long)r * lda + c] = 0.0;
  }
}

// out[0] = 2 * sum(slots[0:count]) in a fixed order (deterministic).
__global__ void logdet_reduce_kernel(const double* slots, int count, double* out) {
  __shared__ double part[256];
  const int tid = threadIdx.x;
  const int per = (count + 255) / 256;
  double acc = 0.0;
  for (int i = tid * per; i < min(count, (tid + 1) * per); ++i) acc += slots[i];
  part[tid] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s) part[tid] += part[tid + s];
    __syncthreads();
  }
  if (tid == 0) out[0] = 2.0 * part[0];
}

int launch_leaf(double* A, long long lda, int n, double* winv, double* ldslot, int* info, int code,
                int mode, cudaStream_t st) {
  leaf_kernel<<<1, 256, 0, st>>>(A, lda, n, winv, ldslot, info, code, mode);
  count_launch();
  return (int)cudaGetLastError();
}

int launch_zero_upper(double* A, long long lda, int n, const int* info, cudaStream_t st) {
  if (n <= 1) return 0;
  const long long total = (long long)n * n;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  zero_upper_kernel<<<blocks, 256, 0, st>>>(A, lda, n, info);
  count_launch();
  return (int)cudaGetLastError();
}

int launch_logdet_reduce(const double* slots, int count, double* out, cudaStream_t st) {
  logdet_reduce_kernel<<<1, 256, 0, st>>>(slots, count, out);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace stbta
