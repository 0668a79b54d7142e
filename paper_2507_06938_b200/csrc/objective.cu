// Device half of the INLA objective f_obj around the BTA factorizations.
//
//   stbta_assemble     theta-dependent values of Q_p / Q_c written straight
//                      into BTA storage (reference: model.py:196-248 value map,
//                      coreg.py:80-121 joint assembly, inla.py:264-283 Q_c,
//                      coreg.py:250-276 map_to_bta incl. the zero fill)
//   stbta_rhs_combine  A^T (tau o y) in BTA order                (inla.py:313-315)
//   stbta_quadform     mu^T Q_p mu from the same entry list      (inla.py:369)
//   stbta_residual     per-process sum (y - A mu)^2              (inla.py:363-367)
//
// Assembly layout.  Every structural nonzero e of the lower BTA envelope is
// described ONCE at evaluator construction: its flat storage offset (sorted
// ascending), the process pair p(e) of its coregional block and a source
// index s(e) into a basis table B[s][t] (T terms per source entry).  For any
// theta the host reduces the model to a coefficient table coef[p][t], and
//   value(e) = sum_t coef[p(e)][t] * B[s(e)][t].
// The kernel walks the BTA storage in 16 KB tiles: each tile is zeroed in
// shared memory, the (sorted) entries falling into it are scattered there,
// and the tile is streamed out with 16-byte stores — the zero fill and the
// scatter are one coalesced pass over HBM.
#include "../../include/stbta.h"
#include "common.cuh"

namespace stbta {

constexpr int ASM_TILE = 2048;  // doubles per storage tile (16 KB)

struct EntryTable {
  const long long* offsets;   // [E] sorted flat offsets into BTA storage
  const int* pair;            // [E] coefficient row
  const int* src;             // [E] basis row
  const double* basis;        // [S][T]
  const double* coef;         // [P][T]
  int T;
};

STBTA_DEV double entry_value(const EntryTable& t, long long e) {
  const double* bv = t.basis + (long long)t.src[e] * t.T;
  const double* cv = t.coef + (long long)t.pair[e] * t.T;
  double v = 0.0;
  for (int k = 0; k < t.T; ++k) v += cv[k] * bv[k];
  return v;
}

__global__ void __launch_bounds__(256) assemble_kernel(double* __restrict__ data, long long nstore,
                                                       const long long* __restrict__ tile_start,
                                                       long long ntiles, EntryTable t) {
  __shared__ __align__(16) double tile[ASM_TILE];
  for (long long ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const long long base = ti * ASM_TILE;
    for (int k = threadIdx.x; k < ASM_TILE; k += 256) tile[k] = 0.0;
    __syncthreads();
    const long long e0 = tile_start[ti], e1 = tile_start[ti + 1];
    for (long long e = e0 + threadIdx.x; e < e1; e += 256) {
      STBTA_CHECK(t.offsets[e] >= base && t.offsets[e] - base < ASM_TILE && t.offsets[e] < nstore);
      tile[t.offsets[e] - base] = entry_value(t, e);
    }
    __syncthreads();
    const long long len = min((long long)ASM_TILE, nstore - base);
    if (len == ASM_TILE) {
      double2* dst = reinterpret_cast<double2*>(data + base);
      const double2* srcv = reinterpret_cast<const double2*>(tile);
      for (int k = threadIdx.x; k < ASM_TILE / 2; k += 256) dst[k] = srcv[k];
    } else {
      for (int k = threadIdx.x; k < len; k += 256) data[base + k] = tile[k];
    }
    __syncthreads();
  }
}

// Decode a flat BTA offset into (row, col) of the permuted matrix and the
// symmetric weight (1 on diagonal blocks / tip, 2 on lower / arrow blocks).
STBTA_DEV void decode(long long off, int n, int b, int a, long long& row, long long& col,
                      double& w) {
  const long long bb = (long long)b * b;
  const long long base_lower = n * bb;
  const long long base_arrow = base_lower + (long long)(n - 1) * bb;
  const long long base_tip = base_arrow + (long long)n * a * b;
  if (off < base_lower) {
    const long long t = off / bb, r = off % bb;
    row = t * b + r / b; col = t * b + r % b; w = 1.0;
  } else if (off < base_arrow) {
    const long long q = off - base_lower, t = q / bb, r = q % bb;
    row = (t + 1) * b + r / b; col = t * b + r % b; w = 2.0;
  } else if (off < base_tip) {
    const long long q = off - base_arrow, ab = (long long)a * b, t = q / ab, r = q % ab;
    row = (long long)n * b + r / b; col = t * b + r % b; w = 2.0;
  } else {
    const long long q = off - base_tip;
    row = (long long)n * b + q / a; col = (long long)n * b + q % a; w = 1.0;
  }
}

__global__ void __launch_bounds__(256) quadform_kernel(EntryTable t, long long nent, int n, int b,
                                                       int a, const double* __restrict__ x,
                                                       double* partial) {
  double acc = 0.0;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < nent; e += (long long)gridDim.x * 256) {
    long long r, c;
    double w;
    decode(t.offsets[e], n, b, a, r, c, w);
    acc += w * entry_value(t, e) * x[r] * x[c];
  }
  acc = warp_sum(acc);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += ws[k];
    partial[blockIdx.x] = s;
  }
}

// out[slot] = sum of partial[0:count] in index order
__global__ void ordered_sum_kernel(const double* partial, int count, double* out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < count; ++k) s += partial[k];
    out[0] = s;
  }
}

// out[e] = sum_i tau[i] * U[i][e]   (fixed process order)
__global__ void rhs_combine_kernel(double* __restrict__ out, const double* __restrict__ U,
                                   const double* __restrict__ tau, int nv, long long N) {
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < N; e += (long long)gridDim.x * 256) {
    double s = 0.0;
    for (int i = 0; i < nv; ++i) s += tau[i] * U[i * N + e];
    out[e] = s;
  }
}

// per-row squared residual of y - A x; rows of process i are [seg[i], seg[i+1])
__global__ void __launch_bounds__(256) residual_kernel(const long long* __restrict__ indptr,
                                                       const int* __restrict__ indices,
                                                       const double* __restrict__ vals, long long nrows,
                                                       const double* __restrict__ y,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ sq) {
  for (long long r = blockIdx.x * 256LL + threadIdx.x; r < nrows; r += (long long)gridDim.x * 256) {
    double ax = 0.0;
    for (long long k = indptr[r]; k < indptr[r + 1]; ++k) ax += vals[k] * x[indices[k]];
    const double d = y[r] - ax;
    sq[r] = d * d;
  }
}

// out[i] = sum over rows of process i, fixed order: one warp per process
__global__ void segment_sum_kernel(const double* sq, const long long* seg, int nseg, double* out) {
  const int i = blockIdx.x;
  if (i >= nseg) return;
  double s = 0.0;
  for (long long r = seg[i] + threadIdx.x; r < seg[i + 1]; r += 32) s += sq[r];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[i] = s;
}

}  // namespace stbta

using namespace stbta;

static inline int grid_for(long long work, int per_block, int cap) {
  long long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

extern "C" {

int stbta_assemble_tile_elems(void) { return ASM_TILE; }

int stbta_assemble(double* data, long long nstore, const long long* tile_start, const long long* offsets,
                   const int* pair, const int* src, const double* basis, const double* coef, int nterms,
                   void* stream) {
  if (data == nullptr || nstore <= 0 || tile_start == nullptr || nterms < 1) return STBTA_EARG;
  const long long ntiles = (nstore + ASM_TILE - 1) / ASM_TILE;
  EntryTable t{offsets, pair, src, basis, coef, nterms};
  assemble_kernel<<<grid_for(ntiles, 1, 148 * 16), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      data, nstore, tile_start, ntiles, t);
  count_launch();
  return (int)cudaGetLastError();
}

int stbta_quadform(const long long* offsets, const int* pair, const int* src, const double* basis,
                   const double* coef, int nterms, long long nentries, int n, int b, int a,
                   const double* x, double* partial, int npartial, double* out, void* stream) {
  if (npartial < 1 || out == nullptr) return STBTA_EARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  EntryTable t{offsets, pair, src, basis, coef, nterms};
  const int g = grid_for(nentries, 256, npartial);
  quadform_kernel<<<g, 256, 0, st>>>(t, nentries, n, b, a, x, partial);
  count_launch();
  ordered_sum_kernel<<<1, 32, 0, st>>>(partial, g, out);
  count_launch();
  return (int)cudaGetLastError();
}

int stbta_rhs_combine(double* out, const double* U, const double* tau, int nv, long long N,
                      void* stream) {
  rhs_combine_kernel<<<grid_for(N, 256, 148 * 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      out, U, tau, nv, N);
  count_launch();
  return (int)cudaGetLastError();
}

int stbta_residual(const long long* indptr, const int* indices, const double* vals, long long nrows,
                   const double* y, const double* x, const long long* seg, int nseg, double* sq,
                   double* out, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nrows > 0) {
    residual_kernel<<<grid_for(nrows, 256, 148 * 8), 256, 0, st>>>(indptr, indices, vals, nrows, y,
                                                                   x, sq);
    count_launch();
  }
  if (nseg > 0) {
    segment_sum_kernel<<<nseg, 32, 0, st>>>(sq, seg, nseg, out);
    count_launch();
  }
  return (int)cudaGetLastError();
}

}  // extern "C"
