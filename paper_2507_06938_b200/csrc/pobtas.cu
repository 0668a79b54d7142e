// POBTAS: forward / backward block substitution against a POBTAF factor.
//
// Reference: bta.forward_substitute (pkg/src/stinla/bta.py:249-275),
// bta.backward_substitute (bta.py:278-302), bta.solve (bta.py:305-307).
//
// B200 mapping.  The block-bidiagonal part of L (diag + lower blocks) is a
// banded lower-triangular matrix; each sweep is ONE persistent-style launch
// over 64-row chunks.  A chunk takes a ticket from an atomic counter (so a
// chunk only ever waits on chunks that are already running: no deadlock),
// streams its row band of L from HBM (prefetched into registers before it waits
// on the producer flag of the matching solution chunk), then solves its 64x64
// diagonal tile in a warp.  The only sequential part is that 64x64 tile and a
// flag hand-off; everything else streams the factor at HBM rate.  The arrow
// rows / tip (a <= 64) are a fixed-order reduction plus an a x a solve.
#include "../../include/stbta.h"
#include "common.cuh"
#include "stbta_internal.cuh"

namespace stbta {

constexpr int CH = 64;     // chunk rows (== LEAF)
constexpr int NRMAX = 8;   // right-hand sides per sweep launch

struct SweepArgs {
  const double* diag;
  const double* lower;
  const double* arrow;
  const double* tip;
  int n, b, a, nck, has_arrow;
  double* x;          // rhs / solution, row-major (dim x ldx), columns [0, ncols)
  long long ldx;
  int ncols;
  int* flags;         // one per chunk, zeroed before the launch
  int* ticket;        // zeroed before the launch
};

STBTA_DEV int acquire_ld(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
STBTA_DEV void release_st(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
STBTA_DEV void wait_flag(const int* f) {
  if (threadIdx.x == 0) {
    while (acquire_ld(f) == 0) __nanosleep(64);
  }
  __syncthreads();
}

// ------------------------------------------------------------ forward sweep
// chunk (i, j): rows ib + 64j + [0, rows).  y_R = L_RR^-1 (r_R - sum_deps L_R,D y_D)
__global__ void __launch_bounds__(256) fwd_sweep_kernel(SweepArgs p) {
  __shared__ int s_k;
  __shared__ double ys[CH][NRMAX];
  __shared__ double Ls[CH][CH + 1];
  __shared__ double accs[CH][NRMAX];
  const int tid = threadIdx.x;
  if (tid == 0) s_k = atomicAdd(p.ticket, 1);
  __syncthreads();
  const int k = s_k;
  const int i = k / p.nck, j = k % p.nck;
  const int b = p.b;
  const int rows = min(CH, b - j * CH);
  const long long grow0 = (long long)i * b + (long long)j * CH;
  const int rr = tid >> 2, q = tid & 3;
  const int nc = p.ncols;

  double acc[NRMAX];
#pragma unroll
  for (int r = 0; r < NRMAX; ++r) acc[r] = 0.0;

  // dependency list: all chunks of block i-1 (through lower[i-1]), then chunks
  // 0..j-1 of block i (through diag[i])
  const int ndep = (i > 0 ? p.nck : 0) + j;
  for (int d = 0; d < ndep; ++d) {
    int bi, bj;
    const double* M;
    if (i > 0 && d < p.nck) {
      bi = i - 1; bj = d; M = p.lower + (long long)(i - 1) * b * b;
    } else {
      bi = i; bj = d - (i > 0 ? p.nck : 0); M = p.diag + (long long)i * b * b;
    }
    const int c0 = bj * CH;
    const int dcols = min(CH, b - c0);
    // prefetch this thread's 16 entries of the L row band before waiting
    double lv[16];
    const bool row_ok = rr < rows;
    const double* mrow = M + (long long)(j * CH + rr) * b + c0 + q * 16;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int col = q * 16 + t;
      lv[t] = (row_ok && col < dcols) ? __ldg(mrow + t) : 0.0;
    }
    wait_flag(p.flags + bi * p.nck + bj);
    const long long drow0 = (long long)bi * b + c0;
    for (int e = tid; e < CH * NRMAX; e += 256) {
      const int t = e / NRMAX, r = e % NRMAX;
      ys[t][r] = (t < dcols && r < nc) ? __ldcg(p.x + (drow0 + t) * p.ldx + r) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
      for (int r = 0; r < NRMAX; ++r) acc[r] -= lv[t] * ys[q * 16 + t][r];
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < NRMAX; ++r) {
    acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 1);
    acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 2);
  }
  if (q == 0) {
#pragma unroll
    for (int r = 0; r < NRMAX; ++r)
      accs[rr][r] = (rr < rows && r < nc) ? __ldcg(p.x + (grow0 + rr) * p.ldx + r) + acc[r] : 0.0;
  }
  const double* Dt = p.diag + (long long)i * b * b + (long long)(j * CH) * b + j * CH;
  for (int e = tid; e < CH * CH; e += 256) {
    const int r = e / CH, c = e % CH;
    Ls[r][c] = (r < rows && c <= r) ? Dt[(long long)r * b + c] : 0.0;
  }
  __syncthreads();
  if (tid < 32) {  // warp substitution, lanes own rows lane and lane+32
    const int l = tid;
    double v0[NRMAX], v1[NRMAX];
#pragma unroll
    for (int r = 0; r < NRMAX; ++r) { v0[r] = accs[l][r]; v1[r] = accs[l + 32][r]; }
    for (int t = 0; t < rows; ++t) {
      const double inv = 1.0 / Ls[t][t];
      const double m0 = Ls[l][t], m1 = Ls[l + 32][t];
#pragma unroll
      for (int r = 0; r < NRMAX; ++r) {
        const double own = (t < 32) ? v0[r] : v1[r];
        const double yt = __shfl_sync(0xffffffffu, own, t & 31) * inv;
        if (l == (t & 31)) { if (t < 32) v0[r] = yt; else v1[r] = yt; }
        if (l > t) v0[r] -= m0 * yt;
        if (l + 32 > t) v1[r] -= m1 * yt;
      }
    }
#pragma unroll
    for (int r = 0; r < NRMAX; ++r) {
      if (r < nc) {
        if (l < rows) p.x[(grow0 + l) * p.ldx + r] = v0[r];
        if (l + 32 < rows) p.x[(grow0 + l + 32) * p.ldx + r] = v1[r];
      }
    }
    __syncwarp();
    if (tid == 0) {
      __threadfence();
      release_st(p.flags + k, 1);
    }
  }
}

// ----------------------------------------------------------- backward sweep
// chunk (i, j) in reverse order: x_R = L_RR^-T (y_R - sum L_D,R^T x_D - A_R^T x_tip)
__global__ void __launch_bounds__(256) bwd_sweep_kernel(SweepArgs p, const double* xtip) {
  __shared__ int s_k;
  __shared__ double xs[CH][NRMAX];
  __shared__ double big[CH * (CH + 1)];  // partial sums first, then the diagonal tile
  double(*Ls)[CH + 1] = reinterpret_cast<double(*)[CH + 1]>(big);
  double(*part)[CH][NRMAX] = reinterpret_cast<double(*)[CH][NRMAX]>(big);
  const int tid = threadIdx.x;
  const int total = p.n * p.nck;
  if (tid == 0) s_k = total - 1 - atomicAdd(p.ticket, 1);
  __syncthreads();
  const int k = s_k;
  const int i = k / p.nck, j = k % p.nck;
  const int b = p.b;
  const int cols = min(CH, b - j * CH);  // rows of this chunk == columns of L used
  const long long grow0 = (long long)i * b + (long long)j * CH;
  const int c = tid & 63, rq = tid >> 6;
  const int nc = p.ncols;

  double acc[NRMAX];
#pragma unroll
  for (int r = 0; r < NRMAX; ++r) acc[r] = 0.0;

  // dependencies, earliest-finished first: chunks of block i+1 (through
  // lower[i]) from the last one down, then chunks j+1.. of block i (diag[i])
  const int nnext = (i + 1 < p.n) ? p.nck : 0;
  const int nself = p.nck - 1 - j;
  for (int d = 0; d < nnext + nself; ++d) {
    int bi, bj;
    const double* M;
    if (d < nnext) {
      bi = i + 1; bj = p.nck - 1 - d; M = p.lower + (long long)i * b * b;
    } else {
      bi = i; bj = p.nck - 1 - (d - nnext); M = p.diag + (long long)i * b * b;
    }
    const int r0 = bj * CH;
    const int drows = min(CH, b - r0);
    double lv[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int rloc = rq * 16 + t;
      lv[t] = (c < cols && rloc < drows) ? __ldg(M + (long long)(r0 + rloc) * b + j * CH + c) : 0.0;
    }
    wait_flag(p.flags + bi * p.nck + bj);
    const long long drow0 = (long long)bi * b + r0;
    for (int e = tid; e < CH * NRMAX; e += 256) {
      const int t = e / NRMAX, r = e % NRMAX;
      xs[t][r] = (t < drows && r < nc) ? __ldcg(p.x + (drow0 + t) * p.ldx + r) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
#pragma unroll
      for (int r = 0; r < NRMAX; ++r) acc[r] -= lv[t] * xs[rq * 16 + t][r];
    }
    __syncthreads();
  }
  // arrow coupling: x_R -= arrow[i][:, R]^T x_tip  (bta.py:297-298)
  if (p.has_arrow && rq == 0 && c < cols) {
    const double* A = p.arrow + (long long)i * p.a * b + j * CH + c;
    for (int t = 0; t < p.a; ++t) {
      const double av = A[(long long)t * b];
#pragma unroll
      for (int r = 0; r < NRMAX; ++r)
        if (r < nc) acc[r] -= av * xtip[t * NRMAX + r];
    }
  }
#pragma unroll
  for (int r = 0; r < NRMAX; ++r) part[rq][c][r] = acc[r];
  __syncthreads();
  double v0[NRMAX], v1[NRMAX];
  const int l = tid & 31;
  if (tid < 32) {
#pragma unroll
    for (int r = 0; r < NRMAX; ++r) {
      const double y0 = (l < cols && r < nc) ? __ldcg(p.x + (grow0 + l) * p.ldx + r) : 0.0;
      const double y1 = (l + 32 < cols && r < nc) ? __ldcg(p.x + (grow0 + l + 32) * p.ldx + r) : 0.0;
      v0[r] = y0 + ((part[0][l][r] + part[1][l][r]) + (part[2][l][r] + part[3][l][r]));
      v1[r] = y1 + ((part[0][l + 32][r] + part[1][l + 32][r]) +
                    (part[2][l + 32][r] + part[3][l + 32][r]));
    }
  }
  __syncthreads();
  const double* Dt = p.diag + (long long)i * b * b + (long long)(j * CH) * b + j * CH;
  for (int e = tid; e < CH * CH; e += 256) {
    const int r = e / CH, cc = e % CH;
    Ls[r][cc] = (r < cols && cc <= r) ? Dt[(long long)r * b + cc] : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    for (int t = cols - 1; t >= 0; --t) {
      const double inv = 1.0 / Ls[t][t];
      const double m0 = Ls[t][l], m1 = Ls[t][l + 32];  // (L^T)[l][t] = L[t][l]
#pragma unroll
      for (int r = 0; r < NRMAX; ++r) {
        const double own = (t < 32) ? v0[r] : v1[r];
        const double xt = __shfl_sync(0xffffffffu, own, t & 31) * inv;
        if (l == (t & 31)) { if (t < 32) v0[r] = xt; else v1[r] = xt; }
        if (l < t) v0[r] -= m0 * xt;
        if (l + 32 < t) v1[r] -= m1 * xt;
      }
    }
#pragma unroll
    for (int r = 0; r < NRMAX; ++r) {
      if (r < nc) {
        if (l < cols) p.x[(grow0 + l) * p.ldx + r] = v0[r];
        if (l + 32 < cols) p.x[(grow0 + l + 32) * p.ldx + r] = v1[r];
      }
    }
    __syncwarp();
    if (tid == 0) {
      __threadfence();
      release_st(p.flags + k, 1);
    }
  }
}

// -------------------------------------------------------------- arrow / tip
// partial[g][t][r] = sum over this CTA's columns of arrow[t][col] * y[col][r]
__global__ void __launch_bounds__(256) arrow_partial_kernel(SweepArgs p, double* partial,
                                                            int cols_per_cta) {
  const int tid = threadIdx.x;
  const long long N = (long long)p.n * p.b;
  const long long c_beg = (long long)blockIdx.x * cols_per_cta;
  const long long c_end = min(N, c_beg + cols_per_cta);
  const int a = p.a, nc = p.ncols;
  for (int t = 0; t < a; ++t) {
    for (int r = 0; r < nc; ++r) {
      double s = 0.0;
      for (long long col = c_beg + tid; col < c_end; col += 256) {
        const long long blk = col / p.b, cc = col % p.b;
        s += p.arrow[(blk * a + t) * p.b + cc] * p.x[col * p.ldx + r];
      }
      s = warp_sum(s);
      __shared__ double wsum[8];
      if ((tid & 31) == 0) wsum[tid >> 5] = s;
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < 8; ++w) tot += wsum[w];
        partial[((long long)blockIdx.x * a + t) * NRMAX + r] = tot;
      }
      __syncthreads();
    }
  }
}

// mode 0 (forward): y_tip = L_tip^-1 (r_tip - sum_g partial[g]);  mode 1: x_tip = L_tip^-T y_tip.
// Works in place on the tip segment of x (any arrow size) and writes a packed
// copy xtip[a][NRMAX] for the backward sweep's arrow coupling.
__global__ void tip_solve_kernel(SweepArgs p, const double* partial, int nparts, double* xtip,
                                 int mode) {
  const int r = threadIdx.x;
  if (r >= p.ncols) return;
  const int a = p.a;
  const long long base = (long long)p.n * p.b;
  double* v = p.x + base * p.ldx + r;  // v[t * ldx]
  const long long ld = p.ldx;
  if (mode == 0 && p.has_arrow && partial != nullptr) {
    for (int t = 0; t < a; ++t) {
      double tot = 0.0;
      for (int g = 0; g < nparts; ++g) tot += partial[((long long)g * a + t) * NRMAX + r];
      v[t * ld] -= tot;
    }
  }
  if (mode == 0) {
    for (int t = 0; t < a; ++t) {
      double s = v[t * ld];
      for (int u = 0; u < t; ++u) s -= p.tip[(long long)t * a + u] * v[u * ld];
      v[t * ld] = s / p.tip[(long long)t * a + t];
    }
  } else {
    for (int t = a - 1; t >= 0; --t) {
      double s = v[t * ld];
      for (int u = t + 1; u < a; ++u) s -= p.tip[(long long)u * a + t] * v[u * ld];
      v[t * ld] = s / p.tip[(long long)t * a + t];
    }
  }
  for (int t = 0; t < a; ++t) xtip[t * NRMAX + r] = v[t * ld];
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
static constexpr int ARROW_PARTS = 148 * 2;

struct PobtasWs {
  int* flags;
  int* ticket;
  double* partial;
  double* xtip;
};

static size_t pobtas_ws(int n, int b, int a, char* base, PobtasWs* o) {
  const int nck = ceil_div(b, CH);
  size_t off = 0;
  const size_t f = align_up((size_t)n * nck * sizeof(int));
  const size_t t = align_up(sizeof(int) * 2);
  const size_t pa = align_up((size_t)ARROW_PARTS * (a > 0 ? a : 1) * NRMAX * sizeof(double));
  const size_t xt = align_up((size_t)(a > 0 ? a : 1) * NRMAX * sizeof(double));
  if (o) {
    o->flags = reinterpret_cast<int*>(base);
    o->ticket = reinterpret_cast<int*>(base + f);
    o->partial = reinterpret_cast<double*>(base + f + t);
    o->xtip = reinterpret_cast<double*>(base + f + t + pa);
  }
  off = f + t + pa + xt;
  return off;
}

static int run_sweeps(const SweepArgs& base_args, int mode, const PobtasWs& ws, cudaStream_t st) {
  SweepArgs p = base_args;
  const int total = p.n * p.nck;
  const size_t fbytes = (size_t)total * sizeof(int);
  int e;
  if (mode == 0 || mode == 1) {
    if ((e = (int)cudaMemsetAsync(p.flags, 0, fbytes, st))) return e;
    if ((e = (int)cudaMemsetAsync(p.ticket, 0, sizeof(int), st))) return e;
    fwd_sweep_kernel<<<total, 256, 0, st>>>(p);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
    if (p.a > 0) {
      int parts = 0;
      if (p.has_arrow) {
        const long long N = (long long)p.n * p.b;
        const int cpc = (int)((N + ARROW_PARTS - 1) / ARROW_PARTS);
        parts = (int)((N + cpc - 1) / cpc);
        arrow_partial_kernel<<<parts, 256, 0, st>>>(p, ws.partial, cpc);
        count_launch();
        if ((e = (int)cudaGetLastError())) return e;
      }
      tip_solve_kernel<<<1, NRMAX, 0, st>>>(p, ws.partial, parts, ws.xtip, 0);
      count_launch();
      if ((e = (int)cudaGetLastError())) return e;
    }
  }
  if (mode == 0 || mode == 2) {
    if (p.a > 0) {
      tip_solve_kernel<<<1, NRMAX, 0, st>>>(p, nullptr, 0, ws.xtip, 1);
      count_launch();
      if ((e = (int)cudaGetLastError())) return e;
    }
    if ((e = (int)cudaMemsetAsync(p.flags, 0, fbytes, st))) return e;
    if ((e = (int)cudaMemsetAsync(p.ticket, 0, sizeof(int), st))) return e;
    bwd_sweep_kernel<<<total, 256, 0, st>>>(p, ws.xtip);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
  }
  return 0;
}

}  // namespace stbta

using namespace stbta;

extern "C" {

size_t stbta_pobtas_workspace_bytes(int n, int b, int a, int nrhs) {
  (void)nrhs;
  if (n < 1 || b < 1 || a < 0) return 0;
  return pobtas_ws(n, b, a, nullptr, nullptr);
}

int stbta_pobtas(const double* factor, int n, int b, int a, int has_arrow, double* rhs, int nrhs,
                 int mode, void* workspace, size_t workspace_bytes, void* stream) {
  if (factor == nullptr || rhs == nullptr || n < 1 || b < 1 || a < 0 ||
      nrhs < 1 || mode < 0 || mode > 2)
    return STBTA_EARG;
  if (workspace_bytes < stbta_pobtas_workspace_bytes(n, b, a, nrhs)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtasWs ws;
  pobtas_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  const long long bb = (long long)b * b;
  SweepArgs p{};
  p.diag = factor;
  p.lower = factor + n * bb;
  p.arrow = p.lower + (long long)(n - 1) * bb;
  p.tip = p.arrow + (long long)n * a * b;
  p.n = n; p.b = b; p.a = a;
  p.nck = ceil_div(b, CH);
  p.has_arrow = has_arrow && a > 0;
  p.ldx = nrhs;
  p.flags = ws.flags;
  p.ticket = ws.ticket;
  for (int c0 = 0; c0 < nrhs; c0 += NRMAX) {
    p.x = rhs + c0;
    p.ncols = nrhs - c0 < NRMAX ? nrhs - c0 : NRMAX;
    int e = run_sweeps(p, mode, ws, st);
    if (e) return e;
  }
  return 0;
}

}  // extern "C"
