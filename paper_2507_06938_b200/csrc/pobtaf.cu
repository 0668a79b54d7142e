// POBTAF: in-place block Cholesky of an SPD BTA matrix (C ABI).
//
// Reference: bta.factorize (pkg/src/stinla/bta.py:177-235), per time block i
//   diag[i]    = chol(diag[i])                                  (bta.py:206)
//   lower[i]   = lower[i] diag[i]^-T,  arrow[i] = arrow[i] diag[i]^-T  (213-219)
//   diag[i+1] -= lower[i] lower[i]^T;  arrow[i+1] -= arrow[i] lower[i]^T;
//   tip       -= arrow[i] arrow[i]^T                             (222-227)
// then tip = chol(tip) (bta.py:228-232), and logdet (bta.py:238-246).
//
// B200 mapping: the panel S_i = [lower[i]; arrow[i]] is one segmented operand,
// so the TRSM is one recursive DMMA sweep over b + a rows and the Schur update
// of [diag[i+1]; arrow[i+1]; tip] is ONE lower-triangular DMMA launch with
// K = b.  Log-det partials are written per 64-leaf and summed once in a fixed
// order; failures go to a device word, so the whole factorization is issued
// without a host synchronisation.
#include <cstring>

#include "../../include/stbta.h"
#include "stbta_internal.cuh"

namespace stbta {

struct BtaView {
  double *diag, *lower, *arrow, *tip;
  int n, b, a;
  explicit BtaView(double* data, int n_, int b_, int a_) : n(n_), b(b_), a(a_) {
    const long long bb = (long long)b * b;
    diag = data;
    lower = diag + n * bb;
    arrow = lower + (long long)(n - 1) * bb;
    tip = arrow + (long long)n * a * b;
  }
  double* D(int i) const { return diag + (long long)i * b * b; }
  double* Lo(int i) const { return lower + (long long)i * b * b; }
  double* Ar(int i) const { return arrow + (long long)i * a * b; }
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct PobtafWs {
  double* winv;
  double* slots;
  int nslots;
};

static size_t pobtaf_ws(int n, int b, int a, char* base, PobtafWs* out) {
  const int nl = leaves_of(b > a ? b : a);
  const int nslots = n * leaves_of(b) + (a > 0 ? leaves_of(a) : 0);
  size_t off = 0;
  const size_t w = align_up((size_t)nl * LEAF * LEAF * sizeof(double));
  const size_t s = align_up((size_t)(nslots > 0 ? nslots : 1) * sizeof(double));
  if (out) {
    out->winv = reinterpret_cast<double*>(base + off);
    out->slots = reinterpret_cast<double*>(base + off + w);
    out->nslots = nslots;
  }
  off += w + s;
  return off;
}

}  // namespace stbta

using namespace stbta;

extern "C" {

const char* stbta_version(void) { return "stbta 0.1.0 (sm_100a, FP64 DMMA)"; }

long long stbta_storage_elems(int n, int b, int a) {
  return (long long)n * b * b + (long long)(n - 1) * b * b + (long long)n * a * b +
         (long long)a * a;
}

size_t stbta_pobtaf_workspace_bytes(int n, int b, int a) {
  if (n < 1 || b < 1 || a < 0) return 0;
  return pobtaf_ws(n, b, a, nullptr, nullptr);
}

int stbta_pobtaf(double* data, int n, int b, int a, int use_arrow, double* logdet_out, int* info,
                 void* workspace, size_t workspace_bytes, void* stream) {
  if (data == nullptr || n < 1 || b < 1 || a < 0 || info == nullptr) return STBTA_EARG;
  if (workspace_bytes < stbta_pobtaf_workspace_bytes(n, b, a)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtafWs ws;
  pobtaf_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  BtaView m(data, n, b, a);
  const bool arrow = use_arrow && a > 0;
  const int lb = leaves_of(b);

  int e = (int)cudaMemsetAsync(info, 0, sizeof(int), st);
  if (e) return e;
  DenseCtx c{st, info, ws.winv, ws.slots};

  for (int i = 0; i < n; ++i) {
    e = potrf_rec(c, m.D(i), b, b, 0, i * lb, i + 1);
    if (e) return e;
    e = launch_zero_upper(m.D(i), b, b, info, st);
    if (e) return e;
    // panel S_i = [lower[i]; arrow[i]]  :=  S_i L_ii^-T
    SegMat S;
    int rows = 0;
    if (i < n - 1) {
      S = arrow ? seg2(m.Lo(i), b, b, m.Ar(i), b) : seg1(m.Lo(i), b);
      rows = b + (arrow ? a : 0);
    } else if (arrow) {
      S = seg1(m.Ar(i), b);
      rows = a;
    }
    if (rows == 0) continue;
    e = trsm_rlt_rec(c, S, rows, m.D(i), b, b, 0);
    if (e) return e;
    // Schur update of [diag[i+1]; arrow[i+1] | tip] by S_i S_i^T (lower part)
    GemmArgs g{};
    g.A = S;
    g.B = S;
    g.M = rows;
    g.N = rows;
    g.K = b;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.c_lower = 1;
    g.info = info;
    g.batch = 1;
    if (i < n - 1) {
      g.C = seg2(m.D(i + 1), b, b, m.Ar(i + 1), b);
      g.C.p2 = m.tip;
      g.C.ld2 = a;
      g.C.c0 = b;
    } else {
      g.C = seg1(m.tip, a);
    }
    e = gemm_launch(g, false, true, st);
    if (e) return e;
  }
  if (a > 0) {
    e = potrf_rec(c, m.tip, a, a, 0, n * lb, n + 1);
    if (e) return e;
    e = launch_zero_upper(m.tip, a, a, info, st);
    if (e) return e;
  }
  if (logdet_out != nullptr) {
    e = launch_logdet_reduce(ws.slots, ws.nslots, logdet_out, st);
    if (e) return e;
  }
  return 0;
}

int stbta_dgemm(int ta, int tb, int M, int N, int K, double alpha, const double* A, long long lda,
                const double* B, long long ldb, double beta, double* C, long long ldc,
                void* stream) {
  if (M < 0 || N < 0 || K < 0) return STBTA_EARG;
  GemmArgs g{};
  g.A = seg1(const_cast<double*>(A), lda);
  g.B = seg1(const_cast<double*>(B), ldb);
  g.C = seg1(C, ldc);
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha; g.beta = beta;
  g.batch = 1;
  return gemm_launch(g, ta != 0, tb != 0, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
