// CTA-level FP64 DMMA tile product for the persistent task-graph kernels:
//
//   acc(BM x BN) = A(BM x K) * B(BN x K)^T        ("NT": both operands K-contiguous)
//
// Operands are row sets of BTA storage (row r at p + r*ld).  K is staged
// through a STAGES-deep cp.async ring of BK-wide slabs in shared memory
// (16-byte copies when rows are 16-byte aligned, 8-byte otherwise; rows >=
// `rows` and columns >= K are zero-filled), and every warp accumulates its
// WM x WN sub-tile as (WM/8) x (WN/8) DMMA.8x8x4 fragments.  A 4-double row
// pad makes every fragment load conflict-free (two wavefronts per 256 B).
#pragma once

#include "common.cuh"

namespace stbta {

struct Opnd {
  const double* p;
  long long ld;
  int rows;  // valid rows (rest read as zero)
  int vec;   // 16-byte copies allowed
};

template <int BM_, int BN_, int WM_, int WN_, int NT_, int BK_ = 16, int ST_ = 4>
struct MmaCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, NT = NT_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static_assert(WARPS_M * WARPS_N * 32 == NT, "warp layout must cover the CTA");
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int BK = BK_, STAGES = ST_, LDS = BK + 4;
  // [k][m] (k-major) staging of an operand stored K x M in memory
  static constexpr int LDA_KM = BM + 4, LDB_KM = BN + 4;
  static constexpr int A_STAGE = (BM * LDS > BK * LDA_KM ? BM * LDS : BK * LDA_KM);
  static constexpr int B_STAGE = (BN * LDS > BK * LDB_KM ? BN * LDS : BK * LDB_KM);
  static constexpr int SMEM_DOUBLES = STAGES * (A_STAGE + B_STAGE);
};

// Slab of an operand stored k-major (element (row, k) at p[k * ld + row]):
// BK k-rows x ROWS columns into sm[k][row] with row stride ROWS + 4.
template <int ROWS, int NT, int BK>
STBTA_DEV void load_slab_km(double* sm, const Opnd& o, int k0, int K) {
  constexpr int LD = ROWS + 4;
  const int tid = threadIdx.x;
  if (o.vec) {
    constexpr int PAIRS = BK * ROWS / 2;
#pragma unroll
    for (int e = tid; e < PAIRS; e += NT) {
      const int k = e / (ROWS / 2), c = (e % (ROWS / 2)) * 2;
      const int gk = k0 + k;
      int bytes = 0;
      const double* src = o.p;
      if (gk < K && c < o.rows) {
        bytes = (c + 1 < o.rows) ? 16 : 8;
        src = o.p + (long long)gk * o.ld + c;
      }
      cp_async16(sm + k * LD + c, src, bytes);
    }
  } else {
    constexpr int ELEMS = BK * ROWS;
#pragma unroll
    for (int e = tid; e < ELEMS; e += NT) {
      const int k = e / ROWS, c = e % ROWS;
      const int gk = k0 + k;
      const bool ok = gk < K && c < o.rows;
      cp_async8(sm + k * LD + c, ok ? o.p + (long long)gk * o.ld + c : o.p, ok);
    }
  }
}

template <int ROWS, int NT, int BK = 16>
STBTA_DEV void load_slab(double* sm, const Opnd& o, int k0, int K) {
  constexpr int LDS = BK + 4;
  constexpr int HP = BK / 2;  // 16-byte pairs per row
  const int tid = threadIdx.x;
  if (o.vec) {
    constexpr int PAIRS = ROWS * HP;
#pragma unroll
    for (int e = tid; e < PAIRS; e += NT) {
      const int r = e / HP, c = (e % HP) * 2;
      const int gc = k0 + c;
      int bytes = 0;
      const double* src = o.p;
      if (r < o.rows && gc < K) {
        bytes = (gc + 1 < K) ? 16 : 8;
        src = o.p + (long long)r * o.ld + gc;
      }
      cp_async16(sm + r * LDS + c, src, bytes);
    }
  } else {
    constexpr int ELEMS = ROWS * BK;
#pragma unroll
    for (int e = tid; e < ELEMS; e += NT) {
      const int r = e / BK, c = e % BK;
      const int gc = k0 + c;
      const bool ok = r < o.rows && gc < K;
      cp_async8(sm + r * LDS + c, ok ? o.p + (long long)r * o.ld + gc : o.p, ok);
    }
  }
}

// acc += A * B^T over k in [0, K).  `n_active`: warps whose first output
// column is >= n_active skip the arithmetic (triangular strips).  All threads
// of the CTA must call; smem holds Cfg::SMEM_DOUBLES doubles.  Ends with a
// __syncthreads so the caller may reuse shared memory.
struct NoInit {
  STBTA_DEV void operator()() const {}
};

// `init` runs after the prologue's slab copies are issued (e.g. the
// accumulator's C-tile load), so its latency overlaps theirs.
template <class Cfg, bool NEG = false, int DBG = 0, bool AKM = false, bool BKM = false,
          class Init = NoInit>
STBTA_DEV void tile_mma(double (&acc)[Cfg::MF][Cfg::NF][2], const Opnd& A, const Opnd& B, int K,
                        int n_active, double* smem, int kbeg = 0, const Init& init = Init()) {
  constexpr int MF = Cfg::MF, NF = Cfg::NF, BK = Cfg::BK, ST = Cfg::STAGES, LDS = Cfg::LDS;
  double* As = smem;
  double* Bs = smem + ST * Cfg::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const bool active = wn0 < n_active;
  const int ktiles = (K - kbeg + BK - 1) / BK;
  auto load_stage = [&](int slot, int k0) {
    if (AKM) load_slab_km<Cfg::BM, Cfg::NT, Cfg::BK>(As + slot * Cfg::A_STAGE, A, k0, K);
    else load_slab<Cfg::BM, Cfg::NT, Cfg::BK>(As + slot * Cfg::A_STAGE, A, k0, K);
    if (BKM) load_slab_km<Cfg::BN, Cfg::NT, Cfg::BK>(Bs + slot * Cfg::B_STAGE, B, k0, K);
    else load_slab<Cfg::BN, Cfg::NT, Cfg::BK>(Bs + slot * Cfg::B_STAGE, B, k0, K);
  };

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < ktiles) load_stage(s, kbeg + s * BK);
    cp_async_commit();
  }
  init();
  for (int kt = 0; kt < ktiles; ++kt) {
    if (DBG != 1) {  // DBG 1: no waits/barriers (timing experiment only)
      cp_async_wait<ST - 2>();
      __syncthreads();
    }
    const int nt = kt + ST - 1;
    if (DBG != 2 && nt < ktiles) load_stage(nt % ST, kbeg + nt * BK);  // DBG 2: no loads
    cp_async_commit();
    if (active) {
      const double* as = As + (kt % ST) * Cfg::A_STAGE;
      const double* bs = Bs + (kt % ST) * Cfg::B_STAGE;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int k = ks * 4 + tq;
        double af[MF], bf[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i)
          af[i] = AKM ? as[k * Cfg::LDA_KM + wm0 + i * 8 + gq] : as[(wm0 + i * 8 + gq) * LDS + k];
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const double bv =
              BKM ? bs[k * Cfg::LDB_KM + wn0 + j * 8 + gq] : bs[(wn0 + j * 8 + gq) * LDS + k];
          bf[j] = NEG ? -bv : bv;
        }
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
          for (int j = 0; j < NF; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

template <class Cfg>
STBTA_DEV void acc_zero(double (&acc)[Cfg::MF][Cfg::NF][2]) {
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// acc = C[m][n] for m < rows, n < cols (and n <= m + diag when lower), else 0.
// All loads are issued before any use, so their latency overlaps.
template <class Cfg>
STBTA_DEV void acc_load(double (&acc)[Cfg::MF][Cfg::NF][2], const double* C, long long ldc,
                        int rows, int cols, int lower, int diag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const bool vec = ((uintptr_t)C % 16 == 0) && (ldc % 2 == 0);
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i) {
    const int m = wm0 + i * 8 + gq;
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) {
      const int n0 = wn0 + j * 8 + 2 * tq;
      const double* src = C + (long long)m * ldc + n0;
      const bool full = vec && m < rows && n0 + 1 < cols && !(lower && n0 + 1 > m + diag);
      if (full) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src));
        acc[i][j][0] = v.x;
        acc[i][j][1] = v.y;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int nn = n0 + e;
          const bool ok = m < rows && nn < cols && !(lower && nn > m + diag);
          acc[i][j][e] = ok ? __ldcg(src + e) : 0.0;
        }
      }
    }
  }
}

// Epilogue: C[m][n] (op)= acc for m < rows, n < cols, and n <= m + diag when
// lower != 0.  op: 0 -> C = alpha*acc ; 1 -> C += alpha*acc.
template <class Cfg>
STBTA_DEV void acc_store(const double (&acc)[Cfg::MF][Cfg::NF][2], double* C, long long ldc,
                         int rows, int cols, int lower, int diag, int op, double alpha) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const bool vec = ((uintptr_t)C % 16 == 0) && (ldc % 2 == 0);
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i) {
    const int m = wm0 + i * 8 + gq;
    if (m >= rows) continue;
    double* crow = C + (long long)m * ldc;
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) {
      const int n0 = wn0 + j * 8 + 2 * tq;
      if (vec && !op && n0 + 1 < cols && !(lower && n0 + 1 > m + diag)) {
        *reinterpret_cast<double2*>(crow + n0) = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        continue;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nn = n0 + e;
        if (nn >= cols || (lower && nn > m + diag)) continue;
        double v = alpha * acc[i][j][e];
        if (op) v += __ldcg(crow + nn);
        crow[nn] = v;
      }
    }
  }
}

}  // namespace stbta

// ---------------------------------------------------------------------------
// Bulk-copy variant for full tiles (rows == BM/BN, K % BK == 0, 16-byte rows):
// warp 0 streams each BK-wide row segment with one cp.async.bulk (TMA engine,
// completion counted on a per-stage "full" mbarrier); warps release a stage
// on its "empty" mbarrier, so there is no CTA-wide barrier per K slab and the
// load issue costs 8 instructions per lane per slab instead of ~20 per thread.
// `slab` is the CTA's running slab counter (identical in every thread); it
// selects stage = slab % ST and the mbarrier parities, so the ring carries
// over from one task to the next.
namespace stbta {

STBTA_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

STBTA_DEV void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
STBTA_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
STBTA_DEV void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
STBTA_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
STBTA_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
STBTA_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

}  // namespace stbta
