// TMA-staged variant of tile_mma for 128 x 128 tiles whose operands are both
// K-contiguous row sets of a region described by a CUtensorMap (POBTAF UPDATE):
//
//   acc(128 x 128) (+)= A(128 x K) * B(128 x K)^T,   K % 32 == 0 or the K range
//   ending at the tensor's last column (the partial slab is zero-filled)
//
// Thread 0 streams each 32-wide K slab of A and B with four
// cp.async.bulk.tensor.2d copies (16 x 128 boxes, 128-byte swizzle) onto a
// per-stage mbarrier (complete_tx), so the global->shared traffic bypasses the
// LSU pipe that feeds the DMMA fragment loads; the 128-byte swizzle makes the
// 8x4 fragment reads conflict-free without padding.  Rows beyond the tile
// (partial tiles) come in as whatever lies there and only feed output rows /
// columns the caller does not store; columns >= the tensor width read as zero.
// The k-steps read the slab columns in the permuted order of tma_kp(), which
// keeps the fragment reads conflict-free.
#pragma once

#include <cuda.h>

#include "tile_mma.cuh"

namespace stbta {

struct TmaOpnd {
  const CUtensorMap* map;  // nullptr: not TMA-eligible
  int row, col;            // tile origin in the tensor (row, first K column)
};

constexpr int TMA_ST = 3;                      // pipeline stages
constexpr int TMA_HALF = 128 * 16;             // doubles per 16-column box
constexpr int TMA_OPND = 2 * TMA_HALF;         // one operand, one 32-wide slab
constexpr int TMA_STAGE = 2 * TMA_OPND;        // A + B
constexpr unsigned TMA_STAGE_BYTES = TMA_STAGE * 8;
constexpr int TMA_SMEM_DOUBLES = TMA_ST * TMA_STAGE + 128;  // + 1 KB alignment slack

STBTA_DEV void tma_load_2d(double* dst, const CUtensorMap* map, int col, int row,
                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}

// Offset of element (r, kp) of one operand's 32-wide slab (r = rb + gq, rb % 8
// == 0): row-major operands are two 16 x 128 boxes, k-major ones eight 16 x 32
// boxes, both 128-byte swizzled (16-byte chunk index ^= 128-byte row & 7).
template <bool KM>
STBTA_DEV int tma_off(int r, int kp) {
  if (!KM) return (kp >> 4) * TMA_HALF + r * 16 + ((((kp & 15) >> 1) ^ (r & 7)) << 1) + (kp & 1);
  return (r >> 4) * 512 + kp * 16 + ((((r & 15) >> 1) ^ (kp & 7)) << 1) + (r & 1);
}

// Physical slab column read by k-step ks (0..7) in lane quad position tq:
// kp = KB[ks] ^ O[tq], KB = {0,1,4,5,16,17,20,21}, O = {0,3,12,15} -- a
// permutation of 0..31 (the same for A and B, so the product is unchanged)
// under which every 64-bit fragment read is conflict-free in BOTH layouts:
// each half-warp (4 rows x 4 quads) must hit 16 distinct bank pairs, which
// needs kp bits {0,3} (row-major) and {1,2} (k-major) to take all four values
// across the quad (checked exhaustively in tests/test_host_logic.py).
// o4 = O[tq] = (tq & 1) * 3 + (tq >> 1) * 12.
STBTA_DEV int tma_kp(int ks, int o4) {
  return ((ks & 1) + ((ks >> 1) & 1) * 4 + (ks >> 2) * 16) ^ o4;
}

// 1 KB-aligned staging base inside `smem` (128-byte swizzle atoms are 1 KB).
STBTA_DEV double* tma_stage_base(double* smem) {
  const unsigned a = smem_u32(smem);
  return smem + (((a + 1023u) & ~1023u) - a) / 8;
}

// Call once per CTA before the first tile_mma_tma (thread 0 initialises).
// bars[0, TMA_ST): stage full (TMA bytes landed); bars[TMA_ST, 2 TMA_ST):
// stage consumed (one arrival per warp), which thread 0 waits on before it
// refills the stage -- so the warps never meet at a CTA barrier per slab.
constexpr int TMA_NBARS = 2 * TMA_ST;
STBTA_DEV void tma_bars_init(unsigned long long* bars) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < TMA_ST; ++s) mbar_init(bars + s, 1);
    for (int s = 0; s < TMA_ST; ++s) mbar_init(bars + TMA_ST + s, blockDim.x >> 5);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

// `phase`: per-stage parity bits, identical in all threads, carried across
// calls: bit s = full-barrier phase of stage s, bit 8 + s = uses of stage s
// consumed so far (mod 2), i.e. the consumed-barrier phase.
// Output rows >= mv / columns >= nv are not wanted by the caller: the warps'
// 8 x 8 fragments lying entirely beyond them skip their loads and DMMAs
// (partial last tiles, e.g. b = 5025 -> 33 columns, and the few arrow rows
// of an arrowhead tile row, a <= 8 of 128), which frees the SM's DMMA pipe
// for the useful fragments.
template <class Cfg>
STBTA_DEV int valid_frags(int v, int w0, int nf) {
  return min(nf, max(0, (v - w0 + 7) >> 3));
}

template <class Cfg, bool NEG = false, class Init = NoInit>
STBTA_DEV void tile_mma_tma(double (&acc)[Cfg::MF][Cfg::NF][2], const TmaOpnd& A,
                            const TmaOpnd& B, int K, double* smem, unsigned long long* bars,
                            unsigned& phase, const Init& init = Init(), int mv = 128,
                            int nv = 128) {
  static_assert(Cfg::BM == 128 && Cfg::BN == 128, "TMA path is laid out for 128 x 128 tiles");
  constexpr int MF = Cfg::MF, NF = Cfg::NF;
  double* base = tma_stage_base(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int nk = (K + 31) / 32;  // a partial last slab must end at the tensor edge (zero fill)
  const int mfv = valid_frags<Cfg>(mv, wm0, MF), nfv = valid_frags<Cfg>(nv, wn0, NF);
  const bool full = (mfv == MF) && (nfv == NF);
  auto issue = [&](int kt) {  // thread 0
    double* st = base + (kt % TMA_ST) * TMA_STAGE;
    unsigned long long* bar = bars + kt % TMA_ST;
    mbar_expect_tx(bar, TMA_STAGE_BYTES);
    const int k0 = kt * 32;
    tma_load_2d(st, A.map, A.col + k0, A.row, bar);
    tma_load_2d(st + TMA_HALF, A.map, A.col + k0 + 16, A.row, bar);
    tma_load_2d(st + TMA_OPND, B.map, B.col + k0, B.row, bar);
    tma_load_2d(st + TMA_OPND + TMA_HALF, B.map, B.col + k0 + 16, B.row, bar);
  };
  if (tid == 0) {
    // earlier generic-proxy shared-memory writes (other task kinds) before async writes
    asm volatile("fence.proxy.async;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < TMA_ST - 1; ++s)
      if (s < nk) issue(s);
  }
  init();
  const int o4 = (tq & 1) * 3 + (tq >> 1) * 12;  // see tma_kp()
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TMA_ST;
    mbar_wait(bars + s, (phase >> s) & 1u);
    phase ^= 1u << s;
    if (tid == 0 && kt + TMA_ST - 1 < nk) {
      // the stage refilled now was consumed at kt - 1: wait until every warp
      // has arrived on its consumed barrier (that use's phase completes)
      const int sr = (kt + TMA_ST - 1) % TMA_ST;
      if (kt >= 1) mbar_wait(bars + TMA_ST + sr, ((phase >> (8 + sr)) & 1u) ^ 1u);
      issue(kt + TMA_ST - 1);
    }
    const double* as = base + s * TMA_STAGE;
    const double* bs = as + TMA_OPND;
    if (full) {
      // fragments double-buffered in registers: k-step ks+1's loads are
      // issued before k-step ks's DMMAs, so their latency is off the pipe
      double af[2][MF], bf[2][NF];
      auto frag_load = [&](int ks, int b) {
        const int kp = tma_kp(ks, o4);
#pragma unroll
        for (int i = 0; i < MF; ++i) af[b][i] = as[tma_off<false>(wm0 + i * 8 + gq, kp)];
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const double bv = bs[tma_off<false>(wn0 + j * 8 + gq, kp)];
          bf[b][j] = NEG ? -bv : bv;
        }
      };
      frag_load(0, 0);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks + 1 < 8) frag_load(ks + 1, (ks + 1) & 1);
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
          for (int j = 0; j < NF; ++j)
            dmma884(acc[i][j][0], acc[i][j][1], af[ks & 1][i], bf[ks & 1][j]);
      }
    } else if (mfv > 0 && nfv > 0) {  // warp-uniform: only the wanted fragments
#pragma unroll 1
      for (int ks = 0; ks < 8; ++ks) {
        const int kp = tma_kp(ks, o4);
        double af[MF], bf[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) af[i] = i < mfv ? as[tma_off<false>(wm0 + i * 8 + gq, kp)] : 0.0;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const double bv = j < nfv ? bs[tma_off<false>(wn0 + j * 8 + gq, kp)] : 0.0;
          bf[j] = NEG ? -bv : bv;
        }
#pragma unroll
        for (int i = 0; i < MF; ++i) {
          if (i >= mfv) break;
#pragma unroll
          for (int j = 0; j < NF; ++j)
            if (j < nfv) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
    }
    __syncwarp();  // the warp's reads of stage s are done (arrive releases them)
    if (lane == 0) mbar_arrive(bars + TMA_ST + s);
    phase ^= 1u << (8 + s);
  }
  __syncthreads();
}

}  // namespace stbta

// ---------------------------------------------------------------------------
// General orientation (POBTASI tile jobs): each operand is either row-major
// (element (r, k) at p[r*ld + k]: tensor {K, rows, blocks}, 16 x 128 boxes) or
// k-major (element (r, k) at p[k*ld + r]: tensor {rows, K, blocks}, 16 x 32
// boxes), 128-byte swizzle in both cases.  To keep the fragment reads
// conflict-free for BOTH layouts, k-step ks reads physical slab columns
// kp = KB[ks] + {0, 1, 4, 5}[tq] (a permutation of 0..31, identical for A and
// B, so the product is unchanged): kp's bit 0 alternates across the lane
// quads (row-major: the two 8-byte halves of a chunk) and bit 2 alternates
// (k-major: the swizzle XOR moves between chunk groups).
namespace stbta {

struct TmaOpnd3 {
  const CUtensorMap* map;  // nullptr: not TMA-eligible
  int r0;                  // first row (m or n) of the tile
  int blk;                 // block index (3rd tensor dimension)
};

STBTA_DEV void tma_load_3d(double* dst, const CUtensorMap* map, int c0, int c1, int c2,
                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}

template <bool KM>
STBTA_DEV void tma_issue_opnd(double* dst, const TmaOpnd3& o, int k0, unsigned long long* bar) {
  if (!KM) {
    tma_load_3d(dst, o.map, k0, o.r0, o.blk, bar);
    tma_load_3d(dst + TMA_HALF, o.map, k0 + 16, o.r0, o.blk, bar);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) tma_load_3d(dst + i * 512, o.map, o.r0 + 16 * i, k0, o.blk, bar);
  }
}

// acc += A * B^T over k in [kbeg, K), (K - kbeg) % 32 == 0.
template <class Cfg, bool AKM, bool BKM>
STBTA_DEV void tile_mma_tma3(double (&acc)[Cfg::MF][Cfg::NF][2], const TmaOpnd3& A,
                             const TmaOpnd3& B, int kbeg, int K, double* smem,
                             unsigned long long* bars, unsigned& phase, int mv = 128,
                             int nv = 128) {
  static_assert(Cfg::BM == 128 && Cfg::BN == 128, "TMA path is laid out for 128 x 128 tiles");
  constexpr int MF = Cfg::MF, NF = Cfg::NF;
  double* base = tma_stage_base(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int nk = (K - kbeg) / 32;
  const int mfv = valid_frags<Cfg>(mv, wm0, MF), nfv = valid_frags<Cfg>(nv, wn0, NF);
  const bool full = (mfv == MF) && (nfv == NF);
  auto issue = [&](int kt) {  // thread 0
    double* st = base + (kt % TMA_ST) * TMA_STAGE;
    unsigned long long* bar = bars + kt % TMA_ST;
    mbar_expect_tx(bar, TMA_STAGE_BYTES);
    tma_issue_opnd<AKM>(st, A, kbeg + kt * 32, bar);
    tma_issue_opnd<BKM>(st + TMA_OPND, B, kbeg + kt * 32, bar);
  };
  if (tid == 0) {
    asm volatile("fence.proxy.async;\n" ::: "memory");
#pragma unroll
    for (int s = 0; s < TMA_ST - 1; ++s)
      if (s < nk) issue(s);
  }
  const int o4 = (tq & 1) * 3 + (tq >> 1) * 12;  // see tma_kp()
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TMA_ST;
    mbar_wait(bars + s, (phase >> s) & 1u);
    phase ^= 1u << s;
    if (tid == 0 && kt + TMA_ST - 1 < nk) {
      // the stage refilled now was consumed at kt - 1: wait until every warp
      // has arrived on its consumed barrier (that use's phase completes)
      const int sr = (kt + TMA_ST - 1) % TMA_ST;
      if (kt >= 1) mbar_wait(bars + TMA_ST + sr, ((phase >> (8 + sr)) & 1u) ^ 1u);
      issue(kt + TMA_ST - 1);
    }
    const double* as = base + s * TMA_STAGE;
    const double* bs = as + TMA_OPND;
    if (full) {
      // fragments double-buffered in registers (as tile_mma_tma)
      double af[2][MF], bf[2][NF];
      auto frag_load = [&](int ks, int b) {
        const int kp = tma_kp(ks, o4);
#pragma unroll
        for (int i = 0; i < MF; ++i) af[b][i] = as[tma_off<AKM>(wm0 + i * 8 + gq, kp)];
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[b][j] = bs[tma_off<BKM>(wn0 + j * 8 + gq, kp)];
      };
      frag_load(0, 0);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks + 1 < 8) frag_load(ks + 1, (ks + 1) & 1);
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
          for (int j = 0; j < NF; ++j)
            dmma884(acc[i][j][0], acc[i][j][1], af[ks & 1][i], bf[ks & 1][j]);
      }
    } else if (mfv > 0 && nfv > 0) {  // warp-uniform: only the wanted fragments
#pragma unroll 1
      for (int ks = 0; ks < 8; ++ks) {
        const int kp = tma_kp(ks, o4);
        double af[MF], bf[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) af[i] = i < mfv ? as[tma_off<AKM>(wm0 + i * 8 + gq, kp)] : 0.0;
#pragma unroll
        for (int j = 0; j < NF; ++j) bf[j] = j < nfv ? bs[tma_off<BKM>(wn0 + j * 8 + gq, kp)] : 0.0;
#pragma unroll
        for (int i = 0; i < MF; ++i) {
          if (i >= mfv) break;
#pragma unroll
          for (int j = 0; j < NF; ++j)
            if (j < nfv) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
    }
    __syncwarp();  // the warp's reads of stage s are done (arrive releases them)
    if (lane == 0) mbar_arrive(bars + TMA_ST + s);
    phase ^= 1u << (8 + s);
  }
  __syncthreads();
}

}  // namespace stbta
