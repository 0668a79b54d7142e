// Tile-engine variants measured against the product's TMA engine
// (tools/mb_tile.py; not used by the product kernels): per-row bulk copies
// with full / empty mbarriers, and a warp-specialised cp.async producer.
#pragma once

#include "../tile_mma.cuh"

namespace stbta {

// bars: 2*ST mbarriers (full[0..ST), empty[ST..2ST)), initialised with
// full = 1 arrival, empty = NT/32 arrivals, before the first use.
template <class Cfg>
STBTA_DEV void bulk_bars_init(unsigned long long* bars) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(bars + s, 1);
      mbar_init(bars + Cfg::STAGES + s, Cfg::NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

template <class Cfg, bool NEG = false>
STBTA_DEV void tile_mma_bulk(double (&acc)[Cfg::MF][Cfg::NF][2], const double* A, long long lda,
                             const double* B, long long ldb, int K, double* smem,
                             unsigned long long* bars, unsigned& slab) {
  constexpr int MF = Cfg::MF, NF = Cfg::NF, BK = Cfg::BK, ST = Cfg::STAGES, LDS = Cfg::LDS;
  constexpr unsigned ROWB = BK * 8;
  constexpr unsigned STAGE_TX = (Cfg::BM + Cfg::BN) * ROWB;
  double* As = smem;
  double* Bs = smem + ST * Cfg::A_STAGE;
  unsigned long long* full = bars;
  unsigned long long* empty = bars + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
  const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int nslab = K / BK;

  auto produce = [&](int i) {  // warp 0 only
    const unsigned c = slab + i;
    const int st = c % ST;
    if (c >= ST) mbar_wait(empty + st, ((c / ST) - 1) & 1);
    if (lane == 0) mbar_expect_tx(full + st, STAGE_TX);
    __syncwarp();
    const int k0 = i * BK;
    for (int r = lane; r < Cfg::BM; r += 32)
      bulk_g2s(As + st * Cfg::A_STAGE + r * LDS, A + (long long)r * lda + k0, ROWB, full + st);
    for (int r = lane; r < Cfg::BN; r += 32)
      bulk_g2s(Bs + st * Cfg::B_STAGE + r * LDS, B + (long long)r * ldb + k0, ROWB, full + st);
  };

  if (warp == 0) {
    fence_proxy_async();  // smem last written through the generic proxy
    const int pre = nslab < ST ? nslab : ST;
    for (int i = 0; i < pre; ++i) produce(i);
  }
  for (int i = 0; i < nslab; ++i) {
    const unsigned c = slab + i;
    const int st = c % ST;
    mbar_wait(full + st, (c / ST) & 1);
    const double* as = As + st * Cfg::A_STAGE;
    const double* bs = Bs + st * Cfg::B_STAGE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + tq;
      double af[MF], bf[NF];
#pragma unroll
      for (int ii = 0; ii < MF; ++ii) af[ii] = as[(wm0 + ii * 8 + gq) * LDS + k];
#pragma unroll
      for (int j = 0; j < NF; ++j)
        bf[j] = NEG ? -bs[(wn0 + j * 8 + gq) * LDS + k] : bs[(wn0 + j * 8 + gq) * LDS + k];
#pragma unroll
      for (int ii = 0; ii < MF; ++ii)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma884(acc[ii][j][0], acc[ii][j][1], af[ii], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
    if (warp == 0 && i + ST < nslab) produce(i + ST);
  }
  slab += nslab;
}

}  // namespace stbta

// ---------------------------------------------------------------------------
// Warp-specialised variant: one producer warp streams the K slabs with
// cp.async and signals a per-stage "full" mbarrier (cp.async.mbarrier.arrive),
// the Cfg::NT/32 consumer warps wait on it, run the DMMA fragments and release
// the stage on its "empty" mbarrier -- no CTA-wide barrier per slab.  The CTA
// has Cfg::NT + 32 threads; the producer is the last warp.  Full tiles only
// (rows == BM/BN, 16-byte aligned rows, K % BK == 0).
namespace stbta {

STBTA_DEV void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

template <class Cfg>
STBTA_DEV void ws_bars_init(unsigned long long* bars) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(bars + s, 32);                          // full: one arrive per producer lane
      mbar_init(bars + Cfg::STAGES + s, Cfg::NT / 32);  // empty: one per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

// acc += A * B^T (NT) over k in [0, K); `slab` is the CTA's running slab
// counter (same value in every thread) that carries the mbarrier phases.
template <class Cfg, bool NEG = false>
STBTA_DEV void tile_mma_ws(double (&acc)[Cfg::MF][Cfg::NF][2], const double* A, long long lda,
                           const double* B, long long ldb, int K, double* smem,
                           unsigned long long* bars, unsigned& slab) {
  constexpr int MF = Cfg::MF, NF = Cfg::NF, BK = Cfg::BK, ST = Cfg::STAGES, LDS = Cfg::LDS;
  double* As = smem;
  double* Bs = smem + ST * Cfg::A_STAGE;
  unsigned long long* full = bars;
  unsigned long long* empty = bars + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nslab = K / BK;
  if (warp == Cfg::NT / 32) {  // ---- producer
    constexpr int HP = BK / 2;
    for (int i = 0; i < nslab; ++i) {
      const unsigned c = slab + i;
      const int st = c % ST;
      if (c >= ST) mbar_wait(empty + st, ((c / ST) - 1) & 1);
      const int k0 = i * BK;
      double* as = As + st * Cfg::A_STAGE;
      double* bs = Bs + st * Cfg::B_STAGE;
#pragma unroll 4
      for (int e = lane; e < Cfg::BM * HP; e += 32) {
        const int r = e / HP, cc = (e % HP) * 2;
        cp_async16(as + r * LDS + cc, A + (long long)r * lda + k0 + cc, 16);
      }
#pragma unroll 4
      for (int e = lane; e < Cfg::BN * HP; e += 32) {
        const int r = e / HP, cc = (e % HP) * 2;
        cp_async16(bs + r * LDS + cc, B + (long long)r * ldb + k0 + cc, 16);
      }
      cp_async_mbar_arrive(full + st);
    }
  } else {  // ---- consumers
    const int gq = lane >> 2, tq = lane & 3;
    const int wm0 = (warp % Cfg::WARPS_M) * Cfg::WM;
    const int wn0 = (warp / Cfg::WARPS_M) * Cfg::WN;
    for (int i = 0; i < nslab; ++i) {
      const unsigned c = slab + i;
      const int st = c % ST;
      mbar_wait(full + st, (c / ST) & 1);
      const double* as = As + st * Cfg::A_STAGE;
      const double* bs = Bs + st * Cfg::B_STAGE;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int k = ks * 4 + tq;
        double af[MF], bf[NF];
#pragma unroll
        for (int ii = 0; ii < MF; ++ii) af[ii] = as[(wm0 + ii * 8 + gq) * LDS + k];
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const double bv = bs[(wn0 + j * 8 + gq) * LDS + k];
          bf[j] = NEG ? -bv : bv;
        }
#pragma unroll
        for (int ii = 0; ii < MF; ++ii)
#pragma unroll
          for (int j = 0; j < NF; ++j) dmma884(acc[ii][j][0], acc[ii][j][1], af[ii], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
  }
  slab += nslab;
}

}  // namespace stbta

