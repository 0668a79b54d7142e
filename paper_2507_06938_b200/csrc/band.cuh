// Tile geometry of the lower band of a BTA matrix, shared by the persistent
// POBTAF / POBTASI task-graph kernels.
//
// The lower triangle of a BTA matrix (reference BTAMatrix, bta.py:50-89) is a
// banded matrix of bandwidth ~2b plus dense arrow rows.  We cut it into
// T x T tiles (T = 128): block time t owns tile rows/cols t*nbt .. t*nbt+nbt-1
// (the last one partial when b % T != 0), and the arrow rows are tile rows
// n*nbt .. n*nbt+nat-1.  A tile (R, C), R >= C, lives in exactly one storage
// region of the flat buffer:
//   R, C in block t          -> diag[t]   (ld b)
//   R in t+1, C in t         -> lower[t]  (ld b)
//   R arrow, C in block t    -> arrow[t]  (ld b)
//   R, C arrow               -> tip       (ld a)
// "Panel" s is tile column s; its band rows are the tile rows below it that
// the block elimination touches (rest of block t, block t+1, and the arrow
// rows when the arrow is active) -- exactly the rows of the reference's
// per-block updates (bta.py:204-227), refined to tile granularity.
#pragma once

#include "common.cuh"

namespace stbta {

constexpr int TT = 128;  // tile size
constexpr int TS = 32;   // strip (row sub-tile) size
constexpr int NSTRIP = TT / TS;

struct Band {
  double* data;  // flat BTA storage (unused when the region pointers are set)
  double *dg, *lw, *ar, *tp;  // diag (n,b,b) | lower (n-1,b,b) | arrow (n,a,b) | tip (a,a)
  int n, b, a;
  int ldb;       // row stride of the diag / lower / arrow blocks (b, or b+1 padded)
  int nbt;       // tiles per time block
  int nat;       // arrow tiles
  int S;         // panels = n*nbt + nat
  int SP;        // panels actually eliminated (S, or nfact*nbt for a partial factorization)
  int use_arrow; // arrow rows take part in the block eliminations
  int vec_b;     // b even: rows of diag/lower/arrow are 16-byte aligned
  int vec_a;     // tip rows 16-byte aligned (a even and b even)
  int chunk;     // POBTAF: panels per chunked update (0: default by block width)
  int look;      // POBTAF: per-panel look-ahead window (0: default)
  int remainder; // POBTAF: remainder chunks inside the window (-1: default)
};

STBTA_DEV bool is_arrow_tile(const Band& g, int R) { return R >= g.n * g.nbt; }

// rows / cols of a tile (partial last tile of a block or of the arrow)
STBTA_DEV int tile_extent(const Band& g, int R) {
  if (R >= g.n * g.nbt) {
    const int q = R - g.n * g.nbt;
    return min(TT, g.a - q * TT);
  }
  const int j = R % g.nbt;
  return min(TT, g.b - j * TT);
}

struct TilePtr {
  double* p;
  long long ld;
  int vec;
};

// storage of tile (R, C), R >= C in the band
STBTA_DEV TilePtr tile_ptr(const Band& g, int R, int C) {
  const long long b = g.ldb;            // row stride
  const long long bb = (long long)g.b * b;  // block stride
  double* diag = g.dg;
  double* lower = g.lw;
  double* arrow = g.ar;
  double* tip = g.tp;
  TilePtr t;
  const int NB = g.n * g.nbt;
  // a tile of the lower band: C <= R < S; block tiles on the diagonal or
  // first sub-diagonal block; arrow rows against any block column or the tip
  STBTA_CHECK(C >= 0 && R >= C && R < g.S);
  STBTA_CHECK(R >= NB || C >= NB || (R / g.nbt - C / g.nbt == 0 || R / g.nbt - C / g.nbt == 1));
  if (C >= NB) {  // tip
    const int qr = R - NB, qc = C - NB;
    t.p = tip + (long long)qr * TT * g.a + qc * TT;
    t.ld = g.a;
    t.vec = g.vec_a;
    return t;
  }
  const int tc = C / g.nbt, jc = C % g.nbt;
  if (R >= NB) {
    const int qr = R - NB;
    t.p = arrow + (long long)tc * g.a * b + (long long)qr * TT * b + jc * TT;  // arrow block: a x ldb
  } else {
    const int tr = R / g.nbt, jr = R % g.nbt;
    double* base = (tr == tc) ? diag + (long long)tc * bb : lower + (long long)tc * bb;
    t.p = base + (long long)jr * TT * b + jc * TT;
  }
  t.ld = b;
  t.vec = g.vec_b;
  return t;
}

// Upper-triangle mirror tile (C, R) of a same-block tile (R > C): diag storage.
STBTA_DEV TilePtr tile_ptr_upper(const Band& g, int R, int C) {
  const long long b = g.ldb;
  const int NB = g.n * g.nbt;
  STBTA_CHECK(R > C && R < g.S && ((R >= NB && C >= NB) || (R < NB && R / g.nbt == C / g.nbt)));
  if (C >= NB) {  // tip
    TilePtr p;
    p.p = g.tp + (long long)(C - NB) * TT * g.a + (R - NB) * TT;
    p.ld = g.a;
    p.vec = g.vec_a;
    return p;
  }
  const int t = C / g.nbt, jr = R % g.nbt, jc = C % g.nbt;
  TilePtr p;
  p.p = g.dg + (long long)t * g.b * b + (long long)jc * TT * b + jr * TT;
  p.ld = b;
  p.vec = g.vec_b;
  return p;
}

// number of band rows of panel s and the i-th band row
STBTA_DEV int band_rows(const Band& g, int s, int* contiguous) {
  const int NB = g.n * g.nbt;
  if (s >= NB) {
    *contiguous = g.S - s - 1;
    return g.S - s - 1;
  }
  const int t = s / g.nbt;
  const int end = min(t + 2, g.n) * g.nbt;  // exclusive block-row end
  const int mb = end - s - 1;
  *contiguous = mb;
  return mb + (g.use_arrow ? g.nat : 0);
}
STBTA_DEV int band_row(const Band& g, int s, int i, int mb) {
  return i < mb ? s + 1 + i : g.n * g.nbt + (i - mb);
}

// Number of panels s' < s whose block elimination updates tile (R, C)
// (R >= C, C > s' ).  Used both as the ordering ticket of the update by panel
// s and, with s = C, as the count after which the tile is fully updated.
STBTA_DEV int n_updates(const Band& g, int R, int C, int s) {
  const int NB = g.n * g.nbt;
  const int hi = min(s, C);
  if (C >= NB) {  // tip tile: every block panel (if the arrow is active), then arrow panels
    int cnt = g.use_arrow ? min(hi, NB) : 0;
    if (hi > NB) cnt += hi - NB;
    return cnt;
  }
  const int tc = C / g.nbt;
  int lo = max(0, (tc - 1) * g.nbt);
  if (R >= NB) {
    if (!g.use_arrow) return 0;
  } else {
    const int tr = R / g.nbt;
    lo = max(lo, (tr - 1) * g.nbt);
  }
  return max(0, hi - lo);
}

// Dependency counter of (strip q of tile row R, tile column C).
STBTA_DEV int* counter(const Band& g, int* ctr, int R, int q, int C) {
  const int NB = g.n * g.nbt;
  if (R < NB) {
    const int tr = R / g.nbt;
    const int rel = C - (tr - 1) * g.nbt;  // in [0, 2 nbt)
    return ctr + ((long long)(R * NSTRIP + q) * (2 * g.nbt) + rel);
  }
  const long long base = (long long)NB * NSTRIP * 2 * g.nbt;
  return ctr + base + (long long)((R - NB) * NSTRIP + q) * g.S + C;
}

inline long long counter_elems(int n, int nbt, int nat, int S) {
  return (long long)n * nbt * NSTRIP * 2 * nbt + (long long)nat * NSTRIP * S;
}

// Region pointers of the reference's flat layout.
inline void band_set_flat(Band& g, double* data) {
  g.ldb = g.b;
  const long long bb = (long long)g.b * g.b;
  g.data = data;
  g.dg = data;
  g.lw = data ? data + (long long)g.n * bb : nullptr;
  g.ar = data ? g.lw + (long long)(g.n - 1) * bb : nullptr;
  g.tp = data ? g.ar + (long long)g.n * g.a * g.b : nullptr;
}

// ------------------------------------------------------------- sync helpers
STBTA_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
STBTA_DEV int ld_volatile(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin until *p >= target or the abort word is set.  Returns false on abort.
STBTA_DEV bool spin_geq(const int* p, int target, const int* abort_flag) {
  int it = 0;
  while (ld_acquire(p) < target) {
    if (ld_volatile(abort_flag)) return false;
    if (++it > 8) __nanosleep(32);
  }
  return true;
}

}  // namespace stbta
