// POBTAS: forward / backward block substitution against a POBTAF factor.
//
// Reference: bta.forward_substitute (pkg/src/stinla/bta.py:249-275),
// bta.backward_substitute (bta.py:278-302), bta.solve (bta.py:305-307).
//
// B200 mapping.  The block-bidiagonal part of L is a banded lower-triangular
// matrix cut into 128-row tiles (band.cuh geometry).  Each sweep is ONE
// launch in which a CTA takes tile R from an atomic ticket (so it only ever
// waits on tiles already claimed) and
//   1. streams the matrix blocks coupling R to its dependencies (tiles of the
//      previous / next time block and of its own block) through a 4-stage
//      cp.async ring of 32-column (32-row) slices -- the factor is read
//      exactly once per sweep at HBM rate, prefetched before the dependency's
//      solution is even ready;
//   2. folds each dependency's solution in, in a fixed order (deterministic),
//      as soon as that tile publishes it (acquire flag);
//   3. solves its 128x128 diagonal triangle in 32-row blocks (warp-level
//      substitution + block updates) and publishes the tile (release flag).
// The arrow rows become per-tile partial products summed in tile order by the
// tip kernel, which also solves L_tip (reference bta.py:263-273, 288-300).
#include "../../include/stbta.h"
#include "band.cuh"
#include "common.cuh"
#include "potrf_tile.cuh"

namespace stbta {

constexpr int PS_NT = 256;
constexpr int NR = 8;      // right-hand sides per sweep launch
constexpr int SL = 32;     // slice width
constexpr int PST = 4;     // ring stages
constexpr int F_LD = SL;               // forward slice: 128 rows x 32 cols, 16-byte chunks swizzled
constexpr int B_LD = 128;              // backward slice: 32 rows x 128 cols (read along rows)
constexpr int STAGE = 128 * F_LD > SL * B_LD ? 128 * F_LD : SL * B_LD;
// forward slice element (r, q): chunk (q >> 1) of row r stored at chunk (q >> 1) ^ (r & 7), so
// the 16-byte reads of 8 consecutive rows at one chunk hit 8 distinct bank quads
STBTA_DEV int fsw(int r, int q) { return r * F_LD + ((((q >> 1) ^ (r & 7))) << 1) + (q & 1); }
constexpr int P_LD = 129;              // coupling block in shared memory
constexpr int WPK = 128 * 129 / 2;     // packed lower 128 x 128
constexpr int PS_SMEM_DOUBLES = WPK + 128 * P_LD + 128 * NR + 128 * NR;
static_assert(PST * STAGE <= 128 * P_LD, "ring must fit in the coupling-block region");

STBTA_DEV int pk(int r, int c) { return r * (r + 1) / 2 + c; }

struct SweepArgs {
  Band g;
  double* x;      // rhs / solution, row-major (dim x ldx), columns [0, ncols)
  long long ldx;
  int ncols;
  int ntile;      // n * nbt block tiles
  int* flags;     // one per tile, zeroed before the launch
  int* ticket;    // zeroed before the launch
  double* part;   // arrow partials [ntile][a][NR] (forward)
  const double* xtip;  // packed x_tip [a][NR] (backward)
  double* push;   // [ntile][128][NR]: coupling contribution pushed to the next tile
  int* flags2;    // one per tile: its second-neighbour push is ready
  double* push2;  // [ntile][128][NR]: coupling contribution pushed two tiles ahead
  unsigned long long* prof;  // optional debug timers (slots 20..23)
  const double* winv;  // [ntile][WPK]: packed inverses of the diagonal tiles
};

// ---------------------------------------------------------------- pre-pass
// W_R = L_RR^-1 for every diagonal tile, packed lower (row-major), through
// the in-CTA blocked inversion of potrf_tile.cuh.
__global__ void __launch_bounds__(PS_NT, 1) inv_tiles_kernel(Band g, double* winv) {
  extern __shared__ __align__(16) double sm[];
  double* T = sm;
  const int R = blockIdx.x;
  const int tid = threadIdx.x;
  const int ext = tile_extent(g, R);
  const TilePtr tp = tile_ptr(g, R, R);
  for (int e = tid; e < 128 * 128; e += PS_NT) {
    const int r = e >> 7, c = e & 127;
    double v;
    if (r < ext && c < ext) v = (c <= r) ? __ldg(tp.p + (long long)r * tp.ld + c) : 0.0;
    else v = (r == c) ? 1.0 : 0.0;
    T[r * INV_LD + c] = v;
  }
  __syncthreads();
  invert_tile_smem<PS_NT>(sm);
  double* out = winv + (long long)R * WPK;
  for (int e = tid; e < WPK; e += PS_NT) {
    int r = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    if ((r + 1) * (r + 2) / 2 <= e) ++r;
    if (r * (r + 1) / 2 > e) --r;
    out[e] = inv_tile_at(sm, r, e - r * (r + 1) / 2);
  }
}

// One 32-wide slice of dependency tile k into a ring stage (16-byte copies
// when the rows are 16-byte aligned, zero fill outside the tile).
template <bool FWD>
STBTA_DEV void load_slice(double* ring_st, const Band& g, int R, int k, int sl, int extR,
                          int extK) {
  const int tid = threadIdx.x;
  if (FWD) {
    // M = tile (R, k): rows r < extR, cols sl*32 + q (q < 32, < extK)
    const TilePtr t = tile_ptr(g, R, k);
    const int c0 = sl * SL;
    const bool vec = ((uintptr_t)t.p % 16 == 0) && (t.ld % 2 == 0);
    if (vec) {
      for (int e = tid; e < 128 * SL / 2; e += PS_NT) {
        const int r = e >> 4, q = (e & 15) * 2;
        int bytes = 0;
        const double* src = t.p;
        if (r < extR && c0 + q < extK) {
          bytes = (c0 + q + 1 < extK) ? 16 : 8;
          src = t.p + (long long)r * t.ld + c0 + q;
        }
        cp_async16(ring_st + fsw(r, q), src, bytes);
      }
    } else {
      for (int e = tid; e < 128 * SL; e += PS_NT) {
        const int r = e >> 5, q = e & 31;
        const bool ok = r < extR && c0 + q < extK;
        cp_async8(ring_st + fsw(r, q), ok ? t.p + (long long)r * t.ld + c0 + q : t.p, ok);
      }
    }
  } else {
    // M = tile (k, R): rows sl*32 + q of tile k (q < 32, < extK), cols r < extR
    const TilePtr t = tile_ptr(g, k, R);
    const int r0 = sl * SL;
    const bool vec = ((uintptr_t)t.p % 16 == 0) && (t.ld % 2 == 0);
    if (vec) {
      for (int e = tid; e < SL * 128 / 2; e += PS_NT) {
        const int q = e >> 6, r = (e & 63) * 2;
        int bytes = 0;
        const double* src = t.p;
        if (r0 + q < extK && r < extR) {
          bytes = (r + 1 < extR) ? 16 : 8;
          src = t.p + (long long)(r0 + q) * t.ld + r;
        }
        cp_async16(ring_st + q * B_LD + r, src, bytes);
      }
    } else {
      for (int e = tid; e < SL * 128; e += PS_NT) {
        const int q = e >> 7, r = e & 127;
        const bool ok = r0 + q < extK && r < extR;
        cp_async8(ring_st + q * B_LD + r, ok ? t.p + (long long)(r0 + q) * t.ld + r : t.p, ok);
      }
    }
  }
}

// out[r] (r < 128, c < NR) = sum_q M(r, q) v[q], M given by an accessor; the
// 256 threads split q in halves, partial sums combined in a fixed order.
template <int NRC, class F>
STBTA_DEV void gemv128(double* out, const double* v, double* tmp, F M) {
  const int tid = threadIdx.x, r = tid & 127, h = tid >> 7;
  double s[NRC];
#pragma unroll
  for (int c = 0; c < NRC; ++c) s[c] = 0.0;
#pragma unroll 4
  for (int qq = 0; qq < 64; ++qq) {
    const int q = h * 64 + qq;
    const double m = M(r, q);
#pragma unroll
    for (int c = 0; c < NRC; ++c) s[c] = fma(m, v[q * NR + c], s[c]);
  }
  if (h == 1) {
#pragma unroll
    for (int c = 0; c < NRC; ++c) tmp[r * NR + c] = s[c];
  }
  __syncthreads();
  if (h == 0) {
#pragma unroll
    for (int c = 0; c < NRC; ++c) out[r * NR + c] = s[c] + tmp[r * NR + c];
  }
  __syncthreads();
}

template <bool FWD, int NRC>
__global__ void __launch_bounds__(PS_NT, 1) sweep_kernel(SweepArgs p) {
  extern __shared__ __align__(16) double sm[];
  double* Wp = sm;                   // packed W of this tile
  double* Pb = Wp + WPK;             // ring for the pulled dependencies, then the push block
  double* ybuf = Pb + 128 * P_LD;    // dependency solution / this tile's solution, 128 x NR
  double* accb = ybuf + 128 * NR;    // right-hand side, 128 x NR
  double* ring = Pb;
  __shared__ int s_k;
  const Band& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_k = atomicAdd(p.ticket, 1);
  __syncthreads();
  const int R = FWD ? s_k : p.ntile - 1 - s_k;
  const int i = R / g.nbt;
  const int extR = tile_extent(g, R);
  const long long row0 = (long long)i * g.b + (long long)(R % g.nbt) * 128;
  const int nc = p.ncols;
  unsigned long long t0 = 0, t1 = 0, t2 = 0;
  if (p.prof && tid == 0) t0 = pt_timer();

  // packed inverse of the diagonal tile (own cp.async group, waited on late)
  {
    const double* src = p.winv + (long long)R * WPK;
    for (int e = tid; e < WPK / 2; e += PS_NT) cp_async16(Wp + 2 * e, src + 2 * e, 16);
    cp_async_commit();
  }

  // pulled dependencies: forward k in [lo, R-1) ascending; backward k in (R+1, hi] descending
  // (the adjacent tile is pushed: it sends its coupling product with its flag)
  // The two nearest tiles push: R-1 (R+1 backward) with its flag, R-2 (R+2)
  // right after its flag -- so the tile folded latest is R-3, three periods
  // before R publishes, and the pulled fold leaves the sweep's recurrence.
  int kfirst, nk, crit, crit2;
  if (FWD) {
    const int lo = max(0, (i - 1) * g.nbt);
    kfirst = lo;
    crit = R - 1;  // -1 for the first tile
    crit2 = (R - 2 >= lo) ? R - 2 : -1;
    nk = max(0, R - 1 - lo) - (crit2 >= 0 ? 1 : 0);
  } else {
    const int hi = min((i + 2) * g.nbt, p.ntile) - 1;
    kfirst = hi;
    crit = (R + 1 < p.ntile) ? R + 1 : -1;
    crit2 = (R + 2 <= hi) ? R + 2 : -1;
    nk = max(0, hi - R - 1) - (crit2 >= 0 ? 1 : 0);
  }
  auto dep = [&](int d) { return FWD ? kfirst + d : kfirst - d; };
  auto nsl = [&](int k) { return (tile_extent(g, k) + SL - 1) / SL; };

  const int r = tid & 127, h = tid >> 7;
  double acc[NRC];
#pragma unroll
  for (int c = 0; c < NRC; ++c) acc[c] = 0.0;

  if (!FWD && g.use_arrow && h == 0 && r < extR) {  // x_R -= arrow[i][:, R]^T x_tip
    const double* arrow = g.ar + (long long)i * g.a * g.ldb;
    const int col = (R % g.nbt) * 128 + r;
    for (int t = 0; t < g.a; ++t) {
      const double av = arrow[(long long)t * g.ldb + col];
#pragma unroll
      for (int c = 0; c < NRC; ++c)
        if (c < nc) acc[c] -= av * p.xtip[t * NR + c];
    }
  }

  int total = 0;
  for (int d = 0; d < nk; ++d) total += nsl(dep(d));
  int pd = 0, ps = 0;
  auto issue = [&](int stage) {
    if (pd < nk) {
      const int k = dep(pd);
      load_slice<FWD>(ring + stage * STAGE, g, R, k, ps, extR, tile_extent(g, k));
      if (++ps == nsl(k)) { ps = 0; ++pd; }
    }
    cp_async_commit();
  };
  for (int s = 0; s < PST - 1; ++s) issue(s);

  int cd = 0, cs = 0;
  for (int it = 0; it < total; ++it) {
    const int k = dep(cd);
    if (cs == 0) {
      __syncthreads();
      if (tid == 0) {
        while (ld_acquire(p.flags + k) == 0) __nanosleep(20);
      }
      __syncthreads();
      const long long krow0 = (long long)(k / g.nbt) * g.b + (long long)(k % g.nbt) * 128;
      const int extK = tile_extent(g, k);
      for (int e = tid; e < 128 * NRC; e += PS_NT) {
        const int q = e / NRC, c = e % NRC;
        ybuf[q * NR + c] = (q < extK && c < nc) ? __ldcg(p.x + (krow0 + q) * p.ldx + c) : 0.0;
      }
    }
    cp_async_wait<PST - 2>();
    __syncthreads();
    issue((it + PST - 1) % PST);
    const double* rs = ring + (it % PST) * STAGE;
    const int q0 = cs * SL;
#pragma unroll 4
    for (int qq = 0; qq < SL / 2; qq += 2) {
      const int q = h * (SL / 2) + qq;
      double m0, m1;
      if (FWD) {
        const double2 v = *reinterpret_cast<const double2*>(rs + fsw(r, q));
        m0 = v.x;
        m1 = v.y;
      } else {
        m0 = rs[q * B_LD + r];
        m1 = rs[(q + 1) * B_LD + r];
      }
      const double* yq = ybuf + (q0 + q) * NR;
#pragma unroll
      for (int c = 0; c < NRC; ++c) acc[c] = fma(-m1, yq[NR + c], fma(-m0, yq[c], acc[c]));
    }
    if (++cs == nsl(k)) { cs = 0; ++cd; }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (p.prof && tid == 0) t1 = pt_timer();

  // prefetch the push block: forward tile (R+1, R) [rows of R+1 x cols of R],
  // backward tile (R, R-1) [rows of R x cols of R-1]
  const int pushto = FWD ? ((R + 1 < p.ntile) ? R + 1 : -1) : R - 1;
  if (pushto >= 0) {
    const TilePtr t = FWD ? tile_ptr(g, R + 1, R) : tile_ptr(g, R, R - 1);
    const int nr = FWD ? tile_extent(g, R + 1) : extR;
    const int ncl = FWD ? extR : tile_extent(g, R - 1);
    for (int e = tid; e < 128 * 128; e += PS_NT) {
      const int rr = e >> 7, cc = e & 127;
      if (rr < nr && cc < ncl) cp_async8(Pb + rr * P_LD + cc, t.p + (long long)rr * t.ld + cc, true);
      else Pb[rr * P_LD + cc] = 0.0;
    }
  }
  cp_async_commit();

  // accb = rhs + pulled contributions (h0 then h1, fixed order)
  if (h == 0) {
#pragma unroll
    for (int c = 0; c < NR; ++c)
      accb[r * NR + c] = (c < NRC && r < extR && c < nc) ? __ldcg(p.x + (row0 + r) * p.ldx + c) + acc[c < NRC ? c : 0] : 0.0;
  }
  __syncthreads();
  if (h == 1) {
#pragma unroll
    for (int c = 0; c < NRC; ++c) accb[r * NR + c] += (r < extR && c < nc) ? acc[c] : 0.0;
  }
  // the second neighbour's pushed contribution (ready a period earlier)
  if (crit2 >= 0) {
    if (tid == 0) {
      while (ld_acquire(p.flags2 + crit2) == 0) __nanosleep(10);
    }
    __syncthreads();
    if (h == 0) {
      const double* u = p.push2 + (long long)R * 128 * NR;
#pragma unroll
      for (int c = 0; c < NRC; ++c) accb[r * NR + c] -= (r < extR && c < nc) ? __ldcg(u + r * NR + c) : 0.0;
    }
  }
  // the adjacent (critical) tile's pushed contribution
  if (crit >= 0) {
    if (tid == 0) {
      while (ld_acquire(p.flags + crit) == 0) __nanosleep(10);
    }
    __syncthreads();
    if (h == 0) {
      const double* u = p.push + (long long)R * 128 * NR;
#pragma unroll
      for (int c = 0; c < NRC; ++c) accb[r * NR + c] -= (r < extR && c < nc) ? __ldcg(u + r * NR + c) : 0.0;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  if (p.prof && tid == 0) t2 = pt_timer();
  // y = W acc (forward)  /  x = W^T acc (backward); result in ybuf
  if (FWD)
    gemv128<NRC>(ybuf, accb, ybuf, [&](int rr, int q) { return q <= rr ? Wp[pk(rr, q)] : 0.0; });
  else
    gemv128<NRC>(ybuf, accb, ybuf, [&](int rr, int q) { return q >= rr ? Wp[pk(q, rr)] : 0.0; });
  // push: forward u = L_{R+1,R} y  ->  push[R+1];  backward v = L_{R,R-1}^T x -> push[R-1]
  if (pushto >= 0) {
    if (FWD)
      gemv128<NRC>(accb, ybuf, accb, [&](int rr, int q) { return Pb[rr * P_LD + q]; });
    else
      gemv128<NRC>(accb, ybuf, accb, [&](int rr, int q) { return Pb[q * P_LD + rr]; });
    double* dst = p.push + (long long)pushto * 128 * NR;
    for (int e = tid; e < 128 * NR; e += PS_NT) dst[e] = accb[e];
  }
  // publish the solution
  for (int e = tid; e < extR * NR; e += PS_NT) {
    const int rr = e / NR, c = e % NR;
    if (c < nc) p.x[(row0 + rr) * p.ldx + c] = ybuf[e];
  }
  if (FWD && g.use_arrow) {  // arrow partials: part[R][t][c] = sum_r arrow[i][t][R0 + r] y[r][c]
    const double* arrow = g.ar + (long long)i * g.a * g.ldb;
    const int col0 = (R % g.nbt) * 128;
    for (int t = warp; t < g.a; t += PS_NT / 32) {
      double s[NRC];
#pragma unroll
      for (int c = 0; c < NRC; ++c) s[c] = 0.0;
      for (int rr = lane; rr < extR; rr += 32) {
        const double av = arrow[(long long)t * g.ldb + col0 + rr];
#pragma unroll
        for (int c = 0; c < NRC; ++c) s[c] = fma(av, ybuf[rr * NR + c], s[c]);
      }
#pragma unroll
      for (int c = 0; c < NRC; ++c) {
        const double v = warp_sum(s[c]);
        if (lane == 0) p.part[((long long)R * g.a + t) * NR + c] = v;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicExch(p.flags + R, 1);
    if (p.prof) {
      const unsigned long long t3 = pt_timer();
      atomicAdd(p.prof + 20, 1ull);
      atomicAdd(p.prof + 21, t1 - t0);
      atomicAdd(p.prof + 22, t2 - t1);
      atomicAdd(p.prof + 23, t3 - t2);
    }
  }
  // off the critical step: the second-neighbour push, straight from global
  // memory (forward u = L_{R+2,R} y_R to R+2; backward v = L_{R,R-2}^T x_R to R-2)
  int to2 = -1;
  if (FWD) {
    if (R + 2 < p.ntile && R >= max(0, ((R + 2) / g.nbt - 1) * g.nbt)) to2 = R + 2;
  } else {
    if (R - 2 >= 0 && R <= min(((R - 2) / g.nbt + 2) * g.nbt, p.ntile) - 1) to2 = R - 2;
  }
  if (to2 >= 0) {
    double* dst = p.push2 + (long long)to2 * 128 * NR;
    if (FWD) {  // stage L_{R+2,R} in the (free) push-block buffer, then the 128-row gemv
      const TilePtr t = tile_ptr(g, R + 2, R);
      const int nr = tile_extent(g, R + 2);
      for (int e = tid; e < 128 * 128; e += PS_NT) {  // row layout of the push block
        const int rr = e >> 7, cc = e & 127;
        const bool ok = rr < nr && cc < extR;
        cp_async8(Pb + rr * P_LD + cc, ok ? t.p + (long long)rr * t.ld + cc : t.p, ok);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      gemv128<NRC>(accb, ybuf, accb, [&](int rr, int q) { return Pb[rr * P_LD + q]; });
      for (int e = tid; e < 128 * NR; e += PS_NT) dst[e] = accb[e];
    } else {  // thread per output column (coalesced rows), halves over the rows
      const TilePtr t = tile_ptr(g, R, R - 2);
      const int ncl = tile_extent(g, R - 2);
      double sacc[NRC];
#pragma unroll
      for (int c = 0; c < NRC; ++c) sacc[c] = 0.0;
      if (r < ncl)
        for (int rr = h * 64; rr < min(extR, h * 64 + 64); ++rr) {
          const double m = __ldcg(t.p + (long long)rr * t.ld + r);
#pragma unroll
          for (int c = 0; c < NRC; ++c) sacc[c] = fma(m, ybuf[rr * NR + c], sacc[c]);
        }
      double* tmp = accb;  // accb is no longer needed
      if (h == 1) {
#pragma unroll
        for (int c = 0; c < NRC; ++c) tmp[r * NR + c] = sacc[c];
      }
      __syncthreads();
      if (h == 0) {
#pragma unroll
        for (int c = 0; c < NRC; ++c) dst[r * NR + c] = sacc[c] + tmp[r * NR + c];
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicExch(p.flags2 + R, 1);
    }
  }
}

// mode 0 (forward): y_tip = L_tip^-1 (r_tip - sum_R part[R]);  mode 1: x_tip = L_tip^-T y_tip.
// In place on the tip segment of x (any arrow size); writes a packed copy
// xtip[a][NR] for the backward sweep's arrow coupling.
__global__ void tip_solve_kernel(SweepArgs p, int nparts, double* xtip, int mode) {
  const int c = threadIdx.x;
  if (c >= p.ncols) return;
  const Band& g = p.g;
  const int a = g.a;
  const long long base = (long long)g.n * g.b;
  const double* tip = g.tp;
  double* v = p.x + base * p.ldx + c;
  const long long ld = p.ldx;
  if (mode == 0 && g.use_arrow) {
    for (int t = 0; t < a; ++t) {
      double tot = 0.0;
      for (int R = 0; R < nparts; ++R) tot += p.part[((long long)R * a + t) * NR + c];
      v[t * ld] -= tot;
    }
  }
  if (mode == 0) {
    for (int t = 0; t < a; ++t) {
      double s = v[t * ld];
      for (int u = 0; u < t; ++u) s -= tip[(long long)t * a + u] * v[u * ld];
      v[t * ld] = s / tip[(long long)t * a + t];
    }
  } else {
    for (int t = a - 1; t >= 0; --t) {
      double s = v[t * ld];
      for (int u = t + 1; u < a; ++u) s -= tip[(long long)u * a + t] * v[u * ld];
      v[t * ld] = s / tip[(long long)t * a + t];
    }
  }
  for (int t = 0; t < a; ++t) xtip[t * NR + c] = v[t * ld];
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct PobtasWs {
  int* flags;
  int* flags2;
  int* ticket;
  double* part;
  double* xtip;
  double* push;
  double* push2;
  double* winv;
};

static size_t pobtas_ws(int n, int b, int a, char* base, PobtasWs* o) {
  const int ntile = n * ((b + 127) / 128);
  const size_t f = align_up((size_t)(2 * ntile + 2) * sizeof(int));
  const size_t pa = align_up((size_t)ntile * (a > 0 ? a : 1) * NR * sizeof(double));
  const size_t xt = align_up((size_t)(a > 0 ? a : 1) * NR * sizeof(double));
  const size_t pu = align_up((size_t)ntile * 128 * NR * sizeof(double));  // push and push2
  const size_t wi = (size_t)ntile * WPK * sizeof(double);
  if (o) {
    o->flags = reinterpret_cast<int*>(base);
    o->flags2 = o->flags + ntile;
    o->ticket = o->flags + 2 * ntile;
    o->part = reinterpret_cast<double*>(base + f);
    o->xtip = reinterpret_cast<double*>(base + f + pa);
    o->push = reinterpret_cast<double*>(base + f + pa + xt);
    o->push2 = reinterpret_cast<double*>(base + f + pa + xt + pu);
    o->winv = reinterpret_cast<double*>(base + f + pa + xt + 2 * pu);
  }
  return f + pa + xt + 2 * pu + wi;
}

static int run_sweeps(SweepArgs p, int mode, const PobtasWs& ws, cudaStream_t st) {
  const size_t fbytes = (size_t)(2 * p.ntile + 1) * sizeof(int);  // flags, flags2, ticket
  const size_t smem = PS_SMEM_DOUBLES * sizeof(double);
  const size_t ismem = INV_SMEM_DOUBLES * sizeof(double);
  static std::atomic<unsigned long long> attr_mask{0};  // per device
  if (attr_pending(attr_mask)) {
    int e1 = (int)cudaFuncSetAttribute(sweep_kernel<true, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int e2 = (int)cudaFuncSetAttribute(sweep_kernel<false, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e1 |= (int)cudaFuncSetAttribute(sweep_kernel<true, NR>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e2 |= (int)cudaFuncSetAttribute(sweep_kernel<false, NR>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int e3 = (int)cudaFuncSetAttribute(inv_tiles_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem);
    if (e1) return e1;
    if (e2) return e2;
    if (e3) return e3;
    attr_mark(attr_mask);
  }
  int e;
  inv_tiles_kernel<<<p.ntile, PS_NT, ismem, st>>>(p.g, ws.winv);
  count_launch();
  if ((e = (int)cudaGetLastError())) return e;
  if (mode == 0 || mode == 1) {
    if ((e = zero_async(p.flags, fbytes, st))) return e;
    if (p.ncols == 1) sweep_kernel<true, 1><<<p.ntile, PS_NT, smem, st>>>(p);
    else sweep_kernel<true, NR><<<p.ntile, PS_NT, smem, st>>>(p);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
    if (p.g.a > 0) {
      tip_solve_kernel<<<1, NR, 0, st>>>(p, p.ntile, ws.xtip, 0);
      count_launch();
      if ((e = (int)cudaGetLastError())) return e;
    }
  }
  if (mode == 0 || mode == 2) {
    if (p.g.a > 0) {
      tip_solve_kernel<<<1, NR, 0, st>>>(p, 0, ws.xtip, 1);
      count_launch();
      if ((e = (int)cudaGetLastError())) return e;
    }
    if ((e = zero_async(p.flags, fbytes, st))) return e;
    if (p.ncols == 1) sweep_kernel<false, 1><<<p.ntile, PS_NT, smem, st>>>(p);
    else sweep_kernel<false, NR><<<p.ntile, PS_NT, smem, st>>>(p);
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
  if (factor == nullptr) return STBTA_EARG;
  const long long bb = (long long)b * b;
  const double* lower = factor + (long long)n * bb;
  const double* arrow = lower + (long long)(n - 1) * bb;
  const double* tip = arrow + (long long)n * a * b;
  return stbta_pobtas_ex(factor, lower, arrow, tip, n, b, a, b, has_arrow, rhs, nrhs, mode,
                         workspace, workspace_bytes, stream);
}

int stbta_pobtas_ex(const double* diag, const double* lower, const double* arrow,
                    const double* tip, int n, int b, int a, int ldb, int has_arrow, double* rhs,
                    int nrhs, int mode, void* workspace, size_t workspace_bytes, void* stream) {
  if (diag == nullptr || rhs == nullptr || n < 1 || b < 1 || a < 0 || nrhs < 1 || mode < 0 ||
      mode > 2 || ldb < b)
    return STBTA_EARG;
  if ((n > 1 && lower == nullptr) || (a > 0 && (arrow == nullptr || tip == nullptr)))
    return STBTA_EARG;
  if (workspace_bytes < stbta_pobtas_workspace_bytes(n, b, a, nrhs)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PobtasWs ws;
  pobtas_ws(n, b, a, reinterpret_cast<char*>(workspace), &ws);
  SweepArgs p{};
  Band& g = p.g;
  g.n = n; g.b = b; g.a = a;
  g.ldb = ldb;
  g.dg = const_cast<double*>(diag);
  g.lw = const_cast<double*>(lower);
  g.ar = const_cast<double*>(arrow);
  g.tp = const_cast<double*>(tip);
  g.data = g.dg;
  g.nbt = (b + 127) / 128;
  g.nat = a > 0 ? (a + 127) / 128 : 0;
  g.S = n * g.nbt + g.nat;
  g.SP = g.S;
  g.use_arrow = has_arrow && a > 0;
  g.vec_b = 0;
  g.vec_a = 0;
  p.ntile = n * g.nbt;
  p.ldx = nrhs;
  p.flags = ws.flags;
  p.flags2 = ws.flags2;
  p.push2 = ws.push2;
  p.ticket = ws.ticket;
  p.part = ws.part;
  p.xtip = ws.xtip;
  p.push = ws.push;
  p.winv = ws.winv;
  p.prof = debug_profile();
  for (int c0 = 0; c0 < nrhs; c0 += NR) {
    p.x = rhs + c0;
    p.ncols = nrhs - c0 < NR ? nrhs - c0 : NR;
    int e = run_sweeps(p, mode, ws, st);
    if (e) return e;
  }
  return 0;
}

}  // extern "C"
