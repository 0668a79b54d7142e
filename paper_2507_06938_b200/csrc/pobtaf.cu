// POBTAF: in-place block Cholesky of an SPD BTA matrix as ONE persistent
// task-graph kernel (C ABI).
//
// Reference: bta.factorize (pkg/src/stinla/bta.py:177-235), per time block i
//   diag[i]    = chol(diag[i])                                  (bta.py:206)
//   lower[i]   = lower[i] diag[i]^-T,  arrow[i] = arrow[i] diag[i]^-T  (213-219)
//   diag[i+1] -= lower[i] lower[i]^T;  arrow[i+1] -= arrow[i] lower[i]^T;
//   tip       -= arrow[i] arrow[i]^T                             (222-227)
// then tip = chol(tip) (bta.py:228-232), and logdet (bta.py:238-246).
//
// B200 mapping.  The same elimination, refined to 128-wide panels of the
// lower band (band.cuh), is a DAG of four task kinds:
//   POTRF(s)        Cholesky + inverse W_s of diagonal tile s (one CTA)
//   TRSM(s,R,q)     32-row strip q of tile (R,s) := strip W_s^T   (DMMA)
//   UPDATE(s,R,C)   tile (R,C) -= X_R X_C^T, X = panel s tiles     (DMMA)
//   STRIP(s,R,q)    lower part of strip q of diagonal tile (R,R)   (DMMA)
// A persistent kernel (one CTA per SM) claims tasks from an atomic ticket in
// a fixed topological order with one panel of look-ahead:
//   P(0) U0(0) | P(1) Urest(0) U0(1) | P(2) Urest(1) U0(2) | ...
// (U0 = updates of the next panel's column, Urest = the rest).  A task only
// waits (acquire-spin on per-strip counters) for tasks with smaller tickets,
// which are already running, so the schedule cannot deadlock; every tile is
// updated in panel order, so results are bitwise deterministic.  A non-SPD
// pivot sets info (1 + time block, n+1 for the tip) and an abort word that
// drains the kernel.  Log-det partials per panel are summed in a fixed order.
#include <cub/block/block_scan.cuh>
#include <cstdlib>
#include <cstring>

#include "../../include/stbta.h"
#include "band.cuh"
#include "potrf_tile.cuh"
#include "tile_mma.cuh"
#include "tma_mma.cuh"
#include "memops.cuh"

namespace stbta {

constexpr int DAG_NT = 256;
using Cfg128 = MmaCfg<128, 128, 64, 32, DAG_NT, 32, 2>;
using Cfg32 = MmaCfg<32, 128, 32, 16, DAG_NT>;
constexpr int TRSM_SMEM_DOUBLES = 32 * 132 + 128 * 132 + 4 * 32 * PT_WLD;
constexpr int cmax(int x, int y) { return x > y ? x : y; }
constexpr int DAG_SMEM_DOUBLES =
    cmax(cmax(cmax(PT_SMEM_DOUBLES, TRSM_SMEM_DOUBLES), Cfg128::SMEM_DOUBLES), TMA_SMEM_DOUBLES);
constexpr int W_SLOT = 4 * 32 * 32;  // per panel: the four W_kk^T blocks
constexpr size_t DAG_SMEM_BYTES = DAG_SMEM_DOUBLES * sizeof(double);

// Ticket order, eight groups per panel s (the critical chain first, then the
// second-row look-ahead, then the bulk of the previous panel, then this
// panel's remaining TRSMs and column s+1):
//   G0 TRSM(s, s+1, q)          the next diagonal tile's strips   [critical]
//   G1 STRIP(s-1, s+1, q)       previous panel's update of that tile
//   G2 STRIP(s, s+1, q)         this panel's update of it  -> POTRF(s+1)
//   G3 TRSM(s, r1, q)           r1 = second band row (= s+2 inside a block)
//   G4 UPDATE(s-1, r1, s+1), UPDATE(s, r1, s+1)   -> TRSM(s+1, r1) = G0(s+1)
//   G5 E(s-1) \ (G1, G4)        bulk updates of panel s-1, columns >= s+1
//   G6 TRSM(s, R, q), R beyond r1
//   G7 UPDATE(s, R, s+1), R beyond r1
// Every task depends only on tasks of earlier groups (or the panel worker's
// POTRF, which depends only on earlier groups), so ticket order is a
// topological order and spinning never deadlocks.
enum { T_POTRF = 0, T_TRSM = 1, T_UPD = 2, T_STRIP = 3 };
constexpr int NGRP = 8;
constexpr int PROF_TL = 64;  // debug profile: per-panel timeline (12 slots) from here
struct DagWs {
  int* gstart;   // G + 1 group starts
  int* ctr;      // dependency counters
  double* W;     // S slots of W_SLOT doubles (diagonal-block inverses)
  double* slots; // S log-det partials
  int* ticket;
  int* abort_flag;
  int* role;     // first CTA to arrive becomes the panel (POTRF) worker
  int G;
  unsigned long long* prof;  // optional: per task type {count, wait ns, exec ns}
  const unsigned* ready;     // optional: per time block upload flags (stbta_upload_blocks)
  unsigned epoch;            // ... a block is resident once ready[t] - epoch >= 0
};

// Upload chunk holding tile (R, C): chunk t = {diag[t], lower[t], arrow[t]},
// the tip travels with the first chunk (every block's arrow updates it).
STBTA_DEV int tile_chunk(const Band& g, int C) {
  return C < g.n * g.nbt ? C / g.nbt : 0;
}

// Wait until the chunk of tile column C is resident (pipelined host upload).
STBTA_DEV bool wait_resident(const Band& g, const DagWs& ws, int C) {
  if (ws.ready == nullptr) return true;
  const unsigned* p = ws.ready + tile_chunk(g, C);
  int it = 0;
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    if ((int)(v - ws.epoch) >= 0) return true;
    if (ld_volatile(ws.abort_flag)) return false;
    // back off: many CTAs may poll the same flag while a chunk is in flight
    __nanosleep(it < 4 ? 128 : 1024);
    ++it;
  }
}

STBTA_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// does panel p = s-1 update tile (s+1, s+1)?  (then G1(s) holds its strips)
STBTA_DEV bool g1_active(const Band& g, int s) {
  if (s < 1) return false;
  int mb;
  const int mp = band_rows(g, s - 1, &mb);
  return mp >= 2 && band_row(g, s - 1, 1, mb) == s + 1;
}

// Chunked updates: tile (R, C) is first needed when panel C is factored, so
// the updates of an aligned chunk of CHUNK consecutive panels p of one block
// whose last panel is at least LOOK panels before C are applied as ONE task
// with K = CHUNK*128 (one C-tile load/store and one pipeline fill per chunk
// instead of per panel).  Updates close to the panel front (the next LOOK
// columns, which the critical chain needs one panel at a time) stay per panel.
// CHUNK panels per fused update: 8 for wide blocks (many tile columns), else 4.
// LOOK >= 2 is required: G1 issues panel s-1's update of tile (s+1, s+1) on
// its own, so that tile must never be part of a chunk.
STBTA_DEV int look(const Band& g) { return g.look > 0 ? g.look : (g.nbt >= 24 ? 2 : 3); }
STBTA_DEV int chunk_k(const Band& g) { return g.chunk > 0 ? g.chunk : (g.nbt >= 24 ? 8 : 4); }
STBTA_DEV bool remainder_chunks(const Band& g) {
  return g.remainder >= 0 ? g.remainder != 0 : g.nbt >= 24;
}
STBTA_DEV int chunk_first(const Band& g, int p) {
  const int t = p / g.nbt, j = p - t * g.nbt;
  return t * g.nbt + (j / chunk_k(g)) * chunk_k(g);
}
STBTA_DEV int chunk_end(const Band& g, int p) {
  return min(chunk_first(g, p) + chunk_k(g) - 1, (p / g.nbt + 1) * g.nbt - 1);
}
STBTA_DEV bool chunk_last(const Band& g, int p) { return p == chunk_end(g, p); }
STBTA_DEV bool cross_col(const Band& g, int p, int C) {
  if (p >= g.n * g.nbt) return false;
  return C >= chunk_end(g, p) + 1 + look(g);
}

// How panel p's update of tile column C is issued:
//   1  per panel (the last LOOK panels before C, and arrow panels),
//   2  as part of a chunk task (s0 = chunk_first(p)) issued at this panel:
//      an aligned chunk at its last panel when all of it is >= LOOK panels
//      before C, else the remainder [chunk_first(p), C - LOOK - 1] at panel
//      C - LOOK - 1 -- so every column gets at most LOOK single-panel
//      updates, each issued LOOK panels ahead of its use,
//   0  not at this panel (it is in a chunk task issued elsewhere).
// The remainder chunks only pay for wide blocks (the C3 block size: 1.6% on
// POBTAF); with narrow ones (C2) the window is all per-panel, as before.
STBTA_DEV int col_mode(const Band& g, int p, int C) {
  if (p >= g.n * g.nbt) return 1;
  if (cross_col(g, p, C)) return chunk_last(g, p) ? 2 : 0;
  if (C <= p + look(g) || !remainder_chunks(g)) return 1;
  return p == C - look(g) - 1 ? 2 : 0;
}

// Does panel p = s-1 update tile (r1, s+1), r1 = second band row of s?  Then
// that update is hoisted from the bulk (G5) to the front of G4, ahead of
// panel s's own update of the tile (never chunked: its column is s+1).
STBTA_DEV bool g4_prev(const Band& g, int s) {
  if (s < 1 || s >= g.SP) return false;
  int mb, mbp;
  const int m = band_rows(g, s, &mb);
  if (m < 2) return false;
  const int mp = band_rows(g, s - 1, &mbp);
  return mp >= 3 && band_row(g, s - 1, 1, mbp) == s + 1 &&
         band_row(g, s - 1, 2, mbp) == band_row(g, s, 1, mb);
}

STBTA_DEV int group_size(const Band& g, int kind, int s) {
  int mb;
  if (s >= g.SP) {  // trailing groups: only the last eliminated panel's bulk (G1, G5)
    if (kind != 1 && kind != 5) return 0;
  }
  const int m = s < g.S ? band_rows(g, s, &mb) : 0;
  switch (kind) {
    case 0: return m >= 1 ? NSTRIP : 0;
    case 1: return g1_active(g, s) ? NSTRIP : 0;
    case 2: return m >= 1 ? NSTRIP : 0;
    case 3: return m >= 2 ? NSTRIP : 0;
    case 4: return (m >= 2 ? 1 : 0) + (g4_prev(g, s) ? 1 : 0);
    case 5: {
      if (s < 1) return 0;
      const int p = s - 1;
      const int mp = band_rows(g, p, &mb);
      int e = 0;
      for (int j = 1; j < mp; ++j) {
        if (col_mode(g, p, band_row(g, p, j, mb)) == 0) continue;
        e += NSTRIP + (mp - 1 - j);
      }
      return e - (g1_active(g, s) ? NSTRIP : 0) - (g4_prev(g, s) ? 1 : 0);
    }
    case 6: return m >= 3 ? NSTRIP * (m - 2) : 0;
    default: return m >= 3 ? m - 2 : 0;
  }
}

// one extra (partial) group set after the last eliminated panel carries its bulk updates
inline int n_groups(int SP) { return NGRP * SP + 6; }

// one CTA of 1024 threads: gstart[gi] = sum of sizes of groups < gi
__global__ void __launch_bounds__(1024) dag_setup_kernel(Band g, DagWs ws) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int G = ws.G;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < G; base += 1024) {
    const int gi = base + threadIdx.x;
    int sz = 0;
    if (gi < G) sz = group_size(g, gi % NGRP, gi / NGRP);
    int ex, tot;
    Scan(tmp).ExclusiveSum(sz, ex, tot);
    if (gi < G) ws.gstart[gi] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) ws.gstart[G] = carry;
}

struct Task {
  int type, s, R, C, q;
  int s0;  // first panel of a chunked update (== s otherwise)
};


// Group containing ticket t (gstart[lo] <= t < gstart[lo+1]): a 32-ary search
// by one full warp (3 dependent load rounds instead of ~13 for a binary search).
STBTA_DEV int find_group(const DagWs& ws, int t) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = ws.G;  // invariant: gstart[lo] <= t < gstart[hi]
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) / 32;
    const int idx = lo + (lane + 1) * step;
    const bool le = idx < hi && __ldg(ws.gstart + idx) <= t;
    const int cnt = __popc(__ballot_sync(0xffffffffu, le));
    const int nlo = lo + cnt * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  return lo;
}

STBTA_DEV Task decode(const Band& g, const DagWs& ws, int t, int lo) {
  const int kind = lo % NGRP, s = lo / NGRP;
  int local = t - __ldg(ws.gstart + lo);
  Task k{};
  k.s0 = -1;
  switch (kind) {
    case 0: k.type = T_TRSM; k.s = s; k.R = s + 1; k.q = local; return k;
    case 1: k.type = T_STRIP; k.s = s - 1; k.R = k.C = s + 1; k.q = local; return k;
    case 2: k.type = T_STRIP; k.s = s; k.R = k.C = s + 1; k.q = local; return k;
    case 3:
    case 6: {
      int mb;
      band_rows(g, s, &mb);
      const int off = kind == 3 ? 1 : 2;
      k.type = T_TRSM; k.s = s; k.R = band_row(g, s, off + local / NSTRIP, mb); k.q = local % NSTRIP;
      return k;
    }
    case 4: {
      int mb;
      band_rows(g, s, &mb);
      k.type = T_UPD; k.R = band_row(g, s, 1, mb); k.C = s + 1;
      k.s = (local == 0 && g4_prev(g, s)) ? s - 1 : s;
      return k;
    }
    case 7: {
      int mb;
      band_rows(g, s, &mb);
      k.type = T_UPD; k.s = s; k.R = band_row(g, s, 2 + local, mb); k.C = s + 1;
      return k;
    }
    default: break;
  }
  // G5: E(p), p = s-1, columns j = 1..mp-1; column 1's strips are in G1 when active
  const int p = s - 1;
  int mb;
  const int mp = band_rows(g, p, &mb);
  const bool skip = g1_active(g, s);
  const int hoist = g4_prev(g, s) ? 1 : 0;  // UPDATE(p, band_row 2, band_row 1) is in G4
  k.s = p;
  for (int j = 1; j < mp; ++j) {
    const int c = band_row(g, p, j, mb);
    const int mode = col_mode(g, p, c);
    if (mode == 0) continue;
    k.s0 = mode == 2 ? chunk_first(g, p) : p;
    const int ns = (j == 1 && skip) ? 0 : NSTRIP;
    const int hj = j == 1 ? hoist : 0;
    const int cnt = ns + (mp - 1 - j) - hj;
    if (local < cnt) {
      if (local < ns) { k.type = T_STRIP; k.R = k.C = c; k.q = local; return k; }
      k.type = T_UPD;
      k.R = band_row(g, p, j + 1 + hj + (local - ns), mb);
      k.C = c;
      return k;
    }
    local -= cnt;
  }
  k.type = -1;  // unreachable
  return k;
}

STBTA_DEV int need(const Band& g, int R, int C) { return n_updates(g, R, C, C); }

// Tensor maps of the diag / lower / arrow regions (rows x b, row stride ldb),
// 16 x 128 boxes, 128-byte swizzle; ok[i] == 0 when a region is not eligible.
struct TmaMaps {
  CUtensorMap m[3];
  int ok[3];
};

STBTA_DEV TmaOpnd tile_tma(const Band& g, const TmaMaps& tm, int R, int C) {
  TmaOpnd o{nullptr, 0, 0};
  const int NB = g.n * g.nbt;
  if (C >= NB) return o;  // tip: no map
  const int tc = C / g.nbt, jc = C % g.nbt;
  o.col = jc * TT;
  int r;
  if (R >= NB) {
    r = 2;
    o.row = tc * g.a + (R - NB) * TT;
  } else {
    const int tr = R / g.nbt, jr = R % g.nbt;
    r = (tr == tc) ? 0 : 1;
    o.row = tc * g.b + jr * TT;
  }
  if (tm.ok[r]) o.map = &tm.m[r];
  return o;
}

// The panel worker: POTRF(s) for s = 0..S-1 in order, on one dedicated CTA
// (its instruction cache stays warm with the factorization code, and the
// panel chain never queues behind bulk updates).  Returns false on abort.
STBTA_DEV bool potrf_worker(const Band& g, const DagWs& ws, int* info, double* smem) {
  __shared__ int s_ok, s_fail;
  __shared__ double s_logdet;
  const int tid = threadIdx.x;
  const int NB = g.n * g.nbt;
  for (int s = 0; s < g.SP; ++s) {
    const int w = tile_extent(g, s);
    unsigned long long t0 = 0, t1 = 0;
    if (ws.prof != nullptr && tid == 0) t0 = gtimer();
    if (tid == 0) { s_ok = 1; s_fail = 0; }
    __syncthreads();
    // strips 0..NSTRIP-2 of the tile are loaded as soon as each is final (the
    // STRIP tasks of one panel finish in strip order: strip q is 32(q+1)
    // columns wide), overlapping the wait for the last one
    double* T = smem;
    const TilePtr tp = tile_ptr(g, s, s);
    auto load_strip = [&](int q) {
      const int warp = tid >> 5, lane = tid & 31;
      for (int r = 32 * q + warp; r < min(w, 32 * q + 32); r += DAG_NT / 32) {
        const double* src = tp.p + (long long)r * tp.ld;
        for (int c = lane; c <= r; c += 32) cp_async8(T + r * PT_LD + c, src + c, true);
      }
    };
    if (tid == NSTRIP) {
      const unsigned long long tw0 = ws.prof ? gtimer() : 0;
      if (!wait_resident(g, ws, s)) s_ok = 0;
      if (ws.prof) {
        unsigned long long* tlp = ws.prof + PROF_TL + (long long)s * 12;
        tlp[10] = tw0;
        tlp[11] = gtimer();
      }
    }
    for (int q = 0; q < NSTRIP; ++q) {
      if (tid == 0 && !spin_geq(counter(g, ws.ctr, s, q, s), need(g, s, s), ws.abort_flag)) s_ok = 0;
      __syncthreads();
      if (!s_ok) return false;
      load_strip(q);
    }
    if (ws.prof != nullptr && tid == 0) t1 = gtimer();
    {
      double* WT = T + 128 * PT_LD;
      double* scratch = WT + 4 * 32 * PT_WLD;
      cp_async_commit();
      if (w < 128) {  // identity padding of a partial tile
        for (int e = tid; e < 128 * 128; e += DAG_NT) {
          const int r = e >> 7, c = e & 127;
          if (r >= w || c >= w) T[r * PT_LD + c] = (r == c) ? 1.0 : 0.0;
        }
      }
      cp_async_wait<0>();
      __syncthreads();
      unsigned long long ph[4] = {0, 0, 0, 0};
      const unsigned long long tl = (ws.prof && tid == 0) ? gtimer() : 0;
      const int fail = potrf_tile_smem<DAG_NT>(T, WT, scratch, &s_logdet, &s_fail,
                                               ws.prof ? ph : nullptr);
      if (fail) {
        if (tid == 0) {
          const int code = (s < NB) ? 1 + s / g.nbt : 1 + g.n;
          atomicCAS(info, 0, code);
          __threadfence();
          atomicExch(ws.abort_flag, 1);
        }
        return false;
      }
      // First what the TRSM tasks read: the strictly-lower 32-blocks of L and
      // the W_kk^T blocks; the diagonal 32-blocks and the zero upper part are
      // stored after the signal (nobody reads them inside the kernel).
      {
        const int warp = tid >> 5, lane = tid & 31;
        for (int r = 32 + warp; r < w; r += DAG_NT / 32) {
          double* dst = tp.p + (long long)r * tp.ld;
          const int cend = min(w, r & ~31);
          for (int c = lane; c < cend; c += 32) dst[c] = T[r * PT_LD + c];
        }
      }
      double* Wg = ws.W + (long long)s * W_SLOT;
      for (int e = tid; e < W_SLOT; e += DAG_NT) {
        const int kb = e >> 10, c = (e >> 5) & 31, i = e & 31;
        Wg[e] = WT[kb * 32 * PT_WLD + c * PT_WLD + i];
      }
      if (tid == 0) ws.slots[s] = s_logdet;
      __syncthreads();
      if (ws.prof && tid == 0) {
        const unsigned long long te = gtimer();
        for (int k = 0; k < 3; ++k) atomicAdd(ws.prof + 12 + k, ph[k]);
        atomicAdd(ws.prof + 16, (te - tl) - (ph[0] + ph[1] + ph[2]));
        atomicAdd(ws.prof + 17, tl - t1);
      }
      if (tid == 0) {
        __threadfence();
        for (int q = 0; q < NSTRIP; ++q) atomicAdd(counter(g, ws.ctr, s, q, s), 1);
        if (ws.prof) {
          const unsigned long long tend = gtimer();
          atomicAdd(ws.prof + 0, 1ull);
          atomicAdd(ws.prof + 1, t1 - t0);
          atomicAdd(ws.prof + 2, tend - t1);
          unsigned long long* tlp = ws.prof + PROF_TL + (long long)s * 12;
          tlp[0] = t0; tlp[1] = t1; tlp[2] = tend;
        }
      }
      {  // the rest of the tile: diagonal 32-blocks of L and zeros above them
        const int warp = tid >> 5, lane = tid & 31;
        for (int r = warp; r < w; r += DAG_NT / 32) {
          double* dst = tp.p + (long long)r * tp.ld;
          for (int c = (r & ~31) + lane; c < w; c += 32) dst[c] = (c <= r) ? T[r * PT_LD + c] : 0.0;
        }
      }
    }
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(DAG_NT, 1) pobtaf_dag_kernel(Band g, DagWs ws, int* info,
                                                              const __grid_constant__ TmaMaps tm) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_ticket, s_ok;
  __shared__ Task s_task;
  const int tid = threadIdx.x;
  const int total = ws.gstart[ws.G];
  const int NB = g.n * g.nbt;
  __shared__ int s_role;
  if (tid == 0) s_role = atomicAdd(ws.role, 1);
  __syncthreads();
  if (s_role == 0) {
    potrf_worker(g, ws, info, smem);
    return;
  }
  __shared__ unsigned long long s_tbars[TMA_NBARS];
  tma_bars_init(s_tbars);
  unsigned tphase = 0;

  for (;;) {
    if (tid < 32) {
      int t = 0;
      if (tid == 0) t = atomicAdd(ws.ticket, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      int grp = 0;
      if (t < total) grp = find_group(ws, t);
      if (tid == 0) {
        s_ticket = t;
        if (t < total) {
          Task tk2 = decode(g, ws, t, grp);
          if (tk2.s0 < 0) tk2.s0 = tk2.s;
          s_task = tk2;
        }
        s_ok = 1;
      }
    }
    __syncthreads();
    if (s_ticket >= total) break;
    const Task tk = s_task;
    const int s = tk.s;
    const int w = tile_extent(g, s);  // panel width = K of every product
    unsigned long long t0 = 0, t1 = 0;
    if (ws.prof != nullptr && tid == 0) t0 = gtimer();

    // UPDATE: pull the C tile toward L2 while the dependencies are awaited, so
    // the accumulator load after them does not pay the HBM latency (a stale
    // copy is harmless: L2 is the point of coherence for the final writes)
    if (tk.type == T_UPD) {
      const TilePtr cp0 = tile_ptr(g, tk.R, tk.C);
      const int er = tile_extent(g, tk.R), ec = tile_extent(g, tk.C);
      const int lines = (ec * 8 + 127) / 128;  // 128-byte lines per row
      for (int e = tid; e < er * lines; e += DAG_NT) {
        const int r = e / lines, l = e - r * lines;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cp0.p + (long long)r * cp0.ld + l * 16));
      }
    }

    // ------------------------------------------------------ dependencies
    {
      const int* p = nullptr;
      int target = 0;
      if (tk.type == T_TRSM) {
        if (tid < NSTRIP) { p = counter(g, ws.ctr, s, tid, s); target = need(g, s, s) + 1; }
        else if (tid == NSTRIP) { p = counter(g, ws.ctr, tk.R, tk.q, s); target = need(g, tk.R, s); }
      } else if (tk.type == T_UPD) {
        const int np = s - tk.s0 + 1, nd = NSTRIP * np;  // panels s0..s
        if (tid < nd) {
          const int sp = tk.s0 + tid / NSTRIP;
          p = counter(g, ws.ctr, tk.R, tid % NSTRIP, sp); target = need(g, tk.R, sp) + 1;
        } else if (tid < 2 * nd) {
          const int sp = tk.s0 + (tid - nd) / NSTRIP;
          p = counter(g, ws.ctr, tk.C, (tid - nd) % NSTRIP, sp); target = need(g, tk.C, sp) + 1;
        } else if (tid < 2 * nd + NSTRIP) {
          p = counter(g, ws.ctr, tk.R, tid - 2 * nd, tk.C); target = n_updates(g, tk.R, tk.C, tk.s0);
        }
      } else {  // T_STRIP
        const int np = s - tk.s0 + 1;
        if (tid < NSTRIP * np) {
          const int sp = tk.s0 + tid / NSTRIP, q = tid % NSTRIP;
          if (q <= tk.q) { p = counter(g, ws.ctr, tk.R, q, sp); target = need(g, tk.R, sp) + 1; }
        } else if (tid == 64) {
          p = counter(g, ws.ctr, tk.R, tk.q, tk.R); target = n_updates(g, tk.R, tk.R, tk.s0);
        }
      }
      if (p != nullptr && !spin_geq(p, target, ws.abort_flag)) s_ok = 0;
      if (tid == 96 && !wait_resident(g, ws, tk.type == T_UPD ? tk.C : tk.type == T_STRIP ? tk.R : s))
        s_ok = 0;
      __syncthreads();
      if (!s_ok) break;
    }
    if (ws.prof != nullptr && tid == 0) t1 = gtimer();

    // ------------------------------------------------------ execute
    if (tk.type == T_TRSM) {
      const int ext = tile_extent(g, tk.R);
      const int r0 = tk.q * TS;
      const int rows = min(TS, ext - r0);
      if (rows > 0) {
        constexpr int XLD = 132;
        double* X = smem;                 // 32 x XLD
        constexpr int TLD = 132;          // 4 mod 16: conflict-free fragment reads
        double* Ls = X + 32 * XLD;        // 128 x TLD (strictly lower blocks used)
        double* WT = Ls + 128 * TLD;      // 4 x 32 x PT_WLD
        const TilePtr xp = tile_ptr(g, tk.R, s);
        const TilePtr lp = tile_ptr(g, s, s);
        double* Xg = xp.p + (long long)r0 * xp.ld;
        const bool xv = ((uintptr_t)Xg % 16 == 0) && (xp.ld % 2 == 0);
        const bool lv = ((uintptr_t)lp.p % 16 == 0) && (lp.ld % 2 == 0);
        if (xv) {  // 16-byte copies (zero fill past the tile)
          for (int e = tid; e < 32 * 64; e += DAG_NT) {
            const int r = e >> 6, c = (e & 63) * 2;
            const int bytes = (r < rows && c < w) ? ((c + 1 < w) ? 16 : 8) : 0;
            cp_async16(X + r * XLD + c, bytes ? Xg + (long long)r * xp.ld + c : Xg, bytes);
          }
        } else {
          for (int e = tid; e < 32 * 128; e += DAG_NT) {
            const int r = e >> 7, c = e & 127;
            if (r < rows && c < w) cp_async8(X + r * XLD + c, Xg + (long long)r * xp.ld + c, true);
            else X[r * XLD + c] = 0.0;
          }
        }
        if (lv) {  // strictly-lower 32-blocks: 6 blocks of 32 x 32
          for (int e = tid; e < 6 * 32 * 16; e += DAG_NT) {
            // blocks (1,0) (2,0) (2,1) (3,0) (3,1) (3,2)
            const int blk = e >> 9, rr = (e >> 4) & 31, cc = (e & 15) * 2;
            const int br = blk < 1 ? 1 : (blk < 3 ? 2 : 3);
            const int bc = blk - br * (br - 1) / 2;
            const int r = br * 32 + rr, c = bc * 32 + cc;
            const int bytes = (r < w && c < w) ? ((c + 1 < w) ? 16 : 8) : 0;
            cp_async16(Ls + r * TLD + c, bytes ? lp.p + (long long)r * lp.ld + c : lp.p, bytes);
          }
        } else {
          for (int e = tid; e < 128 * 128; e += DAG_NT) {
            const int r = e >> 7, c = e & 127;
            if ((r >> 5) > (c >> 5)) {  // strictly-lower 32-blocks
              if (r < w && c < w) cp_async8(Ls + r * TLD + c, lp.p + (long long)r * lp.ld + c, true);
              else Ls[r * TLD + c] = 0.0;
            }
          }
        }
        const double* Wg = ws.W + (long long)s * W_SLOT;
        for (int e = tid; e < W_SLOT; e += DAG_NT) {
          const int kb = e >> 10, c = (e >> 5) & 31, i = e & 31;
          cp_async8(WT + kb * 32 * PT_WLD + c * PT_WLD + i, Wg + e, true);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        unsigned long long ta = 0, tb = 0;
        if (ws.prof && tid == 0) ta = gtimer();
        trsm_strip_smem<DAG_NT, XLD, TLD>(X, Ls, WT, w);
        if (ws.prof && tid == 0) {
          tb = gtimer();
          atomicAdd(ws.prof + 18, ta - t1);
          atomicAdd(ws.prof + 19, tb - ta);
        }
        for (int e = tid; e < rows * w; e += DAG_NT) {
          const int r = e / w, c = e - r * w;
          Xg[(long long)r * xp.ld + c] = X[r * XLD + c];
        }
        const bool same_block = (tk.R < NB) ? (s < NB && tk.R / g.nbt == s / g.nbt) : (s >= NB);
        if (same_block) {
          // clear the mirrored strict-upper strip of the diagonal block / tip
          const TilePtr up = tile_ptr_upper(g, tk.R, s);
          for (int e = tid; e < w * rows; e += DAG_NT) {
            const int r = e / rows, c = e % rows;
            up.p[(long long)r * up.ld + r0 + c] = 0.0;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(counter(g, ws.ctr, tk.R, tk.q, s), 1);
      }
    } else if (tk.type == T_UPD) {
      // panels s0..s of one block: their tile columns are contiguous in storage
      const int kw = (s - tk.s0) * TT + w;
      const TilePtr rp = tile_ptr(g, tk.R, tk.s0);
      const TilePtr cp = tile_ptr(g, tk.C, tk.s0);
      const TilePtr tp = tile_ptr(g, tk.R, tk.C);
      const int er = tile_extent(g, tk.R), ec = tile_extent(g, tk.C);
      double acc[Cfg128::MF][Cfg128::NF][2];
      const Opnd A{rp.p, rp.ld, er, rp.vec};
      const Opnd B{cp.p, cp.ld, ec, cp.vec};
      // the C tile loads overlap the first operand slabs' copies
      auto cload = [&] { acc_load<Cfg128>(acc, tp.p, tp.ld, er, ec, 0, 0); };
      const TmaOpnd ta = tile_tma(g, tm, tk.R, tk.s0), tb = tile_tma(g, tm, tk.C, tk.s0);
      if (ta.map != nullptr && tb.map != nullptr && (kw % 32 == 0 || ta.col + kw == g.b))
        tile_mma_tma<Cfg128, true>(acc, ta, tb, kw, smem, s_tbars, tphase, cload, er, ec);
      else
        tile_mma<Cfg128, true>(acc, A, B, kw, 128, smem, 0, cload);
      if (ws.prof && tid == 0) atomicAdd(ws.prof + 22, gtimer() - t1);
      acc_store<Cfg128>(acc, tp.p, tp.ld, er, ec, 0, 0, 0, 1.0);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        for (int q = 0; q < NSTRIP; ++q) atomicAdd(counter(g, ws.ctr, tk.R, q, tk.C), s - tk.s0 + 1);
      }
    } else {  // T_STRIP
      unsigned long long ta = 0;
      const int ext = tile_extent(g, tk.R);
      const int r0 = tk.q * TS;
      const int rows = min(TS, ext - r0);
      const int kw = (s - tk.s0) * TT + w;
      if (rows > 0) {
        const TilePtr xp = tile_ptr(g, tk.R, tk.s0);
        const TilePtr tp = tile_ptr(g, tk.R, tk.R);
        const int ncol = min(r0 + TS, ext);
        double acc[Cfg32::MF][Cfg32::NF][2];
        const Opnd A{xp.p + (long long)r0 * xp.ld, xp.ld, rows, xp.vec};
        const Opnd B{xp.p, xp.ld, ncol, xp.vec};
        tile_mma<Cfg32, true>(acc, A, B, kw, ncol, smem, 0, [&] {
          acc_load<Cfg32>(acc, tp.p + (long long)r0 * tp.ld, tp.ld, rows, ncol, 1, r0);
        });
        if (ws.prof && tid == 0) {
          ta = gtimer();
          atomicAdd(ws.prof + 20, ta - t1);
        }
        acc_store<Cfg32>(acc, tp.p + (long long)r0 * tp.ld, tp.ld, rows, ncol, 1, r0, 0, 1.0);
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(counter(g, ws.ctr, tk.R, tk.q, tk.R), s - tk.s0 + 1);
      }
    }
    if (ws.prof != nullptr && tid == 0) {
      const unsigned long long t2 = gtimer();
      if ((tk.type == T_TRSM || tk.type == T_STRIP) && tk.R == tk.s + 1 && tk.s + 1 < g.SP) {
        unsigned long long* tlp = ws.prof + PROF_TL + (long long)tk.s * 12 + (tk.type == T_TRSM ? 3 : 6);
        atomicMax(tlp + 0, t0); atomicMax(tlp + 1, t1); atomicMax(tlp + 2, t2);
      }
      if (tk.type == T_STRIP && tk.R == tk.s + 2 && tk.s + 2 < g.SP)
        atomicMax(ws.prof + PROF_TL + (long long)(tk.s + 1) * 12 + 9, t2);
      // updates of tile (C+1, C) (the tile TRSM(C, C+1) solves): slot 10 = claim of the
      // latest one, slot 11 = its completion, for panel C
      if (tk.type == T_UPD && tk.R == tk.C + 1 && tk.C < g.SP) {
        atomicMax(ws.prof + PROF_TL + (long long)tk.C * 12 + 10, t0);
        atomicMax(ws.prof + PROF_TL + (long long)tk.C * 12 + 11, t2);
      }
      atomicAdd(ws.prof + 3 * tk.type, 1ull);
      atomicAdd(ws.prof + 3 * tk.type + 1, t1 - t0);
      atomicAdd(ws.prof + 3 * tk.type + 2, t2 - t1);
    }
    __syncthreads();
  }
}

// out[0] = 2 * sum(slots[0:count]) in a fixed order (deterministic).
__global__ void dag_logdet_kernel(const double* slots, int count, double* out) {
  __shared__ double part[256];
  const int tid = threadIdx.x;
  const int per = (count + 255) / 256;
  double acc = 0.0;
  for (int i = tid * per; i < min(count, (tid + 1) * per); ++i) acc += slots[i];
  part[tid] = acc;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (tid < k) part[tid] += part[tid + k];
    __syncthreads();
  }
  if (tid == 0) out[0] = 2.0 * part[0];
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static bool al16(const void* p) { return ((uintptr_t)p % 16) == 0; }

// nfact < 0: full factorization (all blocks and the tip).  0 <= nfact <= n:
// factorize only the first nfact time blocks (partial elimination); the
// remaining blocks and the tip receive their updates but stay unfactored.
static Band make_band(const double* const* regions, int n, int b, int a, int use_arrow,
                      int nfact, int ldb) {
  Band g{};
  g.n = n; g.b = b; g.a = a;
  g.ldb = ldb;
  g.nbt = (b + TT - 1) / TT;
  g.nat = a > 0 ? (a + TT - 1) / TT : 0;
  g.S = n * g.nbt + g.nat;
  g.SP = (nfact < 0) ? g.S : nfact * g.nbt;
  g.use_arrow = use_arrow && a > 0;
  if (regions != nullptr) {
    g.dg = const_cast<double*>(regions[0]);
    g.lw = const_cast<double*>(regions[1]);
    g.ar = const_cast<double*>(regions[2]);
    g.tp = const_cast<double*>(regions[3]);
    g.data = g.dg;
  }
  // tuning overrides (experiments; defaults by block width in look / chunk_k)
  static const int env_chunk = [] { const char* v = getenv("STBTA_CHUNK"); return v ? atoi(v) : 0; }();
  static const int env_look = [] { const char* v = getenv("STBTA_LOOK"); return v ? atoi(v) : 0; }();
  static const int env_rem = [] { const char* v = getenv("STBTA_REMAINDER"); return v ? atoi(v) : -1; }();
  g.chunk = env_chunk;
  g.look = env_look >= 2 ? env_look : 0;  // LOOK >= 2 is required (G1)
  g.remainder = env_rem;
  const bool base16 = al16(g.dg) && (n < 2 || al16(g.lw)) && (a == 0 || al16(g.ar));
  g.vec_b = base16 && (ldb % 2 == 0);
  g.vec_a = g.vec_b && (a % 2 == 0) && (a == 0 || al16(g.tp));
  return g;
}

// workspace: gstart | ctr, ticket, abort (one memset) | slots | W
static size_t dag_ws(const Band& g, char* base, DagWs* o, size_t* zero_bytes) {
  const int G = n_groups(g.SP);
  const size_t gs = align_up((size_t)(G + 1) * sizeof(int));
  const long long nctr = counter_elems(g.n, g.nbt, g.nat, g.S);
  const size_t cz = align_up((size_t)(nctr + 3) * sizeof(int));
  const size_t sl = align_up((size_t)g.S * sizeof(double));
  const size_t wb = (size_t)g.S * W_SLOT * sizeof(double);
  if (o) {
    o->gstart = reinterpret_cast<int*>(base);
    o->ctr = reinterpret_cast<int*>(base + gs);
    o->ticket = o->ctr + nctr;
    o->abort_flag = o->ticket + 1;
    o->role = o->ticket + 2;
    o->slots = reinterpret_cast<double*>(base + gs + cz);
    o->W = reinterpret_cast<double*>(base + gs + cz + sl);
    o->G = G;
    o->prof = nullptr;
    o->ready = nullptr;
    o->epoch = 0;
  }
  if (zero_bytes) *zero_bytes = cz;
  return gs + cz + sl + wb;
}

// One 2D tensor map per storage region (diag, lower, arrow): width b columns,
// height = the region's rows, row stride ldb doubles.  Disabled (ok = 0) when
// the driver entry point is missing, rows are not 16-byte aligned (odd ldb),
// or STBTA_NO_TMA=1 is set.
static void make_tma_maps(const Band& g, TmaMaps* tm) {
  memset(tm, 0, sizeof(*tm));
  static const bool off = [] {
    const char* v = getenv("STBTA_NO_TMA");
    return v && v[0] == '1';
  }();
  TensorMapEncodeFn enc = tensor_map_encode();
  if (off || enc == nullptr || !g.vec_b) return;
  const double* base[3] = {g.dg, g.lw, g.ar};
  const long long rows[3] = {(long long)g.n * g.b, (long long)(g.n - 1) * g.b,
                             g.use_arrow ? (long long)g.n * g.a : 0};
  for (int r = 0; r < 3; ++r) {
    if (base[r] == nullptr || rows[r] <= 0 || ((uintptr_t)base[r] % 16) != 0) continue;
    const cuuint64_t dims[2] = {(cuuint64_t)g.b, (cuuint64_t)rows[r]};
    const cuuint64_t strides[1] = {(cuuint64_t)g.ldb * sizeof(double)};
    const cuuint32_t box[2] = {16, 128};
    const cuuint32_t es[2] = {1, 1};
    const CUresult e = enc(&tm->m[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base[r]),
                           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    tm->ok[r] = (e == CUDA_SUCCESS) ? 1 : 0;
  }
}

static int sm_count() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}

}  // namespace stbta

using namespace stbta;

extern "C" {

const char* stbta_version(void) { return "stbta 0.2.0 (sm_100a, FP64 DMMA task-graph)"; }

long long stbta_storage_elems(int n, int b, int a) {
  return (long long)n * b * b + (long long)(n - 1) * b * b + (long long)n * a * b +
         (long long)a * a;
}

size_t stbta_pobtaf_workspace_bytes(int n, int b, int a) {
  if (n < 1 || b < 1 || a < 0) return 0;
  const Band g = make_band(nullptr, n, b, a, 1, -1, b);
  return dag_ws(g, nullptr, nullptr, nullptr);
}

int stbta_pobtaf(double* data, int n, int b, int a, int use_arrow, double* logdet_out, int* info,
                 void* workspace, size_t workspace_bytes, void* stream) {
  if (data == nullptr) return STBTA_EARG;
  const long long bb = (long long)b * b;
  double* diag = data;
  double* lower = data + (long long)n * bb;
  double* arrow = lower + (long long)(n - 1) * bb;
  double* tip = arrow + (long long)n * a * b;
  return stbta_pobtaf_ex(diag, lower, arrow, tip, n, b, a, b, use_arrow, -1, logdet_out, info,
                         workspace, workspace_bytes, stream);
}

static int pobtaf_impl(double* diag, double* lower, double* arrow, double* tip, int n, int b, int a,
                       int ldb, int use_arrow, int nfact, double* logdet_out, int* info,
                       const unsigned* ready, unsigned epoch, void* workspace,
                       size_t workspace_bytes, void* stream);

int stbta_pobtaf_ex(double* diag, double* lower, double* arrow, double* tip, int n, int b, int a,
                    int ldb, int use_arrow, int nfact, double* logdet_out, int* info,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return pobtaf_impl(diag, lower, arrow, tip, n, b, a, ldb, use_arrow, nfact, logdet_out, info,
                     nullptr, 0u, workspace, workspace_bytes, stream);
}

int stbta_pobtaf_ready(double* data, int n, int b, int a, int use_arrow, double* logdet_out,
                       int* info, const unsigned* ready, unsigned epoch, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (data == nullptr || ready == nullptr) return STBTA_EARG;
  const long long bb = (long long)b * b;
  double* lower = data + (long long)n * bb;
  double* arrow = lower + (long long)(n - 1) * bb;
  double* tip = arrow + (long long)n * a * b;
  return pobtaf_impl(data, lower, arrow, tip, n, b, a, b, use_arrow, -1, logdet_out, info, ready,
                     epoch, workspace, workspace_bytes, stream);
}

}  // extern "C"

static int pobtaf_impl(double* diag, double* lower, double* arrow, double* tip, int n, int b, int a,
                       int ldb, int use_arrow, int nfact, double* logdet_out, int* info,
                       const unsigned* ready, unsigned epoch, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (diag == nullptr || n < 1 || b < 1 || a < 0 || info == nullptr || nfact > n || ldb < b)
    return STBTA_EARG;
  if ((n > 1 && lower == nullptr) || (a > 0 && (arrow == nullptr || tip == nullptr)))
    return STBTA_EARG;
  if (workspace_bytes < stbta_pobtaf_workspace_bytes(n, b, a)) return STBTA_EWORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double* regions[4] = {diag, lower, arrow, tip};
  const Band g = make_band(regions, n, b, a, use_arrow, nfact, ldb);
  if (g.SP == 0) {  // nothing to eliminate
    int e = zero_async(info, sizeof(int), st);
    if (!e && logdet_out) e = zero_async(logdet_out, sizeof(double), st);
    return e;
  }
  DagWs ws;
  size_t zbytes = 0;
  dag_ws(g, reinterpret_cast<char*>(workspace), &ws, &zbytes);
  ws.prof = debug_profile();
  ws.ready = ready;
  ws.epoch = epoch;
  static std::atomic<unsigned long long> attr_mask{0};  // per device
  if (attr_pending(attr_mask)) {
    int e = (int)cudaFuncSetAttribute(pobtaf_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)DAG_SMEM_BYTES);
    if (e) return e;
    attr_mark(attr_mask);
  }
  int e = zero_async(info, sizeof(int), st);
  if (e) return e;
  if ((e = zero_async(ws.ctr, zbytes, st))) return e;
  dag_setup_kernel<<<1, 1024, 0, st>>>(g, ws);
  count_launch();
  if ((e = (int)cudaGetLastError())) return e;
  TmaMaps tm;
  make_tma_maps(g, &tm);
  pobtaf_dag_kernel<<<sm_count(), DAG_NT, DAG_SMEM_BYTES, st>>>(g, ws, info, tm);
  count_launch();
  if ((e = (int)cudaGetLastError())) return e;
  if (logdet_out != nullptr) {
    dag_logdet_kernel<<<1, 256, 0, st>>>(ws.slots, g.SP, logdet_out);
    count_launch();
    if ((e = (int)cudaGetLastError())) return e;
  }
  return 0;
}
