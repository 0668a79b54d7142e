/*
 * stbta tools library (libstbta_tools.so): micro-benchmarks and debug probes
 * used by tools/ only -- NOT part of the drop-in boundary (include/stbta.h).
 */
#ifndef STBTA_TOOLS_H
#define STBTA_TOOLS_H

#include "stbta.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C = alpha * op(A) * op(B) + beta * C on the FP64 DMMA engine (row-major,
 * op = transpose when ta/tb != 0). */
int stbta_dgemm(int ta, int tb, int M, int N, int K, double alpha, const double* A, long long lda,
                const double* B, long long ldb, double beta, double* C, long long ldc,
                void* stream);
/* *out (device u64) = %globaltimer (ns) when this point of `stream` runs. */
int stbta_debug_globaltimer(unsigned long long* out, void* stream);
/* `grid` CTAs each run `reps` tile products C_t -= A_t B_t^T (128x128, depth K)
 * of CTA shape `variant`. */
int stbta_debug_tile_bench(int variant, const double* A, const double* B, double* C, int ntile,
                           int reps, int grid, int K, void* stream);
/* `grid` CTAs each factorize + invert the SPD 128x128 tile A `reps` times; ph
 * (6 u64) receives CTA 0's phase times in ns. */
int stbta_debug_potrf_bench(const double* A, double* out, int reps, int grid,
                            unsigned long long* ph, void* stream);
/* Cross-SM flag round trips from CTA 0 to every other CTA (one per SM, `reps`
 * each; flags: 64 * SMs zeroed ints): out[4k..4k+3] = ping written (CTA 0
 * %globaltimer), ping seen (CTA k), pong seen (CTA 0), smid of k. */
int stbta_debug_timer_skew(int reps, int* flags, long long* out, void* stream);
/* clock cycles of `iters` dependent DMMA (which=0) or DFMA (1) on one warp. */
int stbta_debug_latency(int which, int iters, double* scratch, long long* cycles, void* stream);
/* DMMA throughput with shared-memory fragment loads (mode 0 LDS.64, 1 LDS.128,
 * 2 none); FLOPs = grid*8*iters*8*32*512. */
int stbta_debug_lds_bench(int mode, int iters, int grid, double* out, void* stream);
/* blocks x 256 threads, each thread iters*8 DFMA: FLOPs = blocks*256*iters*16. */
int stbta_probe_dfma(int blocks, int iters, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STBTA_TOOLS_H */
