/*
 * stbta — B200-native (sm_100a) BTA structured solver, C ABI.
 *
 * Drop-in boundary for the reference's solver layer (stinla, pure Python on
 * numpy/scipy).  Every pointer argument is a DEVICE pointer
 * unless stated otherwise, every entry point is stream-ordered on `stream`
 * (a cudaStream_t passed as void*), never synchronises, holds no global
 * mutable state and is re-entrant for distinct streams and workspaces.
 *
 * Storage: one flat FP64 buffer per BTA matrix, in the reference order
 *   diag (n,b,b) | lower (n-1,b,b) [block (i+1,i)] | arrow (n,a,b) | tip (a,a)
 * all row-major  (reference BTAMatrix, pkg/src/stinla/bta.py:50-89).
 *
 * Return value: 0 on success, >0 a cudaError_t from a launch, <0 an argument
 * error (STBTA_EARG / STBTA_EWORKSPACE).  Numerical failure (a non-positive
 * pivot, the reference's FactorizationError, bta.py:17-31) is NOT a return
 * code: it is written to the device word *info as 1 + block index (n for the
 * tip, so info == n+1), read back by the caller at its single sync point.
 */
#ifndef STBTA_H
#define STBTA_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STBTA_EARG (-1)
#define STBTA_EWORKSPACE (-2)

/* Library version string (host). */
const char* stbta_version(void);

/* Number of FP64 elements of the flat BTA buffer: n*b*b+(n-1)*b*b+n*a*b+a*a
 * (reference BTAMatrix.__init__, bta.py:69-72). */
long long stbta_storage_elems(int n, int b, int a);

/* ---------------------------------------------------------------- POBTAF --
 * In-place block Cholesky of an SPD BTA matrix.
 * Replaces: bta.factorize (pkg/src/stinla/bta.py:177-235) + bta.logdet
 * (bta.py:238-246).  use_arrow = 0 skips all arrow work exactly like the
 * reference's `use_arrow = a > 0 and np.any(arrow)` (bta.py:200-202); the tip
 * is still factorized when a > 0 (bta.py:228-232).
 * logdet_out (device double) = 2 * sum log diag(L), fixed summation order.
 * info (device int) is zeroed first, then set on failure.
 * workspace: >= stbta_pobtaf_workspace_bytes(n,b,a) bytes of device memory. */
size_t stbta_pobtaf_workspace_bytes(int n, int b, int a);
int stbta_pobtaf(double* data, int n, int b, int a, int use_arrow, double* logdet_out, int* info,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Region-pointer form of POBTAF (diag (n,b,b), lower (n-1,b,b), arrow (n,a,b),
 * tip (a,a) may live in separate buffers; the block rows may be padded to a
 * row stride ldb >= b, e.g. b+1 for odd b so every row is 16-byte aligned)
 * with a partial-elimination count:
 * nfact < 0 is the full factorization; 0 <= nfact <= n factorizes only the
 * first nfact time blocks, leaving the later blocks and the tip updated by
 * their Schur complement but unfactored, and
 * logdet_out covering the eliminated blocks only (time partitions of
 * bta_dist.d_factorize, reference bta_dist.py:174-254). */
int stbta_pobtaf_ex(double* diag, double* lower, double* arrow, double* tip, int n, int b, int a,
                    int ldb, int use_arrow, int nfact, double* logdet_out, int* info,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- POBTAS --
 * Triangular solves against a POBTAF factor, in place on rhs (dim x nrhs,
 * row-major, dim = n*b+a).  mode 0: L L^T x = r (bta.solve, bta.py:305-307);
 * 1: L y = r (forward_substitute, bta.py:249-275); 2: L^T x = r
 * (backward_substitute, bta.py:278-302).  has_arrow = BTAFactor.has_arrow. */
size_t stbta_pobtas_workspace_bytes(int n, int b, int a, int nrhs);
int stbta_pobtas(const double* factor, int n, int b, int a, int has_arrow, double* rhs, int nrhs,
                 int mode, void* workspace, size_t workspace_bytes, void* stream);

/* Region-pointer form of POBTAS (block row stride ldb >= b). */
int stbta_pobtas_ex(const double* diag, const double* lower, const double* arrow,
                    const double* tip, int n, int b, int a, int ldb, int has_arrow, double* rhs,
                    int nrhs, int mode, void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------------------------- POBTASI --
 * Selected inversion: the BTA-pattern entries of (L L^T)^-1 written to `inv`
 * (a separate buffer of the same layout; X_ii stored full symmetric).
 * Replaces: bta.selected_invert (pkg/src/stinla/bta.py:310-359). */
size_t stbta_pobtasi_workspace_bytes(int n, int b, int a);
int stbta_pobtasi(const double* factor, double* inv, int n, int b, int a, int has_arrow,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Region-pointer form of POBTASI.  nstart < 0 is the full selected inversion;
 * 0 <= nstart <= n continues a recursion whose blocks nstart.. (X diag /
 * lower / arrow) and X_tip are already in the output
 * (partition interiors of bta_dist.d_selected_invert, bta_dist.py:461-602). */
int stbta_pobtasi_ex(const double* Ld, const double* Ll, const double* La, const double* Lt,
                     double* Xd, double* Xl, double* Xa, double* Xt, int n, int b, int a,
                     int has_arrow, int nstart, void* workspace, size_t workspace_bytes,
                     void* stream);

/* ----------------------------------------- pipelined host <-> device I/O --
 * The reference keeps matrices in host memory (numpy); a host-resident BTA
 * matrix used through the device path (BTAMatrix(host data) -> factorize ->
 * solve -> selected_invert -> host inverse, bta.py:50-359) is moved in time-
 * block chunks overlapped with the compute instead of before / after it.
 * Requires the driver's stream memory operations (cuStreamWriteValue32 /
 * cuStreamWaitValue32, resolved at run time):
 *   stbta_stream_memops_supported: 1 when available (else the entry points
 *     below return cudaErrorNotSupported).
 *   stbta_upload_blocks: copy the flat buffer src_host (PINNED host memory)
 *     to dst on `stream` in chunks {diag[t], lower[t], arrow[t]} (the tip with
 *     the first chunk), writing ready[t] = epoch after chunk t has landed.
 *   stbta_pobtaf_ready: stbta_pobtaf whose task graph starts at once and waits
 *     per task for ready[chunk] - epoch >= 0 of the block it touches; `stream`
 *     must NOT wait for the upload stream (that is the point), and the upload
 *     must not wait for `stream` after this launch.
 *   stbta_pobtasi_stream_out: stbta_pobtasi on `stream`, plus block-wise
 *     device->host copies of the inverse into host_out (PINNED, flat layout)
 *     on copy_stream, each gated on the recursion's completion counter of that
 *     block; record an event on copy_stream to know when host_out is final. */
int stbta_stream_memops_supported(void);
int stbta_upload_blocks(double* dst, const double* src_host, int n, int b, int a, unsigned* ready,
                        unsigned epoch, void* stream);
int stbta_pobtaf_ready(double* data, int n, int b, int a, int use_arrow, double* logdet_out,
                       int* info, const unsigned* ready, unsigned epoch, void* workspace,
                       size_t workspace_bytes, void* stream);
int stbta_pobtasi_stream_out(const double* factor, double* inv, double* host_out, int n, int b,
                             int a, int has_arrow, void* workspace, size_t workspace_bytes,
                             void* stream, void* copy_stream);

/* ------------------------------------------------ W-based POBTAS (solve) --
 * The block inverses W_t = L_tt^-1 (and W_tip) that POBTASI computes first
 * can be computed once per factor and shared between the triangular solves
 * and the selected inversion:
 *   stbta_pobtasi_prepare: W into a POBTASI workspace (stbta_pobtasi_workspace_bytes).
 *   stbta_pobtas_w: same contract as stbta_pobtas (bta.solve / forward_substitute /
 *     backward_substitute, bta.py:249-307) but each block step is a GEMV with W_t
 *     (y_t = W_t (r_t - L_{t,t-1} y_{t-1}), x_t = W_t^T (...)) in one cooperative
 *     kernel; si_workspace = the prepared POBTASI workspace, workspace of
 *     stbta_pobtas_w_workspace_bytes.
 *   stbta_pobtasi_prepared: stbta_pobtasi (host_out NULL) or
 *     stbta_pobtasi_stream_out (host_out pinned) on a prepared workspace; skips
 *     the W pre-pass. */
int stbta_pobtasi_prepare(const double* factor, int n, int b, int a, void* workspace,
                          size_t workspace_bytes, void* stream);
size_t stbta_pobtas_w_workspace_bytes(int n, int b, int a);
int stbta_pobtas_w(const double* factor, int n, int b, int a, int has_arrow, double* rhs,
                   int nrhs, int mode, const void* si_workspace, void* workspace,
                   size_t workspace_bytes, void* stream);
int stbta_pobtasi_prepared(const double* factor, double* inv, double* host_out, int n, int b,
                           int a, int has_arrow, void* workspace, size_t workspace_bytes,
                           void* stream, void* copy_stream);

/* ------------------------------------------------------ Q assembly / f_obj --
 * stbta_assemble: write the theta-dependent values of a precision matrix into
 * a BTA buffer of nstore elements, zero everywhere else.  Replaces the value
 * map of model.spatio_temporal_precision / build_univariate_prior
 * (pkg/src/stinla/model.py:196-248), coreg.assemble_joint_precision
 * (coreg.py:80-121), ObjectiveEvaluator._conditional_matrix (inla.py:264-283)
 * and coreg.map_to_bta incl. its zero fill (coreg.py:250-276):
 *   data[offsets[e]] = sum_t coef[pair[e]*nterms + t] * basis[src[e]*nterms + t]
 * offsets (int64, strictly increasing) come from PermutationMap.bind
 * (coreg.py:186-241); tile_start[k] = first e with offsets[e] >= k*TILE,
 * k = 0..ceil(nstore/TILE), TILE = stbta_assemble_tile_elems(). */
int stbta_assemble_tile_elems(void);
int stbta_assemble(double* data, long long nstore, const long long* tile_start,
                   const long long* offsets, const int* pair, const int* src, const double* basis,
                   const double* coef, int nterms, void* stream);
/* out[0] = x^T Q x over the symmetric matrix described by the same entry
 * list (lower BTA envelope, off-diagonal blocks counted twice); x in BTA
 * order.  Replaces `mu @ (prior_matrix @ mu)` (inla.py:369).  partial: npartial
 * doubles of scratch; summation order fixed. */
int stbta_quadform(const long long* offsets, const int* pair, const int* src, const double* basis,
                   const double* coef, int nterms, long long nentries, int n, int b, int a,
                   const double* x, double* partial, int npartial, double* out, void* stream);
/* out[e] = sum_i tau[i] * U[i*N + e], i < nv: the conditional-mean right-hand
 * side design^T (noise * y) in BTA order (inla.py:313-315). */
int stbta_rhs_combine(double* out, const double* U, const double* tau, int nv, long long N,
                      void* stream);
/* out[i] = sum_{r in [seg[i], seg[i+1])} (y[r] - (A x)[r])^2 for the CSR design
 * A (columns already in BTA order); sq: nrows doubles of scratch
 * (inla.py:363-367). */
int stbta_residual(const long long* indptr, const int* indices, const double* vals,
                   long long nrows, const double* y, const double* x, const long long* seg,
                   int nseg, double* sq, double* out, void* stream);

/* --------------------------------------------- time-partitioned solver --
 * Coupling products of the partitioned solve (S3): the thin products that
 * join a partition's interior solve to the reduced separator system
 * (replaces the `@` / `np.einsum` couplings of bta_dist.d_solve,
 * pkg/src/stinla/bta_dist.py:370-458):
 *   Y_j += alpha * op(A_j) X_j, j < nbatch        (reduce == 0)
 *   Y   += alpha * sum_j op(A_j) X_j, j ascending (reduce != 0)
 * A_j: m x n row-major, row stride lda, batch stride strideA;
 * op(A) = A (trans == 0: X_j n x k, Y_j m x k) or A^T (trans != 0: X_j m x k,
 * Y_j n x k); X / Y rows are k wide with row strides ldx / ldy >= k and batch
 * strides strideX / strideY (0 broadcasts X).  Fixed summation order
 * (bitwise reproducible).  workspace >= stbta_couple_workspace_bytes(...). */
size_t stbta_couple_workspace_bytes(int trans, int nbatch, int m, int n, int reduce);
int stbta_couple(int trans, int nbatch, int m, int n, int k, double alpha, const double* A,
                 long long lda, long long strideA, const double* X, long long ldx,
                 long long strideX, double* Y, long long ldy, long long strideY, int reduce,
                 void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------- instrumentation --
 * Kernel launches issued by this library since load (host counter; bench.py
 * reports the difference over its timed region as gpu_launches). */
long long stbta_launch_count(void);
/* FP64 peak probes (bench.py's roofline denominator; MEASURED_PEAKS.json has
 * no FP64 entry).  blocks x 256 threads; FLOPs = blocks*8*iters*16*512 for
 * the DMMA.8x8x4 probe and blocks*256*iters*16 for the DFMA probe. */
/* Debug hook: device buffer of 12 u64 into which POBTAF accumulates, per task
 * kind (POTRF, TRSM, UPDATE, STRIP), {count, ns waiting, ns executing};
 * NULL disables (the default). */
void stbta_debug_set_profile(unsigned long long* buf);
/* Launch blocks x 256 threads, each warp issuing iters*16 DMMA.8x8x4:
 * FLOPs = blocks*8*iters*16*512. */
int stbta_probe_dmma(int blocks, int iters, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STBTA_H */
