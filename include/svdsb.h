/*
 * svdsb.h -- C ABI of the B200-native PHSVDS hot path (libsvdsb.so).
 *
 * Everything below is plain C: opaque handles, raw pointers, 64-bit sizes,
 * int status codes.  No torch / C++ types cross this boundary, so the same
 * library can be bound from ctypes (what the Python package does), cgo, JNI
 * or N-API.  See INTEGRATION.md for the binding stubs.
 *
 * Conventions (PRIMME's, fixed as stable API by the reference spec,
 * /root/reference/SPEC.md:183 and PAPER.md:701-709):
 *   - dense blocks are column-major fp64 with an explicit leading dimension
 *     (x, ldx): element (i, j) lives at x[i + j*ldx];
 *   - every pointer named x/y/v/w/... is a DEVICE pointer unless the
 *     parameter name ends in _host;
 *   - every call is asynchronous on the caller's CUDA stream (`stream`,
 *     a cudaStream_t passed as void*; NULL = legacy default stream) unless
 *     documented otherwise;
 *   - return value 0 = success, < 0 = error; svdsb_last_error() returns the
 *     message of the last failure on the calling thread.
 *
 * Reference interfaces each entry point replaces are cited per function
 * (paths relative to /root/reference).
 */
#ifndef SVDSB_H
#define SVDSB_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVDSB_OK 0
#define SVDSB_ERR_ARG (-1)      /* invalid argument (maps to ValueError)   */
#define SVDSB_ERR_CUDA (-2)     /* CUDA runtime failure                    */
#define SVDSB_ERR_ALLOC (-3)    /* device/host allocation failure          */
#define SVDSB_ERR_RANGE (-4)    /* size beyond the int32-index device layout */
#define SVDSB_ERR_FORMAT (-5)   /* malformed Matrix Market input (MatrixMarketError) */
#define SVDSB_ERR_IO (-6)       /* file cannot be opened / read / written (OSError) */

typedef struct svdsb_ctx svdsb_ctx;  /* per-stream workspace for reductions */
typedef struct svdsb_csr svdsb_csr;  /* device CSR of A plus stored A^T     */

/* ------------------------------------------------------------------ */
/* library / context                                                   */

int svdsb_version(void);
const char *svdsb_last_error(void);
/* Number of kernels this library launched since load (the bench's
 * gpu_launches evidence). */
int64_t svdsb_launch_count(void);
/* Adds n to that counter: a CUDA-graph replay of n captured library kernels
 * is n launches the host no longer makes one by one. */
int64_t svdsb_note_launches(int64_t n);
/* Kernel-variant knob for measurement tools (key < 17; value 0 = default
 * dispatch).  Not part of the reference interface.  Set it before the
 * first solve: CUDA graphs captured earlier keep the kernels they were
 * captured with. */
int svdsb_tune_set(int key, int value);

/* Status plumbing: asynchronous device->host copy on `stream` (dst should be
 * pinned) and a stream synchronisation -- the single per-iteration host
 * round trip of the solver. */
int svdsb_d2h(void *dst_host, const void *src, size_t bytes, void *stream);
int svdsb_stream_sync(void *stream);

/* CUDA-graph capture of a launch sequence on a non-default `stream`
 * (thread-local capture mode), instantiation + upload, replay and release.
 * The solver captures the device work of one Davidson iteration once per
 * shape and replays it (eigensolver.py:563-700's per-iteration kernels). */
int svdsb_graph_begin(void *stream);
int svdsb_graph_end(void *stream, void **exec_out);
/* Ends the capture and, when exec_in is not NULL, updates that executable
 * graph in place with the captured one (same topology -- e.g. the same
 * iteration on a new matrix of the same shape); falls back to a fresh
 * instantiation (*exec_out != exec_in, the caller releases exec_in). */
int svdsb_graph_end_update(void *stream, void *exec_in, void **exec_out);
int svdsb_graph_launch(void *exec, void *stream);
int svdsb_graph_destroy(void *exec);

/* A context owns the device workspace used by the deterministic two-level
 * reductions (per-CTA partials + a ticket counter).  One context per stream
 * in flight. */
int svdsb_ctx_create(int device, svdsb_ctx **out);
int svdsb_ctx_destroy(svdsb_ctx *ctx);

/* ------------------------------------------------------------------ */
/* sparse matrix: replaces SparseMatrixCsr (pkg/src/itersvd/matio.py:22-123) */

#define SVDSB_CSR_TRANSPOSE 1   /* also build CSR(A^T) on device          */

/* Upload a host CSR in the reference layout (int64 row_ptr[m+1], int64
 * col_idx[nnz] strictly increasing per row, fp64 values[nnz]); validates
 * like SparseMatrixCsr.__init__ (matio.py:35-52), stores int32 indices on
 * device, and with SVDSB_CSR_TRANSPOSE builds CSR(A^T) equal bit for bit to
 * SparseMatrixCsr.from_coo(n, m, col_idx, rows, values) (matio.py:63-92).
 * Synchronises `stream` before returning. */
int svdsb_csr_create_host(svdsb_ctx *ctx, int64_t m, int64_t n, int64_t nnz,
                          const int64_t *row_ptr_host,
                          const int64_t *col_idx_host,
                          const double *values_host, int flags, void *stream,
                          svdsb_csr **out);
/* Assemble from COO triplets already on device (int64 rows/cols, fp64
 * vals) with SparseMatrixCsr.from_coo semantics (matio.py:63-92): entries
 * sorted by (row, col), duplicates summed in ascending input order. */
int svdsb_csr_create_coo_device(svdsb_ctx *ctx, int64_t m, int64_t n,
                                int64_t ntrip, const int64_t *rows,
                                const int64_t *cols, const double *vals,
                                int flags, void *stream, svdsb_csr **out);
/* As above, with the values possibly still being copied to the device on
 * another stream: `vals_ready` (a cudaEvent_t recorded after that copy, or
 * NULL) is waited on by `stream` just before the duplicate sums, the first
 * use of `vals` -- the key build, sort and scans of the indices overlap the
 * copy (SparseMatrixCsr.from_coo from host arrays, matio.py:63-92). */
int svdsb_csr_create_coo_device_ev(svdsb_ctx *ctx, int64_t m, int64_t n,
                                   int64_t ntrip, const int64_t *rows,
                                   const int64_t *cols, const double *vals,
                                   void *vals_ready, int flags, void *stream,
                                   svdsb_csr **out);
int svdsb_csr_destroy(svdsb_csr *a);
int svdsb_csr_shape(const svdsb_csr *a, int64_t *m, int64_t *n, int64_t *nnz);
/* Derived device layouts of a handle (tests / tools; not part of the
 * reference interface).  key 0: slices of the forward sliced-ELL copy (0
 * until a 2..4-column product built it); 1: operand rows the forward b = 4
 * kernel keeps in shared memory (0: hot-column copy not built); 2: column
 * blocks of the stored transpose. */
int svdsb_csr_layout_info(const svdsb_csr *a, int key, int64_t *out);
/* Copy CSR(A) (transpose = 0) or CSR(A^T) (transpose = 1) back to host in
 * the reference's int64/fp64 layout (bit-exactness checks).  Synchronous. */
int svdsb_csr_export_host(const svdsb_csr *a, int transpose,
                          int64_t *row_ptr_host, int64_t *col_idx_host,
                          double *values_host);

/* Borrow the device arrays of CSR(A) (transpose = 0) or CSR(A^T): int32
 * row_ptr[rows+1], int32 col[nnz], fp64 val[nnz].  Valid until destroy. */
int svdsb_csr_device_arrays(const svdsb_csr *a, int transpose,
                            const int **row_ptr, const int **col,
                            const double **val);

/* y = op(A) x for a block of `block` columns: the PRIMME matrixMatvec
 * contract; replaces spmv_block (matio.py:126-155) and
 * SvdOperator.apply / apply_t (operators.py:117-129).
 * transpose = 0: x is n x block, y is m x block; transpose = 1: A^T.
 * Summation order per output element reproduces the reference bit for bit
 * for rows that fit one tile: forward = p0 + numpy-pairwise(p1..) of the
 * rounded products (np.add.reduceat), transpose = left-to-right over
 * ascending rows (np.add.at).  Rows longer than a tile use a deterministic
 * chunked reduction instead. */
int svdsb_matvec(svdsb_ctx *ctx, const svdsb_csr *a, int transpose,
                 const double *x, int64_t ldx, double *y, int64_t ldy,
                 int block, void *stream);
/* Normal-equations operator without forming it (make_normal_operator,
 * operators.py:163-172): side 0 -> y = A^T (A x) (dimension n),
 * side 1 -> y = A (A^T x) (dimension m).  tmp: scratch of the inner
 * dimension x block (ldtmp). */
int svdsb_apply_normal(svdsb_ctx *ctx, const svdsb_csr *a, int side,
                       const double *x, int64_t ldx, double *y, int64_t ldy,
                       int block, double *tmp, int64_t ldtmp, void *stream);
/* Augmented operator [0 A^T; A 0] on stacked [v (n); u (m)] vectors
 * (make_augmented_operator, operators.py:175-190): y[:n] = A^T x[n:],
 * y[n:] = A x[:n]. */
int svdsb_apply_augmented(svdsb_ctx *ctx, const svdsb_csr *a, const double *x,
                          int64_t ldx, double *y, int64_t ldy, int block,
                          void *stream);

/* Point-Jacobi diagonal (jacobi_precond_on_normal, operators.py:225-249):
 * side 0 -> squared column norms (column_sq_norms, matio.py:115-118),
 * side 1 -> squared row norms (row_sq_norms, matio.py:120-123); each clamped
 * below at EPS * max.  d has n (side 0) or m (side 1) entries. Bit-exact. */
int svdsb_precond_diag(svdsb_ctx *ctx, const svdsb_csr *a, int side,
                       double *d, void *stream);
/* The unclamped squared norms of svdsb_precond_diag (column_sq_norms /
 * row_sq_norms, matio.py:115-123): the per-rank partial of the sharded
 * Jacobi diagonal, summed over ranks and clamped by the caller (dist.py). */
int svdsb_row_sq(svdsb_ctx *ctx, const svdsb_csr *a, int side, double *d,
                 void *stream);
/* y = x ./ d (applyPreconditioner; the lambda at
 * operators.py:249).  y may alias x. */
int svdsb_diag_solve(int64_t dim, const double *d, const double *x,
                     int64_t ldx, double *y, int64_t ldy, int block,
                     void *stream);

/* ------------------------------------------------------------------ */
/* tall-skinny fp64 kernels (kernels.py, eigensolver.py dense work).      */
/* Up to SVDSB_MAX_BLOCKS column blocks can be passed as one concatenated */
/* operand [X_0 | X_1 | ...] (the `against` lists of kernels.py:47-51).   */

#define SVDSB_MAX_BLOCKS 4

/* C (ldc) = [X_0|X_1|..]^T Y : (sum cols) x b, deterministic two-level
 * reduction.  Replaces b.T @ v (kernels.py:50), V^T W (eigensolver.py:351,
 * :690).  If norms2 != NULL also writes ||Y[:,j]||^2 (before anything). */
int svdsb_gram(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs,
               const int64_t *ldxs, const int *cols, const double *y,
               int64_t ldy, int b, double *c, int64_t ldc, double *norms2,
               void *stream);
/* Y -= [X_0|X_1|..] C  (C device, (sum cols) x b, ldc); then, if norms2
 * != NULL, norms2[j] = ||Y[:,j]||^2 of the updated block.  One classical
 * Gram-Schmidt projection (kernels.py:47-51 / :497-499). */
int svdsb_project_out(svdsb_ctx *ctx, int64_t dim, int nblk,
                      const double *const *xs, const int64_t *ldxs,
                      const int *cols, const double *c, int64_t ldc, double *y,
                      int64_t ldy, int b, double *norms2, void *stream);
/* Y = alpha * X C + beta * Y ; X dim x g, C (device) g x s.  Replaces
 * V @ coefs (eigensolver.py:526-527), V @ y (:390, :710, :760).  beta == 0
 * never reads Y.  Y may alias X only exactly (y == x, ldy == ldx: the
 * in-place restart V <- V C) with s <= min(g, 32), alpha 1, beta 0; any
 * other overlap is undefined. */
int svdsb_ts_gemm(svdsb_ctx *ctx, int64_t dim, const double *x, int64_t ldx,
                  int g, const double *c, int64_t ldc, int s, double alpha,
                  double beta, double *y, int64_t ldy, void *stream);
/* Fused Ritz candidates (eigensolver.py:385-394): for j < p
 *   X[:,j] = V Yc[:,j], OX[:,j] = W Yc[:,j], R[:,j] = OX[:,j] - lam[j] X[:,j]
 * writes R (and X / OX when non-NULL) and rn2[j] = ||R[:,j]||^2.
 * lam, yc, rn2 are device arrays. */
int svdsb_ritz_residual(svdsb_ctx *ctx, int64_t dim, const double *v,
                        int64_t ldv, const double *w, int64_t ldw, int g,
                        const double *yc, int64_t ldyc, const double *lam,
                        int p, double *r, int64_t ldr, double *x, int64_t ldx,
                        double *ox, int64_t ldox, double *rn2, void *stream);
/* out[j] = ||X[:,j]||^2 (deterministic). */
int svdsb_col_norms2(svdsb_ctx *ctx, int64_t dim, const double *x,
                     int64_t ldx, int b, double *out, void *stream);
/* Column dot products out[j] = X[:,j] . Y[:,j]. */
int svdsb_col_dots(svdsb_ctx *ctx, int64_t dim, const double *x, int64_t ldx,
                   const double *y, int64_t ldy, int b, double *out,
                   void *stream);
/* Y[:,j] = X[:,j] * f(s[j]) with s a DEVICE array: mode 0 multiply,
 * mode 1 divide, mode 2 divide by sqrt (normalise from a squared norm).
 * Columns whose factor is 0 (mode 1/2) are left untouched.  Y may alias X. */
int svdsb_scale_cols(int64_t dim, const double *x, int64_t ldx, int b,
                     const double *s, int mode, double *y, int64_t ldy,
                     void *stream);
/* Y = alpha X + beta Y elementwise on dim x b. */
int svdsb_axpby(int64_t dim, int b, double alpha, const double *x,
                int64_t ldx, double beta, double *y, int64_t ldy,
                void *stream);
/* Device-indexed column gather: with f = *first (a device int),
 * Y[:, c] = X[:, f + c] (divided elementwise by d when d != NULL, exactly
 * as svdsb_diag_solve) for c < ncols and f + c < limit.  The column index
 * lives on the device so captured iteration graphs need not be re-captured
 * when the selected Ritz candidate changes (eigensolver.py:598-607 picks
 * the first unconverged one; :520-527 keeps its +k neighbours). */
int svdsb_gather_cols(int64_t dim, const double *x, int64_t ldx,
                      const int *first, int ncols, int limit,
                      const double *d, double *y, int64_t ldy, void *stream);
/* Iteration status straight into pinned (UVA-mapped) host memory:
 * host_dst[0:gn] = lams, [gn:gn+p] = rn2, [gn+p:gn+p+8] = state; the host
 * reads it after an event on `stream` (the per-iteration status read of
 * eigensolver.py:563-607). */
int svdsb_status_pack(const double *lams, int gn, const double *rn2, int p,
                      const double *state, double *host_dst, void *stream);
/* As svdsb_status_pack with nstate consecutive 8-double DGKS records (one
 * per column of a block expansion): host_dst receives gn + p + 8*nstate. */
int svdsb_status_pack_n(const double *lams, int gn, const double *rn2, int p,
                        const double *state, int nstate, double *host_dst,
                        void *stream);
/* Standard-normal block out[r + c*ldo] (r < rows, c < cols) for global rows
 * row0 .. row0+rows-1 of a cols-wide block: element (R, c) is a pure
 * function of (seed, R*cols + c) (Philox4x32-10 counter RNG, Box-Muller), so
 * a row-partitioned caller gets the slices of one global block.  Replaces
 * the host draw rng.standard_normal((N, cols)) of eigensolver.py:283-292
 * for large N (a different stream: same distribution, not the same bits). */
int svdsb_randn(uint64_t seed, int64_t row0, int64_t rows, int cols,
                double *out, int64_t ldo, void *stream);
/* *dst = v on the stream (stream-ordered scalar update for the above). */
int svdsb_set_int(int *dst, int v, void *stream);
/* Stage-2 split statistics of candidate vectors on the stacked layout
 * [v (nsplit); u (dim-nsplit)] (hybrid.py:226-241, :413-423): for each
 * column j writes 6 sums to out[6j..6j+5]:
 *   ||r_v||^2, r_v.x_v, ||x_v||^2, ||r_u||^2, r_u.x_u, ||x_u||^2 */
int svdsb_split_stats(svdsb_ctx *ctx, int64_t dim, int64_t nsplit,
                      const double *r, int64_t ldr, const double *x,
                      int64_t ldx, int b, double *out, void *stream);

/* Exact stage-2 split residual from the split statistics (hybrid.py:
 * 226-241): with nv = ||x_v||, nu = ||x_u||, sigma = |lam[j]| (lam device),
 *   e1 = r_u/nv + (lam/nv - sigma/nu) x_u   (= A v^ - sigma u^)
 *   e2 = r_v/nu + (lam/nu - sigma/nv) x_v   (= A^T u^ - sigma v^)
 * out[j] = ||e1||^2 + ||e2||^2, formed elementwise (no cancellation).
 * stats: the 6-per-column output of svdsb_split_stats (device).  Columns
 * with nv == 0 or nu == 0 get out[j] = +inf. */
/* The whole single-column expansion orthonormalisation in one launch (basis
 * of <= 40 columns): x = R[:, *ci] (./ d when d != NULL, as
 * svdsb_diag_solve), the +k coefficient copy prev[:g, :kk] = Y[:g, *ci ...]
 * (when prev != NULL), then up to `passes` device-decided CGS passes as
 * svdsb_cgs_pass and x /= final norm; `state` receives the DGKS record
 * (svdsb_dgks_begin layout).  Replaces the orthonormalize / _expand
 * sequence of eigensolver.py:666-700 + kernels.py:54-133 for one column.
 * Uses a software grid barrier: the grid is at most one CTA per SM
 * (queried, not assumed) and the launch is cooperative, so it fails with
 * SVDSB_ERR_CUDA instead of hanging when the CTAs cannot be co-resident. */
int svdsb_cgs_fused(svdsb_ctx *ctx, int64_t dim, int nblk,
                    const double *const *xs, const int64_t *ldxs,
                    const int *cols, const double *rsrc, int64_t ldr,
                    const int *ci, const double *d, double *x,
                    const double *yin, int64_t ldyin, int g, int kk,
                    double *prev, int64_t ldprev, int passes, double *state,
                    void *stream);
/* Device-decided iterated CGS of a block of b new columns v (in place, on
 * entry the preconditioned expansion directions, on exit orthonormal),
 * the reference's column loop (kernels.py:54-133, eigensolver.py:666-700)
 * with its first pass split: the projection against the prior blocks runs
 * for all b columns at once (one Gram + one projection over the basis
 * instead of b of each), then column j finishes pass 1 against the block's
 * columns 0..j-1 and takes up to passes-1 further passes against
 * [prior, v[:, :j]] as svdsb_cgs_pass; the DGKS decision of pass 1 uses
 * |v_j| before the batched projection.  state: b 8-double records
 * (svdsb_cgs_pass layout); a column still active or collapsed after
 * `passes` (state[0] != 0 or state[5] == 0) must be redone by the caller.
 * cwork >= total*b + 3*b + total doubles (total = prior columns). */
int svdsb_cgs_block(svdsb_ctx *ctx, int64_t dim, int nblk,
                    const double *const *xs, const int64_t *ldxs,
                    const int *cols, double *v, int64_t ldv, int b,
                    double *cwork, double *state, int passes, void *stream);
/* 1 when svdsb_cgs_fused can run on the current device (cooperative launch
 * supported, kernel fits an SM); callers use svdsb_cgs_pass otherwise. */
int svdsb_cgs_fused_supported(void);
/* Device-resident iterated CGS for ONE new column v (kernels.py:54-133
 * without the host round trip).  state: 8 doubles [active, pass,
 * collapses, orig, prev, final, |v|^2 before, |v|^2 after];
 * svdsb_dgks_begin arms it, every svdsb_cgs_pass (Gram + projection, the
 * second kernel's last CTA applies the DGKS 1/sqrt(2) / collapse rule)
 * is a no-op once the column is final, so a caller queues a fixed number
 * of passes and checks state later.  cwork: >= sum(cols) doubles.
 * Operands must be 16-byte aligned with even leading dimensions. */
int svdsb_dgks_begin(double *state, void *stream);
int svdsb_cgs_pass(svdsb_ctx *ctx, int64_t dim, int nblk,
                   const double *const *xs, const int64_t *ldxs,
                   const int *cols, double *v, double *cwork, double *state,
                   int first_pass, void *stream);
int svdsb_split_residual(svdsb_ctx *ctx, int64_t dim, int64_t nsplit,
                         const double *r, int64_t ldr, const double *x,
                         int64_t ldx, int b, const double *lam,
                         const double *stats, double *out, void *stream);

/* ------------------------------------------------------------------ */
/* small dense kernels (one CTA; g <= SVDSB_SMALL_MAX)                     */

#define SVDSB_SMALL_MAX 64

#define SVDSB_ORDER_ASC 0       /* np.linalg.eigh order                     */
#define SVDSB_ORDER_DESC 1      /* argsort(-lams, stable)  (eigensolver.py:256) */
#define SVDSB_ORDER_INTERIOR 2  /* _interior_order (eigensolver.py:148-154) */

/* Symmetric eigendecomposition of the g x g matrix H (ldh), reordered per
 * `order` (shift used by INTERIOR): w[g] values, Y (ldy) orthonormal
 * eigenvector columns.  Replaces sym_eig (kernels.py:136-145) +
 * extract_rayleigh_ritz (eigensolver.py:362-367).  Cyclic Jacobi in fp64. */
int svdsb_syev_small(int g, const double *h, int64_t ldh, int order,
                     double shift, double *w, double *y, int64_t ldy,
                     void *stream);
/* Warm-started version of svdsb_syev_small for a projection that grew by b
 * bordering rows/columns: given H[:g0,:g0] = Y0 diag(l0) Y0^T (y0 g0 x g0,
 * l0 g0; y0 == NULL means Y0 = I and l0 = diag(H), the state right after a
 * thick restart that kept Ritz vectors), returns the eigendecomposition of
 * H[:g0+b,:g0+b] ordered like svdsb_syev_small.  Each border is absorbed as
 * an arrowhead matrix through its secular equation (deflation + Gu-Eisenstat
 * couplings), O(g^2) per border.  y / w may alias y0 / l0. */
int svdsb_syev_update(int g0, int b, const double *h, int64_t ldh,
                      const double *y0, int64_t ldy0, const double *l0,
                      int order, double shift, double *w, double *y,
                      int64_t ldy, void *stream);
/* Refined extraction (eigensolver.py:369-380): y = right singular vector
 * of the smallest singular value of the g x g matrix R (ldr), lam = y^T H y.
 * One-sided Jacobi SVD.  sv (optional, g) receives singular values desc. */
int svdsb_refined_small(int g, const double *r, int64_t ldr, const double *h,
                        int64_t ldh, double *y, double *lam, double *sv,
                        void *stream);
/* Thick-restart coefficient selection (eigensolver.py:485-515 with
 * _coef_gs :438-459 and _padded_prev :461-469): the priority list
 * [yfirst (optional)] + the ny ordered Ritz coefficient columns of yall
 * is orthonormalised in order against `exclude` (optional g-vector),
 * 2 modified Gram-Schmidt passes, dropping norms <= 1e-8, keeping at most
 * `retain`; then up to max(min(plus_k, gmax-1-kept), 0) previous
 * coefficient columns (prev, prev_g x nprev, zero padded to g; skipped
 * when prev_g > g) against [exclude] + kept.  Result g x s in out (ldo);
 * s written to count_dev[0] (device int). */
int svdsb_restart_coefs(int g, int gmax, const double *yfirst,
                        const double *yall, int64_t ldy, int ny, int retain,
                        const double *exclude, const double *prev,
                        int64_t ldp, int nprev, int prev_g, int plus_k,
                        double *out, int64_t ldo, int *count_dev,
                        void *stream);
/* Hout (s x s) = sym(C^T H C), C g x s (eigensolver.py:528-531). */
int svdsb_project_small(int g, int s, const double *h, int64_t ldh,
                        const double *c, int64_t ldc, double *hout,
                        int64_t ldho, void *stream);
/* Thin QR of M = R Y (R g x g, Y g x s) with nonnegative diag:
 * qy (g x s), ry (s x s)  (qr_restart, kernels.py:225-242). */
int svdsb_qr_small(int g, int s, const double *r, int64_t ldr,
                   const double *yc, int64_t ldy, double *qy, int64_t ldq,
                   double *ry, int64_t ldry, void *stream);
/* Insert the Gram block hc ((g+b) x b, ldhc) as new columns g..g+b-1 of the
 * symmetric projection H (eigensolver.py:690-694). */
int svdsb_h_insert(int g, int b, const double *hc, int64_t ldhc, double *h,
                   int64_t ldh, void *stream);
/* H (g x g) = sym(G) (eigensolver.py:349-352). */
int svdsb_h_symmetrize(int g, const double *gm, int64_t ldg, double *h,
                       int64_t ldh, void *stream);

/* ------------------------------------------------------------------ */
/* One single-column GD+k iteration, all launches in one call (the body of */
/* the solver's captured iteration graph; eigensolver.py:563-700): fused   */
/* CGS expansion of the candidate *ci into V[:, g], W[:, g] = A^T A V[:, g] */
/* (csr, side as svdsb_apply_normal), H column, warm RR update            */
/* (svdsb_syev_update with g0 / y0 / l0), Ritz residuals of p candidates, */
/* status into pinned host memory.  See csrc/gdk.cu.                       */
typedef struct svdsb_gdk_iter_args {
  int64_t n;
  double *v; int64_t ldv;          /* basis, n x (g+1) used */
  double *w; int64_t ldw;          /* its image */
  int g;                            /* columns before the expansion */
  const double *rsrc; int64_t ldr;  /* candidate residual block */
  const int *ci;                    /* device candidate index */
  const double *d;                  /* Jacobi diagonal or NULL */
  const double *yin; int64_t ldyin; /* Ritz coefficients (for the +k copy) */
  int kk; double *prev; int64_t ldprev;
  int passes; double *dgks;         /* DGKS state (8 doubles) */
  const svdsb_csr *csr; int side; double *tmp; int64_t ldtmp;
  double *hc; int64_t ldhc; double *h; int64_t ldh;
  int g0; const double *y0; int64_t ldy0; const double *l0;
  int order; double shift;
  double *lout; double *yout; int64_t ldyout;
  int p; double *rout; int64_t ldrout; double *rn2;
  double *status_host;
} svdsb_gdk_iter_args;

int svdsb_gdk_iteration(svdsb_ctx *ctx, const svdsb_gdk_iter_args *args,
                        void *stream);

/* ------------------------------------------------------------------ */
/* JDQMR inner solver (PRIMME's QMRs on the Jacobi-Davidson correction    */
/* equation; the paper's stage-2 method, PAPER.md:765-767, 897 -- the      */
/* reference runs GD+k only):                                */
/*   P (Op - sigma I) P t = -r,  P = I - Q Q^T, Q (n x nq, nq <= 32)       */
/* orthonormal, optional point-Jacobi K^-1 = 1 ./ dg applied as P K^-1 P.  */
/* The caller owns every vector (device, length n, contiguous).  The      */
/* operator product w = Op d is the caller's (the CSR SpMV entry points)  */
/* between phase 0 and each phase 1:                                       */
/*   phase 0: setup from r (state inputs SIGMA, RITZ, RNORM, MAXIT, TOL_E, */
/*            ETOL_FRAC, LFAC must be written first, svdsb_jd_state_size() */
/*            doubles);                                                     */
/*   phase 1: one QMRs step after w = Op d: scalars, t/g updates, the     */
/*            eigen-residual estimate of x + t and the device-side stop    */
/*            test; `cond` (from svdsb_while_begin, or 0) is set to 0 when */
/*            the inner solve is done.                                     */
/* The solution accumulates in t.  State slots: 0 SIGMA, 14 ERES, 16 IT,   */
/* 17 MAXIT, 18 TOL_E, 19 ETOL_FRAC, 20 STOP (reason), 21 RITZ, 22 RNORM,  */
/* 25 LFAC (see csrc/jdqmr.cu).                                           */
typedef struct svdsb_jd_vecs {
  const double *r;   /* outer residual (input)                     */
  const double *dg;  /* Jacobi diagonal or NULL                    */
  double *rc, *g, *t, *dl, *z, *d, *w;  /* QMRs work vectors, t = solution */
} svdsb_jd_vecs;

int svdsb_jd_state_size(void);
int svdsb_jd_phase(svdsb_ctx *ctx, int phase, int64_t n,
                   const svdsb_jd_vecs *vecs, const double *q, int64_t ldq,
                   int nq, double *state, uint64_t cond, void *stream);
/* Capture a CUDA graph whose single node is a WHILE loop: launches made on
 * `stream` between begin and end form the loop body, which repeats while
 * the conditional handle *cond_out (pass it to svdsb_jd_phase) is nonzero;
 * it is 1 at every launch of the instantiated graph.  PDL is off inside the
 * body.  Launch / destroy with svdsb_graph_launch / svdsb_graph_destroy. */
int svdsb_while_begin(void *stream, uint64_t *cond_out);
int svdsb_while_end(void *stream, void **exec_out);

/* ------------------------------------------------------------------ */
/* Matrix Market ingestion (host side; replaces read_matrix_market /     */
/* write_matrix_market / write_dense_market, matio.py:170-258).          */
/* The reader is two calls: the header (shape, stored entry count,       */
/* layout), then the entries into caller-owned host arrays of exactly    */
/* `entries` elements (0-based rows/cols; array files column-major).     */
/* A malformed file returns SVDSB_ERR_FORMAT with *err_line = the        */
/* 1-based line the reference names and the reference's message in      */
/* svdsb_last_error().  Symmetric expansion and device assembly are the  */
/* caller's (svdsb_csr_create_coo_device sums duplicates in input order).*/

int svdsb_mm_read_header(const char *path, int64_t *m, int64_t *n,
                         int64_t *entries, int *is_array, int *symmetric,
                         int64_t *err_line);
int svdsb_mm_read_entries(const char *path, int64_t entries,
                          int64_t *rows_host, int64_t *cols_host,
                          double *vals_host, int64_t *err_line);
/* "coordinate real general", values as %.17g (matio.py:244-251). */
int svdsb_mm_write_coo(const char *path, int64_t m, int64_t n, int64_t nnz,
                       const int64_t *row_ptr_host, const int64_t *col_host,
                       const double *vals_host);
/* "array real general", column-major (matio.py:254-262). */
int svdsb_mm_write_array(const char *path, int64_t m, int64_t n,
                         const double *a_host, int64_t lda);

#ifdef __cplusplus
}
#endif
#endif /* SVDSB_H */
