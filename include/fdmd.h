/* fdmd.h — C ABI of the B200-native DMD hot path (libfdmd.so).
 *
 * The reference (`flowdmd`, arXiv 2502.05339) is pure Python over
 * numpy/LAPACK; its hot path has no FFI of its own. Each entry point below
 * replaces the numpy/LAPACK call sites the reference makes on that path
 * (file:line relative to /root/reference/pkg/src/flowdmd/):
 *
 *   fdmd_tall_gemm     M @ G, M @ W (linalg.py:82,85), Q @ Ub (linalg.py:88),
 *                      Xp @ (V/S) and P @ W (dmd.py:255,258), U @ B.T (dmd.py:414)
 *                      — and the CholeskyQR replacement of np.linalg.qr (linalg.py:82,85)
 *   fdmd_tall_gram     M.conj().T @ Q (linalg.py:84), Q.conj().T @ M (linalg.py:86),
 *                      U.conj().T @ P (dmd.py:256); Gram Y^T Y of CholeskyQR2
 *   fdmd_colmajor_dot  pinv(phi) @ u (runtime.py:52,199), pinv(phi) @ B_i (dmd.py:489)
 *   fdmd_decode        cols @ coeff / (phi @ z).real (runtime.py:88-99) — batched
 *   fdmd_table_apply   decode_table() column construction (dmd.py:92-120) and the
 *                      normalise/phase-canonicalise step of _order_and_pair (dmd.py:191-206)
 *   fdmd_residual      provenance["residual"] (dmd.py:269-272)
 *   fdmd_geev          np.linalg.eig in eig_small (linalg.py:120) — cuSOLVER Xgeev
 *   fdmd_synth3d       BASELINE.json configs 1-4 snapshot generator (device)
 *   fdmd_rsvd          randomized_svd (linalg.py:62-90) as one call (sketch, power
 *                      iterations, CholeskyQR2, projection, svd, canonical signs, lift)
 *   fdmd_dmd_fit       exact_dmd (dmd.py:240-274) / optdmd + _varpro_lm (dmd.py:277-455)
 *                      as one call over a device-owned SnapshotMatrix (fdmd_mat_upload)
 *   fdmd_model_*       ReducedModel.phi (dmd.py:53-77, chunked), decode (runtime.py:66-99);
 *   fdmd_encode        encode (runtime.py:47-52) — model handles from fdmd_dmd_fit
 *   fdmd_mac_*         2-D serving / guided upscaling: frame planes (server.py:205-214),
 *                      density transport (solver.py:133-150), injection and the
 *                      guide projection (upres.py:21-50, 154-169)
 *
 * Conventions: every pointer argument is DEVICE memory unless named *_host;
 * `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 * asynchronous on `stream` except fdmd_geev (returns after the solve).
 * Status: 0 = OK; negative = error, message via fdmd_last_error() (thread-local).
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with FDMD_ERR_CUDA.
 */
#ifndef FDMD_H_
#define FDMD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDMD_OK 0
#define FDMD_ERR_INVALID (-1)     /* maps to ValueError */
#define FDMD_ERR_CUDA (-2)        /* CUDA runtime failure */
#define FDMD_ERR_SOLVER (-3)      /* cuSOLVER failure -> ConvergenceError */
#define FDMD_ERR_WORKSPACE (-4)   /* workspace too small */

#define FDMD_F32 0
#define FDMD_F64 1
#define FDMD_ROW 0 /* element (i, k) at p[i*ld + k] */
#define FDMD_COL 1 /* element (i, k) at p[k*ld + i] */

int fdmd_version(void);
const char* fdmd_last_error(void);
int fdmd_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

#define FDMD_B_UPPER 1 /* tall_gemm flag: B is upper triangular (CholeskyQR's R^-1) */
#define FDMD_SHARE_SMS 2 /* tall_gemm flag: leave 8 SMs free for small work on another stream */

/* C[n x N] = A[n x K] * B[K x N]. A: f32/f64, ROW/COL. B: f64 row-major (ld ldb).
 * C: f32/f64 ROW/COL, may be NULL (statistics only). FP64 DMMA accumulation.
 * pair_stats (optional, length 3*(N/2), N even): for unit u = columns (2u, 2u+1)
 * read as (Re, Im): [sum_i |c_i|^2, max_i |c_i|^2, first argmax i + row_offset]. */
size_t fdmd_tall_gemm_workspace(int64_t n, int N);
int fdmd_tall_gemm(const void* A, int a_dtype, int a_layout, int64_t lda,
                   const double* B, int64_t ldb,
                   void* C, int c_dtype, int c_layout, int64_t ldc,
                   int64_t n, int K, int N, int flags,
                   double* pair_stats, int64_t row_offset,
                   void* workspace, size_t workspace_bytes, void* stream);

/* C = A[n x K] * B[K x N] (A row-major f32/f64, FP64 DMMA) written as the fp16
 * hi/lo planes of C * scale (row-major n x ldu, ldu = round_up(N, 8) <= 256,
 * padding columns zero): the operand format of fdmd_tc_decode_ex. Replaces
 * the lift U = Q Ub (linalg.py:88) when Q = S M is implicit. */
int fdmd_tall_gemm_planes(const void* A, int a_dtype, int64_t lda, const double* B, int64_t ldb,
                          void* uh, void* ul, int64_t ldu, double scale,
                          int64_t n, int K, int N, int flags, void* stream);

/* C[K1 x K2] (f64 row-major, ld ldc) = beta*C + A[n x K1]^T B[n x K2].
 * Deterministic fixed-order split reduction. symmetric=1 requires A==B, K1==K2. */
size_t fdmd_tall_gram_workspace(int64_t n, int K1, int K2);
int fdmd_tall_gram(const void* A, int a_dtype, int a_layout, int64_t lda,
                   const void* B, int b_dtype, int b_layout, int64_t ldb,
                   double* C, int64_t ldc, double beta,
                   int64_t n, int K1, int K2, int symmetric,
                   void* workspace, size_t workspace_bytes, void* stream);

/* C (K x (K+1), f64, row stride ldc) = beta*C + [A^T A | A^T a_K] over the rows of a
 * row-major f32/f64 A with at least K + 1 columns (a_K = column K): the snapshot
 * Gram X^T X together with the border X^T s_m of S^T S in ONE pass over S — what
 * the projection B = Q^T M takes from a Gram when Q = X M1 (reference
 * linalg.py:82-86, `Q.T @ M` after the power loop). The border rides in the
 * symmetric panel kernel as 5 extra 8x8 blocks per diagonal warp tile;
 * operands that kernel cannot take run the symmetric Gram + fdmd_tall_tdot.
 * Deterministic fixed-order split reduction. */
size_t fdmd_tall_gram_bordered_workspace(int64_t n, int K);
int fdmd_tall_gram_bordered(const void* A, int dtype, int64_t lda, double* C, int64_t ldc, double beta,
                            int64_t n, int K, void* workspace, size_t workspace_bytes, void* stream);

/* Host-side view of the panel-Gram schedule for a K x K (symmetric / bordered) Gram
 * over n rows of elt_bytes elements: info[9] = {ok, partitions, cost (sum over
 * partitions of the busiest SM sub-partition, in 8x8 DMMA blocks per k-step), cuts,
 * row splits, K1p, K2p, border block column, blocks}; tiles (may be NULL) receives
 * {i0, j0, kind, 8*partition+warp} per warp tile. Returns the tile count. No device work. */
int fdmd_gram_plan_info(int64_t n, int K, int symmetric, int border, int elt_bytes, int* info, int* tiles,
                        int max_tiles);

/* y[k] = beta*y[k] + sum_i A[i*lda + k] v[i*ldv]  (k < K): A^T v over the rows of a
 * row-major f32/f64 A, v strided in the same dtype (e.g. a column of A), f64 out,
 * fixed-order (deterministic) split sums. The border X^T s_m of the snapshot Gram
 * S^T S next to X^T X (linalg.py:82-86: Q^T M with Q = X M1). */
size_t fdmd_tall_tdot_workspace(int64_t n, int K);
int fdmd_tall_tdot(const void* A, int dtype, int64_t lda, const void* v, int64_t ldv,
                   int64_t n, int K, double* y, double beta,
                   void* workspace, size_t workspace_bytes, void* stream);

/* Reconstruction: out[f*ldo + i] = sum_k D[k*ldd + i] * coef[k*ldcoef + f]
 * for f < B frames, i < n rows, k < r table columns. D, coef, out share dtype. */
int fdmd_decode(const void* D, int dtype, int64_t ldd, const void* coef, int ldcoef,
                void* out, int64_t ldo, int64_t n, int r, int B, void* stream);

/* y[k*nv + v] = sum_i D[k*ldd + i] * U[v*ldu + i]  (k < r, v < nv <= 8), f64 out. */
size_t fdmd_colmajor_dot_workspace(int64_t n, int r, int nv);
int fdmd_colmajor_dot(const void* D, int d_dtype, int64_t ldd,
                      const void* U, int u_dtype, int64_t ldu,
                      int64_t n, int r, int nv, double* y,
                      void* workspace, size_t workspace_bytes, void* stream);

/* D[j*ldd + i] = alpha[j]*R[(2*src[j])*ldr + i] + beta[j]*R[(2*src[j]+1)*ldr + i]. */
int fdmd_table_apply(const void* R, int r_dtype, int64_t ldr, const int* src,
                     const double* alpha, const double* beta,
                     void* D, int d_dtype, int64_t ldd, int64_t n, int ncols, void* stream);

/* In place: R[j*ldr + i] <- alpha[j]*R[(2*src[j])*ldr + i] + beta[j]*R[(2*src[j]+1)*ldr + i]
 * for j < ncols <= nraw (each block stages its rows of all nraw columns first). */
int fdmd_table_apply_inplace(void* R, int dtype, int64_t ldr, int nraw, const int* src,
                             const double* alpha, const double* beta, int ncols, int64_t n, void* stream);

/* out[0] = sum_i sum_{j<T} (S[i*lds + 1 + j] - sum_k D[k*ldd+i] F[k*T+j])^2,
 * out[1] = sum_i sum_{j<T} S[i*lds + 1 + j]^2  (out: 2 doubles, device). */
size_t fdmd_residual_workspace(int64_t n);
int fdmd_residual(const void* S, int s_dtype, int64_t lds, const void* D, int d_dtype, int64_t ldd,
                  const double* F, int r, int T, int64_t n, double* out,
                  void* workspace, size_t workspace_bytes, void* stream);

/* Thin SVD of a small row-major f64 device matrix B (l x T, l <= T, row stride ldb):
 * B = Ub diag(s) Vh with ubt = Ub^T (l x l row-major), s (l, descending), vh (l x T
 * row-major) — `np.linalg.svd(B, full_matrices=False)` of randomized_svd (reference
 * linalg.py:87) and of the DMDc sketches. cuSOLVER gesvdp, stream-ordered (no host
 * synchronisation); *info_dev (device int) receives cuSOLVER's info; B is destroyed. */
int fdmd_svd_small(double* B, int64_t ldb, int l, int T, double* ubt, double* s_out, double* vh, int* info_dev,
                   void* stream);

/* Real nonsymmetric eigendecomposition (cuSOLVER Xgeev). A: n x n column-major
 * f64 (overwritten). Outputs: w_host (2n doubles: re, im interleaved),
 * vr_host (n x n column-major, LAPACK packing: a complex pair occupies columns
 * j (real part) and j+1 (imaginary part)); vr_host = NULL computes the
 * eigenvalues only (the OptDMD initial guess, dmd.py:387). Synchronous. */
int fdmd_geev(int n, double* A, double* w_host, double* vr_host, void* stream);

/* tcgen05 batched reconstruction (FP32-accurate 2-way FP16 split, see
 * csrc/fdmd_tc_decode.cuh). Basis planes uh/ul: row-major n x ldu halves
 * (ldu % 8 == 0) of U * 2^su; coefficient planes ch/cl: frame-major nf x ldk
 * halves; fscale[f] = 2^-(su + sc_f); out[f*ldo + i] fp32. r <= 256.
 * fdmd_split_basis builds uh/ul from a column-major fp32 table (r x n, ld ldd);
 * fdmd_split_coef builds ch/cl/fscale from coefficients (r x nf, row-major).
 * Replace the per-frame `cols @ coeff` of runtime.py:88 for batches. */
int fdmd_split_basis(const float* D, int64_t ldd, int64_t n, int r, float scale, void* uh, void* ul, int64_t ldu,
                     void* stream);
int fdmd_split_coef(const float* coef, int ldc, int r, int nf, float su_inv, void* ch, void* cl, int ldk,
                    float* fscale, void* stream);
/* fp16 hi/lo planes (row-major n x ldu) of a row-major fp64 tall matrix
 * (n x K, ld lda) scaled by `scale` — the sketch basis Q for the tcgen05
 * lift U = Q Ub (linalg.py:88) and modes Q (Ub B^T) (dmd.py:414). */
int fdmd_split_rows_f64(const double* A, int64_t lda, int64_t n, int K, double scale, void* uh, void* ul,
                        int64_t ldu, void* stream);
/* same for an fp32 or fp64 row-major matrix (dtype FDMD_F32 / FDMD_F64): the
 * snapshot matrix S for the tcgen05 exact-DMD modes X' (V S^-1 W) (dmd.py:255,258) */
int fdmd_split_rows(const void* A, int dtype, int64_t lda, int64_t n, int K, double scale, void* uh, void* ul,
                    int64_t ldu, void* stream);
/* Per unit u of a column-major fp32 table (columns 2u, 2u+1 = Re, Im):
 * out[3u..3u+2] = [sum |phi|^2, max |phi|^2, first argmax + row_offset] —
 * the normalisation / phase-pivot statistics of _order_and_pair (dmd.py:189-206). */
size_t fdmd_pair_stats_workspace(int64_t n, int units);
int fdmd_pair_stats(const float* raw, int64_t ld, int64_t n, int units, int64_t row_offset, double* out,
                    void* workspace, size_t workspace_bytes, void* stream);
int fdmd_tc_decode(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch, const void* cl,
                   int ldk, int nf, const float* fscale, float* out, int64_t ldo, void* stream);
/* same, with flags: FDMD_SHARE_SMS leaves 8 SMs to work on another stream
 * (the OptDMD eigen / variable-projection solves overlapping the lift) */
int fdmd_tc_decode_ex(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch, const void* cl,
                      int ldk, int nf, const float* fscale, float* out, int64_t ldo, int flags, void* stream);

/* fdmd_tc_decode of a modes product (columns 2u, 2u+1 = Re, Im of mode u; `U @ B.T`, reference
 * dmd.py:414) with the normalisation / phase-pivot statistics of `_order_and_pair`
 * (dmd.py:189-206: the first largest-|.| entry of each mode) taken in the frame epilogue:
 * st[3u] = sum_i |phi_u[i]|^2 (f64 running sums of f32 32-row partials), st[3u + 1] =
 * max_i |phi_u[i]|^2, st[3u + 2] = first row attaining it + row_offset — what
 * fdmd_pair_stats reads back from the table. *fused = 1 when the CTA-pair kernel ran (nf > 128) and filled st;
 * 0 = frames only (the caller then runs fdmd_pair_stats over the table). */
int fdmd_tc_decode_pairstats(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                             const void* cl, int ldk, int nf, const float* fscale, float* out, int64_t ldo,
                             int64_t row_offset, double* st, int* fused, void* stream);

/* tc_decode (CTA-pair kernel, nf <= 256) writing its result as the fp16
 * hi/lo planes of a row-major n x ldp matrix scaled by pscale (ldp % 8 == 0,
 * ldp >= nf; columns [nf, ldp) are written as zeros): the lift U = Q Ub
 * (linalg.py:88) straight into the planes of the config-4 basis. */
int fdmd_tc_decode_planes(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                          const void* cl, int ldk, int nf, const float* fscale, void* out_h, void* out_l,
                          int64_t ldp, float pscale, int flags, void* stream);

/* ---- 2-D MAC-grid serving / guided upscaling ----
 * State layout (grid.py:1-18): u block ny x (nx+1), then v block (ny+1) x nx. */
#define FDMD_MAC_VELOCITY 0
#define FDMD_MAC_SPEED 1

/* Fused decode -> cell-centred planes. Replaces ModelServer.frame_payload's
 * decode(model, z) + unflatten + centring (+ speed) (server.py:205-214).
 * D: column-major decode table (ncol x n_state, ld ldd, dtype F32/F64);
 * coef: ncol f64 table coefficients (device). out: f64, VELOCITY -> 2 planes
 * [uc; vc] of ny x nx, SPEED -> 1 plane sqrt(uc^2 + vc^2). */
int fdmd_mac_decode(const void* D, int dtype, int64_t ldd, int ncol, const double* coef, int nx, int ny,
                    int field, double* out, void* stream);

/* Semi-Lagrangian transport of a cell-centred scalar q (ny x nx f64) for
 * one step dt through the flat MAC velocity `vel` (dtype F32/F64).
 * Replaces advect_semi_lagrangian(vel, ScalarField, dt) (solver.py:167-171,
 * 133-150 with maccormack=False) as used by server.py:232 and runtime.py:259. */
int fdmd_mac_advect(const void* vel, int dtype, int nx, int ny, double h, double dt, const double* q, double* q_out,
                    void* stream);

/* Nearest-face prolongation of nv coarse states (ld_low apart) onto the
 * fine grid (ld_fine apart): build_inject(high, factor) @ L (upres.py:21-50, 121). */
int fdmd_mac_inject(const double* low, int nx_high, int ny_high, int factor, int nv, int64_t ld_low,
                    int64_t ld_fine, double* fine, void* stream);

/* Guide-consistency projection x = H + A^T (A A^T)^-1 (L - A H) for the
 * face-averaging downsample A (grid.py:195-236); A A^T = gram_diag * I.
 * Replaces build_projector + constrained_project (upres.py:140-169). */
int fdmd_mac_project(const double* H, const double* L, int nx_high, int ny_high, int factor, double gram_diag,
                     double* x, void* stream);

/* ---- 2-D smoke solver (reference solver.py) --------
 * vel: flat MAC state (f64, u block then v block); cell arrays ny x nx f64;
 * solid: ny x nx uint8 (NULL = no obstacles); closed/open: boundary kind. */
#define FDMD_SOL_REDUCE_BLOCKS 296
int fdmd_sol_mask(double* vel, int nx, int ny, const unsigned char* solid, int closed, void* stream);
/* apply_solid_mask (grid.py:264-272) */
int fdmd_sol_advect(const double* vel, const double* q, int which, int nx, int ny, double h, double dt,
                    int maccormack, double* scratch, double* out, void* stream);
/* _advect_array (solver.py:133-150): which 0 = u, 1 = v, 2 = cell centres;
 * scratch holds 3 arrays of q's size (MacCormack predictor and extrema). */
int fdmd_sol_emit(double* dens, double* temp, int nx, int ny, double h, double cx, double cy, double r2, double dadd,
                  double tadd, void* stream);                                  /* _emit (solver.py:323-334) */
int fdmd_sol_buoyancy(double* vel, const double* dens, const double* temp, int nx, int ny, double alpha, double beta,
                      double dt, void* stream);                                /* add_body_forces (solver.py:181-194) */
int fdmd_sol_vorticity(double* vel, int nx, int ny, double h, double eps, double dt, double* scratch, void* stream);
/* vorticity_confinement (solver.py:197-222), scratch = 3 cell arrays */
int fdmd_sol_reduce(const double* a, const double* b, const unsigned char* solid, int64_t n, int op, double* part,
                    double* out, void* stream);
/* op 0: sum a*b (np.vdot), 1: max |a|, 2: sum of a over fluid cells; fixed
 * order; part holds FDMD_SOL_REDUCE_BLOCKS doubles; *out is device memory. */
int fdmd_sol_rhs(const double* vel, int nx, int ny, double h, const unsigned char* solid, int closed, double nfluid,
                 double* b, double* part, double* sum, void* stream);
/* b = -divergence (0 on solids), mean-free on fluid cells when closed (solver.py:262-268) */
int fdmd_sol_poisson(const double* p, int nx, int ny, double h2, const unsigned char* solid, int open, double* out,
                     void* stream);                                            /* _apply_poisson (solver.py:248-258) */
int fdmd_sol_cg_step(double* p, double* r, const double* d, const double* Ad, double alpha, int64_t n, void* stream);
int fdmd_sol_cg_dir(double* d, const double* r, double beta, int64_t n, void* stream);
int fdmd_sol_cg_single(const double* b, double* p, double* r, double* d, double* Ad, int nx, int ny, double h2,
                       const unsigned char* solid, int open, double cg_tol, int max_iters, double* status,
                       void* stream);
/* The complete CG loop of _project (solver.py:270-309) in one 1024-thread CTA
 * for grids <= 131072 cells; status (device, 4 doubles) = final max|r|,
 * iterations, ran-out flag, max|b|. */
int fdmd_sol_pressure_apply(double* vel, const double* p, int nx, int ny, double h, const unsigned char* solid,
                            int open, void* stream);                           /* _project tail (solver.py:311-315) */

/* Randomized SVD of X (n x T, f32/f64 row-major, ld ldx) in one call —
 * randomized_svd(M, r, oversample=l-r, power_iters=q) of linalg.py:62-90 with
 * the host-drawn Omega (T x l f64 row-major, default_rng(seed).standard_normal).
 * Outputs: sigma_host (r), V_host (T x r row-major), U (device, column-major
 * r x n f64, ld ldu >= n), canonicalised as linalg.py:29-44. Synchronous.
 * Requires r <= l <= min(T, 256). */
int fdmd_rsvd(const void* X, int x_dtype, int64_t ldx, int64_t n, int T, int r, int l, int q,
              const double* omega_host, double* sigma_host, double* V_host, double* U, int64_t ldu,
              void* stream);

/* ---- Fit / model handles ----------------------------------
 * The whole exact-DMD / OptDMD fit, the mode matrix, encode and decode as C
 * calls over plain host buffers, for a binding without this package's Python
 * layer. A context owns one device and a pool of streams;
 * every call takes a stream from the pool for its duration, so concurrent
 * calls from several host threads (the reference server's request threads,
 * server.py:57-67) are safe. Host buffers are caller-owned; calls are
 * synchronous on return. Complex values are interleaved (re, im) doubles. */
typedef struct fdmd_ctx fdmd_ctx;
typedef struct fdmd_mat fdmd_mat;
typedef struct fdmd_model fdmd_model;

#define FDMD_METHOD_EXACT 0 /* exact_dmd (dmd.py:240-274) */
#define FDMD_METHOD_OPT 1   /* optdmd (dmd.py:366-436) */

int fdmd_ctx_create(int device, int n_streams, fdmd_ctx** out);
int fdmd_ctx_destroy(fdmd_ctx* ctx);
/* SnapshotMatrix(states) (dmd.py:26-50): host C-order n x m (row stride
 * ld_host elements, FDMD_F32 / FDMD_F64) -> a device-owned row-major copy.
 * ValueError semantics: n >= 1, m >= 2, every entry finite. */
int fdmd_mat_upload(fdmd_ctx* ctx, const void* host, int dtype, int64_t n, int64_t m, int64_t ld_host,
                    fdmd_mat** out);
int fdmd_mat_free(fdmd_mat* mat);
/* exact_dmd(data, r, svd_mode="randomized", seed) / optdmd(data, r, init,
 * LMConfig(max_iters=lm_max_iters), svd_mode="randomized", seed) on the
 * snapshot columns X = states[:, :-1], X' = states[:, 1:]:
 * omega_host = default_rng(seed).standard_normal((T, l)) (T = m - 1,
 * l = r + oversample, linalg.py:76), q power iterations. OPT only:
 * init_lam_host (2r, NULL = exact-DMD eigenvalues, dmd.py:387), jitter_host
 * (r values default_rng(seed).random(r) for the collapse retry,
 * dmd.py:394-399; NULL = fail on collapse). Outputs sigma_host (r), lam_host
 * (2r) and the model (modes on the device, table dtype = states dtype). */
int fdmd_dmd_fit(fdmd_ctx* ctx, const fdmd_mat* states, double dt, int r, int l, int q, const double* omega_host,
                 int method, int lm_max_iters, const double* init_lam_host, const double* jitter_host,
                 double* sigma_host, double* lam_host, fdmd_model** out);
/* Augmented DMDc (the package's dmd.dmdc_fit; Proctor et al. 2016, SURVEY.md
 * §8(c) "C2 restatement"): controls_host ell x T row-major (u_j for j < T);
 * a rank-r_aug sketch of [X; Upsilon] (omega_aug_host T x l_aug) and the
 * output basis U_hat = a rank-r sketch of X' (omega_out_host T x l).
 * Outputs sigma_aug_host (r_aug), lam_host (2r), reduced_b_host (r x ell
 * complex, interleaved) = pinv(phi) U_hat B~ / dt, the ControlOperator matrix
 * runtime.step_forced consumes (runtime.py:164-200), and the model. */
int fdmd_dmdc_fit(fdmd_ctx* ctx, const fdmd_mat* states, const double* controls_host, int ell, double dt, int r_aug,
                  int l_aug, int r, int l, int q, const double* omega_aug_host, const double* omega_out_host,
                  double* sigma_aug_host, double* lam_host, double* reduced_b_host, fdmd_model** out);
int fdmd_model_info(const fdmd_model* model, int64_t* n, int* r, double* dt, int* converged);
/* the variable-projection objective history (provenance["objective_history"]);
 * returns its length, copies min(length, cap) values */
int fdmd_model_history(const fdmd_model* model, double* out, int cap);
/* rows [row0, row0 + rows) of phi (n x r complex, C-order) -> out_c128 (rows x 2r doubles) */
int fdmd_model_phi_to_host(fdmd_ctx* ctx, const fdmd_model* model, int64_t row0, int64_t rows, double* out_c128);
/* encode: z = pinv(phi) u (runtime.py:47-52); u_host n doubles, z_host 2r */
int fdmd_encode(fdmd_ctx* ctx, const fdmd_model* model, const double* u_host, double* z_host);
/* decode: frames[f] = Re(phi z_f) (runtime.py:66-99) for B states (z_host B x 2r)
 * -> out_host (B x n doubles, C-order) */
int fdmd_model_decode(fdmd_ctx* ctx, const fdmd_model* model, const double* z_host, int B, double* out_host);
int fdmd_model_free(fdmd_model* model);

/* FP64 tensor-pipe (DMMA.8x8x4) throughput probe on the current device:
 * a register-only mma.sync f64 loop lasting ~`seconds`/4; writes TFLOP/s.
 * The fit's roofline denominator (MEASURED_PEAKS.json has no FP64 figure). */
int fdmd_dmma_peak(double seconds, double* tflops);

/* Pitched 2-D copy (cudaMemcpy2DAsync; kind = cudaMemcpyKind, 4 = default/UVA):
 * uploads a host n x m snapshot block into a padded row-major device buffer. */
int fdmd_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                int kind, void* stream);

/* Synthetic separable 3D snapshots (see synth.py). Tables f64 on device. */
int fdmd_synth3d(const double* sx, const double* sy, const double* sz, const double* Am,
                 int K, int C, int N, int m, double noise, uint64_t key,
                 int64_t row0, int64_t rows, void* out, int out_dtype, int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDMD_H_ */
