/*
 * mgpu.h -- C-ABI of the B200 (sm_100a) SPAI + shifted-system PCG library.
 *
 * This is the drop-in boundary for the hot path of the reference
 * (/root/reference/proj, arXiv 1606.01216 AIRGA):  assembling the shifted
 * operators A(s) = s^2 M + s D + K, building / updating / applying the SPAI
 * preconditioner chain, and the right-preconditioned CG solves of A(s) X = F.
 * Every entry point names the reference interface it replaces (file:line
 * relative to /root/reference/proj).  Plain pointers and sizes only.
 *
 * Conventions (all follow the reference's):
 *   - CSR: int64 row_ptr[nrows+1], int32 col_idx[nnz] strictly increasing per
 *     row, double values[nnz] with no stored exact zeros   (include/mor/sparse.hpp:12-22)
 *   - dense blocks are n x m column-major                   (include/mor/dense.hpp:14-37)
 *   - preconditioner chains are listed NEWEST FIRST, [Q_z, ..., Q_2, P]
 *     and applied oldest first                               (include/mor/spai.hpp:63-79)
 *   - FP64 everywhere; no tensor cores; no CPU fallback: a call that cannot
 *     run on the device fails with MGPU_ERR_CUDA / MGPU_ERR_UNSUPPORTED.
 *
 * Errors: every call returns an mgpu_status.  The exception class the
 * reference would throw maps 1:1 (include/mor/errors.hpp:13-59):
 *   ArgumentError -> MGPU_ERR_ARG, StagnationError(column) -> MGPU_ERR_STAGNATION,
 *   BreakdownError(iteration) -> MGPU_ERR_BREAKDOWN, NumericalError -> MGPU_ERR_NUMERICAL.
 * mgpu_last_error() returns the payload (column / iteration, plus the RHS
 * column and point index for batched solves) and a message shaped like the
 * reference's what().  Exhausting maxit is NOT an error (converged = 0),
 * exactly as in krylov.cpp:128-137.
 *
 * Threading: a context is bound to one device and one CUDA stream and must be
 * used by one host thread at a time; independent contexts are independent
 * (one per GPU for shift sharding).
 */
#ifndef MGPU_H
#define MGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mgpu_status
{
  MGPU_OK = 0,
  MGPU_ERR_ARG = 1,         /* mor::ArgumentError     */
  MGPU_ERR_STAGNATION = 2,  /* mor::StagnationError   */
  MGPU_ERR_BREAKDOWN = 3,   /* mor::BreakdownError    */
  MGPU_ERR_NUMERICAL = 4,   /* mor::NumericalError    */
  MGPU_ERR_UNSUPPORTED = 5, /* shape outside the kernels' envelope (message says which) */
  MGPU_ERR_CUDA = 6,        /* CUDA runtime / launch failure */
  MGPU_ERR_NCCL = 7,
} mgpu_status;

typedef enum mgpu_memkind
{
  MGPU_HOST = 0,   /* pointer is host memory (pageable or pinned) */
  MGPU_DEVICE = 1, /* pointer is device memory on the context's device */
} mgpu_memkind;

typedef struct mgpu_ctx mgpu_ctx; /* device + stream + scratch arena + last error */
typedef struct mgpu_csr mgpu_csr; /* device-resident CSR matrix */

/* ------------------------------------------------------------------ context */

/* stream: a cudaStream_t to run on, or NULL for a library-owned stream. */
int mgpu_ctx_create(int device, void *stream, mgpu_ctx **out);
int mgpu_ctx_destroy(mgpu_ctx *ctx);
int mgpu_ctx_synchronize(mgpu_ctx *ctx);
/* Copies the last error's message (NUL-terminated, truncated to cap) and
 * payload: index = column (stagnation) or iteration (breakdown), rhs_column
 * and point for batched solves (-1 when not applicable). */
int mgpu_last_error(const mgpu_ctx *ctx, int64_t *index, int64_t *rhs_column, int64_t *point, char *msg, size_t cap);
const char *mgpu_status_string(int status);
/* Number of kernels this context has launched so far (for bench gpu_launches). */
int64_t mgpu_launch_count(const mgpu_ctx *ctx);
/* Device-side duration (ms, CUDA events on the context stream) of the last
 * mgpu_cg_solve* kernel region and the number of CG iterations it ran. */
int mgpu_last_cg_timing(const mgpu_ctx *ctx, double *ms, int64_t *iterations);

/* CG kernel selection.  0 = automatic: when every operator and factor has
 * bandwidth <= 64 and chains have <= 8 factors, the cluster-resident kernel
 * (one thread-block cluster per shifted system, operators in shared memory)
 * if the systems fit on chip, else the fused banded grid kernel (2 grid
 * barriers per iteration); otherwise the general CSR kernel.
 * 1 = always the general kernel, 2 = the banded grid kernel (no cluster),
 * 3 = cluster kernel v1 only (vectors in shared memory; v2 keeps them in
 * registers and is preferred for single right-hand sides), 4 = the streaming
 * kernel (TMA bulk copies into double-buffered shared memory; the automatic
 * choice for banded systems too large for the cluster kernels).
 * mgpu_last_cg_path reports 2 (cluster v2), 3 (cluster v1), 4 (stream),
 * 0 (banded grid) or 1 (general). */
int mgpu_ctx_set_cg_path(mgpu_ctx *ctx, int path);
int mgpu_last_cg_path(const mgpu_ctx *ctx);

/* Per-context tuning / diagnostic options (no environment variables are read by the library).
 * Defaults are the measured best choices; the others exist for the A/B experiments in DESIGN.md. */
typedef enum mgpu_option
{
  MGPU_OPT_RETIRED0 = 0,        /* (was the x~ update placement; the deferred update is the only schedule now) */
  MGPU_OPT_RETIRED1 = 1,        /* (was the point-serial schedule; measured slower, removed -- DESIGN.md 5) */
  MGPU_OPT_STREAM_CHUNK = 2,    /* cg_stream: forced chunk rows (0 = planner, default) */
  MGPU_OPT_STREAM_RING = 3,     /* cg_stream: forced ring depth with MGPU_OPT_STREAM_CHUNK (2..4) */
  MGPU_OPT_STREAM_SAME_CHB = 4, /* cg_stream: phase B on phase A's chunk height (default 0) */
  MGPU_OPT_CLUSTER_CS = 5,      /* cg_cluster_v2: forced cluster size (0 = planner, default) */
  MGPU_OPT_CLUSTER_ASYNC = 6,   /* cg_cluster_v2: st.async + mbarrier exchange (default 1; 0 = cluster barriers) */
  MGPU_OPT_PROFILE_PHASES = 7,  /* clock64 per-phase totals of the CG kernels (default 0; read with mgpu_phase_profile) */
  MGPU_OPT_QR_UNBLOCKED = 8,    /* thin_qr: column-at-a-time schedule instead of compact WY (default 0) */
  MGPU_OPT_LS_GROUP = 9,        /* LS-SPAI: skip the lane-per-column kernels (default 0) */
  MGPU_OPT_STREAM_TILES = 10,   /* cg_stream: row-slab x point tiles, the points of a slab processed at the same time (default 1: where a tile holds >= 16 chunks; 2: always; 0: one contiguous row range per block) */
  MGPU_OPT_RETIRED2 = 11,       /* (was a traffic experiment switch of cg_stream; removed) */
  MGPU_OPT_SEQ_SPARSE = 12,     /* sequential MR-SPAI: sparse row-list kernel at every size (default 0: dense-factor kernel up to n = 4096) */
  MGPU_OPT_COUNT = 13,
} mgpu_option;
int mgpu_ctx_set_option(mgpu_ctx *ctx, int option, int64_t value);
int mgpu_ctx_get_option(const mgpu_ctx *ctx, int option, int64_t *value);
/* Copies the 16 clock64 phase totals (MGPU_OPT_PROFILE_PHASES) and resets them. */
int mgpu_phase_profile(mgpu_ctx *ctx, long long *out16);

/* Device scratch buffers for callers that keep results on the device between calls (the drop-in
 * backend's batched solve, read back point by point).  Stream-ordered on the context stream;
 * mgpu_memcpy synchronises the stream before returning (MGPU_HOST: dst is host memory). */
int mgpu_buffer_alloc(mgpu_ctx *ctx, size_t bytes, void **out);
int mgpu_buffer_free(mgpu_ctx *ctx, void *p);
int mgpu_memcpy_d2h(mgpu_ctx *ctx, void *host_dst, const void *dev_src, size_t bytes);
int mgpu_memcpy_h2d(mgpu_ctx *ctx, void *dev_dst, const void *host_src, size_t bytes);

/* ------------------------------------------------------------------ CSR I/O */

/* Replaces constructing a mor::SparseMatrix (sparse.hpp:16-46).  The host
 * arrays are copied (H2D) and may be reused on return.  The CSR invariants
 * are validated on the device (MGPU_ERR_ARG on violation, cf. sparse.cpp:108-138). */
int mgpu_csr_upload(mgpu_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *row_ptr,
                    const int32_t *col_idx, const double *values, mgpu_csr **out);
/* Several host CSR matrices at once (same validation as mgpu_csr_upload): every copy and
 * check is queued before one read-back; out[q] receives matrix q. */
int mgpu_csr_upload_batch(mgpu_ctx *ctx, int count, const int64_t *nrows, const int64_t *ncols, const int64_t *nnz,
                          const int64_t *const *row_ptr, const int32_t *const *col_idx, const double *const *values,
                          mgpu_csr **out);
/* Same, from device pointers already on the context's device (copied). */
int mgpu_csr_upload_device(mgpu_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *row_ptr,
                           const int32_t *col_idx, const double *values, mgpu_csr **out);
/* Shape of the matrix as the reference would store it: stored exact zeros
 * (the LS-SPAI kernels keep the pattern fixed) are dropped on download. */
int mgpu_csr_info(mgpu_ctx *ctx, const mgpu_csr *a, int64_t *nrows, int64_t *ncols, int64_t *nnz);
int mgpu_csr_download(mgpu_ctx *ctx, const mgpu_csr *a, int64_t *row_ptr, int32_t *col_idx, double *values);
/* Binary CSR sidecar (the reference interchanges Matrix Market text, model_io.cpp:154-351):
 * "MGCSR\0\0\1", int64 nrows, ncols, nnz, row_ptr, col_idx (int32), values (f64), little-endian.
 * write stores the download view; read validates like mgpu_csr_upload. */
int mgpu_csr_write(mgpu_ctx *ctx, const mgpu_csr *a, const char *path);
int mgpu_csr_read(mgpu_ctx *ctx, const char *path, mgpu_csr **out);
/* Raw device view (no zero dropping) for callers that stay on the device. */
int mgpu_csr_device_view(const mgpu_csr *a, int64_t *nrows, int64_t *nnz, const int64_t **row_ptr,
                         const int32_t **col_idx, const double **values);
int mgpu_csr_free(mgpu_csr *a);

/* ------------------------------------------------------------ core kernels */

/* sparse.cpp:167-218 sp_add_scaled: a*A + b*B on the union pattern, no FMA
 * contraction, exact zeros dropped. */
int mgpu_sp_add_scaled(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double a, double b, mgpu_csr **out);
/* system.cpp:64-68 shifted_operator, batched over l shifts:
 * out[i] = sp_add(sp_add(M, D, s_i^2, s_i), K, 1, 1), bitwise identical to the reference. */
int mgpu_shifted_operators(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int l,
                           const double *shifts, mgpu_csr **out);
/* sparse.cpp:220-249 transpose (rows of the result ascending, like the reference). */
int mgpu_transpose(mgpu_ctx *ctx, const mgpu_csr *A, mgpu_csr **out);
/* sparse.cpp:251-296: trace(A), trace_inner(A, B) with a fixed-order device
 * reduction (deterministic; trace_inner(A,B) == trace_inner(B,A) bitwise). */
int mgpu_trace(mgpu_ctx *ctx, const mgpu_csr *A, double *out);
int mgpu_trace_inner(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double *out);
/* sparse.cpp:140-158 spmv_into: y = A x (x, y device pointers). */
int mgpu_spmv(mgpu_ctx *ctx, const mgpu_csr *A, const double *x, double *y);
/* spai.cpp:361-373 chain_apply: y = Q_z(...(Q_2(P x))). factors newest first.
 * x, y: n-vectors in `where` memory. */
int mgpu_chain_apply(mgpu_ctx *ctx, int z, const mgpu_csr *const *factors, const double *x, double *y,
                     mgpu_memkind where);

/* spai.cpp:375-409 chain_quality: sqrt((n / samples) sum_k ||(I - K P_chain) g_k||^2) over
 * `samples` unit-norm Gaussian probes from std::mt19937_64(seed) + std::normal_distribution
 * (the reference's stream; default seed 42, spai.hpp:84-85).  factors newest first (z may be 0). */
int mgpu_chain_quality(mgpu_ctx *ctx, int z, const mgpu_csr *const *factors, const mgpu_csr *K, int64_t samples,
                       uint64_t seed, double *out);

/* ------------------------------------------------------------------ SPAI */

typedef enum mgpu_spai_mode
{
  MGPU_SPAI_SEQUENTIAL = 0, /* spai.hpp:38-42 (device: sparse row lists of the built columns, any n) */
  MGPU_SPAI_FROZEN = 1,
} mgpu_spai_mode;

/* spai.cpp:314-331 spai_build (MR-SPAI, Alg. 2): P = alpha I refined per
 * column until ||e_j - K p_j|| <= tol.  col_residual (host, n, optional)
 * receives SpaiFactor::target_frob_residual.  Stagnation reports the LOWEST
 * failing column, as the reference's sequential column loop would. */
int mgpu_spai_build(mgpu_ctx *ctx, const mgpu_csr *K, double tol, int64_t max_col_iters, int mode, mgpu_csr **P,
                    double *col_residual);
/* spai.cpp:333-350 spai_update (Alg. 4): Q minimising ||K_old - K_new Q||_F. */
int mgpu_spai_update(mgpu_ctx *ctx, const mgpu_csr *K_old, const mgpu_csr *K_new, double tol, int64_t max_col_iters,
                     int mode, mgpu_csr **Q, double *col_residual);

typedef enum mgpu_ls_pattern
{
  MGPU_PATTERN_A = 0,  /* J_j = pattern of row j of A               */
  MGPU_PATTERN_A2 = 1, /* J_j = pattern of row j of the symbolic A*A */
  /* flag, OR-ed into the pattern: column-equilibrated LS.  Every column c of S = A(I,J) is scaled
   * by r_c = 1 / ||S_c|| (in-order dot, one division) before the QR and the solution by r_c after
   * the back-substitution.  Same least-squares minimiser; it avoids thin_qr's global rank flush
   * (sigma <= 1e-12 ||S||_F, dense.cpp:162-179), which on the Hermite beam declares every column
   * rank-deficient from n = 2e5 (A^2 pattern) / 4e5 (A pattern) because the theta-dof columns
   * scale like h^2.  The oracle restates it in oracle.c orc_spai_ls / ref_shim.cpp ref_spai_ls. */
  MGPU_LS_COLSCALE = 0x10,
} mgpu_ls_pattern;

/* Static-pattern least-squares SPAI (north star subsystem 1; not in the
 * reference, whose closest relative is spai_build, spai.cpp:314): per column j
 * min ||e_j - A(I,J) m||, J from `pattern`, I = rows of A(:,J), solved by
 * Householder QR in FP64, one warp per column.  K_old != NULL gives the update
 * factor (rhs K_old(I, j), cf. spai.cpp:333).  Rank deficiency ->
 * MGPU_ERR_NUMERICAL naming the column. */
int mgpu_spai_ls(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *K_old, int pattern, mgpu_csr **P);
/* Batched LS-SPAI over l operators (one launch for all shifts). */
int mgpu_spai_ls_batched(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, const mgpu_csr *const *K_old, int pattern,
                         mgpu_csr **P);

/* Sparse x sparse product C = A * B on the device (north star subsystem 2:
 * collapsing a chain [Q, P] into one factor Q*P, cf. spai.cpp:361-373).
 * Exact zeros are dropped. */
int mgpu_spgemm(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, mgpu_csr **C);

/* ------------------------------------------------------------------ CG */

typedef struct mgpu_cg_out
{
  /* all optional (NULL = not wanted); layout [point][column][row] = n x m
   * column-major per point, in `where` memory */
  double *X;          /* BlockSolveResult::X                   (krylov.hpp:44-51) */
  double *recurrence; /* BlockSolveResult::recurrence_residuals */
  double *true_res;   /* BlockSolveResult::true_residuals       */
  /* host arrays of l*m entries */
  int64_t *iterations; /* per column iterations (krylov.cpp:115)              */
  int *converged;      /* per column converged flag                           */
  int *status;         /* per column MGPU_OK / MGPU_ERR_BREAKDOWN              */
  int64_t *breakdown_iteration; /* iteration index of a breakdown, else -1     */
  /* optional host history [point][column][history_cap]: recurrence ||r||/||b|| per iteration */
  double *history;
  int64_t history_cap;
} mgpu_cg_out;

/* krylov.cpp:28-174 pcg_solve / block_solve, batched over l shifted systems
 * and m right-hand sides:  for every point p and column c, CG on A_p P_p with
 * x~0 = 0, the true-residual confirm / restart branch, the breakdown guard
 * (d,w) <= 1e-30 (d,d), maxit, and solution = P_p x~.  All recurrences run in
 * one persistent cooperative kernel with the control flow on the device.
 *   A[p]             : l operators (n x n)
 *   chains[p*z + f]  : z factors per point, newest first (z may be 0: P = I)
 *   B                : rhs, [point][column][row]; ldb_point = elements between
 *                      points (0 = the same n x m block for every point)
 * Returns MGPU_ERR_BREAKDOWN for the first (point, column) that broke down,
 * with the payload the reference's block_solve would carry (krylov.cpp:160-163);
 * other columns still complete and are reported in `out`. */
int mgpu_cg_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains, int64_t n,
                  int64_t m, const double *B, int64_t ldb_point, double rtol, int64_t maxit, mgpu_memkind where,
                  mgpu_cg_out *out);

/* The path in one call (CgBackend::prepare + a solve of every point, airga.cpp:108-181):
 * out[i] = shifted_operator(M, D, K, shifts[i]) (system.cpp:64-68), its LS-SPAI factor on
 * `pattern` (MGPU_PATTERN_A / MGPU_PATTERN_A2, or -1 for P = I), then mgpu_cg_solve over the
 * l points with B / ldb_point / out as there.  Operators and factors are temporaries.
 * phase_ms (optional, 3 doubles): device time of assembly, SPAI, and the solve call. */
int mgpu_shifted_solve(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int l,
                       const double *shifts, int pattern, const double *B, int64_t m, int64_t ldb_point, double rtol,
                       int64_t maxit, mgpu_memkind where, mgpu_cg_out *out, double *phase_ms);

/* ------------------------------------------------------------ model input */

/* Host-side model generators for benchmarks and tests (not on the hot path).
 * Reference chain model: model_io.cpp:18-87 beam_generate.  Hermite
 * cantilever: BASELINE.json configs.  Output arrays are
 * malloc'd; release with mgpu_host_free. */
typedef struct mgpu_host_csr
{
  int64_t nrows, ncols, nnz;
  int64_t *row_ptr;
  int32_t *col_idx;
  double *values;
} mgpu_host_csr;
int mgpu_model_chain(int64_t n, double alpha, double beta, double stiffness_scale, double mass_scale,
                     int consistent_mass, mgpu_host_csr *M, mgpu_host_csr *D, mgpu_host_csr *K);
int mgpu_model_hermite(int64_t ne, double E, double I, double rho, double area, double L, double alpha, double beta,
                       mgpu_host_csr *M, mgpu_host_csr *D, mgpu_host_csr *K);
void mgpu_host_free(mgpu_host_csr *a);
/* Page-locks / releases a host range the caller keeps alive (cudaHostRegister): uploads from it
 * then run as DMA at the link rate instead of through the driver's staging buffers.  The
 * drop-in backend's C entry points pin their copy of M, D, K (re-uploaded on every prepare). */
int mgpu_host_pin(mgpu_ctx *ctx, void *ptr, size_t bytes);
int mgpu_host_unpin(mgpu_ctx *ctx, void *ptr);
/* Device-side generation of the same Hermite cantilever: M, D, K assembled in HBM,
 * bitwise equal to mgpu_model_hermite (row-parallel element sums in element order, exact zeros dropped). */
int mgpu_model_hermite_device(mgpu_ctx *ctx, int64_t ne, double E, double I, double rho, double area, double L,
                              double alpha, double beta, mgpu_csr **M, mgpu_csr **D, mgpu_csr **K);


/* ------------------------------------------------------------------ global Arnoldi + projection */

/* dense.cpp:153-246 thin_qr: A (rows x cols, column-major) -> Q (rows x cols), R (cols x cols), rank
 * (Householder; columns with sigma <= rank_tol ||A||_F are flushed to zero, R's diagonal made
 * nonnegative).  rows >= cols (MGPU_ERR_ARG otherwise), cols <= 1024 on the device. */
int mgpu_thin_qr(mgpu_ctx *ctx, int64_t rows, int64_t cols, const double *A, double rank_tol, double *Q, double *R,
                 int64_t *rank, mgpu_memkind where);

/* airga.cpp:485-500 project_reduce: V (n x r, column-major, orthonormal basis) ->
 *   Mh, Dh, Kh (r x r) = V^T S V,  Fh (r x m) = V^T F,  Cph, Cvh (q x r) = Cp V, Cv V
 * (Cp, Cv: q x n column-major; m = 0 skips F, q = 0 skips Cp / Cv).  All dense buffers in `where` memory. */
int mgpu_project_reduce(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t r,
                        const double *V, int64_t m, const double *F, int64_t q, const double *Cp, const double *Cv,
                        double *Mh, double *Dh, double *Kh, double *Fh, double *Cph, double *Cvh, mgpu_memkind where);

/* Row-slab form of mgpu_project_reduce for a row-distributed basis: M, D, K are the slab's
 * p rows (global column indices), Vext holds global basis rows [ext0, ext0 + next) (the slab's rows
 * [row0, row0 + p) plus a halo covering every column the slab touches), F the slab's p x m rows and
 * Cp / Cv its q x p columns.  Outputs are this slab's partial sums (an all-reduce over slabs gives
 * mgpu_project_reduce's result). */
int mgpu_project_reduce_slab(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t row0,
                             int64_t ext0, int64_t next, int64_t r, const double *Vext, int64_t m, const double *F,
                             int64_t q, const double *Cp, const double *Cv, double *Mh, double *Dh, double *Kh,
                             double *Fh, double *Cph, double *Cvh, mgpu_memkind where);

/* airga.cpp:456-473 arnoldi_deflate: two sweeps of X -= <B_t, X> B_t over the nblocks basis blocks
 * (each `len` values, the same shape as X); gammas[t] = sum of both sweeps' coefficients.
 * X and blocks in `where` memory, gammas on the host. */
int mgpu_arnoldi_deflate(mgpu_ctx *ctx, int64_t len, double *X, int nblocks, const double *const *blocks,
                         double *gammas, mgpu_memkind where);

/* ------------------------------------------------------------------ NVLink / NCCL data plane */

/* One NCCL rank per context (one process per GPU).  Rank 0 creates the id (128 bytes) and the
 * caller distributes it (torch.distributed, MPI, a file); every rank then calls mgpu_comm_init. */
int mgpu_comm_unique_id(void *id128);
int mgpu_comm_init(mgpu_ctx *ctx, const void *id128, int nranks, int rank);
int mgpu_comm_destroy(mgpu_ctx *ctx);
/* In-place sum over ranks of a device buffer (synchronous). */
int mgpu_comm_allreduce_sum(mgpu_ctx *ctx, double *buf, int64_t count);
/* This rank's balanced row slab [row0, row0 + p) of an n-row basis and its halo-extended range
 * [ext0, ext0 + next) (h rows each side, clipped). */
int mgpu_comm_rows(mgpu_ctx *ctx, int64_t n, int64_t h, int64_t *row0, int64_t *p, int64_t *ext0, int64_t *next);
/* Arnoldi-block redistribution after the shift-sharded solves: this rank holds the full-length
 * columns col_ids[c_local] (host ids, global) of an n x R block in X_local (device, n x c_local
 * column-major); Vext (device, next x R column-major) receives rows [ext0, ext0 + next) of all R
 * columns.  Grouped ncclSend / ncclRecv, no host staging. */
int mgpu_comm_columns_to_rows(mgpu_ctx *ctx, int64_t n, int64_t h, int64_t c_local, const int64_t *col_ids,
                              const double *X_local, int64_t R, double *Vext);
/* airga.cpp:485-500 project_reduce over the row-distributed basis: M, D, K are the full operators
 * (replicated), Vext this rank's extended slab (h >= the operators' bandwidth), F (n x m) and Cp, Cv
 * (q x n) the full input / output maps in `where` memory.  Slab partials on the device
 * (mgpu_project_reduce_slab) + one ncclAllReduce; every rank receives the reduced matrices. */
int mgpu_comm_project_reduce(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t h,
                             int64_t r, const double *Vext, int64_t m, const double *F, int64_t q, const double *Cp,
                             const double *Cv, double *Mh, double *Dh, double *Kh, double *Fh, double *Cph,
                             double *Cvh, mgpu_memkind where);
/* max |i - j| over the stored entries (the halo the projection needs). */
int mgpu_csr_bandwidth(mgpu_ctx *ctx, const mgpu_csr *a, int64_t *bw);

#ifdef __cplusplus
}
#endif

#endif /* MGPU_H */
