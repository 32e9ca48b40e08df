/*
 * mor_cuda.h -- C entry points of the drop-in SolveBackend (libmor_cuda.so).
 *
 * The reference selects its solve backend through mor::make_backend (src/airga.cpp:358-365) and
 * drives it through the three SolveBackend methods (include/mor/airga.hpp:136-145):
 *   prepare(sys, points, outer, records)  ->  mor_cuda_backend_prepare
 *   solve(point_index, rhs)               ->  mor_cuda_backend_solve
 *   provides_residuals()                  ->  always true for this backend
 * These functions wrap a mor::CudaCgBackend (paper_1606_01216_b200/host/cuda_backend.hpp) for
 * callers that cannot use the C++ class: a ctypes / cgo / JNI host, and bench.py's end-to-end leg,
 * which drives the reference's own call sequence (prepare, then solve(i, F) for every point, as
 * zeroth_moments does, airga.cpp:374-381) with host buffers.
 *
 * Status codes are mgpu.h's (MGPU_OK, MGPU_ERR_ARG, ...); the message of the reference exception
 * the C++ backend raised is copied into msg.  Host arrays are borrowed for the call.
 */
#ifndef MOR_CUDA_H
#define MOR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mor_cuda_backend mor_cuda_backend;

/* solver: 1 cg_plain, 2 cg_spai, 3 cg_spai_update (AirgaConfig::Solver, airga.hpp:42-48);
 * algorithm: 0 MR-SPAI (reference spai_build / spai_update), 1 LS-SPAI with ls_pattern
 * (MGPU_PATTERN_A / MGPU_PATTERN_A2, | MGPU_LS_COLSCALE); spai_mode: 0 sequential, 1 frozen;
 * maxit_override > 0 replaces cg_maxit_factor * n; flags: MOR_CUDA_SPECULATIVE (batch-solve sys.F in
 * prepare, CudaBackendOptions::speculative_solve), MOR_CUDA_COLLAPSE (collapse the update chain into
 * one factor with a device SpGEMM, CudaBackendOptions::collapse). */
#define MOR_CUDA_SPECULATIVE 1
#define MOR_CUDA_COLLAPSE 2
int mor_cuda_backend_create(int device, int solver, int algorithm, int ls_pattern, double spai_tol,
                            int64_t spai_max_col_iters, int spai_mode, double cg_rtol, int64_t cg_maxit_factor,
                            int64_t maxit_override, int64_t update_start_iteration, int flags,
                            mor_cuda_backend **out, char *msg, size_t cap);
/* Shift sharding over several devices in one process (mor::MultiDeviceCgBackend): point i is
 * prepared and solved on devices[i % ndev]; the devices prepare concurrently. */
int mor_cuda_backend_create_multi(int ndev, const int *devices, int solver, int algorithm, int ls_pattern,
                                  double spai_tol, int64_t spai_max_col_iters, int spai_mode, double cg_rtol,
                                  int64_t cg_maxit_factor, int64_t maxit_override, int64_t update_start_iteration,
                                  int flags, mor_cuda_backend **out, char *msg, size_t cap);
void mor_cuda_backend_destroy(mor_cuda_backend *b);

/* The SecondOrderSystem the backend prepares (system.hpp:15-33): M, D, K as CSR (n x n), F as
 * n x m column-major.  Copied into the backend's mor::SecondOrderSystem. */
int mor_cuda_backend_set_system(mor_cuda_backend *b, int64_t n, int64_t nnz_m, const int64_t *m_rp,
                                const int32_t *m_ci, const double *m_v, int64_t nnz_d, const int64_t *d_rp,
                                const int32_t *d_ci, const double *d_v, int64_t nnz_k, const int64_t *k_rp,
                                const int32_t *k_ci, const double *k_v, int64_t m, const double *F, char *msg,
                                size_t cap);

/* SolveBackend::prepare (airga.cpp:108-164).  record_seconds (optional, l entries): the
 * PrecondRecord seconds of each point. */
int mor_cuda_backend_prepare(mor_cuda_backend *b, int l, const double *points, int64_t outer,
                             double *record_seconds, char *msg, size_t cap);

/* SolveBackend::solve (airga.cpp:166-181) for one point: rhs n x m column-major; X, REC, TR
 * (n x m column-major, optional) receive BlockSolveResult::X / recurrence_residuals /
 * true_residuals; iterations (m, optional) and all_converged (optional). */
int mor_cuda_backend_solve(mor_cuda_backend *b, int64_t point_index, int64_t m, const double *rhs, double *X,
                           double *REC, double *TR, int64_t *iterations, int *all_converged, char *msg, size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* MOR_CUDA_H */
