// SPDX-License-Identifier: Apache-2.0
//
// C entry points over mor::CudaCgBackend (include/mor_cuda.h).  Marshalling only: every flop
// runs in libmgpu.so.
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "cuda_backend.hpp"
#include "mgpu.h"
#include "mor/errors.hpp"
#include "mor_cuda.h"

struct mor_cuda_backend
{
  std::unique_ptr<mor::CudaCgBackend> impl;         // one device
  std::unique_ptr<mor::MultiDeviceCgBackend> multi; // or shift-sharded over several
  mor::SolveBackend &backend() { return multi ? static_cast<mor::SolveBackend &>(*multi) : *impl; }
  mor::SecondOrderSystem sys;
  int64_t n = 0;
  // host ranges of `sys` that are page-locked (mgpu_host_pin): prepare() re-uploads M, D, K every
  // time, from pinned memory that is a DMA at the link rate
  std::vector<void *> pinned;
  void unpin()
  {
    for (void *p : pinned)
      mgpu_host_unpin(nullptr, p);
    pinned.clear();
  }
  ~mor_cuda_backend() { unpin(); }
};

namespace
{
void put(char *msg, size_t cap, const std::string &s)
{
  if (msg && cap)
  {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(msg, s.data(), k);
    msg[k] = '\0';
  }
}

// mor:: exception -> mgpu status (include/mor/errors.hpp:13-59 <-> mgpu.h)
template <class F>
int guarded(char *msg, size_t cap, F &&f)
{
  try
  {
    f();
    put(msg, cap, "");
    return MGPU_OK;
  }
  catch (const mor::StagnationError &e)
  {
    put(msg, cap, e.what());
    return MGPU_ERR_STAGNATION;
  }
  catch (const mor::BreakdownError &e)
  {
    put(msg, cap, e.what());
    return MGPU_ERR_BREAKDOWN;
  }
  catch (const mor::NumericalError &e)
  {
    put(msg, cap, e.what());
    return MGPU_ERR_NUMERICAL;
  }
  catch (const mor::ArgumentError &e)
  {
    put(msg, cap, e.what());
    return MGPU_ERR_ARG;
  }
  catch (const std::exception &e)
  {
    put(msg, cap, e.what());
    return MGPU_ERR_CUDA;
  }
}

mor::SparseMatrix csr(int64_t n, int64_t nnz, const int64_t *rp, const int32_t *ci, const double *v)
{
  mor::SparseMatrix A;
  A.nrows = n;
  A.ncols = n;
  A.row_ptr.assign(rp, rp + n + 1);
  A.col_idx.assign(ci, ci + nnz);
  A.values.assign(v, v + nnz);
  return A;
}
} // namespace

extern "C" {

namespace
{
void settings(int solver, int algorithm, int ls_pattern, double spai_tol, int64_t spai_max_col_iters, int spai_mode,
              double cg_rtol, int64_t cg_maxit_factor, int64_t maxit_override, int64_t update_start_iteration,
              int flags, mor::CudaSolveSettings &s, mor::CudaBackendOptions &o)
{
  if (solver < 1 || solver > 3 || algorithm < 0 || algorithm > 1)
    throw mor::ArgumentError("mor_cuda_backend_create: bad argument");
  s.solver = solver == 1   ? mor::AirgaConfig::Solver::cg_plain
             : solver == 2 ? mor::AirgaConfig::Solver::cg_spai
                           : mor::AirgaConfig::Solver::cg_spai_update;
  s.spai_tol = spai_tol;
  s.spai_max_col_iters = spai_max_col_iters;
  s.spai_mode = spai_mode == 0 ? mor::SpaiOptions::Mode::sequential : mor::SpaiOptions::Mode::frozen;
  s.cg_rtol = cg_rtol;
  s.cg_maxit_factor = cg_maxit_factor;
  s.update_start_iteration = update_start_iteration;
  o.algorithm = algorithm == 1 ? mor::cuda::SpaiAlgorithm::ls : mor::cuda::SpaiAlgorithm::mr;
  o.ls_pattern = ls_pattern;
  o.speculative_solve = (flags & MOR_CUDA_SPECULATIVE) != 0;
  o.collapse = (flags & MOR_CUDA_COLLAPSE) != 0;
  o.maxit_override = maxit_override;
}
} // namespace

int mor_cuda_backend_create(int device, int solver, int algorithm, int ls_pattern, double spai_tol,
                            int64_t spai_max_col_iters, int spai_mode, double cg_rtol, int64_t cg_maxit_factor,
                            int64_t maxit_override, int64_t update_start_iteration, int flags,
                            mor_cuda_backend **out, char *msg, size_t cap)
{
  return mor_cuda_backend_create_multi(1, &device, solver, algorithm, ls_pattern, spai_tol, spai_max_col_iters,
                                       spai_mode, cg_rtol, cg_maxit_factor, maxit_override, update_start_iteration,
                                       flags, out, msg, cap);
}

int mor_cuda_backend_create_multi(int ndev, const int *devices, int solver, int algorithm, int ls_pattern,
                                  double spai_tol, int64_t spai_max_col_iters, int spai_mode, double cg_rtol,
                                  int64_t cg_maxit_factor, int64_t maxit_override, int64_t update_start_iteration,
                                  int flags, mor_cuda_backend **out, char *msg, size_t cap)
{
  return guarded(msg, cap, [&] {
    if (!out || ndev < 1 || !devices)
      throw mor::ArgumentError("mor_cuda_backend_create: bad argument");
    mor::CudaSolveSettings s;
    mor::CudaBackendOptions o;
    settings(solver, algorithm, ls_pattern, spai_tol, spai_max_col_iters, spai_mode, cg_rtol, cg_maxit_factor,
             maxit_override, update_start_iteration, flags, s, o);
    auto b = std::make_unique<mor_cuda_backend>();
    if (ndev == 1)
    {
      o.device = devices[0];
      b->impl = std::make_unique<mor::CudaCgBackend>(s, o);
    }
    else
      b->multi = std::make_unique<mor::MultiDeviceCgBackend>(s, o, std::vector<int>(devices, devices + ndev));
    *out = b.release();
  });
}

void mor_cuda_backend_destroy(mor_cuda_backend *b) { delete b; }

int mor_cuda_backend_set_system(mor_cuda_backend *b, int64_t n, int64_t nnz_m, const int64_t *m_rp,
                                const int32_t *m_ci, const double *m_v, int64_t nnz_d, const int64_t *d_rp,
                                const int32_t *d_ci, const double *d_v, int64_t nnz_k, const int64_t *k_rp,
                                const int32_t *k_ci, const double *k_v, int64_t m, const double *F, char *msg,
                                size_t cap)
{
  return guarded(msg, cap, [&] {
    if (!b || n < 0 || m < 0 || (m > 0 && !F))
      throw mor::ArgumentError("mor_cuda_backend_set_system: bad argument");
    b->unpin(); // the old arrays go away with the assignments below
    b->sys.M = csr(n, nnz_m, m_rp, m_ci, m_v);
    b->sys.D = csr(n, nnz_d, d_rp, d_ci, d_v);
    b->sys.K = csr(n, nnz_k, k_rp, k_ci, k_v);
    for (mor::SparseMatrix *A : {&b->sys.M, &b->sys.D, &b->sys.K})
    {
      auto pin = [&](void *p, size_t bytes) {
        if (bytes >= (size_t(1) << 20) && mgpu_host_pin(nullptr, p, bytes) == MGPU_OK) // (small systems: not worth a registration)
          b->pinned.push_back(p);
      };
      pin(A->row_ptr.data(), sizeof(A->row_ptr[0]) * A->row_ptr.size());
      pin(A->col_idx.data(), sizeof(A->col_idx[0]) * A->col_idx.size());
      pin(A->values.data(), sizeof(A->values[0]) * A->values.size());
    }
    b->sys.F = mor::DenseMatrix(n, m);
    if (m > 0)
      std::memcpy(b->sys.F.values.data(), F, sizeof(double) * static_cast<size_t>(n * m));
    b->n = n;
  });
}

int mor_cuda_backend_prepare(mor_cuda_backend *b, int l, const double *points, int64_t outer,
                             double *record_seconds, char *msg, size_t cap)
{
  return guarded(msg, cap, [&] {
    if (!b || l < 0 || (l > 0 && !points))
      throw mor::ArgumentError("mor_cuda_backend_prepare: bad argument");
    std::vector<mor::PrecondRecord> recs;
    b->backend().prepare(b->sys, std::vector<double>(points, points + l), outer, &recs);
    if (record_seconds)
      for (const auto &r : recs)
        if (r.point_index >= 0 && r.point_index < l)
          record_seconds[r.point_index] = r.seconds;
  });
}

int mor_cuda_backend_solve(mor_cuda_backend *b, int64_t point_index, int64_t m, const double *rhs, double *X,
                           double *REC, double *TR, int64_t *iterations, int *all_converged, char *msg, size_t cap)
{
  return guarded(msg, cap, [&] {
    if (!b || !rhs || m < 0)
      throw mor::ArgumentError("mor_cuda_backend_solve: bad argument");
    mor::CudaCgBackend *part = b->impl.get();
    int64_t local = point_index;
    if (b->multi && point_index >= 0)
    {
      const auto own = b->multi->owner(point_index);
      part = &b->multi->part(own.first);
      local = own.second;
    }
    if (part->cached(local, rhs, m)) // prepare's batched solve: one device -> host copy per array
    {
      bool conv = false;
      part->take_cached(local, X, REC, TR, iterations, &conv);
      if (all_converged)
        *all_converged = conv ? 1 : 0;
      return;
    }
    mor::DenseMatrix B(b->n, m);
    std::memcpy(B.values.data(), rhs, sizeof(double) * static_cast<size_t>(b->n * m));
    mor::BlockSolveResult r = b->backend().solve(point_index, B);
    const size_t bytes = sizeof(double) * static_cast<size_t>(b->n * m);
    if (X)
      std::memcpy(X, r.X.values.data(), bytes);
    if (REC)
      std::memcpy(REC, r.recurrence_residuals.values.data(), bytes);
    if (TR)
      std::memcpy(TR, r.true_residuals.values.data(), bytes);
    if (iterations)
      std::copy(r.iterations.begin(), r.iterations.end(), iterations);
    if (all_converged)
      *all_converged = r.all_converged ? 1 : 0;
  });
}

} // extern "C"
