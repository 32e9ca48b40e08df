// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C entry points over the UNMODIFIED reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/).  Python tests and bench.py's reference arm load the result,
// oracle/_ref/libmorref.so, with ctypes.  Every function forwards to the
// reference API it names; nothing here re-implements reference arithmetic.
//
// Status codes follow include/mgpu.h (MGPU_OK, MGPU_ERR_*), so a test can
// compare the reference's exception class with the CUDA path's status word.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "mor/airga.hpp"
#include "mor/dense.hpp"
#include "mor/errors.hpp"
#include "mor/kernels.hpp"
#include "mor/krylov.hpp"
#include "mor/model_io.hpp"
#include "mor/sparse.hpp"
#include "mor/spai.hpp"
#include "mor/system.hpp"

extern "C" {

// Borrowed (input) or malloc-owned (output) CSR triple.
typedef struct ref_csr
{
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  int64_t *row_ptr;
  int32_t *col_idx;
  double *values;
} ref_csr;

typedef struct ref_err
{
  int64_t index; // column / iteration payload of the exception
  char msg[512];
} ref_err;
}

namespace
{

enum Status
{
  OK = 0,
  ERR_ARG = 1,
  ERR_STAGNATION = 2,
  ERR_BREAKDOWN = 3,
  ERR_NUMERICAL = 4,
  ERR_OTHER = 9,
};

mor::SparseMatrix to_mor(const ref_csr *a)
{
  mor::SparseMatrix m;
  m.nrows = a->nrows;
  m.ncols = a->ncols;
  m.row_ptr.assign(a->row_ptr, a->row_ptr + a->nrows + 1);
  m.col_idx.assign(a->col_idx, a->col_idx + a->nnz);
  m.values.assign(a->values, a->values + a->nnz);
  return m;
}

void to_ref(const mor::SparseMatrix &m, ref_csr *out)
{
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->nnz = m.nnz();
  out->row_ptr = static_cast<int64_t *>(std::malloc(sizeof(int64_t) * (m.nrows + 1)));
  out->col_idx = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * (m.nnz() > 0 ? m.nnz() : 1)));
  out->values = static_cast<double *>(std::malloc(sizeof(double) * (m.nnz() > 0 ? m.nnz() : 1)));
  std::memcpy(out->row_ptr, m.row_ptr.data(), sizeof(int64_t) * (m.nrows + 1));
  if (m.nnz() > 0)
  {
    std::memcpy(out->col_idx, m.col_idx.data(), sizeof(int32_t) * m.nnz());
    std::memcpy(out->values, m.values.data(), sizeof(double) * m.nnz());
  }
}

void set_msg(ref_err *err, const char *what)
{
  if (err != nullptr)
  {
    std::snprintf(err->msg, sizeof err->msg, "%s", what);
  }
}

// Maps the reference's exception taxonomy (errors.hpp:13-103) onto status codes.
template <class F>
int guarded(ref_err *err, F &&body)
{
  if (err != nullptr)
  {
    err->index = -1;
    err->msg[0] = '\0';
  }
  try
  {
    body();
    return OK;
  }
  catch (const mor::StagnationError &e)
  {
    if (err) err->index = e.column;
    set_msg(err, e.what());
    return ERR_STAGNATION;
  }
  catch (const mor::BreakdownError &e)
  {
    if (err) err->index = e.iteration;
    set_msg(err, e.what());
    return ERR_BREAKDOWN;
  }
  catch (const mor::NumericalError &e)
  {
    set_msg(err, e.what());
    return ERR_NUMERICAL;
  }
  catch (const mor::ArgumentError &e)
  {
    set_msg(err, e.what());
    return ERR_ARG;
  }
  catch (const std::exception &e)
  {
    set_msg(err, e.what());
    return ERR_OTHER;
  }
}

mor::PreconditionerChain make_chain(int z, const ref_csr *factors_newest_first)
{
  mor::PreconditionerChain chain;
  // push_newest prepends, so push oldest first.
  for (int f = z - 1; f >= 0; --f)
  {
    mor::SpaiFactor fac;
    fac.matrix = to_mor(&factors_newest_first[f]);
    chain.push_newest(std::move(fac));
  }
  return chain;
}

mor::SpaiOptions make_opts(double tol, int64_t max_col_iters, int mode, int64_t threads)
{
  mor::SpaiOptions o;
  o.tol = tol;
  o.max_col_iters = max_col_iters;
  o.mode = mode == 0 ? mor::SpaiOptions::Mode::sequential : mor::SpaiOptions::Mode::frozen;
  o.threads = threads;
  return o;
}

} // namespace

extern "C" {

void ref_csr_free(ref_csr *a)
{
  std::free(a->row_ptr);
  std::free(a->col_idx);
  std::free(a->values);
  a->row_ptr = nullptr;
  a->col_idx = nullptr;
  a->values = nullptr;
}

// 0 = scalar, 1 = avx2 (kernels_dispatch.cpp:633-641). Returns 1 on success.
int ref_force_kernels(int variant)
{
  return mor::kernels::force_variant(variant == 0 ? mor::kernels::Variant::scalar : mor::kernels::Variant::avx2) ? 1
                                                                                                                 : 0;
}

int ref_beam_generate(int64_t n, double alpha, double beta, double stiffness_scale, double mass_scale,
                      int consistent_mass, ref_csr *M, ref_csr *D, ref_csr *K, ref_err *err)
{
  return guarded(err, [&] {
    mor::ModelSpec spec;
    spec.n = n;
    spec.alpha = alpha;
    spec.beta = beta;
    spec.stiffness_scale = stiffness_scale;
    spec.mass_scale = mass_scale;
    spec.mass = consistent_mass ? mor::ModelSpec::Mass::consistent : mor::ModelSpec::Mass::identity;
    const mor::SecondOrderSystem sys = mor::beam_generate(spec);
    to_ref(sys.M, M);
    to_ref(sys.D, D);
    to_ref(sys.K, K);
  });
}

// Triplets -> CSR through the reference's from_triplets (sum duplicates, drop zeros).
int ref_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t *rows, const int64_t *cols,
                      const double *vals, ref_csr *out, ref_err *err)
{
  return guarded(err, [&] {
    std::vector<mor::SparseMatrix::Triplet> t(static_cast<std::size_t>(count));
    for (int64_t k = 0; k < count; ++k)
    {
      t[static_cast<std::size_t>(k)] = {rows[k], cols[k], vals[k]};
    }
    to_ref(mor::SparseMatrix::from_triplets(nrows, ncols, std::move(t)), out);
  });
}

int ref_sp_add_scaled(const ref_csr *A, const ref_csr *B, double a, double b, ref_csr *out, ref_err *err)
{
  return guarded(err, [&] { to_ref(mor::sp_add_scaled(to_mor(A), to_mor(B), a, b), out); });
}

int ref_shifted_operator(const ref_csr *M, const ref_csr *D, const ref_csr *K, double s, ref_csr *out,
                         ref_err *err)
{
  return guarded(err, [&] {
    mor::SecondOrderSystem sys;
    sys.M = to_mor(M);
    sys.D = to_mor(D);
    sys.K = to_mor(K);
    to_ref(mor::shifted_operator(sys, s), out);
  });
}

int ref_transpose(const ref_csr *A, ref_csr *out, ref_err *err)
{
  return guarded(err, [&] { to_ref(mor::transpose(to_mor(A)), out); });
}

double ref_trace(const ref_csr *A) { return mor::trace(to_mor(A)); }

double ref_trace_inner(const ref_csr *A, const ref_csr *B) { return mor::trace_inner(to_mor(A), to_mor(B)); }

int ref_spmv(const ref_csr *A, const double *x, double *y, ref_err *err)
{
  return guarded(err, [&] {
    const mor::SparseMatrix m = to_mor(A);
    mor::spmv_into(m, std::span<const double>(x, static_cast<std::size_t>(m.ncols)),
                   std::span<double>(y, static_cast<std::size_t>(m.nrows)));
  });
}

// mode: 0 sequential, 1 frozen (spai.hpp:38-42)
int ref_spai_build(const ref_csr *K, double tol, int64_t max_col_iters, int mode, int64_t threads, ref_csr *P,
                   double *col_residual, double *seconds, ref_err *err)
{
  return guarded(err, [&] {
    const mor::SpaiFactor f = mor::spai_build(to_mor(K), make_opts(tol, max_col_iters, mode, threads));
    to_ref(f.matrix, P);
    if (col_residual != nullptr)
    {
      std::memcpy(col_residual, f.target_frob_residual.data(), sizeof(double) * f.target_frob_residual.size());
    }
    if (seconds != nullptr)
    {
      *seconds = f.build_seconds;
    }
  });
}

int ref_spai_update(const ref_csr *K_old, const ref_csr *K_new, double tol, int64_t max_col_iters, int mode,
                    int64_t threads, ref_csr *Q, double *col_residual, double *seconds, ref_err *err)
{
  return guarded(err, [&] {
    const mor::SpaiFactor f =
        mor::spai_update(to_mor(K_old), to_mor(K_new), make_opts(tol, max_col_iters, mode, threads));
    to_ref(f.matrix, Q);
    if (col_residual != nullptr)
    {
      std::memcpy(col_residual, f.target_frob_residual.data(), sizeof(double) * f.target_frob_residual.size());
    }
    if (seconds != nullptr)
    {
      *seconds = f.build_seconds;
    }
  });
}

// factors are given newest first, as PreconditionerChain stores them (spai.hpp:63).
int ref_chain_apply(int z, const ref_csr *factors, int64_t n, const double *v, double *out, ref_err *err)
{
  return guarded(err, [&] {
    const mor::PreconditionerChain chain = make_chain(z, factors);
    const std::vector<double> x = mor::chain_apply(chain, std::span<const double>(v, static_cast<std::size_t>(n)));
    std::memcpy(out, x.data(), sizeof(double) * x.size());
  });
}

double ref_chain_quality(int z, const ref_csr *factors, const ref_csr *K, int64_t samples, uint64_t seed)
{
  const mor::PreconditionerChain chain = make_chain(z, factors);
  return mor::chain_quality(chain, to_mor(K), samples, seed);
}

// pcg_solve with A = from_sparse(A) and P = chain (identity when z == 0),
// exactly how CgBackend::solve wires it (airga.cpp:166-181).
int ref_pcg_solve(const ref_csr *A, int z, const ref_csr *factors, const double *b, double rtol, int64_t maxit,
                  double *solution, double *residual, double *recurrence, int64_t *iterations, int *converged,
                  double *history, int64_t history_cap, int64_t *history_len, ref_err *err)
{
  return guarded(err, [&] {
    const mor::SparseMatrix Am = to_mor(A);
    const int64_t n = Am.nrows;
    const mor::LinearOperator Aop = mor::LinearOperator::from_sparse(Am);
    const mor::PreconditionerChain chain = make_chain(z, factors);
    const mor::LinearOperator P =
        z == 0 ? mor::LinearOperator::identity(n)
               : mor::LinearOperator{[&chain](std::span<const double> v) { return mor::chain_apply(chain, v); }, n};
    const mor::SolveReport rep =
        mor::pcg_solve(Aop, P, std::span<const double>(b, static_cast<std::size_t>(n)), rtol, maxit);
    std::memcpy(solution, rep.solution.data(), sizeof(double) * n);
    std::memcpy(residual, rep.residual.data(), sizeof(double) * n);
    std::memcpy(recurrence, rep.recurrence_residual.data(), sizeof(double) * n);
    *iterations = rep.iterations;
    *converged = rep.converged ? 1 : 0;
    const int64_t h = static_cast<int64_t>(rep.relres_history.size());
    *history_len = h;
    if (history != nullptr)
    {
      std::memcpy(history, rep.relres_history.data(), sizeof(double) * (h < history_cap ? h : history_cap));
    }
  });
}

// B, X, recurrence, true_res: n x m column-major (dense.hpp:14-37).
int ref_block_solve(const ref_csr *A, int z, const ref_csr *factors, int64_t m, const double *B, double rtol,
                    int64_t maxit, double *X, double *recurrence, double *true_res, int64_t *iterations,
                    int *all_converged, ref_err *err)
{
  return guarded(err, [&] {
    const mor::SparseMatrix Am = to_mor(A);
    const int64_t n = Am.nrows;
    const mor::LinearOperator Aop = mor::LinearOperator::from_sparse(Am);
    const mor::PreconditionerChain chain = make_chain(z, factors);
    const mor::LinearOperator P =
        z == 0 ? mor::LinearOperator::identity(n)
               : mor::LinearOperator{[&chain](std::span<const double> v) { return mor::chain_apply(chain, v); }, n};
    mor::DenseMatrix Bm(n, m);
    std::memcpy(Bm.values.data(), B, sizeof(double) * n * m);
    const mor::BlockSolveResult r = mor::block_solve(Aop, P, Bm, rtol, maxit);
    std::memcpy(X, r.X.values.data(), sizeof(double) * n * m);
    std::memcpy(recurrence, r.recurrence_residuals.values.data(), sizeof(double) * n * m);
    std::memcpy(true_res, r.true_residuals.values.data(), sizeof(double) * n * m);
    std::memcpy(iterations, r.iterations.data(), sizeof(int64_t) * m);
    *all_converged = r.all_converged ? 1 : 0;
  });
}

int ref_thin_qr(int64_t rows, int64_t cols, const double *A, double rank_tol, double *Q, double *R, int64_t *rank,
                ref_err *err)
{
  return guarded(err, [&] {
    mor::DenseMatrix a(rows, cols);
    std::memcpy(a.values.data(), A, sizeof(double) * rows * cols);
    const mor::QrResult qr = mor::thin_qr(a, rank_tol);
    std::memcpy(Q, qr.Q.values.data(), sizeof(double) * rows * cols);
    std::memcpy(R, qr.R.values.data(), sizeof(double) * cols * cols);
    *rank = qr.rank;
  });
}

// project_reduce (airga.cpp:485-500) on (M, D, K, F, Cp, Cv) and an assembled basis V (n x r).
int ref_project_reduce(const ref_csr *M, const ref_csr *D, const ref_csr *K, int64_t r, const double *V, int64_t m,
                       const double *F, int64_t q, const double *Cp, const double *Cv, double *Mh, double *Dh,
                       double *Kh, double *Fh, double *Cph, double *Cvh, ref_err *err)
{
  return guarded(err, [&] {
    mor::SecondOrderSystem sys;
    sys.M = to_mor(M);
    sys.D = to_mor(D);
    sys.K = to_mor(K);
    const int64_t n = sys.M.nrows;
    sys.F = mor::DenseMatrix(n, m);
    if (m > 0)
      std::memcpy(sys.F.values.data(), F, sizeof(double) * n * m);
    sys.Cp = mor::DenseMatrix(q, n);
    sys.Cv = mor::DenseMatrix(q, n);
    if (q > 0)
    {
      std::memcpy(sys.Cp.values.data(), Cp, sizeof(double) * q * n);
      std::memcpy(sys.Cv.values.data(), Cv, sizeof(double) * q * n);
    }
    mor::OrthonormalBasis basis;
    basis.assembled = mor::DenseMatrix(n, r);
    std::memcpy(basis.assembled.values.data(), V, sizeof(double) * n * r);
    const mor::ReducedSystem rs = mor::project_reduce(sys, basis);
    std::memcpy(Mh, rs.Mh.values.data(), sizeof(double) * r * r);
    std::memcpy(Dh, rs.Dh.values.data(), sizeof(double) * r * r);
    std::memcpy(Kh, rs.Kh.values.data(), sizeof(double) * r * r);
    if (m > 0)
      std::memcpy(Fh, rs.Fh.values.data(), sizeof(double) * r * m);
    if (q > 0)
    {
      std::memcpy(Cph, rs.Cph.values.data(), sizeof(double) * q * r);
      std::memcpy(Cvh, rs.Cvh.values.data(), sizeof(double) * q * r);
    }
  });
}

// arnoldi_deflate (airga.cpp:456-473): X (rows x cols) against nblocks blocks of the same shape.
int ref_arnoldi_deflate(int64_t rows, int64_t cols, double *X, int nblocks, const double *const *blocks,
                        double *gammas, ref_err *err)
{
  return guarded(err, [&] {
    mor::DenseMatrix x(rows, cols);
    std::memcpy(x.values.data(), X, sizeof(double) * rows * cols);
    std::vector<mor::DenseMatrix> bl;
    for (int t = 0; t < nblocks; ++t)
    {
      bl.emplace_back(rows, cols);
      std::memcpy(bl.back().values.data(), blocks[t], sizeof(double) * rows * cols);
    }
    const std::vector<double> g = mor::arnoldi_deflate(x, bl);
    std::memcpy(X, x.values.data(), sizeof(double) * rows * cols);
    for (int t = 0; t < nblocks; ++t)
      gammas[t] = g[static_cast<std::size_t>(t)];
  });
}

// ---- LS-SPAI from reference primitives (SURVEY.md 8(a') definition) ----
//
// The static-pattern least-squares SPAI is NOT in the reference (north star
// subsystem 1).  This is its CPU restatement assembled from the reference's
// own primitives: transpose (sparse.cpp:220), DenseMatrix, thin_qr
// (dense.cpp:153-246) and from_triplets (sparse.cpp:15-60).  It is the
// reference arm's LS-SPAI and the pin for oracle.c's orc_spai_ls.
// pattern 0 = A's CSR pattern, 1 = symbolic A*A pattern.
int ref_spai_ls(const ref_csr *A_in, const ref_csr *K_old_in, int pattern, ref_csr *P, double *seconds, ref_err *err)
{
  return guarded(err, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    const mor::SparseMatrix A = to_mor(A_in);
    const int64_t n = A.nrows;
    if (A.ncols != n || (K_old_in && (K_old_in->nrows != n || K_old_in->ncols != n)))
    {
      throw mor::ArgumentError("spai_ls: operands must be square with equal shape");
    }
    // pattern | 0x10: column-equilibrated variant (oracle.c orc_spai_ls header): r_c = 1 / ||S_c||,
    // S_c *= r_c before thin_qr, m_c = u_c * r_c after the back-substitution
    const bool colscale = (pattern & 0x10) != 0;
    pattern &= ~0x10;
    // symbolic pattern rows
    std::vector<std::vector<int32_t>> pat(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i)
    {
      auto &row = pat[static_cast<std::size_t>(i)];
      for (int64_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
      {
        if (pattern == 0)
        {
          row.push_back(A.col_idx[k]);
          continue;
        }
        const int32_t t = A.col_idx[k];
        for (int64_t q = A.row_ptr[t]; q < A.row_ptr[t + 1]; ++q)
        {
          row.push_back(A.col_idx[q]);
        }
      }
      std::sort(row.begin(), row.end());
      row.erase(std::unique(row.begin(), row.end()), row.end());
    }
    const mor::SparseMatrix At = mor::transpose(A);
    mor::SparseMatrix Kot;
    if (K_old_in)
    {
      Kot = mor::transpose(to_mor(K_old_in));
    }
    std::vector<int64_t> pos(static_cast<std::size_t>(n), -1);
    std::vector<mor::SparseMatrix::Triplet> trips;
    for (int64_t j = 0; j < n; ++j)
    {
      const auto &J = pat[static_cast<std::size_t>(j)];
      const int64_t nj = static_cast<int64_t>(J.size());
      if (nj == 0)
      {
        continue;
      }
      std::vector<int64_t> I;
      for (const int32_t k : J)
      {
        for (int64_t q = At.row_ptr[k]; q < At.row_ptr[k + 1]; ++q)
        {
          I.push_back(At.col_idx[q]);
        }
      }
      std::sort(I.begin(), I.end());
      I.erase(std::unique(I.begin(), I.end()), I.end());
      const int64_t ni = static_cast<int64_t>(I.size());
      for (int64_t a = 0; a < ni; ++a)
      {
        pos[static_cast<std::size_t>(I[a])] = a;
      }
      if (ni < nj)
      {
        throw mor::NumericalError("spai_ls: rank-deficient least-squares problem in column " + std::to_string(j));
      }
      mor::DenseMatrix S(ni, nj);
      for (int64_t c = 0; c < nj; ++c)
      {
        const int32_t k = J[static_cast<std::size_t>(c)];
        for (int64_t q = At.row_ptr[k]; q < At.row_ptr[k + 1]; ++q)
        {
          S.at(pos[static_cast<std::size_t>(At.col_idx[q])], c) = At.values[q];
        }
      }
      std::vector<double> e(static_cast<std::size_t>(ni), 0.0);
      if (K_old_in)
      {
        for (int64_t q = Kot.row_ptr[j]; q < Kot.row_ptr[j + 1]; ++q)
        {
          const int64_t p = pos[static_cast<std::size_t>(Kot.col_idx[q])];
          if (p >= 0)
          {
            e[static_cast<std::size_t>(p)] = Kot.values[q];
          }
        }
      }
      else if (pos[static_cast<std::size_t>(j)] >= 0)
      {
        e[static_cast<std::size_t>(pos[static_cast<std::size_t>(j)])] = 1.0;
      }
      const auto &ops = mor::kernels::active();
      std::vector<double> dsc(static_cast<std::size_t>(nj), 1.0);
      if (colscale)
      {
        for (int64_t c = 0; c < nj; ++c)
        {
          const double d = std::sqrt(ops.dot(S.col(c), S.col(c), static_cast<std::size_t>(ni)));
          if (d == 0.0)
          {
            throw mor::NumericalError("spai_ls: rank-deficient least-squares problem in column " + std::to_string(j));
          }
          const double r = 1.0 / d;
          dsc[static_cast<std::size_t>(c)] = r;
          for (int64_t i = 0; i < ni; ++i)
          {
            S.at(i, c) = S.at(i, c) * r;
          }
        }
      }
      const mor::QrResult qr = mor::thin_qr(S);
      if (qr.rank < nj)
      {
        throw mor::NumericalError("spai_ls: rank-deficient least-squares problem in column " + std::to_string(j));
      }
      std::vector<double> y(static_cast<std::size_t>(nj)), m(static_cast<std::size_t>(nj));
      for (int64_t c = 0; c < nj; ++c)
      {
        y[static_cast<std::size_t>(c)] = ops.dot(qr.Q.col(c), e.data(), static_cast<std::size_t>(ni));
      }
      for (int64_t k = nj - 1; k >= 0; --k)
      {
        double acc = y[static_cast<std::size_t>(k)];
        for (int64_t q = k + 1; q < nj; ++q)
        {
          acc -= qr.R.at(k, q) * m[static_cast<std::size_t>(q)];
        }
        m[static_cast<std::size_t>(k)] = acc / qr.R.at(k, k);
      }
      if (colscale)
      {
        for (int64_t c = 0; c < nj; ++c)
        {
          m[static_cast<std::size_t>(c)] = m[static_cast<std::size_t>(c)] * dsc[static_cast<std::size_t>(c)];
        }
      }
      for (int64_t c = 0; c < nj; ++c)
      {
        trips.push_back({J[static_cast<std::size_t>(c)], j, m[static_cast<std::size_t>(c)]});
      }
      for (int64_t a = 0; a < ni; ++a)
      {
        pos[static_cast<std::size_t>(I[a])] = -1;
      }
    }
    to_ref(mor::SparseMatrix::from_triplets(n, n, std::move(trips)), P);
    if (seconds != nullptr)
    {
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

// ---- The reference CgBackend through make_backend (airga.cpp:358-365) ----

struct ref_backend
{
  std::unique_ptr<mor::SolveBackend> impl;
  mor::SecondOrderSystem sys;
  std::vector<mor::PrecondRecord> records;
};

// solver: 1 cg_plain, 2 cg_spai, 3 cg_spai_update (airga.hpp:42-48)
ref_backend *ref_backend_create(int solver, double spai_tol, int64_t spai_max_col_iters, int spai_mode, double cg_rtol,
                                int64_t cg_maxit_factor, int64_t update_start_iteration, const ref_csr *M,
                                const ref_csr *D, const ref_csr *K)
{
  auto *b = new ref_backend;
  mor::AirgaConfig cfg;
  cfg.solver = solver == 1   ? mor::AirgaConfig::Solver::cg_plain
               : solver == 2 ? mor::AirgaConfig::Solver::cg_spai
                             : mor::AirgaConfig::Solver::cg_spai_update;
  cfg.spai_tol = spai_tol;
  cfg.spai_max_col_iters = spai_max_col_iters;
  cfg.spai_mode = spai_mode == 0 ? mor::SpaiOptions::Mode::sequential : mor::SpaiOptions::Mode::frozen;
  cfg.cg_rtol = cg_rtol;
  cfg.cg_maxit_factor = cg_maxit_factor;
  cfg.update_start_iteration = update_start_iteration;
  b->impl = mor::make_backend(cfg);
  b->sys.M = to_mor(M);
  b->sys.D = to_mor(D);
  b->sys.K = to_mor(K);
  return b;
}

void ref_backend_destroy(ref_backend *b) { delete b; }

int ref_backend_prepare(ref_backend *b, int64_t l, const double *points, int64_t outer, double *seconds_out,
                        int *kind_out, int64_t *chain_len_out, ref_err *err)
{
  return guarded(err, [&] {
    b->records.clear();
    b->impl->prepare(b->sys, std::vector<double>(points, points + l), outer, &b->records);
    for (std::size_t i = 0; i < b->records.size(); ++i)
    {
      if (seconds_out) seconds_out[i] = b->records[i].seconds;
      if (kind_out) kind_out[i] = b->records[i].kind == mor::SpaiFactor::Kind::base ? 0 : 1;
      if (chain_len_out) chain_len_out[i] = b->records[i].chain_length;
    }
  });
}

int ref_backend_solve(ref_backend *b, int64_t point_index, int64_t n, int64_t m, const double *rhs, double *X,
                      double *recurrence, double *true_res, int64_t *iterations, int *all_converged, ref_err *err)
{
  return guarded(err, [&] {
    mor::DenseMatrix B(n, m);
    std::memcpy(B.values.data(), rhs, sizeof(double) * n * m);
    const mor::BlockSolveResult r = b->impl->solve(point_index, B);
    std::memcpy(X, r.X.values.data(), sizeof(double) * n * m);
    std::memcpy(recurrence, r.recurrence_residuals.values.data(), sizeof(double) * n * m);
    std::memcpy(true_res, r.true_residuals.values.data(), sizeof(double) * n * m);
    std::memcpy(iterations, r.iterations.data(), sizeof(int64_t) * m);
    *all_converged = r.all_converged ? 1 : 0;
  });
}

} // extern "C"
