// SPDX-License-Identifier: Apache-2.0
//
// Host side of the drop-in B200 solve backend (see cuda_backend.hpp).  Pure
// marshalling between the reference's value types and the C-ABI; all
// arithmetic runs in libmgpu.so.  There is no CPU fallback: a missing device
// or an unsupported shape surfaces as an exception.
#include "cuda_backend.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>
#include <string>

#include "mgpu.h"
#include "mor/errors.hpp"

namespace mor
{
namespace
{

using Clock = std::chrono::steady_clock;

// mgpu status -> the reference's exception taxonomy (errors.hpp:13-59).
[[noreturn]] void raise(mgpu_ctx *ctx, int st)
{
  int64_t idx = -1, col = -1, pt = -1;
  char msg[1024] = {0};
  mgpu_last_error(ctx, &idx, &col, &pt, msg, sizeof msg);
  switch (st)
  {
  case MGPU_ERR_ARG: throw ArgumentError(msg);
  case MGPU_ERR_STAGNATION: throw StagnationError(msg, idx);
  case MGPU_ERR_BREAKDOWN: throw BreakdownError(msg, idx);
  case MGPU_ERR_NUMERICAL: throw NumericalError(msg);
  default: throw std::runtime_error(std::string("mgpu (") + mgpu_status_string(st) + "): " + msg);
  }
}

void check(mgpu_ctx *ctx, int st)
{
  if (st != MGPU_OK)
    raise(ctx, st);
}

mgpu_csr *upload(mgpu_ctx *ctx, const SparseMatrix &A)
{
  mgpu_csr *h = nullptr;
  check(ctx, mgpu_csr_upload(ctx, A.nrows, A.ncols, A.nnz(), A.row_ptr.data(), A.col_idx.data(), A.values.data(),
                             &h));
  return h;
}

SparseMatrix download(mgpu_ctx *ctx, const mgpu_csr *m)
{
  SparseMatrix A;
  int64_t nr = 0, nc = 0, nnz = 0;
  check(ctx, mgpu_csr_info(ctx, m, &nr, &nc, &nnz));
  A.nrows = nr;
  A.ncols = nc;
  A.row_ptr.assign(static_cast<std::size_t>(nr + 1), 0);
  A.col_idx.assign(static_cast<std::size_t>(nnz), 0);
  A.values.assign(static_cast<std::size_t>(nnz), 0.0);
  check(ctx, mgpu_csr_download(ctx, m, A.row_ptr.data(), A.col_idx.data(), A.values.data()));
  return A;
}

double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// One batched mgpu_cg_solve for `l` points sharing chain length z.
// status_out: per (point, column) status instead of raising the first breakdown.
std::vector<BlockSolveResult> solve_points(mgpu_ctx *ctx, const std::vector<mgpu_csr *> &A,
                                           const std::vector<mgpu_csr *> &chains_flat, int z, const DenseMatrix &B,
                                           double rtol, std::int64_t maxit, std::vector<int> *status_out = nullptr)
{
  const int l = static_cast<int>(A.size());
  const int64_t n = B.nrows, m = B.ncols;
  const std::size_t blk = static_cast<std::size_t>(n * m);
  std::vector<double> X(blk * l), REC(blk * l), TR(blk * l);
  std::vector<int64_t> it(static_cast<std::size_t>(l * m)), bd(static_cast<std::size_t>(l * m));
  std::vector<int> conv(static_cast<std::size_t>(l * m)), status(static_cast<std::size_t>(l * m));
  mgpu_cg_out out{};
  out.X = X.data();
  out.recurrence = REC.data();
  out.true_res = TR.data();
  out.iterations = it.data();
  out.converged = conv.data();
  out.status = status.data();
  out.breakdown_iteration = bd.data();
  const int st = mgpu_cg_solve(ctx, l, A.data(), z, chains_flat.empty() ? nullptr : chains_flat.data(), n, m,
                               B.values.data(), 0, rtol, maxit, MGPU_HOST, &out);
  if (!(status_out && st == MGPU_ERR_BREAKDOWN))
    check(ctx, st);
  if (status_out)
    *status_out = status;
  std::vector<BlockSolveResult> res(static_cast<std::size_t>(l));
  for (int p = 0; p < l; ++p)
  {
    BlockSolveResult &r = res[static_cast<std::size_t>(p)];
    r.X = DenseMatrix(n, m);
    r.recurrence_residuals = DenseMatrix(n, m);
    r.true_residuals = DenseMatrix(n, m);
    std::copy(X.begin() + p * blk, X.begin() + (p + 1) * blk, r.X.values.begin());
    std::copy(REC.begin() + p * blk, REC.begin() + (p + 1) * blk, r.recurrence_residuals.values.begin());
    std::copy(TR.begin() + p * blk, TR.begin() + (p + 1) * blk, r.true_residuals.values.begin());
    r.iterations.assign(it.begin() + p * m, it.begin() + (p + 1) * m);
    r.all_converged = std::all_of(conv.begin() + p * m, conv.begin() + (p + 1) * m, [](int c) { return c != 0; });
  }
  return res;
}

} // namespace

// ------------------------------------------------------------------ cuda::
namespace cuda
{

Device::Device(int device)
{
  if (mgpu_ctx_create(device, nullptr, &ctx_) != MGPU_OK)
    throw std::runtime_error("mor::cuda: no usable sm_100 device " + std::to_string(device) + " (no CPU fallback)");
}

Device::~Device() { mgpu_ctx_destroy(ctx_); }

DeviceMatrix::DeviceMatrix(Device &dev, const SparseMatrix &A) : dev_(&dev), m_(upload(dev.ctx(), A)) {}
DeviceMatrix::DeviceMatrix(Device &dev, mgpu_csr *adopt) : dev_(&dev), m_(adopt) {}
DeviceMatrix::~DeviceMatrix() { mgpu_csr_free(m_); }
DeviceMatrix::DeviceMatrix(DeviceMatrix &&o) noexcept : dev_(o.dev_), m_(o.m_) { o.m_ = nullptr; }
DeviceMatrix &DeviceMatrix::operator=(DeviceMatrix &&o) noexcept
{
  if (this != &o)
  {
    mgpu_csr_free(m_);
    dev_ = o.dev_;
    m_ = o.m_;
    o.m_ = nullptr;
  }
  return *this;
}
SparseMatrix DeviceMatrix::download() const { return mor::download(dev_->ctx(), m_); }

namespace
{
int mode_of(const SpaiOptions &opts)
{
  return opts.mode == SpaiOptions::Mode::frozen ? MGPU_SPAI_FROZEN : MGPU_SPAI_SEQUENTIAL;
}

SpaiFactor finish_factor(mgpu_ctx *ctx, mgpu_csr *P, std::vector<double> res, Clock::time_point t0,
                         SpaiFactor::Kind kind)
{
  SpaiFactor f;
  f.matrix = mor::download(ctx, P);
  mgpu_csr_free(P);
  f.target_frob_residual = std::move(res);
  f.build_seconds = seconds_since(t0);
  f.kind = kind;
  return f;
}

std::vector<mgpu_csr *> upload_chain(Device &dev, const PreconditionerChain &chain,
                                     std::vector<DeviceMatrix> &keep)
{
  std::vector<mgpu_csr *> h;
  for (const SpaiFactor &f : chain.factors) // newest first, as stored (spai.hpp:63-75)
  {
    keep.emplace_back(dev, f.matrix);
    h.push_back(keep.back().get());
  }
  return h;
}
} // namespace

SpaiFactor spai_build(Device &dev, const SparseMatrix &K, const SpaiOptions &opts)
{
  const auto t0 = Clock::now();
  DeviceMatrix dK(dev, K);
  std::vector<double> res(static_cast<std::size_t>(K.nrows));
  mgpu_csr *P = nullptr;
  check(dev.ctx(), mgpu_spai_build(dev.ctx(), dK.get(), opts.tol, opts.max_col_iters, mode_of(opts), &P, res.data()));
  return finish_factor(dev.ctx(), P, std::move(res), t0, SpaiFactor::Kind::base);
}

SpaiFactor spai_update(Device &dev, const SparseMatrix &K_old, const SparseMatrix &K_new, const SpaiOptions &opts)
{
  const auto t0 = Clock::now();
  DeviceMatrix dO(dev, K_old), dN(dev, K_new);
  std::vector<double> res(static_cast<std::size_t>(K_new.nrows));
  mgpu_csr *Q = nullptr;
  check(dev.ctx(), mgpu_spai_update(dev.ctx(), dO.get(), dN.get(), opts.tol, opts.max_col_iters, mode_of(opts), &Q,
                                    res.data()));
  return finish_factor(dev.ctx(), Q, std::move(res), t0, SpaiFactor::Kind::update);
}

SpaiFactor spai_ls(Device &dev, const SparseMatrix &A, const SparseMatrix *K_old, int pattern)
{
  const auto t0 = Clock::now();
  DeviceMatrix dA(dev, A);
  DeviceMatrix dO;
  if (K_old)
    dO = DeviceMatrix(dev, *K_old);
  mgpu_csr *P = nullptr;
  check(dev.ctx(), mgpu_spai_ls(dev.ctx(), dA.get(), K_old ? dO.get() : nullptr, pattern, &P));
  return finish_factor(dev.ctx(), P, {}, t0, K_old ? SpaiFactor::Kind::update : SpaiFactor::Kind::base);
}

std::vector<double> chain_apply(Device &dev, const PreconditionerChain &chain, std::span<const double> v)
{
  if (chain.empty())
    return std::vector<double>(v.begin(), v.end()); // spai.hpp:77-78
  if (chain.dim() != static_cast<std::int64_t>(v.size()))
    throw ArgumentError("chain_apply: dimension mismatch");
  std::vector<DeviceMatrix> keep;
  const std::vector<mgpu_csr *> h = upload_chain(dev, chain, keep);
  std::vector<double> out(v.size());
  check(dev.ctx(), mgpu_chain_apply(dev.ctx(), static_cast<int>(h.size()), h.data(), v.data(), out.data(), MGPU_HOST));
  return out;
}

double chain_quality(Device &dev, const PreconditionerChain &chain, const SparseMatrix &K, std::int64_t samples,
                     std::uint64_t seed)
{
  if (samples < 1)
    throw ArgumentError("chain_quality: samples must be >= 1"); // spai.cpp:378-381
  std::vector<DeviceMatrix> keep;
  const std::vector<mgpu_csr *> h = chain.empty() ? std::vector<mgpu_csr *>{} : upload_chain(dev, chain, keep);
  const DeviceMatrix dK(dev, K);
  double out = 0.0;
  check(dev.ctx(), mgpu_chain_quality(dev.ctx(), static_cast<int>(h.size()), h.empty() ? nullptr : h.data(), dK.get(),
                                      samples, seed, &out));
  return out;
}

SolveReport pcg_solve(Device &dev, const SparseMatrix &A, const PreconditionerChain &P, std::span<const double> b,
                      double rtol, std::int64_t maxit)
{
  const int64_t n = A.nrows;
  if (A.nrows != A.ncols)
    throw ArgumentError("LinearOperator::from_sparse: matrix must be square");
  if ((!P.empty() && P.dim() != n) || static_cast<int64_t>(b.size()) != n)
    throw ArgumentError("pcg_solve: dimension mismatch");
  DeviceMatrix dA(dev, A);
  std::vector<DeviceMatrix> keep;
  const std::vector<mgpu_csr *> ch = upload_chain(dev, P, keep);
  std::vector<double> x(n), tr(n), rec(n);
  int64_t it = 0, bd = -1;
  int conv = 0, status = 0;
  const int64_t cap = std::min<int64_t>(maxit, int64_t(1) << 20);
  std::vector<double> hist(static_cast<std::size_t>(std::max<int64_t>(cap, 1)));
  mgpu_cg_out out{};
  out.X = x.data();
  out.recurrence = rec.data();
  out.true_res = tr.data();
  out.iterations = &it;
  out.converged = &conv;
  out.status = &status;
  out.breakdown_iteration = &bd;
  out.history = hist.data();
  out.history_cap = cap;
  mgpu_csr *a = dA.get();
  const int st = mgpu_cg_solve(dev.ctx(), 1, &a, static_cast<int>(ch.size()), ch.empty() ? nullptr : ch.data(), n, 1,
                               b.data(), 0, rtol, maxit, MGPU_HOST, &out);
  if (st == MGPU_ERR_BREAKDOWN) // pcg_solve's own message (krylov.cpp:108-111)
    throw BreakdownError("pcg_solve: direction curvature breakdown at iteration " + std::to_string(bd), bd);
  check(dev.ctx(), st);
  SolveReport rep;
  rep.solution = std::move(x);
  rep.residual = std::move(tr);
  rep.recurrence_residual = std::move(rec);
  rep.iterations = it;
  rep.converged = conv != 0;
  hist.resize(static_cast<std::size_t>(std::min(it, cap)));
  rep.relres_history = std::move(hist);
  return rep;
}

BlockSolveResult block_solve(Device &dev, const SparseMatrix &A, const PreconditionerChain &P, const DenseMatrix &B,
                             double rtol, std::int64_t maxit)
{
  if (B.nrows != A.nrows)
    throw ArgumentError("block_solve: right-hand-side rows do not match the operator dimension");
  DeviceMatrix dA(dev, A);
  std::vector<DeviceMatrix> keep;
  const std::vector<mgpu_csr *> ch = upload_chain(dev, P, keep);
  return solve_points(dev.ctx(), {dA.get()}, ch, static_cast<int>(ch.size()), B, rtol, maxit)[0];
}

std::vector<double> SparseApply::operator()(std::span<const double> v) const { return spmv(*A, v); }
std::vector<double> ChainApply::operator()(std::span<const double> v) const { return mor::chain_apply(*chain, v); }

LinearOperator sparse_operator(const SparseMatrix &A)
{
  if (A.nrows != A.ncols)
    throw ArgumentError("LinearOperator::from_sparse: matrix must be square");
  return {SparseApply{&A}, A.nrows};
}

LinearOperator chain_operator(const PreconditionerChain &chain, std::int64_t n)
{
  if (chain.empty())
    return identity_operator(n);
  return {ChainApply{&chain}, n};
}

LinearOperator identity_operator(std::int64_t n) { return {IdentityApply{}, n}; }

namespace
{
// The operator pair as device inputs: A must be a matrix; P a matrix, chain or identity.
struct DeviceOperands
{
  const SparseMatrix *A = nullptr;
  PreconditionerChain chain; // copy of the factors (or the single matrix P)
};

DeviceOperands resolve(const LinearOperator &A, const LinearOperator &P, const char *who)
{
  DeviceOperands d;
  if (const auto *sa = A.apply.target<SparseApply>())
    d.A = sa->A;
  else
    throw ArgumentError(std::string(who) + ": operator not device-resident (build A with mor::cuda::sparse_operator)");
  if (P.apply.target<IdentityApply>())
    return d;
  if (const auto *ca = P.apply.target<ChainApply>())
    d.chain = *ca->chain;
  else if (const auto *sp = P.apply.target<SparseApply>())
  {
    SpaiFactor f;
    f.matrix = *sp->A;
    d.chain.push_newest(std::move(f));
  }
  else
    throw ArgumentError(std::string(who) +
                        ": preconditioner not device-resident (use mor::cuda::chain_operator / sparse_operator / "
                        "identity_operator)");
  if (P.dim != A.dim)
    throw ArgumentError(std::string(who) + ": dimension mismatch");
  return d;
}
} // namespace

SolveReport pcg_solve(Device &dev, const LinearOperator &A, const LinearOperator &P, std::span<const double> b,
                      double rtol, std::int64_t maxit)
{
  const DeviceOperands d = resolve(A, P, "pcg_solve");
  return pcg_solve(dev, *d.A, d.chain, b, rtol, maxit);
}

BlockSolveResult block_solve(Device &dev, const LinearOperator &A, const LinearOperator &P, const DenseMatrix &B,
                             double rtol, std::int64_t maxit)
{
  const DeviceOperands d = resolve(A, P, "block_solve");
  return block_solve(dev, *d.A, d.chain, B, rtol, maxit);
}

QrResult thin_qr(Device &dev, const DenseMatrix &A, double rank_tol)
{
  if (A.nrows < A.ncols)
    throw ArgumentError("thin_qr: requires nrows >= ncols"); // dense.cpp:155-158
  QrResult out;
  out.Q = DenseMatrix(A.nrows, A.ncols);
  out.R = DenseMatrix(A.ncols, A.ncols);
  int64_t rank = 0;
  check(dev.ctx(), mgpu_thin_qr(dev.ctx(), A.nrows, A.ncols, A.values.data(), rank_tol, out.Q.values.data(),
                                out.R.values.data(), &rank, MGPU_HOST));
  out.rank = rank;
  return out;
}

ReducedSystem project_reduce(Device &dev, const SecondOrderSystem &sys, const OrthonormalBasis &basis)
{
  const DenseMatrix &V = basis.assembled;
  const int64_t n = sys.M.nrows, r = V.ncols, m = sys.F.ncols, q = sys.Cp.nrows;
  if (V.nrows != n)
    throw ArgumentError("project_reduce: basis has the wrong row count");
  const DeviceMatrix dM(dev, sys.M), dD(dev, sys.D), dK(dev, sys.K);
  ReducedSystem rs;
  rs.Mh = DenseMatrix(r, r);
  rs.Dh = DenseMatrix(r, r);
  rs.Kh = DenseMatrix(r, r);
  rs.Fh = DenseMatrix(r, m);
  rs.Cph = DenseMatrix(q, r);
  rs.Cvh = DenseMatrix(q, r);
  check(dev.ctx(), mgpu_project_reduce(dev.ctx(), dM.get(), dD.get(), dK.get(), r, V.values.data(), m,
                                       m ? sys.F.values.data() : nullptr, q, q ? sys.Cp.values.data() : nullptr,
                                       q ? sys.Cv.values.data() : nullptr, rs.Mh.values.data(), rs.Dh.values.data(),
                                       rs.Kh.values.data(), m ? rs.Fh.values.data() : nullptr,
                                       q ? rs.Cph.values.data() : nullptr, q ? rs.Cvh.values.data() : nullptr,
                                       MGPU_HOST));
  rs.basis = V; // airga.cpp:495-499
  rs.r = r;
  rs.alpha = sys.alpha;
  rs.beta = sys.beta;
  return rs;
}

std::vector<double> arnoldi_deflate(Device &dev, DenseMatrix &X, std::span<const DenseMatrix> basis_blocks)
{
  std::vector<const double *> ptrs;
  for (const DenseMatrix &b : basis_blocks)
  {
    if (b.nrows != X.nrows || b.ncols != X.ncols)
      throw ArgumentError("trace_inner(dense): shape mismatch"); // dense.cpp:40-43 via trace_inner
    ptrs.push_back(b.values.data());
  }
  std::vector<double> gammas(basis_blocks.size(), 0.0);
  check(dev.ctx(), mgpu_arnoldi_deflate(dev.ctx(), static_cast<int64_t>(X.values.size()), X.values.data(),
                                        static_cast<int>(ptrs.size()), ptrs.empty() ? nullptr : ptrs.data(),
                                        gammas.empty() ? nullptr : gammas.data(), MGPU_HOST));
  return gammas;
}

} // namespace cuda

// ------------------------------------------------------------------ backend
struct CudaCgBackend::State
{
  CudaSolveSettings cfg;
  CudaBackendOptions opt;
  cuda::Device dev;
  int64_t n = 0;
  cuda::DeviceMatrix M, D, K;
  std::vector<cuda::DeviceMatrix> prev_ops;            // operators of the prepared iteration
  std::vector<std::vector<cuda::DeviceMatrix>> chains; // per point, newest first
  std::vector<std::int64_t> zlog;                      // logical chain length per point (collapse)
  // speculative batched solve of sys.F (CudaBackendOptions::speculative_solve): X, recurrence and
  // true residuals of every point stay on the device ([array][point][column][row]) until
  // solve(i, F) reads point i back
  std::vector<double> spec_rhs; // the F it was solved for
  int64_t spec_m = 0;
  void *spec_dev = nullptr;
  std::vector<int64_t> spec_it;
  std::vector<int> spec_conv;
  std::vector<char> spec_ready; // per point: results valid and not yet handed out

  State(const CudaSolveSettings &c, const CudaBackendOptions &o) : cfg(c), opt(o), dev(o.device) {}
  ~State() { drop_spec(); }
  void drop_spec()
  {
    if (spec_dev)
      mgpu_buffer_free(dev.ctx(), spec_dev);
    spec_dev = nullptr;
    spec_ready.clear();
  }
  int64_t maxit() const { return opt.maxit_override > 0 ? opt.maxit_override : cfg.cg_maxit_factor * n; }
};

CudaSolveSettings settings_of(const AirgaConfig &cfg)
{
  CudaSolveSettings s;
  s.solver = cfg.solver;
  s.spai_tol = cfg.spai_tol;
  s.spai_max_col_iters = cfg.spai_max_col_iters;
  s.spai_mode = cfg.spai_mode;
  s.cg_rtol = cfg.cg_rtol;
  s.cg_maxit_factor = cfg.cg_maxit_factor;
  s.update_start_iteration = cfg.update_start_iteration;
  return s;
}

CudaCgBackend::CudaCgBackend(const AirgaConfig &cfg, const CudaBackendOptions &opt)
  : st_(std::make_unique<State>(settings_of(cfg), opt))
{
}

CudaCgBackend::CudaCgBackend(const CudaSolveSettings &cfg, const CudaBackendOptions &opt)
  : st_(std::make_unique<State>(cfg, opt))
{
}

CudaCgBackend::~CudaCgBackend() = default;

// airga.cpp:108-164
void CudaCgBackend::prepare(const SecondOrderSystem &sys, const std::vector<double> &points, std::int64_t outer,
                            std::vector<PrecondRecord> *records)
{
  State &s = *st_;
  mgpu_ctx *ctx = s.dev.ctx();
  s.n = sys.order();
  s.drop_spec();
  // M, D, K are uploaded on every prepare, as the reference rebuilds shifted_operator(sys, s) from
  // sys on every prepare (airga.cpp:110-116): a caller may edit sys between outer iterations.
  {
    const SparseMatrix *src[3] = {&sys.M, &sys.D, &sys.K};
    int64_t nr[3], nc[3], nz[3];
    const int64_t *rp[3];
    const int32_t *ci[3];
    const double *va[3];
    for (int q = 0; q < 3; ++q)
    {
      nr[q] = src[q]->nrows;
      nc[q] = src[q]->ncols;
      nz[q] = src[q]->nnz();
      rp[q] = src[q]->row_ptr.data();
      ci[q] = src[q]->col_idx.data();
      va[q] = src[q]->values.data();
    }
    mgpu_csr *h[3] = {nullptr, nullptr, nullptr};
    check(ctx, mgpu_csr_upload_batch(ctx, 3, nr, nc, nz, rp, ci, va, h));
    s.M = cuda::DeviceMatrix(s.dev, h[0]);
    s.D = cuda::DeviceMatrix(s.dev, h[1]);
    s.K = cuda::DeviceMatrix(s.dev, h[2]);
  }
  const int l = static_cast<int>(points.size());
  std::vector<mgpu_csr *> raw(static_cast<std::size_t>(l), nullptr);
  if (l > 0)
    check(ctx, mgpu_shifted_operators(ctx, s.M.get(), s.D.get(), s.K.get(), l, points.data(), raw.data()));
  std::vector<cuda::DeviceMatrix> fresh;
  for (mgpu_csr *h : raw)
    fresh.emplace_back(s.dev, h);

  if (s.cfg.solver == AirgaConfig::Solver::cg_plain)
  {
    s.chains.clear();
    s.chains.resize(static_cast<std::size_t>(l));
  }
  else
  {
    SpaiOptions opts;
    opts.tol = s.cfg.spai_tol;
    opts.max_col_iters = s.cfg.spai_max_col_iters;
    opts.mode = s.cfg.spai_mode;
    const bool update_mode = s.cfg.solver == AirgaConfig::Solver::cg_spai_update &&
                             outer >= s.cfg.update_start_iteration &&
                             s.prev_ops.size() == static_cast<std::size_t>(l) &&
                             s.chains.size() == static_cast<std::size_t>(l);
    if (!update_mode)
    {
      s.chains.clear();
      s.chains.resize(static_cast<std::size_t>(l));
      s.zlog.assign(static_cast<std::size_t>(l), 0);
    }
    // push_newest (spai.cpp:352-359), or with collapse the product Q P with the collapsed chain
    auto push = [&](int i, mgpu_csr *f) {
      auto &chain = s.chains[static_cast<std::size_t>(i)];
      if (s.opt.collapse && update_mode && !chain.empty())
      {
        cuda::DeviceMatrix q(s.dev, f);
        mgpu_csr *qp = nullptr;
        check(ctx, mgpu_spgemm(ctx, q.get(), chain.front().get(), &qp));
        chain.front() = cuda::DeviceMatrix(s.dev, qp);
      }
      else
        chain.insert(chain.begin(), cuda::DeviceMatrix(s.dev, f));
      return ++s.zlog[static_cast<std::size_t>(i)];
    };
    if (s.opt.algorithm == cuda::SpaiAlgorithm::ls)
    {
      // one batched launch for every point; the per-point record gets the average
      const auto t0 = Clock::now();
      std::vector<mgpu_csr *> olds, outs(static_cast<std::size_t>(l), nullptr);
      for (const auto &o : s.prev_ops)
        olds.push_back(o.get());
      check(ctx, mgpu_spai_ls_batched(ctx, l, raw.data(), update_mode ? olds.data() : nullptr, s.opt.ls_pattern,
                                      outs.data()));
      const double each = seconds_since(t0) / std::max(l, 1);
      for (int i = 0; i < l; ++i)
      {
        const std::int64_t z = push(i, outs[static_cast<std::size_t>(i)]);
        if (records)
        {
          PrecondRecord rec;
          rec.outer = outer;
          rec.point_index = i;
          rec.point = points[static_cast<std::size_t>(i)];
          rec.seconds = each;
          rec.kind = update_mode ? SpaiFactor::Kind::update : SpaiFactor::Kind::base;
          rec.chain_length = z;
          records->push_back(rec);
        }
      }
    }
    else
    {
      const int mode = opts.mode == SpaiOptions::Mode::frozen ? MGPU_SPAI_FROZEN : MGPU_SPAI_SEQUENTIAL;
      for (int i = 0; i < l; ++i)
      {
        PrecondRecord rec;
        rec.outer = outer;
        rec.point_index = i;
        rec.point = points[static_cast<std::size_t>(i)];
        const auto t0 = Clock::now();
        mgpu_csr *f = nullptr;
        if (update_mode)
        {
          check(ctx, mgpu_spai_update(ctx, s.prev_ops[static_cast<std::size_t>(i)].get(), raw[static_cast<std::size_t>(i)],
                                      opts.tol, opts.max_col_iters, mode, &f, nullptr));
          rec.kind = SpaiFactor::Kind::update;
        }
        else
        {
          check(ctx, mgpu_spai_build(ctx, raw[static_cast<std::size_t>(i)], opts.tol, opts.max_col_iters, mode, &f,
                                     nullptr));
          rec.kind = SpaiFactor::Kind::base;
        }
        mgpu_ctx_synchronize(ctx);
        rec.chain_length = push(i, f);
        rec.seconds = seconds_since(t0);
        if (records)
          records->push_back(rec);
      }
    }
  }
  s.prev_ops = std::move(fresh);
  // speculative batched solve of sys.F for every point (one kernel; zeroth_moments asks for
  // exactly these next).  A breakdown is left to the on-demand path, which raises it with the
  // reference's payload; the other points keep their results.
  const int64_t m = sys.F.ncols;
  if (s.opt.speculative_solve && l > 0 && m > 0 && sys.F.nrows == s.n)
  {
    std::vector<mgpu_csr *> A, flat;
    const std::size_t z = s.chains.empty() ? 0 : s.chains[0].size();
    bool uniform = true;
    for (int i = 0; i < l; ++i)
    {
      A.push_back(s.prev_ops[static_cast<std::size_t>(i)].get());
      const std::size_t zi = s.chains.empty() ? 0 : s.chains[static_cast<std::size_t>(i)].size();
      uniform = uniform && zi == z;
      if (!s.chains.empty())
        for (const auto &f : s.chains[static_cast<std::size_t>(i)])
          flat.push_back(f.get());
    }
    if (uniform)
    {
      const std::size_t blk = static_cast<std::size_t>(s.n * m), cnt = static_cast<std::size_t>(l) * m;
      check(ctx, mgpu_buffer_alloc(ctx, (3 * blk * l + blk) * sizeof(double), &s.spec_dev));
      auto *base = static_cast<double *>(s.spec_dev);
      double *Bd = base + 3 * blk * l; // the rhs block, uploaded once
      check(ctx, mgpu_memcpy_h2d(ctx, Bd, sys.F.values.data(), blk * sizeof(double)));
      std::vector<int> status(cnt);
      std::vector<int64_t> bd(cnt);
      s.spec_it.assign(cnt, 0);
      s.spec_conv.assign(cnt, 0);
      mgpu_cg_out out{};
      out.X = base;
      out.recurrence = base + blk * l;
      out.true_res = base + 2 * blk * l;
      out.iterations = s.spec_it.data();
      out.converged = s.spec_conv.data();
      out.status = status.data();
      out.breakdown_iteration = bd.data();
      // the results stay in spec_dev until solve(i, F) reads point i back
      const int st = mgpu_cg_solve(ctx, l, A.data(), static_cast<int>(z), flat.empty() ? nullptr : flat.data(), s.n,
                                   m, Bd, 0, s.cfg.cg_rtol, s.maxit(), MGPU_DEVICE, &out);
      if (st != MGPU_OK && st != MGPU_ERR_BREAKDOWN)
        check(ctx, st);
      s.spec_ready.assign(static_cast<std::size_t>(l), 1);
      for (int i = 0; i < l; ++i)
        for (int64_t c = 0; c < m; ++c)
          if (status[static_cast<std::size_t>(i * m + c)] != MGPU_OK)
            s.spec_ready[static_cast<std::size_t>(i)] = 0; // the on-demand solve raises the breakdown
      s.spec_rhs = sys.F.values;
      s.spec_m = m;
    }
  }
}

// airga.cpp:166-181
BlockSolveResult CudaCgBackend::solve(std::int64_t point_index, const DenseMatrix &rhs)
{
  State &s = *st_;
  if (point_index < 0 || point_index >= static_cast<std::int64_t>(s.prev_ops.size()))
    throw std::out_of_range("CudaCgBackend::solve: point index");
  if (rhs.nrows != s.n)
    throw ArgumentError("block_solve: right-hand-side rows do not match the operator dimension");
  const std::size_t pi = static_cast<std::size_t>(point_index);
  if (cached(point_index, rhs))
  {
    BlockSolveResult r;
    r.X = DenseMatrix(s.n, rhs.ncols);
    r.recurrence_residuals = DenseMatrix(s.n, rhs.ncols);
    r.true_residuals = DenseMatrix(s.n, rhs.ncols);
    r.iterations.assign(static_cast<std::size_t>(rhs.ncols), 0);
    take_cached(point_index, r.X.values.data(), r.recurrence_residuals.values.data(), r.true_residuals.values.data(),
                r.iterations.data(), &r.all_converged);
    return r;
  }
  std::vector<mgpu_csr *> chain;
  if (!s.chains.empty())
    for (const auto &f : s.chains[pi])
      chain.push_back(f.get());
  return solve_points(s.dev.ctx(), {s.prev_ops[pi].get()}, chain, static_cast<int>(chain.size()), rhs, s.cfg.cg_rtol,
                      s.maxit())[0];
}

bool CudaCgBackend::cached(std::int64_t point_index, const DenseMatrix &rhs) const
{
  return rhs.nrows == st_->n && cached(point_index, rhs.values.data(), rhs.ncols);
}

namespace
{
// memcmp == 0 over several host threads: the exact "is this sys.F" test reads 2 x 8 n m bytes per
// solve(i, F) call (configs[3]: 16 calls x 32 MB, ~3 ms each on one thread).
bool same_bytes(const void *a, const void *b, std::size_t bytes)
{
  constexpr std::size_t kPerThread = std::size_t(4) << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t parts = std::min<std::size_t>({std::size_t(8), std::size_t(hw), bytes / kPerThread + 1});
  if (parts <= 1)
    return std::memcmp(a, b, bytes) == 0;
  std::vector<int> eq(parts, 1);
  std::vector<std::thread> th;
  const auto *pa = static_cast<const unsigned char *>(a);
  const auto *pb = static_cast<const unsigned char *>(b);
  for (std::size_t t = 0; t < parts; ++t)
  {
    const std::size_t o0 = bytes * t / parts, o1 = bytes * (t + 1) / parts;
    th.emplace_back([=, &eq] { eq[t] = std::memcmp(pa + o0, pb + o0, o1 - o0) == 0; });
  }
  for (auto &x : th)
    x.join();
  return std::all_of(eq.begin(), eq.end(), [](int v) { return v != 0; });
}
} // namespace

bool CudaCgBackend::cached(std::int64_t point_index, const double *rhs, std::int64_t m) const
{
  const State &s = *st_;
  const std::size_t pi = static_cast<std::size_t>(point_index);
  return point_index >= 0 && pi < s.spec_ready.size() && s.spec_ready[pi] && m == s.spec_m &&
         same_bytes(rhs, s.spec_rhs.data(), sizeof(double) * s.spec_rhs.size());
}

void CudaCgBackend::take_cached(std::int64_t point_index, double *X, double *REC, double *TR, std::int64_t *iterations,
                                bool *all_converged)
{
  State &s = *st_;
  const std::size_t pi = static_cast<std::size_t>(point_index), l = s.spec_ready.size();
  const std::size_t blk = static_cast<std::size_t>(s.n * s.spec_m);
  const auto *base = static_cast<const double *>(s.spec_dev);
  double *dst[3] = {X, REC, TR};
  for (int q = 0; q < 3; ++q)
    if (dst[q])
      check(s.dev.ctx(), mgpu_memcpy_d2h(s.dev.ctx(), dst[q], base + (q * l + pi) * blk, blk * sizeof(double)));
  bool conv = true;
  for (int64_t c = 0; c < s.spec_m; ++c)
  {
    if (iterations)
      iterations[c] = s.spec_it[pi * s.spec_m + c];
    conv = conv && s.spec_conv[pi * s.spec_m + c] != 0;
  }
  if (all_converged)
    *all_converged = conv;
  s.spec_ready[pi] = 0; // handed out once; a repeated request solves again
}

std::vector<BlockSolveResult> CudaCgBackend::solve_all(const DenseMatrix &rhs)
{
  State &s = *st_;
  const int l = static_cast<int>(s.prev_ops.size());
  std::vector<mgpu_csr *> A, flat;
  std::size_t z = s.chains.empty() ? 0 : s.chains[0].size();
  bool uniform = true;
  for (int i = 0; i < l; ++i)
  {
    A.push_back(s.prev_ops[static_cast<std::size_t>(i)].get());
    const std::size_t zi = s.chains.empty() ? 0 : s.chains[static_cast<std::size_t>(i)].size();
    uniform = uniform && zi == z;
    if (!s.chains.empty())
      for (const auto &f : s.chains[static_cast<std::size_t>(i)])
        flat.push_back(f.get());
  }
  if (!uniform)
  {
    std::vector<BlockSolveResult> out;
    for (int i = 0; i < l; ++i)
      out.push_back(solve(i, rhs));
    return out;
  }
  return solve_points(s.dev.ctx(), A, flat, static_cast<int>(z), rhs, s.cfg.cg_rtol, s.maxit());
}

// ------------------------------------------------------------------ multi-device backend
MultiDeviceCgBackend::MultiDeviceCgBackend(const CudaSolveSettings &cfg, const CudaBackendOptions &opt,
                                           std::vector<int> devices)
{
  if (devices.empty())
    throw ArgumentError("MultiDeviceCgBackend: no devices");
  for (int d : devices)
  {
    CudaBackendOptions o = opt;
    o.device = d;
    parts_.push_back(std::make_unique<CudaCgBackend>(cfg, o));
  }
}

MultiDeviceCgBackend::MultiDeviceCgBackend(const AirgaConfig &cfg, const CudaBackendOptions &opt,
                                           std::vector<int> devices)
  : MultiDeviceCgBackend(settings_of(cfg), opt, std::move(devices))
{
}

MultiDeviceCgBackend::~MultiDeviceCgBackend() = default;

std::pair<std::size_t, std::int64_t> MultiDeviceCgBackend::owner(std::int64_t point_index) const
{
  const auto N = static_cast<std::int64_t>(parts_.size());
  return {static_cast<std::size_t>(point_index % N), point_index / N};
}

void MultiDeviceCgBackend::prepare(const SecondOrderSystem &sys, const std::vector<double> &points,
                                   std::int64_t outer, std::vector<PrecondRecord> *records)
{
  const std::size_t N = parts_.size();
  std::vector<std::vector<double>> mine(N);
  for (std::size_t i = 0; i < points.size(); ++i)
    mine[i % N].push_back(points[i]);
  std::vector<std::vector<PrecondRecord>> recs(N);
  std::vector<std::exception_ptr> err(N);
  std::vector<std::thread> th;
  for (std::size_t d = 0; d < N; ++d)
    th.emplace_back([&, d] {
      try
      {
        parts_[d]->prepare(sys, mine[d], outer, &recs[d]);
      }
      catch (...)
      {
        err[d] = std::current_exception();
      }
    });
  for (auto &t : th)
    t.join();
  for (std::size_t d = 0; d < N; ++d) // the lowest device slot's error, as a serial loop would meet first
    if (err[d])
      std::rethrow_exception(err[d]);
  if (records) // global point order, as CgBackend::prepare records them
  {
    std::vector<PrecondRecord> all;
    for (std::size_t d = 0; d < N; ++d)
      for (PrecondRecord r : recs[d])
      {
        r.point_index = r.point_index * static_cast<std::int64_t>(N) + static_cast<std::int64_t>(d);
        all.push_back(r);
      }
    std::sort(all.begin(), all.end(), [](const PrecondRecord &a, const PrecondRecord &b) {
      return a.point_index < b.point_index;
    });
    records->insert(records->end(), all.begin(), all.end());
  }
}

BlockSolveResult MultiDeviceCgBackend::solve(std::int64_t point_index, const DenseMatrix &rhs)
{
  if (point_index < 0)
    throw std::out_of_range("MultiDeviceCgBackend::solve: point index");
  const auto [d, local] = owner(point_index);
  return parts_[d]->solve(local, rhs);
}

std::unique_ptr<SolveBackend> make_cuda_backend(const AirgaConfig &cfg, const CudaBackendOptions &opt)
{
  if (cfg.solver == AirgaConfig::Solver::direct)
    throw ArgumentError("make_cuda_backend: the direct solver has no device backend");
  return std::make_unique<CudaCgBackend>(cfg, opt);
}

} // namespace mor
