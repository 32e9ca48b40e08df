// SPDX-License-Identifier: Apache-2.0
//
// Drop-in B200 solve backend for the reference AIRGA library (namespace mor).
//
// Compiles against the reference's own headers (proj/include/mor/*.hpp) and
// calls the sm_100a kernels through the C-ABI in include/mgpu.h.  Nothing here
// re-implements host-side arithmetic: every flop of prepare() and solve()
// runs on the device.  See INTEGRATION.md for the two-line change to
// make_backend (airga.cpp:358-365) that selects it.
//
//   class CudaCgBackend : public mor::SolveBackend   (airga.hpp:133-145)
//       replaces CgBackend (airga.cpp:103-190): same prepare / solve /
//       provides_residuals contract, same PrecondRecord bookkeeping, same
//       exception types and payloads; plus solve_all() (every point in one
//       batched kernel) and an LS-SPAI option.
//   namespace mor::cuda                               free-function drop-ins
//       spai_build / spai_update      (spai.hpp:53-61)  -> MR-SPAI on the device
//       spai_ls                       (north star LS-SPAI, not in the reference)
//       chain_apply                   (spai.hpp:77-79)
//       chain_quality                 (spai.hpp:81-85)
//       pcg_solve / block_solve       (krylov.hpp:41-56)
//       thin_qr / project_reduce / arnoldi_deflate   (dense.hpp:69, airga.hpp:176-183)
//   The reference's pcg_solve takes LinearOperators wrapping std::function;
//   arbitrary host callables cannot run on the device, so the drop-ins take
//   the SparseMatrix and PreconditionerChain that CgBackend::solve wraps
//   (airga.cpp:168-180) -- the only operators the solve path ever builds.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "mor/airga.hpp"
#include "mor/krylov.hpp"
#include "mor/spai.hpp"

struct mgpu_ctx;
struct mgpu_csr;

namespace mor
{

namespace cuda
{

/// Device context (one GPU, one stream); not shareable across host threads.
class Device
{
public:
  explicit Device(int device = 0);
  ~Device();
  Device(const Device &) = delete;
  Device &operator=(const Device &) = delete;
  mgpu_ctx *ctx() const { return ctx_; }

private:
  mgpu_ctx *ctx_ = nullptr;
};

/// Device-resident CSR (owns an mgpu_csr).
class DeviceMatrix
{
public:
  DeviceMatrix() = default;
  DeviceMatrix(Device &dev, const SparseMatrix &A);
  DeviceMatrix(Device &dev, mgpu_csr *adopt);
  ~DeviceMatrix();
  DeviceMatrix(DeviceMatrix &&o) noexcept;
  DeviceMatrix &operator=(DeviceMatrix &&o) noexcept;
  DeviceMatrix(const DeviceMatrix &) = delete;
  DeviceMatrix &operator=(const DeviceMatrix &) = delete;
  mgpu_csr *get() const { return m_; }
  /// Reference-convention CSR (exact zeros dropped), D2H.
  SparseMatrix download() const;

private:
  Device *dev_ = nullptr;
  mgpu_csr *m_ = nullptr;
};

enum class SpaiAlgorithm
{
  mr, ///< the reference's minimal-residual SPAI (Alg. 2/4), frozen mode
  ls, ///< static-pattern least-squares SPAI (north star subsystem 1)
};

SpaiFactor spai_build(Device &dev, const SparseMatrix &K, const SpaiOptions &opts = {});
SpaiFactor spai_update(Device &dev, const SparseMatrix &K_old, const SparseMatrix &K_new,
                       const SpaiOptions &opts = {});
/// pattern 0: A's pattern, 1: symbolic A*A.  K_old == nullptr builds P.
SpaiFactor spai_ls(Device &dev, const SparseMatrix &A, const SparseMatrix *K_old, int pattern = 0);
std::vector<double> chain_apply(Device &dev, const PreconditionerChain &chain, std::span<const double> v);
/// Stochastic ||I - K P_chain||_F, the reference's probe stream (mt19937_64(seed)).
double chain_quality(Device &dev, const PreconditionerChain &chain, const SparseMatrix &K, std::int64_t samples,
                     std::uint64_t seed = 42);
SolveReport pcg_solve(Device &dev, const SparseMatrix &A, const PreconditionerChain &P, std::span<const double> b,
                      double rtol, std::int64_t maxit);
BlockSolveResult block_solve(Device &dev, const SparseMatrix &A, const PreconditionerChain &P, const DenseMatrix &B,
                             double rtol, std::int64_t maxit);

// ---- LinearOperator overloads (krylov.hpp:41-56 signatures).  The reference's own
// factories return unnamed lambdas a device cannot see into, so operators for the device
// are built with these factories instead: ordinary LinearOperators (they run unchanged in
// the reference's pcg_solve) whose callables are the named types below, recovered here
// with std::function::target<T>().  Any other callable -> ArgumentError.
struct SparseApply
{
  const SparseMatrix *A;
  std::vector<double> operator()(std::span<const double> v) const;
};
struct ChainApply
{
  const PreconditionerChain *chain;
  std::vector<double> operator()(std::span<const double> v) const;
};
struct IdentityApply
{
  std::vector<double> operator()(std::span<const double> v) const { return {v.begin(), v.end()}; }
};
LinearOperator sparse_operator(const SparseMatrix &A);                             // from_sparse (krylov.cpp:19-26)
LinearOperator chain_operator(const PreconditionerChain &chain, std::int64_t n);  // airga.cpp:176-177
LinearOperator identity_operator(std::int64_t n);                                  // identity (krylov.cpp:14-17)
SolveReport pcg_solve(Device &dev, const LinearOperator &A, const LinearOperator &P, std::span<const double> b,
                      double rtol, std::int64_t maxit);
BlockSolveResult block_solve(Device &dev, const LinearOperator &A, const LinearOperator &P, const DenseMatrix &B,
                             double rtol, std::int64_t maxit);

// Global Arnoldi + projection
QrResult thin_qr(Device &dev, const DenseMatrix &A, double rank_tol = 1e-12);                 // dense.hpp:69
ReducedSystem project_reduce(Device &dev, const SecondOrderSystem &sys, const OrthonormalBasis &basis); // airga.hpp:183
std::vector<double> arnoldi_deflate(Device &dev, DenseMatrix &X, std::span<const DenseMatrix> basis_blocks); // airga.hpp:176

} // namespace cuda

/// GPU-only choices on top of AirgaConfig.
struct CudaBackendOptions
{
  int device = 0;
  cuda::SpaiAlgorithm algorithm = cuda::SpaiAlgorithm::mr;
  int ls_pattern = 0; ///< MGPU_PATTERN_A / _A2, optionally | MGPU_LS_COLSCALE
  /// prepare() also solves sys.F for every prepared point in ONE batched kernel and keeps the
  /// results; solve(i, rhs) returns them when rhs is sys.F (bitwise), which is what
  /// zeroth_moments asks for right after prepare (airga.cpp:374-381).  Any other rhs is solved
  /// on demand, as before.
  bool speculative_solve = true;
  /// > 0: CG iteration budget in place of cg_maxit_factor * n (fixed-budget benchmarking; the
  /// factor is an integer multiple of n in AirgaConfig).
  std::int64_t maxit_override = 0;
  /// North-star subsystem 2: in update mode the chain is collapsed after every update into ONE
  /// factor, P <- Q P (device SpGEMM, mgpu_spgemm), instead of growing [Q_z, ..., Q_2, P]
  /// (spai.cpp:352-373).  Records still report the logical chain length.
  bool collapse = false;
};

/// The AirgaConfig fields the CG backend reads (airga.hpp:40-69).  Kept separately so that the
/// backend can be built without an AirgaConfig, whose default initial_points call into the
/// reference library (the C API in include/mor_cuda.h does this).
struct CudaSolveSettings
{
  AirgaConfig::Solver solver = AirgaConfig::Solver::cg_spai;
  double spai_tol = 0.01;
  std::int64_t spai_max_col_iters = 50;
  SpaiOptions::Mode spai_mode = SpaiOptions::Mode::sequential;
  double cg_rtol = 1e-10;
  std::int64_t cg_maxit_factor = 10;
  std::int64_t update_start_iteration = 3;
};
CudaSolveSettings settings_of(const AirgaConfig &cfg);

class CudaCgBackend final : public SolveBackend
{
public:
  CudaCgBackend(const AirgaConfig &cfg, const CudaBackendOptions &opt = {});
  CudaCgBackend(const CudaSolveSettings &cfg, const CudaBackendOptions &opt = {});
  ~CudaCgBackend() override;

  void prepare(const SecondOrderSystem &sys, const std::vector<double> &points, std::int64_t outer,
               std::vector<PrecondRecord> *records) override;
  BlockSolveResult solve(std::int64_t point_index, const DenseMatrix &rhs) override;
  bool provides_residuals() const override { return true; }

  /// Every prepared point against the same rhs block in one batched kernel
  /// (the reference solves point by point, airga.cpp:374-405).
  std::vector<BlockSolveResult> solve_all(const DenseMatrix &rhs);

  /// True when solve(point_index, rhs) would be served from prepare's batched solve.
  bool cached(std::int64_t point_index, const DenseMatrix &rhs) const;
  bool cached(std::int64_t point_index, const double *rhs, std::int64_t m) const; ///< rhs: n x m column-major
  /// Reads that result straight into caller buffers (each optional; n x m column-major) and
  /// marks it handed out -- the C API's path, one device-to-host copy per array.
  void take_cached(std::int64_t point_index, double *X, double *REC, double *TR, std::int64_t *iterations,
                   bool *all_converged);

private:
  struct State;
  std::unique_ptr<State> st_;
};

/// Shift sharding inside one process: one CudaCgBackend -- one context -- per
/// listed device; prepare deals the points out round-robin (point i to device i mod N) and prepares
/// every device concurrently (one host thread each), solve(i, rhs) runs on point i's device.  The
/// shifted systems are independent, so nothing crosses devices on the solve path.
class MultiDeviceCgBackend final : public SolveBackend
{
public:
  MultiDeviceCgBackend(const CudaSolveSettings &cfg, const CudaBackendOptions &opt, std::vector<int> devices);
  MultiDeviceCgBackend(const AirgaConfig &cfg, const CudaBackendOptions &opt, std::vector<int> devices);
  ~MultiDeviceCgBackend() override;

  void prepare(const SecondOrderSystem &sys, const std::vector<double> &points, std::int64_t outer,
               std::vector<PrecondRecord> *records) override;
  BlockSolveResult solve(std::int64_t point_index, const DenseMatrix &rhs) override;
  bool provides_residuals() const override { return true; }

  std::size_t devices() const { return parts_.size(); }
  CudaCgBackend &part(std::size_t d) { return *parts_[d]; }
  /// (device slot, local point index) of a global point index
  std::pair<std::size_t, std::int64_t> owner(std::int64_t point_index) const;

private:
  std::vector<std::unique_ptr<CudaCgBackend>> parts_;
};

std::unique_ptr<SolveBackend> make_cuda_backend(const AirgaConfig &cfg, const CudaBackendOptions &opt = {});

} // namespace mor
