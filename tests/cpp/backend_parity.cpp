// TEST DRIVER (GPU): the reference's CgBackend (make_backend, airga.cpp:358-365)
// against the drop-in CudaCgBackend on the same system and the same
// prepare / solve sequence.  Links the unmodified reference library (oracle/_ref)
// as the checker.  Prints one JSON object; exit code 0 iff every bar holds:
// solutions within 1e-8 relative, iterations within +-2, identical converged
// flags, identical PrecondRecord kind / chain length, identical exception
// class and payload.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "cuda_backend.hpp"
#include "mor/errors.hpp"
#include "mor/kernels.hpp"
#include "mor/model_io.hpp"

using namespace mor;

static double max_rel(const DenseMatrix &a, const DenseMatrix &b)
{
  double num = 0.0, den = 0.0;
  for (std::size_t k = 0; k < a.values.size(); ++k)
  {
    num = std::max(num, std::fabs(a.values[k] - b.values[k]));
    den = std::max(den, std::fabs(b.values[k]));
  }
  return den > 0 ? num / den : num;
}

static int failures = 0;
static double worst_x = 0.0;
static long worst_it = 0;
static int solves = 0;

static void compare_backends(const char *tag, const SecondOrderSystem &sys, AirgaConfig cfg,
                             const std::vector<std::vector<double>> &seq, cuda::SpaiAlgorithm alg)
{
  auto ref = make_backend(cfg);
  CudaBackendOptions opt;
  opt.algorithm = alg;
  CudaCgBackend gpu(cfg, opt);
  for (std::size_t z = 0; z < seq.size(); ++z)
  {
    std::vector<PrecondRecord> rr, gr;
    ref->prepare(sys, seq[z], static_cast<std::int64_t>(z + 1), &rr);
    gpu.prepare(sys, seq[z], static_cast<std::int64_t>(z + 1), &gr);
    if (rr.size() != gr.size())
      ++failures;
    for (std::size_t i = 0; i < rr.size() && i < gr.size(); ++i)
      if (rr[i].kind != gr[i].kind || rr[i].chain_length != gr[i].chain_length)
        ++failures;
    const auto all = gpu.solve_all(sys.F);
    for (std::size_t i = 0; i < seq[z].size(); ++i)
    {
      const BlockSolveResult a = ref->solve(static_cast<std::int64_t>(i), sys.F);
      const BlockSolveResult b = gpu.solve(static_cast<std::int64_t>(i), sys.F);
      const double dx = max_rel(b.X, a.X), dxa = max_rel(all[i].X, a.X);
      const long dit = std::labs(static_cast<long>(a.iterations[0] - b.iterations[0]));
      worst_x = std::max(worst_x, std::max(dx, dxa));
      worst_it = std::max(worst_it, dit);
      ++solves;
      if (!(dx <= 1e-8) || !(dxa <= 1e-8) || dit > 2 || a.all_converged != b.all_converged)
      {
        ++failures;
        std::fprintf(stderr, "%s outer %zu point %zu: dx %.3e dxa %.3e it %ld/%ld conv %d/%d\n", tag, z + 1, i, dx,
                     dxa, static_cast<long>(a.iterations[0]), static_cast<long>(b.iterations[0]), a.all_converged,
                     b.all_converged);
      }
    }
  }
}

int main()
{
  // canonical oracle variant: the scalar kernel table, whose
  // in-order gather_dot the device SpMV replays bit for bit
  kernels::force_variant(kernels::Variant::scalar);
  // T1: the reference's own model family (model_io.cpp:18-87), consistent mass
  ModelSpec spec;
  spec.n = 2000;
  spec.mass = ModelSpec::Mass::consistent;
  spec.stiffness_scale = 1.0;
  const SecondOrderSystem sys = beam_generate(spec);
  const std::vector<std::vector<double>> seq = {{1.0, 10.0, 100.0}, {2.0, 12.0, 90.0}, {3.0, 15.0, 80.0}};
  AirgaConfig cfg;
  cfg.spai_mode = SpaiOptions::Mode::frozen;
  cfg.update_start_iteration = 2;
  cfg.solver = AirgaConfig::Solver::cg_spai_update;
  compare_backends("cg_spai_update", sys, cfg, seq, cuda::SpaiAlgorithm::mr);
  cfg.solver = AirgaConfig::Solver::cg_spai;
  compare_backends("cg_spai", sys, cfg, seq, cuda::SpaiAlgorithm::mr);
  cfg.solver = AirgaConfig::Solver::cg_plain;
  compare_backends("cg_plain", sys, cfg, {{1.0, 50.0}}, cuda::SpaiAlgorithm::mr);
  // the reference default, spai_mode = sequential (d = P r over the built columns): heavy fill,
  // so a smaller system keeps the reference side to seconds
  ModelSpec small = spec;
  small.n = 400;
  const SecondOrderSystem sys_small = beam_generate(small);
  AirgaConfig seq_cfg;
  seq_cfg.spai_mode = SpaiOptions::Mode::sequential;
  seq_cfg.update_start_iteration = 2;
  seq_cfg.solver = AirgaConfig::Solver::cg_spai_update;
  compare_backends("cg_spai_update/sequential", sys_small, seq_cfg, seq, cuda::SpaiAlgorithm::mr);
  seq_cfg.solver = AirgaConfig::Solver::cg_spai;
  compare_backends("cg_spai/sequential", sys_small, seq_cfg, seq, cuda::SpaiAlgorithm::mr);

  cuda::Device dev(0);
  // free-function drop-ins: spai_build / spai_update / chain_apply / pcg_solve / block_solve
  SecondOrderSystem s2 = sys;
  const SparseMatrix A1 = shifted_operator(sys, 10.0), A2 = shifted_operator(sys, 11.0);
  SpaiOptions o;
  o.mode = SpaiOptions::Mode::frozen;
  const SpaiFactor Pr = spai_build(A1, o), Pg = cuda::spai_build(dev, A1, o);
  const SpaiFactor Qr = spai_update(A1, A2, o), Qg = cuda::spai_update(dev, A1, A2, o);
  double dspai = 0.0;
  for (std::size_t k = 0; k < Pr.matrix.values.size() && k < Pg.matrix.values.size(); ++k)
    dspai = std::max(dspai, std::fabs(Pr.matrix.values[k] - Pg.matrix.values[k]) / std::fabs(Pr.matrix.values[k]));
  for (std::size_t k = 0; k < Qr.matrix.values.size() && k < Qg.matrix.values.size(); ++k)
    dspai = std::max(dspai, std::fabs(Qr.matrix.values[k] - Qg.matrix.values[k]) / std::fabs(Qr.matrix.values[k]));
  if (Pr.matrix.col_idx != Pg.matrix.col_idx || Qr.matrix.col_idx != Qg.matrix.col_idx || !(dspai <= 1e-10))
    ++failures;
  PreconditionerChain chr, chg;
  chr.push_newest(Pr);
  chr.push_newest(Qr);
  chg.push_newest(Pg);
  chg.push_newest(Qg);
  std::vector<double> v(2000);
  for (int i = 0; i < 2000; ++i)
    v[static_cast<std::size_t>(i)] = std::sin(0.01 * i);
  const auto ca = chain_apply(chr, v), cb = cuda::chain_apply(dev, chr, v);
  double dchain = 0.0;
  for (std::size_t i = 0; i < ca.size(); ++i)
    dchain = std::max(dchain, std::fabs(ca[i] - cb[i]));
  if (dchain != 0.0) // same factors, in-order SpMV: bitwise
    ++failures;
  // LinearOperator overloads: the same named-functor operators through the reference's
  // pcg_solve (CPU) and the device; foreign callables are refused
  {
    const LinearOperator Aop = cuda::sparse_operator(A2), Pop = cuda::chain_operator(chr, 2000);
    const SolveReport lr = pcg_solve(Aop, Pop, v, 1e-10, 20000);
    const SolveReport lg = cuda::pcg_solve(dev, Aop, Pop, v, 1e-10, 20000);
    double dl = 0.0, nl = 0.0;
    for (std::size_t i = 0; i < lr.solution.size(); ++i)
    {
      dl = std::max(dl, std::fabs(lr.solution[i] - lg.solution[i]));
      nl = std::max(nl, std::fabs(lr.solution[i]));
    }
    if (!(dl <= 1e-8 * nl) || lr.converged != lg.converged)
      ++failures;
    bool refused = false;
    try { (void)cuda::pcg_solve(dev, LinearOperator::from_sparse(A2), Pop, v, 1e-10, 100); }
    catch (const ArgumentError &) { refused = true; }
    if (!refused)
      ++failures;
  }
  // chain_quality: the reference's probe stream, device SpMM + deterministic sums
  const double qr_ref = chain_quality(chr, A2, 8, 42), qr_gpu = cuda::chain_quality(dev, chr, A2, 8, 42);
  const double dq = std::fabs(qr_ref - qr_gpu) / std::fabs(qr_ref);
  if (!(dq <= 1e-12))
    ++failures;
  const auto P = LinearOperator{[&chr](std::span<const double> x) { return chain_apply(chr, x); }, 2000};
  const SolveReport ra = pcg_solve(LinearOperator::from_sparse(A2), P, v, 1e-10, 20000);
  const SolveReport rb = cuda::pcg_solve(dev, A2, chr, v, 1e-10, 20000);
  double dpcg = 0.0, nrm = 0.0;
  for (std::size_t i = 0; i < ra.solution.size(); ++i)
  {
    dpcg = std::max(dpcg, std::fabs(ra.solution[i] - rb.solution[i]));
    nrm = std::max(nrm, std::fabs(ra.solution[i]));
  }
  dpcg /= nrm;
  if (!(dpcg <= 1e-8) || std::labs(static_cast<long>(ra.iterations - rb.iterations)) > 2 ||
      ra.converged != rb.converged || ra.relres_history.size() != static_cast<std::size_t>(ra.iterations) ||
      rb.relres_history.size() != static_cast<std::size_t>(rb.iterations))
    ++failures;
  // global Arnoldi + projection: thin_qr / arnoldi_deflate / project_reduce on solve blocks
  DenseMatrix Vt(2000, 6);
  for (int c = 0; c < 6; ++c)
  {
    const SparseMatrix Ac = shifted_operator(sys, 5.0 + 20.0 * c);
    std::vector<double> rhs(2000, 0.0);
    rhs[static_cast<std::size_t>(c * 300)] = 1.0;
    const SolveReport sr = pcg_solve(LinearOperator::from_sparse(Ac), LinearOperator::identity(2000), rhs, 1e-12, 20000);
    std::copy(sr.solution.begin(), sr.solution.end(), Vt.col(c));
  }
  const QrResult qa = thin_qr(Vt), qb = cuda::thin_qr(dev, Vt);
  auto rel_dense = [](const DenseMatrix &a, const DenseMatrix &b) {
    double num = 0.0, den = 0.0;
    for (std::size_t k = 0; k < a.values.size(); ++k)
    {
      num += (a.values[k] - b.values[k]) * (a.values[k] - b.values[k]);
      den += b.values[k] * b.values[k];
    }
    return std::sqrt(num / (den > 0.0 ? den : 1.0));
  };
  double dproj = std::max(rel_dense(qb.Q, qa.Q), rel_dense(qb.R, qa.R));
  if (qa.rank != qb.rank)
    ++failures;
  DenseMatrix Xd(2000, 6);
  for (std::size_t k = 0; k < Xd.values.size(); ++k)
    Xd.values[k] = std::sin(0.001 * static_cast<double>(k)) + 0.5 * std::cos(0.37 * static_cast<double>(k));
  DenseMatrix Xg = Xd;
  std::vector<DenseMatrix> blocks = {qa.Q};
  const auto ga = arnoldi_deflate(Xd, blocks), gb = cuda::arnoldi_deflate(dev, Xg, blocks);
  dproj = std::max({dproj, rel_dense(Xg, Xd), std::fabs(ga[0] - gb[0]) / std::fabs(ga[0])});
  SecondOrderSystem sysp = sys;
  sysp.F = DenseMatrix(2000, 1);
  sysp.F.at(0, 0) = 1.0;
  sysp.Cp = DenseMatrix(1, 2000);
  sysp.Cv = DenseMatrix(1, 2000);
  sysp.Cp.at(0, 1999) = 1.0;
  OrthonormalBasis ob;
  ob.assembled = qa.Q;
  const ReducedSystem ra_ = project_reduce(sysp, ob), rb_ = cuda::project_reduce(dev, sysp, ob);
  dproj = std::max({dproj, rel_dense(rb_.Mh, ra_.Mh), rel_dense(rb_.Dh, ra_.Dh), rel_dense(rb_.Kh, ra_.Kh),
                    rel_dense(rb_.Fh, ra_.Fh), rel_dense(rb_.Cph, ra_.Cph)});
  if (!(dproj <= 1e-12))
    ++failures;
  // exception parity: MR-SPAI stagnation on the BASELINE Hermite-like stiff case, CG breakdown
  long stag_ref = -1, stag_gpu = -1, bd_ref = -1, bd_gpu = -1;
  ModelSpec stiff = spec;
  stiff.stiffness_scale = 100.0;
  const SparseMatrix As = shifted_operator(beam_generate(stiff), 1.0);
  try { (void)spai_build(As, o); } catch (const StagnationError &e) { stag_ref = e.column; }
  try { (void)cuda::spai_build(dev, As, o); } catch (const StagnationError &e) { stag_gpu = e.column; }
  const SparseMatrix Ad = SparseMatrix::from_triplets(3, 3, {{0, 0, 1.0}, {1, 1, -1.0}, {2, 2, 2.0}});
  const std::vector<double> bd = {1.0, 1.0, 0.0};
  try { (void)pcg_solve(LinearOperator::from_sparse(Ad), LinearOperator::identity(3), bd, 1e-10, 30); }
  catch (const BreakdownError &e) { bd_ref = e.iteration; }
  try { (void)cuda::pcg_solve(dev, Ad, PreconditionerChain{}, bd, 1e-10, 30); }
  catch (const BreakdownError &e) { bd_gpu = e.iteration; }
  if (stag_ref != stag_gpu || stag_ref < 0 || bd_ref != bd_gpu || bd_ref < 0)
    ++failures;
  std::printf("{\"solves\": %d, \"max_rel_x\": %.3e, \"max_iter_diff\": %ld, \"spai_rel\": %.3e, "
              "\"chain_apply_abs\": %.3e, \"chain_quality_rel\": %.3e, \"projection_rel\": %.3e, \"pcg_rel\": %.3e, \"stagnation_col\": [%ld, %ld], "
              "\"breakdown_it\": [%ld, %ld], \"failures\": %d}\n",
              solves, worst_x, worst_it, dspai, dchain, dq, dproj, dpcg, stag_ref, stag_gpu, bd_ref, bd_gpu, failures);
  return failures == 0 ? 0 : 1;
}
