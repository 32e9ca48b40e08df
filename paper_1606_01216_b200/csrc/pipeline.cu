// The hot path in one call: assembly of the l shifted operators (system.cpp:64-68), their
// LS-SPAI factors, and the batched PCG solve (krylov.cpp:141-174) -- what CgBackend::prepare
// followed by a solve of every point does (airga.cpp:108-181), without host round trips
// between the stages beyond the size and status reads each stage needs.  The operators and
// factors are temporaries, released stream-ordered before returning.
#include <vector>

#include "internal.cuh"

using namespace mgpu;

extern "C" {

int mgpu_shifted_solve(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int l,
                       const double *shifts, int pattern, const double *B, int64_t m, int64_t ldb_point, double rtol,
                       int64_t maxit, mgpu_memkind where, mgpu_cg_out *out, double *phase_ms)
{
  if (ctx == nullptr)
    return MGPU_ERR_ARG;
  if (M == nullptr || D == nullptr || K == nullptr || shifts == nullptr || l < 1 ||
      (pattern != -1 && (pattern & ~MGPU_LS_COLSCALE) != MGPU_PATTERN_A &&
       (pattern & ~MGPU_LS_COLSCALE) != MGPU_PATTERN_A2))
    return guard(ctx, [&] { MG_ARG(false, "shifted_solve: bad argument"); });
  cudaStream_t s = ctx->stream;
  cudaEvent_t *ev = ctx->phase_ev; // created once per context
  if (phase_ms)
    for (int k = 0; k < 4; ++k)
      if (!ev[k] && cudaEventCreate(&ev[k]) != cudaSuccess)
        return guard(ctx, [&] { MG_CUDA(cudaGetLastError()); });
  auto rec = [&](int k) {
    if (phase_ms)
      cudaEventRecord(ev[k], s);
  };
  std::vector<mgpu_csr *> ops(static_cast<size_t>(l), nullptr), facs;
  auto release = [&]() {
    for (auto *f : facs)
      mgpu_csr_free(f);
    for (auto *o : ops)
      mgpu_csr_free(o);
  };
  rec(0);
  host_mark("shifted_solve: enter");
  int st = mgpu_shifted_operators(ctx, M, D, K, l, shifts, ops.data());
  host_mark("shifted_solve: operators queued");
  rec(1);
  if (st == MGPU_OK && pattern >= 0)
  {
    facs.assign(static_cast<size_t>(l), nullptr);
    st = mgpu_spai_ls_batched(ctx, l, ops.data(), nullptr, pattern, facs.data());
    if (st != MGPU_OK)
      facs.clear(); // nothing was handed out
  }
  host_mark("shifted_solve: spai returned");
  rec(2);
  if (st == MGPU_OK)
    st = mgpu_cg_solve(ctx, l, ops.data(), pattern >= 0 ? 1 : 0, pattern >= 0 ? facs.data() : nullptr, M->nrows, m, B,
                       ldb_point, rtol, maxit, where, out);
  rec(3);
  if (phase_ms)
  {
    cudaEventSynchronize(ev[3]);
    float t = 0.f;
    for (int k = 0; k < 3; ++k)
      phase_ms[k] = cudaEventElapsedTime(&t, ev[k], ev[k + 1]) == cudaSuccess ? t : -1.0;
  }
  release();
  return st;
}

} // extern "C"
