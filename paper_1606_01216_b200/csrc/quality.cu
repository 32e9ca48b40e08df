// chain_quality (spai.cpp:375-409): stochastic estimate of ||I - K P_chain||_F
// from `samples` unit-norm Gaussian probes, sqrt((n / samples) sum_k ||(I - K P) g_k||^2).
//
// The probes are the reference's own stream: std::mt19937_64(seed) driving
// std::normal_distribution<double>(0, 1), drawn in the same order (sample-major).
// They are generated on the host with the same standard library -- an input,
// like a right-hand side -- and everything after that runs on the device over
// all probes at once:
//   ||g_k||^2 per probe (deterministic tree), g_k /= ||g_k||,
//   the chain (oldest factor first, spai.cpp:368) and K as one SpMM over the
//   n x samples block (each row in CSR order, no FMA: spmv's gather_dot order),
//   e = g - K P g and sum e^2 (deterministic tree; the reference sums serially).
#include <cmath>
#include <cstdint>
#include <random>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace mgpu
{
namespace
{

// y[:, k] = A x[:, k] for k < S (column-major n x S blocks); one thread per (row, probe).
__global__ void spmm_cols(int64_t n, int S, DCsr A, const double *__restrict__ x, double *__restrict__ y)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * S)
    return;
  const int k = static_cast<int>(t / n);
  const int64_t i = t - static_cast<int64_t>(k) * n;
  const double *xk = x + static_cast<int64_t>(k) * n;
  double acc = 0.0;
  for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q)
    acc = __dadd_rn(acc, __dmul_rn(A.v[q], xk[A.ci[q]]));
  y[t] = acc;
}

__global__ void square_cols(int64_t count, const double *__restrict__ g, double *__restrict__ out)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count)
    out[t] = __dmul_rn(g[t], g[t]);
}

__global__ void scale_cols(int64_t n, int S, const double *__restrict__ nrm_sq, double *__restrict__ g)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * S)
    return;
  g[t] = __ddiv_rn(g[t], sqrt(nrm_sq[t / n]));
}

__global__ void residual_sq(int64_t count, const double *__restrict__ g, const double *__restrict__ kpg,
                            double *__restrict__ out)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= count)
    return;
  const double e = __dsub_rn(g[t], kpg[t]);
  out[t] = __dmul_rn(e, e);
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_chain_quality(mgpu_ctx *ctx, int z, const mgpu_csr *const *factors, const mgpu_csr *K, int64_t samples,
                       uint64_t seed, double *out)
{
  return guard(ctx, [&] {
    MG_ARG(K && out && z >= 0 && (z == 0 || factors), "chain_quality: null argument");
    MG_ARG(samples >= 1, "chain_quality: samples must be >= 1"); // spai.cpp:378-381
    const int64_t n = K->nrows;
    for (int f = 0; f < z; ++f)
      MG_ARG(factors[f] && factors[f]->nrows == n && factors[f]->ncols == n, "chain_quality: dimension mismatch");
    MG_ARG(samples <= INT32_MAX, "chain_quality: too many samples");
    const int S = static_cast<int>(samples);
    cudaStream_t s = ctx->stream;
    // ---- probes: the reference's generator, same draw order (spai.cpp:383-393)
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    const int64_t total = n * S;
    std::vector<double> host(static_cast<size_t>(total > 0 ? total : 1));
    for (int64_t t = 0; t < total; ++t)
      host[static_cast<size_t>(t)] = gauss(rng);
    const size_t bytes = sizeof(double) * static_cast<size_t>(total > 0 ? total : 1);
    DBuf g(bytes, s), a(bytes, s), b(bytes, s), nrm(sizeof(double) * S, s), acc(sizeof(double), s);
    MG_CUDA(cudaMemcpyAsync(g.ptr, host.data(), sizeof(double) * total, cudaMemcpyHostToDevice, s));
    if (n > 0)
    {
      // ---- g_k /= ||g_k||
      square_cols<<<blocks_for(total), kThreads, 0, s>>>(total, g.as<double>(), a.as<double>());
      check_launch(ctx, "square_cols");
      for (int k = 0; k < S; ++k)
        det_sum(ctx, a.as<double>() + static_cast<int64_t>(k) * n, n, nrm.as<double>() + k);
      scale_cols<<<blocks_for(total), kThreads, 0, s>>>(n, S, nrm.as<double>(), g.as<double>());
      check_launch(ctx, "scale_cols");
      // ---- P g (oldest factor first), then K P g
      const double *src = g.as<double>();
      double *dst = a.as<double>(), *spare = b.as<double>();
      if (z == 0)
      {
        MG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * total, cudaMemcpyDeviceToDevice, s));
        src = dst;
        std::swap(dst, spare);
      }
      for (int f = z - 1; f >= 0; --f)
      {
        spmm_cols<<<blocks_for(total), kThreads, 0, s>>>(n, S, factors[f]->view(), src, dst);
        check_launch(ctx, "spmm_cols");
        src = dst;
        std::swap(dst, spare);
      }
      spmm_cols<<<blocks_for(total), kThreads, 0, s>>>(n, S, K->view(), src, dst);
      check_launch(ctx, "spmm_cols");
      // ---- sum (g - K P g)^2
      double *sq = dst == a.as<double>() ? b.as<double>() : a.as<double>();
      residual_sq<<<blocks_for(total), kThreads, 0, s>>>(total, g.as<double>(), dst, sq);
      check_launch(ctx, "residual_sq");
      det_sum(ctx, sq, total, acc.as<double>());
    }
    else
      MG_CUDA(cudaMemsetAsync(acc.ptr, 0, sizeof(double), s));
    double h = 0.0;
    MG_CUDA(cudaMemcpyAsync(&h, acc.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    *out = std::sqrt(static_cast<double>(n) / static_cast<double>(samples) * h); // spai.cpp:408
  });
}

} // extern "C"
