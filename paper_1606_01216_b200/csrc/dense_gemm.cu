// Hand-written FP64 GEMM for the projection / thin-QR path: replaces the
// cuBLAS DGEMM the compact-WY thin_qr and project_reduce used.
//
//   C (M x N) = alpha op(A) op(B) + beta C, column-major, op(A) = A or A^T, op(B) = B.
//
// The shapes on this path are tall and skinny: either the inner dimension K is the basis length
// (V^T C, V^T F, C V: K up to 1e7 rows, M, N <= a few hundred) or M is (the rank-32 compact-WY
// update C -= V W).  One kernel covers both: 64 x 64 output tiles, 256 threads with 4 x 4
// accumulators each, K staged through shared memory 16 at a time; when the tile grid alone cannot
// fill the 148 SMs the K range is split across blocks, each block writes its partial tile and a
// second kernel sums the partials in split order (deterministic, no atomics) and applies
// alpha / beta.  FP64 DFMA throughout (the tensor-core FP64 path is not used on this chip).
#include <algorithm>

#include "internal.cuh"

namespace mgpu
{
namespace
{

constexpr int kTM = 64, kTN = 64, kTK = 16, kGT = 256;

template <bool TA>
__global__ void __launch_bounds__(kGT) gemm_tile(int64_t M, int64_t N, int64_t K, int64_t kchunk, double alpha,
                                                 const double *__restrict__ A, int64_t lda,
                                                 const double *__restrict__ B, int64_t ldb, double beta,
                                                 double *__restrict__ C, int64_t ldc, double *__restrict__ part)
{
  __shared__ double As[kTK][kTM + 1];
  __shared__ double Bs[kTK][kTN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4; // 16 x 16 threads, 4 x 4 outputs each
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTM, j0 = static_cast<int64_t>(blockIdx.y) * kTN;
  const int64_t k0 = static_cast<int64_t>(blockIdx.z) * kchunk, k1 = K < k0 + kchunk ? K : k0 + kchunk;
  double acc[4][4] = {};
  for (int64_t kb = k0; kb < k1; kb += kTK)
  {
    // A tile: op(A)(i0 + i, kb + k), i < 64, k < 16 (1024 values, 4 per thread)
    for (int t = threadIdx.x; t < kTM * kTK; t += kGT)
    {
      int i, k;
      if (TA) // A is K x M: consecutive threads along k
      {
        k = t % kTK;
        i = t / kTK;
      }
      else // A is M x K: consecutive threads along i
      {
        i = t % kTM;
        k = t / kTM;
      }
      const int64_t gi = i0 + i, gk = kb + k;
      double v = 0.0;
      if (gi < M && gk < k1)
        v = TA ? A[gi * lda + gk] : A[gk * lda + gi];
      As[k][i] = v;
    }
    // B tile: B(kb + k, j0 + j) (B is K x N, consecutive threads along k)
    for (int t = threadIdx.x; t < kTN * kTK; t += kGT)
    {
      const int k = t % kTK, j = t / kTK;
      const int64_t gk = kb + k, gj = j0 + j;
      Bs[k][j] = (gk < k1 && gj < N) ? B[gj * ldb + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTK; ++k)
    {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
      {
        a[u] = As[k][ty + 16 * u];
        b[u] = Bs[k][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
    {
      const int64_t gi = i0 + ty + 16 * u, gj = j0 + tx + 16 * v;
      if (gi >= M || gj >= N)
        continue;
      if (part) // split K: raw partial, summed by gemm_reduce
        part[(static_cast<int64_t>(blockIdx.z) * N + gj) * M + gi] = acc[u][v];
      else
        C[gj * ldc + gi] = beta == 0.0 ? alpha * acc[u][v] : fma(alpha, acc[u][v], beta * C[gj * ldc + gi]);
    }
}

__global__ void gemm_reduce(int64_t M, int64_t N, int splits, double alpha, const double *__restrict__ part,
                            double beta, double *__restrict__ C, int64_t ldc)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= M * N)
    return;
  const int64_t j = t / M, i = t - j * M;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) // split order: deterministic
    s += part[static_cast<int64_t>(z) * M * N + t];
  C[j * ldc + i] = beta == 0.0 ? alpha * s : fma(alpha, s, beta * C[j * ldc + i]);
}

} // namespace

void gemm(mgpu_ctx *ctx, bool transA, int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
          const double *B, int64_t ldb, double beta, double *C, int64_t ldc)
{
  if (M == 0 || N == 0)
    return;
  cudaStream_t s = ctx->stream;
  const int64_t tm = (M + kTM - 1) / kTM, tn = (N + kTN - 1) / kTN;
  const int64_t want = 2 * static_cast<int64_t>(ctx->num_sms);
  int64_t splits = 1;
  if (tm * tn < want && K > 4 * kTK)
  {
    splits = std::min<int64_t>((want + tm * tn - 1) / (tm * tn), (K + 255) / 256);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, (int64_t{16} << 20) / (M * N))); // <= 128 MB of partials
    splits = std::max<int64_t>(splits, 1);
  }
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + kTK - 1) / kTK * kTK;
  splits = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  if (K == 0)
  {
    kchunk = 0;
    splits = 1;
  }
  DBuf part(splits > 1 ? sizeof(double) * static_cast<size_t>(splits * M * N) : 0, s);
  const dim3 grid(static_cast<unsigned>(tm), static_cast<unsigned>(tn), static_cast<unsigned>(splits));
  if (transA)
    gemm_tile<true><<<grid, kGT, 0, s>>>(M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc,
                                         splits > 1 ? part.as<double>() : nullptr);
  else
    gemm_tile<false><<<grid, kGT, 0, s>>>(M, N, K, kchunk, alpha, A, lda, B, ldb, beta, C, ldc,
                                          splits > 1 ? part.as<double>() : nullptr);
  check_launch(ctx, "gemm_tile");
  if (splits > 1)
  {
    gemm_reduce<<<blocks_for(M * N), kThreads, 0, s>>>(M, N, static_cast<int>(splits), alpha, part.as<double>(), beta,
                                                       C, ldc);
    check_launch(ctx, "gemm_reduce");
  }
}

} // namespace mgpu
