// K-spgemm: C = A * B for device CSR (north star subsystem 2: collapse a
// preconditioner chain [Q_z, ..., P] into one factor, cf. chain_apply,
// spai.cpp:361-373, which instead applies one SpMV per factor).
//
// One thread per row of A; the row of C is accumulated in a small sorted
// register/local buffer (SPAI factors of banded operators have short rows),
// C_ic = sum_k A_ik B_kc with k ascending and no FMA; exact zeros are dropped
// like every reference CSR (sparse.hpp:15).  Two passes: count, then fill.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace mgpu
{
namespace
{

constexpr int kRowCap = 96;

__device__ int product_row(int64_t i, DCsr A, DCsr B, int32_t *cols, double *vals)
{
  int cnt = 0;
  for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q)
  {
    const int32_t k = A.ci[q];
    const double a = A.v[q];
    for (int64_t t = B.rp[k]; t < B.rp[k + 1]; ++t)
    {
      const int32_t c = B.ci[t];
      const double prod = __dmul_rn(a, B.v[t]);
      int lo = 0, hi = cnt; // position of c in the sorted buffer
      while (lo < hi)
      {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < c)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < cnt && cols[lo] == c)
      {
        vals[lo] = __dadd_rn(vals[lo], prod);
        continue;
      }
      if (cnt == kRowCap)
        return -1;
      for (int u = cnt; u > lo; --u)
      {
        cols[u] = cols[u - 1];
        vals[u] = vals[u - 1];
      }
      cols[lo] = c;
      vals[lo] = prod;
      ++cnt;
    }
  }
  return cnt;
}

__global__ void spgemm_count(int64_t n, DCsr A, DCsr B, int64_t *rp, int *overflow)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int32_t cols[kRowCap];
  double vals[kRowCap];
  const int c = product_row(i, A, B, cols, vals);
  int64_t nz = 0;
  if (c < 0)
    atomicOr(overflow, 1);
  for (int u = 0; u < c; ++u)
    nz += vals[u] != 0.0;
  rp[i + 1] = nz;
  if (i == 0)
    rp[0] = 0;
}

__global__ void spgemm_fill(int64_t n, DCsr A, DCsr B, const int64_t *rp, int32_t *ci, double *v)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int32_t cols[kRowCap];
  double vals[kRowCap];
  const int c = product_row(i, A, B, cols, vals);
  int64_t o = rp[i];
  for (int u = 0; u < c; ++u)
    if (vals[u] != 0.0)
    {
      ci[o] = cols[u];
      v[o] = vals[u];
      ++o;
    }
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" int mgpu_spgemm(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, mgpu_csr **C)
{
  return guard(ctx, [&] {
    MG_ARG(A && B && C, "spgemm: null argument");
    MG_ARG(A->ncols == B->nrows, "spgemm: shape mismatch");
    const int64_t n = A->nrows;
    cudaStream_t s = ctx->stream;
    mgpu_csr *out = new mgpu_csr;
    out->ctx = ctx;
    out->nrows = n;
    out->ncols = B->ncols;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->row_ptr), sizeof(int64_t) * (n + 1), s));
    MG_CUDA(cudaMemsetAsync(out->row_ptr, 0, sizeof(int64_t), s));
    DBuf ovf(sizeof(int), s);
    MG_CUDA(cudaMemsetAsync(ovf.ptr, 0, sizeof(int), s));
    if (n > 0)
    {
      spgemm_count<<<blocks_for(n), kThreads, 0, s>>>(n, A->view(), B->view(), out->row_ptr, ovf.as<int>());
      check_launch(ctx, "spgemm_count");
      size_t tmp = 0;
      MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, out->row_ptr + 1, out->row_ptr + 1, n, s));
      DBuf t(tmp, s);
      MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, out->row_ptr + 1, out->row_ptr + 1, n, s));
      count_launch(ctx);
    }
    int h_ovf = 0;
    int64_t nnz = 0;
    MG_CUDA(cudaMemcpyAsync(&h_ovf, ovf.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&nnz, out->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (h_ovf)
    {
      mgpu_csr_free(out);
      throw Error(MGPU_ERR_UNSUPPORTED, "spgemm: a product row has more than 96 entries");
    }
    out->nnz = nnz;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->values), sizeof(double) * (nnz > 0 ? nnz : 1), s));
    if (n > 0)
    {
      spgemm_fill<<<blocks_for(n), kThreads, 0, s>>>(n, A->view(), B->view(), out->row_ptr, out->col_idx, out->values);
      check_launch(ctx, "spgemm_fill");
    }
    if (A->bw >= 0 && B->bw >= 0)
      out->bw = A->bw + B->bw;
    *C = out;
  });
}
