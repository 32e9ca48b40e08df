// K-spgemm: C = A * B for device CSR (north star subsystem 2: collapse a
// preconditioner chain [Q_z, ..., P] into one factor, cf. chain_apply,
// spai.cpp:361-373, which instead applies one SpMV per factor).
//
// One thread per row of A.  Pass 1 bounds each row of C by sum_k |B row k| (no merging); the
// bounds are scanned into a scratch layout, pass 2 accumulates the row into its scratch slice as a
// sorted list (C_ic = sum_k A_ik B_kc with k ascending, products added as they come, no FMA) and
// counts its nonzeros, pass 3 compacts the nonzeros into C.  Exact zeros are dropped like every
// reference CSR (sparse.hpp:15).  No row-length cap: the update chains of the AIRGA sequence
// collapse into factors whose rows widen with every product.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace mgpu
{
namespace
{

__global__ void spgemm_bound(int64_t n, DCsr A, DCsr B, int64_t *bound)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int64_t b = 0;
  for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q)
    b += B.rp[A.ci[q] + 1] - B.rp[A.ci[q]];
  bound[i + 1] = b;
  if (i == 0)
    bound[0] = 0;
}

// Row i of A*B into cols/vals (scratch slice); returns the number of distinct columns and sets
// *nz to the number of nonzero values among them.
__global__ void spgemm_rows(int64_t n, DCsr A, DCsr B, const int64_t *__restrict__ off, int32_t *__restrict__ cols,
                            double *__restrict__ vals, int64_t *__restrict__ uniq, int64_t *__restrict__ nzrow)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int32_t *cl = cols + off[i];
  double *vl = vals + off[i];
  int cnt = 0;
  for (int64_t q = A.rp[i]; q < A.rp[i + 1]; ++q)
  {
    const int32_t k = A.ci[q];
    const double a = A.v[q];
    for (int64_t t = B.rp[k]; t < B.rp[k + 1]; ++t)
    {
      const int32_t c = B.ci[t];
      const double prod = __dmul_rn(a, B.v[t]);
      int lo = 0, hi = cnt; // position of c in the sorted list
      while (lo < hi)
      {
        const int mid = (lo + hi) >> 1;
        if (cl[mid] < c)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo < cnt && cl[lo] == c)
      {
        vl[lo] = __dadd_rn(vl[lo], prod);
        continue;
      }
      for (int u = cnt; u > lo; --u)
      {
        cl[u] = cl[u - 1];
        vl[u] = vl[u - 1];
      }
      cl[lo] = c;
      vl[lo] = prod;
      ++cnt;
    }
  }
  int64_t nz = 0;
  for (int u = 0; u < cnt; ++u)
    nz += vl[u] != 0.0;
  uniq[i] = cnt;
  nzrow[i + 1] = nz;
  if (i == 0)
    nzrow[0] = 0;
}

__global__ void spgemm_compact(int64_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ cols,
                               const double *__restrict__ vals, const int64_t *__restrict__ uniq,
                               const int64_t *__restrict__ rp, int32_t *__restrict__ ci, double *__restrict__ v)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int64_t o = rp[i];
  for (int64_t u = 0; u < uniq[i]; ++u)
  {
    const double x = vals[off[i] + u];
    if (x != 0.0)
    {
      ci[o] = cols[off[i] + u];
      v[o] = x;
      ++o;
    }
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
    auto scan = [&](int64_t *a) { // inclusive scan of a[1 .. n] in place
      size_t tmp = 0;
      MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, a + 1, a + 1, n, s));
      DBuf t(tmp, s);
      MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, a + 1, a + 1, n, s));
      count_launch(ctx);
    };
    DBuf off(sizeof(int64_t) * (n + 1), s), uniq(sizeof(int64_t) * (n > 0 ? n : 1), s);
    MG_CUDA(cudaMemsetAsync(off.ptr, 0, sizeof(int64_t), s));
    int64_t total = 0;
    if (n > 0)
    {
      spgemm_bound<<<blocks_for(n), kThreads, 0, s>>>(n, A->view(), B->view(), off.as<int64_t>());
      check_launch(ctx, "spgemm_bound");
      scan(off.as<int64_t>());
      MG_CUDA(cudaMemcpyAsync(&total, off.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
    }
    DBuf scols(sizeof(int32_t) * (total > 0 ? total : 1), s), svals(sizeof(double) * (total > 0 ? total : 1), s);
    mgpu_csr *out = new mgpu_csr;
    out->ctx = ctx;
    out->nrows = n;
    out->ncols = B->ncols;
    try
    {
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->row_ptr), sizeof(int64_t) * (n + 1), s));
      MG_CUDA(cudaMemsetAsync(out->row_ptr, 0, sizeof(int64_t), s));
      int64_t nnz = 0;
      if (n > 0)
      {
        spgemm_rows<<<blocks_for(n), kThreads, 0, s>>>(n, A->view(), B->view(), off.as<int64_t>(), scols.as<int32_t>(),
                                                       svals.as<double>(), uniq.as<int64_t>(), out->row_ptr);
        check_launch(ctx, "spgemm_rows");
        scan(out->row_ptr);
        MG_CUDA(cudaMemcpyAsync(&nnz, out->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        MG_CUDA(cudaStreamSynchronize(s));
      }
      out->nnz = nnz;
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&out->values), sizeof(double) * (nnz > 0 ? nnz : 1), s));
      if (n > 0)
      {
        spgemm_compact<<<blocks_for(n), kThreads, 0, s>>>(n, off.as<int64_t>(), scols.as<int32_t>(), svals.as<double>(),
                                                          uniq.as<int64_t>(), out->row_ptr, out->col_idx, out->values);
        check_launch(ctx, "spgemm_compact");
      }
    }
    catch (...)
    {
      mgpu_csr_free(out);
      throw;
    }
    if (A->bw >= 0 && B->bw >= 0)
      out->bw = A->bw + B->bw;
    *C = out;
  });
}
