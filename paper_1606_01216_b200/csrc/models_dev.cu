// Device-side beam generation: the BASELINE Hermite
// cantilever (models.cpp:mgpu_model_hermite, n = 2 ne) assembled directly in
// HBM.  The reference path builds ~16 ne triplets and sorts them through
// from_triplets (sparse.cpp:15-60; 29 s at n = 1e7).  Here the structure is
// analytic: dof i belongs to node v = i / 2 + 1, which only elements v - 1
// (as its right node) and v (as its left node) touch, so row i has at most
// the 6 columns 2v-4 .. 2v+1 and each entry is
//     (0 + c_{v-1}) + c_v        in element order (the stable sort's order),
// with exact-zero sums dropped -- the same values, bit for bit, as the host
// generator.  D = alpha M + beta K then goes through the device sp_add_scaled
// (bitwise to sparse.cpp:167-218).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace mgpu
{
namespace
{

struct BeamCoef
{
  double k[4][4]; // kc * kcoef[a][b] factors (kc applied on the device, like the host's kc * kcoef)
  double m[4][4];
  double kc, mc;
};

// value of (row i, column col) in K (which = 0) or M (which = 1), NaN-free; `hit` = any contribution
__device__ __forceinline__ double beam_entry(const BeamCoef &c, int which, int64_t ne, int64_t i, int64_t col,
                                             bool &hit)
{
  const int64_t v = i / 2 + 1;
  const int ai = static_cast<int>(i % 2);
  const double f = which == 0 ? c.kc : c.mc;
  double s = 0.0;
  hit = false;
  // element v - 1: dofs {2v-4, 2v-3, 2v-2, 2v-1}, node v is its right node (local row 2 + ai)
  {
    const int64_t b = col - (2 * v - 4);
    if (b >= 0 && b < 4 && col >= 0)
    {
      const double t = __dmul_rn(f, which == 0 ? c.k[2 + ai][b] : c.m[2 + ai][b]);
      s = __dadd_rn(s, t);
      hit = true;
    }
  }
  // element v (if it exists): dofs {2v-2, 2v-1, 2v, 2v+1}, node v is its left node (local row ai)
  if (v < ne)
  {
    const int64_t b = col - (2 * v - 2);
    if (b >= 0 && b < 4)
    {
      const double t = __dmul_rn(f, which == 0 ? c.k[ai][b] : c.m[ai][b]);
      s = __dadd_rn(s, t);
      hit = true;
    }
  }
  return s;
}

// pass 0: counts (rp[i + 1]); pass 1: fill at rp[i]
template <bool kFill>
__global__ void beam_rows(int64_t ne, int which, BeamCoef c, int64_t *__restrict__ rp, int32_t *__restrict__ ci,
                          double *__restrict__ v)
{
  const int64_t n = 2 * ne;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  const int64_t node = i / 2 + 1;
  int64_t o = kFill ? rp[i] : 0;
  for (int64_t col = 2 * node - 4; col <= 2 * node + 1; ++col)
  {
    if (col < 0 || col >= n)
      continue;
    bool hit;
    const double s = beam_entry(c, which, ne, i, col, hit);
    if (!hit || s == 0.0) // exact zeros are not stored (sparse.cpp:43-50)
      continue;
    if (kFill)
    {
      ci[o] = static_cast<int32_t>(col);
      v[o] = s;
    }
    ++o;
  }
  if (!kFill)
  {
    rp[i + 1] = o;
    if (i == 0)
      rp[0] = 0;
  }
}

mgpu_csr *beam_matrix(mgpu_ctx *ctx, int64_t ne, int which, const BeamCoef &c)
{
  const int64_t n = 2 * ne;
  cudaStream_t s = ctx->stream;
  mgpu_csr *A = new mgpu_csr;
  A->ctx = ctx;
  A->nrows = n;
  A->ncols = n;
  try
  {
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&A->row_ptr), sizeof(int64_t) * (n + 1), s));
    beam_rows<false><<<blocks_for(n), kThreads, 0, s>>>(ne, which, c, A->row_ptr, nullptr, nullptr);
    check_launch(ctx, "beam_rows<count>");
    size_t tmp = 0;
    MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, A->row_ptr + 1, A->row_ptr + 1, n, s));
    DBuf t(tmp, s);
    MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, A->row_ptr + 1, A->row_ptr + 1, n, s));
    count_launch(ctx);
    int64_t nnz = 0;
    MG_CUDA(cudaMemcpyAsync(&nnz, A->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    A->nnz = nnz;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&A->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&A->values), sizeof(double) * (nnz > 0 ? nnz : 1), s));
    beam_rows<true><<<blocks_for(n), kThreads, 0, s>>>(ne, which, c, A->row_ptr, A->col_idx, A->values);
    check_launch(ctx, "beam_rows<fill>");
    A->bw = 3;     // |i - j| <= 3 by construction
    A->maxrow = 6; // at most 6 candidates per row
  }
  catch (...)
  {
    mgpu_csr_free(A);
    throw;
  }
  return A;
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_model_hermite_device(mgpu_ctx *ctx, int64_t ne, double E, double I, double rho, double area, double L,
                              double alpha, double beta, mgpu_csr **M, mgpu_csr **D, mgpu_csr **K)
{
  return guard(ctx, [&] {
    MG_ARG(M && D && K, "hermite model: null argument");
    MG_ARG(ne >= 1 && ne <= (static_cast<int64_t>(INT32_MAX) - 1) / 2, "hermite model: bad arguments");
    // the host generator's scalar arithmetic, verbatim (models.cpp)
    const double h = L / static_cast<double>(ne);
    const double kc = (E * I) / (h * h * h);
    const double mc = (rho * area * h) / 420.0;
    const double hh = h * h;
    const double kcoef[4][4] = {{12.0, 6.0 * h, -12.0, 6.0 * h},
                                {6.0 * h, 4.0 * hh, -6.0 * h, 2.0 * hh},
                                {-12.0, -6.0 * h, 12.0, -6.0 * h},
                                {6.0 * h, 2.0 * hh, -6.0 * h, 4.0 * hh}};
    const double mcoef[4][4] = {{156.0, 22.0 * h, 54.0, -13.0 * h},
                                {22.0 * h, 4.0 * hh, 13.0 * h, -3.0 * hh},
                                {54.0, 13.0 * h, 156.0, -22.0 * h},
                                {-13.0 * h, -3.0 * hh, -22.0 * h, 4.0 * hh}};
    BeamCoef c{};
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b)
      {
        c.k[a][b] = kcoef[a][b];
        c.m[a][b] = mcoef[a][b];
      }
    c.kc = kc;
    c.mc = mc;
    mgpu_csr *hK = beam_matrix(ctx, ne, 0, c);
    mgpu_csr *hM = nullptr, *hD = nullptr;
    try
    {
      hM = beam_matrix(ctx, ne, 1, c);
      const int st = mgpu_sp_add_scaled(ctx, hM, hK, alpha, beta, &hD); // D = alpha M + beta K
      if (st != MGPU_OK)
        throw Error(st, ctx->err_msg);
    }
    catch (...)
    {
      mgpu_csr_free(hK);
      mgpu_csr_free(hM);
      throw;
    }
    *M = hM;
    *D = hD;
    *K = hK;
  });
}

} // extern "C"
