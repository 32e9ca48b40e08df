// Small-n fast path of sequential-mode MR-SPAI (n <= kSeqDenseMaxN; spai_seq.cu, whose sparse
// row lists have no size bound, dispatches here).  The built factor is dense, which lets the WHOLE
// GRID work on every MR step (the sparse chain runs on one block): n = 2000 builds in 186 ms
// against 2086 ms, at the price of O(n) rows reread per step, so the crossover is a few thousand.
//
// K-mr in SEQUENTIAL mode (spai.cpp:113-209 with SpaiOptions::Mode::sequential,
// the reference default): column j's step d = P r applies the columns 0..j-1
// that are already built (spai.cpp:138-158), so columns are processed in
// order.  One cooperative persistent kernel walks the columns; every MR
// iteration is three grid-wide phases:
//
//   d = P r      one warp per row: d_row = sum_{i < j} r_i P(row, i), then the
//                unbuilt self term alpha r_row for row >= j (it follows the
//                built columns in the reference's ascending-i order);
//   w = K d      one thread per row, ascending column (spai.cpp:159-169),
//                with the (w, w) and (w, r) block partials;
//   p += a d, r += (-a) w, ||r||^2 partials (spai.cpp:185-195).
//
// The built part of P is a dense row-major n x n array (a warp reads one row
// coalesced), so the device mode is bounded at n <= kSeqMaxN.  Sums the
// reference takes serially over sorted supports (ww, rw, ||r||^2 and the
// per-row d sum) are fixed-order trees here: deterministic, ~1e-16 relative
// from the serial order.  A dense slot that is not in a Spa's support holds an
// exact zero and contributes an exact zero, so the dense sums equal the sparse
// ones up to that reordering.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <cstdio>
#include <string>

#include "internal.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
mgpu_csr *transpose_csr(mgpu_ctx *ctx, const mgpu_csr *A);

namespace
{

constexpr int kSeqTB = 256;
constexpr int64_t kSeqMaxN = 8192; // (memory bound of the dense factor; the dispatch threshold is lower)

enum SeqFail : int
{
  kSeqOk = 0,
  kSeqStall = 1,       // spai.cpp:129-135
  kSeqZeroCurv = 2,    // spai.cpp:178
  kSeqNonFiniteW = 3,  // spai.cpp:174-177
  kSeqNonFiniteA = 4,  // spai.cpp:181-184
};

struct SeqArgs
{
  int64_t n;
  DCsr K;  // rows: w = K d
  DCsr Kt; // columns of K: initial residual
  DCsr Rt; // columns of the rhs operator (update); rp == nullptr for the build
  double alpha, tol_sq;
  int64_t max_iters;
  double *P; // dense row-major: P[row * n + i] = entry (row, i) of built column i
  double *p, *r, *d, *w;
  double *partial;  // [3][gridDim.x]
  double *residual; // [n]
  int *fail;        // [0] code, [1] spare
  int64_t *fail_col, *fail_iters;
  double *fail_rn;
};

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Block sum of v (fixed tree), result valid in thread 0.
__device__ double block_sum(double v, double *red)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0)
    red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0)
  {
    t = lane < kSeqTB / 32 ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// Sum of partial[0..G) in a fixed order, the same value in every block.
__device__ double grid_total(const double *partial, double *red)
{
  double v = 0.0;
  for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kSeqTB)
    v = __dadd_rn(v, __ldcg(partial + b));
  v = block_sum(v, red);
  if (threadIdx.x == 0)
    red[kSeqTB / 32] = v;
  __syncthreads();
  const double t = red[kSeqTB / 32];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kSeqTB) mr_sequential_dense(SeqArgs a)
{
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double red[kSeqTB / 32 + 1];
  const int64_t n = a.n;
  const int64_t G = gridDim.x;
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * kSeqTB + threadIdx.x;
  const int64_t gs = G * kSeqTB;
  const int lane = threadIdx.x & 31;
  const int64_t gw = gt >> 5, nw = gs >> 5;
  double *ww_part = a.partial, *rw_part = a.partial + G, *rn_part = a.partial + 2 * G;
  auto fail = [&](int code, int64_t j, double rn, int64_t it) {
    if (gt == 0)
    {
      a.fail[0] = code;
      *a.fail_col = j;
      *a.fail_iters = it;
      *a.fail_rn = rn;
    }
  };
  auto rnorm_sq = [&]() {
    double v = 0.0;
    for (int64_t i = gt; i < n; i += gs)
    {
      const double ri = __ldcg(a.r + i);
      v = __dadd_rn(v, __dmul_rn(ri, ri));
    }
    v = block_sum(v, red);
    if (threadIdx.x == 0)
      rn_part[blockIdx.x] = v;
    grid.sync();
    return grid_total(rn_part, red);
  };
  for (int64_t j = 0; j < n; ++j)
  {
    // ---- p = alpha e_j ; r = rhs - alpha K e_j   (spai.cpp:119-122)
    for (int64_t i = gt; i < n; i += gs)
    {
      a.p[i] = i == j ? a.alpha : 0.0;
      a.r[i] = 0.0;
    }
    grid.sync();
    if (a.Rt.rp)
    {
      for (int64_t q = a.Rt.rp[j] + gt; q < a.Rt.rp[j + 1]; q += gs)
        a.r[a.Rt.ci[q]] = __dmul_rn(1.0, a.Rt.v[q]);
    }
    else if (gt == 0)
      a.r[j] = 1.0;
    grid.sync();
    for (int64_t q = a.Kt.rp[j] + gt; q < a.Kt.rp[j + 1]; q += gs)
    {
      const int64_t i = a.Kt.ci[q];
      a.r[i] = __dadd_rn(__ldcg(a.r + i), __dmul_rn(-a.alpha, a.Kt.v[q]));
    }
    grid.sync();
    double rn = rnorm_sq();
    int64_t iters = 0;
    while (rn > a.tol_sq)
    {
      if (iters >= a.max_iters)
      {
        fail(kSeqStall, j, sqrt(rn), iters);
        return;
      }
      // ---- d = P r  (built columns i < j), + alpha r_row for the unbuilt column row >= j
      for (int64_t row = gw; row < n; row += nw)
      {
        const double *prow = a.P + row * n;
        double acc = 0.0;
        for (int64_t i = lane; i < j; i += 32)
          acc = __dadd_rn(acc, __dmul_rn(__ldcg(a.r + i), __ldcg(prow + i)));
        acc = warp_sum(acc);
        if (lane == 0)
        {
          if (row >= j)
          {
            const double rr = __ldcg(a.r + row);
            if (rr != 0.0)
              acc = __dadd_rn(acc, __dmul_rn(a.alpha, rr));
          }
          a.d[row] = acc;
        }
      }
      grid.sync();
      // ---- w = K d, (w, w), (w, r)
      double ww = 0.0, rw = 0.0;
      for (int64_t row = gt; row < n; row += gs)
      {
        double acc = 0.0;
        for (int64_t q = a.K.rp[row]; q < a.K.rp[row + 1]; ++q)
        {
          const double dk = __ldcg(a.d + a.K.ci[q]);
          if (dk != 0.0)
            acc = __dadd_rn(acc, __dmul_rn(dk, a.K.v[q]));
        }
        a.w[row] = acc;
        ww = __dadd_rn(ww, __dmul_rn(acc, acc));
        rw = __dadd_rn(rw, __dmul_rn(acc, __ldcg(a.r + row)));
      }
      ww = block_sum(ww, red);
      rw = block_sum(rw, red);
      if (threadIdx.x == 0)
      {
        ww_part[blockIdx.x] = ww;
        rw_part[blockIdx.x] = rw;
      }
      grid.sync();
      ww = grid_total(ww_part, red);
      rw = grid_total(rw_part, red);
      if (!(ww > 0.0))
      {
        fail(isfinite(ww) ? kSeqZeroCurv : kSeqNonFiniteW, j, sqrt(rn), iters);
        return;
      }
      const double step = rw / ww;
      if (!isfinite(step))
      {
        fail(kSeqNonFiniteA, j, sqrt(rn), iters);
        return;
      }
      for (int64_t i = gt; i < n; i += gs)
      {
        a.p[i] = __dadd_rn(a.p[i], __dmul_rn(step, __ldcg(a.d + i)));
        a.r[i] = __dadd_rn(__ldcg(a.r + i), __dmul_rn(-step, __ldcg(a.w + i)));
      }
      grid.sync();
      rn = rnorm_sq();
      ++iters;
    }
    // ---- column j of P (exact zeros are "not stored", spai.cpp:197-206)
    if (gt == 0)
      a.residual[j] = sqrt(rn);
    for (int64_t row = gt; row < n; row += gs)
      a.P[row * n + j] = a.p[row];
    grid.sync();
  }
}

// CSR of the dense row-major factor: one warp per row, ascending column.
__global__ void dense_row_count(int64_t n, const double *__restrict__ P, int64_t *__restrict__ cnt)
{
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n)
    return;
  int64_t c = 0;
  for (int64_t i = lane; i < n; i += 32)
    c += P[row * n + i] != 0.0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane == 0)
    cnt[row + 1] = c;
}

__global__ void dense_row_fill(int64_t n, const double *__restrict__ P, const int64_t *__restrict__ rp,
                               int32_t *__restrict__ ci, double *__restrict__ v)
{
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n)
    return;
  int64_t out = rp[row];
  for (int64_t i0 = 0; i0 < n; i0 += 32)
  {
    const int64_t i = i0 + lane;
    const double x = i < n ? P[row * n + i] : 0.0;
    const bool nz = x != 0.0;
    const unsigned mask = __ballot_sync(0xffffffffu, nz);
    if (nz)
    {
      const int64_t o = out + __popc(mask & ((1u << lane) - 1u));
      ci[o] = static_cast<int32_t>(i);
      v[o] = x;
    }
    out += __popc(mask);
  }
}

std::string fmt_seq(double v)
{
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v); // std::to_string(double) format
  return buf;
}

} // namespace

// Sequential-mode build / update: K the operator, rhs_src = K_old (update) or null.
mgpu_csr *mr_build_sequential_dense(mgpu_ctx *ctx, const mgpu_csr *K, const mgpu_csr *rhs_src, double alpha, double tol,
                              int64_t max_iters, double *col_residual)
{
  const int64_t n = K->nrows;
  if (n > kSeqMaxN)
    throw Error(MGPU_ERR_UNSUPPORTED, "spai: sequential mode on the device holds the built factor densely (n <= " +
                                          std::to_string(kSeqMaxN) + ", got " + std::to_string(n) +
                                          "); use frozen mode or LS-SPAI");
  cudaStream_t s = ctx->stream;
  mgpu_csr *Kt = transpose_csr(ctx, K);
  mgpu_csr *Rt = nullptr;
  mgpu_csr *P = nullptr;
  try
  {
    Rt = rhs_src ? transpose_csr(ctx, rhs_src) : nullptr;
    const int64_t nn = n > 0 ? n : 1;
    DBuf dense(sizeof(double) * static_cast<size_t>(nn) * nn, s);
    DBuf vec(sizeof(double) * 4 * nn, s), resid(sizeof(double) * nn, s);
    const int G = ctx->num_sms;
    DBuf part(sizeof(double) * 3 * G, s), fl(sizeof(int) * 2, s), fcol(sizeof(int64_t), s), fit(sizeof(int64_t), s),
        frn(sizeof(double), s);
    MG_CUDA(cudaMemsetAsync(fl.ptr, 0, sizeof(int) * 2, s));
    MG_CUDA(cudaMemsetAsync(dense.ptr, 0, sizeof(double) * static_cast<size_t>(nn) * nn, s));
    SeqArgs a{};
    a.n = n;
    a.K = K->view();
    a.Kt = Kt->view();
    a.Rt = Rt ? Rt->view() : DCsr{nullptr, nullptr, nullptr};
    a.alpha = alpha;
    a.tol_sq = tol * tol;
    a.max_iters = max_iters;
    a.P = dense.as<double>();
    a.p = vec.as<double>();
    a.r = a.p + nn;
    a.d = a.r + nn;
    a.w = a.d + nn;
    a.partial = part.as<double>();
    a.residual = resid.as<double>();
    a.fail = fl.as<int>();
    a.fail_col = fcol.as<int64_t>();
    a.fail_iters = fit.as<int64_t>();
    a.fail_rn = frn.as<double>();
    if (n > 0)
    {
      int per_sm = 0;
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mr_sequential_dense, kSeqTB, 0));
      if (per_sm < 1)
        throw Error(MGPU_ERR_CUDA, "spai: sequential kernel cannot be resident");
      void *args[] = {&a};
      MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(mr_sequential_dense), dim3(static_cast<unsigned>(G)),
                                          dim3(kSeqTB), args, 0, s));
      check_launch(ctx, "mr_sequential_dense");
    }
    int hf[2] = {0, 0};
    int64_t col = 0, it = 0;
    double rn = 0.0;
    MG_CUDA(cudaMemcpyAsync(hf, fl.ptr, sizeof hf, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&col, fcol.ptr, sizeof col, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&it, fit.ptr, sizeof it, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&rn, frn.ptr, sizeof rn, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    if (hf[0] != kSeqOk)
    {
      const std::string c = std::to_string(col);
      switch (hf[0])
      {
      case kSeqStall:
        throw Error(MGPU_ERR_STAGNATION,
                    "spai: column " + c + " stalled at ||r|| = " + fmt_seq(rn) + " after " + std::to_string(it) +
                        " iterations (tol " + fmt_seq(tol) + ")",
                    col);
      case kSeqZeroCurv:
        throw Error(MGPU_ERR_STAGNATION, "spai: zero curvature in column " + c + " with ||r|| > tol", col);
      case kSeqNonFiniteW:
        throw Error(MGPU_ERR_NUMERICAL, "spai: non-finite values in column " + c, col);
      default:
        throw Error(MGPU_ERR_NUMERICAL, "spai: non-finite step in column " + c, col);
      }
    }
    P = new mgpu_csr;
    P->ctx = ctx;
    P->nrows = n;
    P->ncols = n;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&P->row_ptr), sizeof(int64_t) * (n + 1), s));
    MG_CUDA(cudaMemsetAsync(P->row_ptr, 0, sizeof(int64_t) * (n + 1), s));
    const unsigned rows_grid = static_cast<unsigned>((n * 32 + kThreads - 1) / kThreads);
    if (n > 0)
    {
      dense_row_count<<<rows_grid, kThreads, 0, s>>>(n, dense.as<double>(), P->row_ptr);
      check_launch(ctx, "dense_row_count");
      size_t tmp = 0;
      MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, P->row_ptr + 1, P->row_ptr + 1, n, s));
      DBuf t(tmp, s);
      MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, P->row_ptr + 1, P->row_ptr + 1, n, s));
      count_launch(ctx);
    }
    int64_t nnz = 0;
    MG_CUDA(cudaMemcpyAsync(&nnz, P->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    P->nnz = nnz;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&P->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&P->values), sizeof(double) * (nnz > 0 ? nnz : 1), s));
    if (n > 0)
    {
      dense_row_fill<<<rows_grid, kThreads, 0, s>>>(n, dense.as<double>(), P->row_ptr, P->col_idx, P->values);
      check_launch(ctx, "dense_row_fill");
    }
    if (col_residual && n > 0)
      MG_CUDA(cudaMemcpyAsync(col_residual, resid.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
  }
  catch (...)
  {
    mgpu_csr_free(P);
    mgpu_csr_free(Kt);
    mgpu_csr_free(Rt);
    throw;
  }
  mgpu_csr_free(Kt);
  mgpu_csr_free(Rt);
  return P;
}

} // namespace mgpu
