// K-mr in SEQUENTIAL mode (spai.cpp:113-209 with SpaiOptions::Mode::sequential, the reference
// default): column j's step d = P r applies the columns 0..j-1 already built (spai.cpp:138-158),
// so columns are processed in order and the build is a serial column chain.  One persistent
// block walks the columns (the chain leaves nothing to spread over SMs but each step's rows);
// the factor is kept SPARSE, so n is bounded only by memory:
//
//   built factor   row lists: row i holds (column, value) of the built columns with an entry in row
//                  i, columns ascending (appended in build order), capacity `cap` per row;
//   supports       every accumulator (p, r, d, w) is a dense n-vector that is zero outside an index
//                  range [lo, hi] tracked per accumulator (the reference's Spa with a sorted
//                  support, spai.cpp:22-68; an index inside the range but outside the support
//                  holds an exact zero and contributes nothing);
//   d = P r        one thread per row of d's range: the row's list entries with a column inside r's
//                  range, ascending, each r_i P(row, i) with r_i != 0, then the unbuilt self term
//                  alpha r_row for row >= j -- per row exactly the reference's ascending-i
//                  accumulation (bitwise);
//   w = K d        one thread per row, K's row in ascending column (spai.cpp:159-169, bitwise);
//   ww, rw, ||r||^2  fixed-order block trees over the ranges (the reference sums serially over the
//                  sorted support: ~1e-16 relative, deterministic);
//   p += a d, r += (-a) w (spai.cpp:185-195), then the column's nonzeros are appended to the row
//   lists and the accumulators cleared over their ranges.
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <cstdio>
#include <string>

#include "internal.cuh"

namespace mgpu
{
mgpu_csr *transpose_csr(mgpu_ctx *ctx, const mgpu_csr *A);
// spai_seq_dense.cu
mgpu_csr *mr_build_sequential_dense(mgpu_ctx *ctx, const mgpu_csr *K, const mgpu_csr *rhs_src, double alpha, double tol,
                                    int64_t max_iters, double *col_residual);
constexpr int64_t kSeqDenseMaxN = 4096;

namespace
{

constexpr int kSeqTB = 1024;

enum SeqFail : int
{
  kSeqOk = 0,
  kSeqStall = 1,      // spai.cpp:129-135
  kSeqZeroCurv = 2,   // spai.cpp:178
  kSeqNonFiniteW = 3, // spai.cpp:174-177
  kSeqNonFiniteA = 4, // spai.cpp:181-184
  kSeqCapacity = 5,   // a row list is full (host retries with a larger capacity)
};

struct SeqArgs
{
  int64_t n;
  DCsr K;  // rows: w = K d
  DCsr Kt; // columns of K: initial residual
  DCsr Rt; // columns of the rhs operator (update); rp == nullptr for the build
  double alpha, tol_sq;
  int64_t max_iters;
  int64_t bwK;        // bandwidth of K (w's range around d's)
  int64_t cap;        // row-list capacity
  int32_t *rl_cnt;    // [n]
  int32_t *rl_col;    // [n * cap]
  double *rl_val;     // [n * cap]
  int64_t *col_lo, *col_hi; // [n] row range of built column i (lo > hi: empty)
  double *p, *r, *d, *w;    // dense, zero outside their ranges
  double *residual;         // [n]
  int *fail;
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

// Block sum (fixed tree), the same value in every thread.
__device__ double block_sum(double v, double *red)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0)
    red[warp] = v;
  __syncthreads();
  double t = lane < kSeqTB / 32 ? red[lane] : 0.0;
  t = warp_sum(t);
  __syncthreads();
  return t;
}

__device__ int64_t block_min(int64_t v, int64_t *red)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    v = min(v, static_cast<int64_t>(__shfl_xor_sync(0xffffffffu, static_cast<long long>(v), off)));
  if (lane == 0)
    red[warp] = v;
  __syncthreads();
  int64_t t = lane < kSeqTB / 32 ? red[lane] : LLONG_MAX;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    t = min(t, static_cast<int64_t>(__shfl_xor_sync(0xffffffffu, static_cast<long long>(t), off)));
  __syncthreads();
  return t;
}

__device__ int64_t block_max(int64_t v, int64_t *red) { return -block_min(-v, red); }

__global__ void __launch_bounds__(kSeqTB, 1) mr_sequential(SeqArgs a)
{
  __shared__ double red[kSeqTB / 32];
  __shared__ int64_t ired[kSeqTB / 32];
  const int64_t n = a.n;
  const int t = threadIdx.x;
  double *p = a.p, *r = a.r, *d = a.d, *w = a.w;
  auto fail = [&](int code, int64_t j, double rn, int64_t it) {
    if (t == 0)
    {
      a.fail[0] = code;
      *a.fail_col = j;
      *a.fail_iters = it;
      *a.fail_rn = rn;
    }
  };
  for (int64_t j = 0; j < n; ++j)
  {
    // ---- p = alpha e_j ; r = rhs - alpha K e_j   (spai.cpp:119-122)
    int64_t r_lo = j, r_hi = j;
    if (t == 0)
      p[j] = a.alpha;
    if (a.Rt.rp)
    {
      for (int64_t q = a.Rt.rp[j] + t; q < a.Rt.rp[j + 1]; q += kSeqTB)
        r[a.Rt.ci[q]] = __dmul_rn(1.0, a.Rt.v[q]);
      if (a.Rt.rp[j + 1] > a.Rt.rp[j])
      {
        r_lo = a.Rt.ci[a.Rt.rp[j]];
        r_hi = a.Rt.ci[a.Rt.rp[j + 1] - 1];
      }
      else
        r_lo = 0, r_hi = -1; // empty (lo > hi)
    }
    else if (t == 0)
      r[j] = 1.0;
    __syncthreads();
    for (int64_t q = a.Kt.rp[j] + t; q < a.Kt.rp[j + 1]; q += kSeqTB)
    {
      const int64_t i = a.Kt.ci[q];
      r[i] = __dadd_rn(r[i], __dmul_rn(-a.alpha, a.Kt.v[q]));
    }
    // ranges: [lo, hi], empty when lo > hi; unite() is the union's hull
    auto unite = [](int64_t &lo, int64_t &hi, int64_t lo2, int64_t hi2) {
      if (lo2 > hi2)
        return;
      if (lo > hi)
      {
        lo = lo2;
        hi = hi2;
        return;
      }
      lo = min(lo, lo2);
      hi = max(hi, hi2);
    };
    if (a.Kt.rp[j + 1] > a.Kt.rp[j])
      unite(r_lo, r_hi, a.Kt.ci[a.Kt.rp[j]], a.Kt.ci[a.Kt.rp[j + 1] - 1]);
    int64_t p_lo = j, p_hi = j, d_lo = 0, d_hi = -1, w_lo = 0, w_hi = -1;
    __syncthreads();
    auto rnorm_sq = [&]() {
      double v = 0.0;
      for (int64_t i = r_lo + t; i <= r_hi; i += kSeqTB)
        v = __dadd_rn(v, __dmul_rn(r[i], r[i]));
      return block_sum(v, red);
    };
    double rn = rnorm_sq();
    int64_t iters = 0;
    while (rn > a.tol_sq)
    {
      if (iters >= a.max_iters)
      {
        fail(kSeqStall, j, sqrt(rn), iters);
        return;
      }
      // ---- d's range: built columns i < j in r's support spread over [col_lo, col_hi]; unbuilt
      // indices contribute to themselves
      int64_t lo = LLONG_MAX, hi = -1;
      for (int64_t i = r_lo + t; i <= r_hi; i += kSeqTB)
      {
        if (r[i] == 0.0)
          continue;
        if (i < j)
        {
          if (a.col_lo[i] <= a.col_hi[i])
          {
            lo = min(lo, a.col_lo[i]);
            hi = max(hi, a.col_hi[i]);
          }
        }
        else
        {
          lo = min(lo, i);
          hi = max(hi, i);
        }
      }
      int64_t nd_lo = block_min(lo, ired), nd_hi = block_max(hi, ired);
      if (nd_lo > nd_hi)
        nd_lo = 0, nd_hi = -1;
      // clear the previous d range, then d = P r over the new one
      for (int64_t i = d_lo + t; i <= d_hi; i += kSeqTB)
        d[i] = 0.0;
      __syncthreads();
      d_lo = nd_lo;
      d_hi = nd_hi;
      const int64_t ib = min(r_hi, j - 1); // built columns inside r's range: [r_lo, ib]
      for (int64_t row = d_lo + t; row <= d_hi; row += kSeqTB)
      {
        const int32_t cnt = a.rl_cnt[row];
        const int32_t *cols = a.rl_col + row * a.cap;
        const double *vals = a.rl_val + row * a.cap;
        int lo2 = 0, hi2 = cnt; // first list entry with column >= r_lo
        while (lo2 < hi2)
        {
          const int mid = (lo2 + hi2) >> 1;
          if (cols[mid] < r_lo)
            lo2 = mid + 1;
          else
            hi2 = mid;
        }
        double acc = 0.0;
        for (int e = lo2; e < cnt && cols[e] <= ib; ++e)
        {
          const double ri = r[cols[e]];
          if (ri != 0.0)
            acc = __dadd_rn(acc, __dmul_rn(ri, vals[e]));
        }
        if (row >= j && row >= r_lo && row <= r_hi)
        {
          const double rr = r[row];
          if (rr != 0.0)
            acc = __dadd_rn(acc, __dmul_rn(a.alpha, rr));
        }
        d[row] = acc;
      }
      __syncthreads();
      // ---- w = K d over d's range plus K's bandwidth; (w, w), (w, r)
      for (int64_t i = w_lo + t; i <= w_hi; i += kSeqTB)
        w[i] = 0.0;
      __syncthreads();
      w_lo = d_lo - a.bwK > 0 ? d_lo - a.bwK : 0;
      w_hi = d_hi + a.bwK < n - 1 ? d_hi + a.bwK : n - 1;
      if (d_lo > d_hi)
        w_lo = 0, w_hi = -1;
      double ww = 0.0, rw = 0.0;
      for (int64_t row = w_lo + t; row <= w_hi; row += kSeqTB)
      {
        double acc = 0.0;
        for (int64_t q = a.K.rp[row]; q < a.K.rp[row + 1]; ++q)
        {
          const int64_t c = a.K.ci[q];
          const double dk = (c >= d_lo && c <= d_hi) ? d[c] : 0.0;
          if (dk != 0.0)
            acc = __dadd_rn(acc, __dmul_rn(dk, a.K.v[q]));
        }
        w[row] = acc;
        ww = __dadd_rn(ww, __dmul_rn(acc, acc));
        const double rv = (row >= r_lo && row <= r_hi) ? r[row] : 0.0;
        rw = __dadd_rn(rw, __dmul_rn(acc, rv));
      }
      ww = block_sum(ww, red);
      rw = block_sum(rw, red);
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
      for (int64_t i = d_lo + t; i <= d_hi; i += kSeqTB)
        p[i] = __dadd_rn(p[i], __dmul_rn(step, d[i]));
      for (int64_t i = w_lo + t; i <= w_hi; i += kSeqTB)
        r[i] = __dadd_rn(r[i], __dmul_rn(-step, w[i]));
      unite(p_lo, p_hi, d_lo, d_hi);
      unite(r_lo, r_hi, w_lo, w_hi);
      __syncthreads();
      rn = rnorm_sq();
      ++iters;
    }
    // ---- column j of P: its nonzeros (spai.cpp:197-206) appended to the row lists
    if (t == 0)
      a.residual[j] = sqrt(rn);
    int64_t clo = LLONG_MAX, chi = -1;
    bool full = false;
    for (int64_t row = p_lo + t; row <= p_hi; row += kSeqTB)
    {
      const double v = p[row];
      if (v == 0.0)
        continue;
      const int32_t c = a.rl_cnt[row];
      if (c >= a.cap)
      {
        full = true;
        continue;
      }
      a.rl_col[row * a.cap + c] = static_cast<int32_t>(j);
      a.rl_val[row * a.cap + c] = v;
      a.rl_cnt[row] = c + 1;
      clo = min(clo, row);
      chi = max(chi, row);
    }
    if (__syncthreads_or(full))
    {
      fail(kSeqCapacity, j, 0.0, 0);
      return;
    }
    clo = block_min(clo, ired);
    chi = block_max(chi, ired);
    if (t == 0)
    {
      a.col_lo[j] = clo <= chi ? clo : 0; // an all-zero column: empty range
      a.col_hi[j] = clo <= chi ? chi : -1;
    }
    // ---- clear the accumulators over their ranges
    for (int64_t i = p_lo + t; i <= p_hi; i += kSeqTB)
      p[i] = 0.0;
    for (int64_t i = r_lo + t; i <= r_hi; i += kSeqTB)
      r[i] = 0.0;
    for (int64_t i = d_lo + t; i <= d_hi; i += kSeqTB)
      d[i] = 0.0;
    for (int64_t i = w_lo + t; i <= w_hi; i += kSeqTB)
      w[i] = 0.0;
    __syncthreads();
  }
}

// Row lists -> CSR (rows keep their ascending columns).
__global__ void rl_fill(int64_t n, int64_t cap, const int32_t *__restrict__ cnt, const int32_t *__restrict__ col,
                        const double *__restrict__ val, const int64_t *__restrict__ rp, int32_t *__restrict__ ci,
                        double *__restrict__ v)
{
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= n)
    return;
  for (int32_t e = 0; e < cnt[row]; ++e)
  {
    ci[rp[row] + e] = col[row * cap + e];
    v[rp[row] + e] = val[row * cap + e];
  }
}

__global__ void rl_counts(int64_t n, const int32_t *__restrict__ cnt, int64_t *__restrict__ rp)
{
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row < n)
    rp[row + 1] = cnt[row];
  if (row == 0)
    rp[0] = 0;
}

std::string fmt_seq(double v)
{
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v); // std::to_string(double) format
  return buf;
}

} // namespace

// Sequential-mode build / update: K the operator, rhs_src = K_old (update) or null.
mgpu_csr *mr_build_sequential(mgpu_ctx *ctx, const mgpu_csr *K, const mgpu_csr *rhs_src, double alpha, double tol,
                              int64_t max_iters, double *col_residual)
{
  const int64_t n = K->nrows;
  // small systems: the dense-factor kernel spreads every MR step over the whole grid
  // (spai_seq_dense.cu; n = 2000: 186 ms against 2086 ms for the single-block sparse chain)
  if (n <= kSeqDenseMaxN && ctx->opt[MGPU_OPT_SEQ_SPARSE] == 0)
    return mr_build_sequential_dense(ctx, K, rhs_src, alpha, tol, max_iters, col_residual);
  cudaStream_t s = ctx->stream;
  mgpu_csr *Kt = transpose_csr(ctx, K);
  mgpu_csr *Rt = nullptr;
  mgpu_csr *P = nullptr;
  try
  {
    Rt = rhs_src ? transpose_csr(ctx, rhs_src) : nullptr;
    const int64_t nn = n > 0 ? n : 1;
    const int64_t bwK = csr_bandwidth(ctx, const_cast<mgpu_csr *>(K));
    // row-list capacity: ~4 GB of lists by default, never more than n; a full list stops the
    // kernel and the build reruns with twice the capacity
    int64_t cap = std::min<int64_t>(nn, std::max<int64_t>(64, (int64_t{4} << 30) / (12 * nn)));
    for (;;)
    {
      DBuf cnt(sizeof(int32_t) * nn, s), lcol(sizeof(int32_t) * static_cast<size_t>(nn * cap), s),
          lval(sizeof(double) * static_cast<size_t>(nn * cap), s), crange(sizeof(int64_t) * 2 * nn, s);
      DBuf vec(sizeof(double) * 4 * nn, s), resid(sizeof(double) * nn, s);
      DBuf fl(sizeof(int) * 2, s), fcol(sizeof(int64_t), s), fit(sizeof(int64_t), s), frn(sizeof(double), s);
      MG_CUDA(cudaMemsetAsync(fl.ptr, 0, sizeof(int) * 2, s));
      MG_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(int32_t) * nn, s));
      MG_CUDA(cudaMemsetAsync(vec.ptr, 0, sizeof(double) * 4 * nn, s));
      SeqArgs a{};
      a.n = n;
      a.K = K->view();
      a.Kt = Kt->view();
      a.Rt = Rt ? Rt->view() : DCsr{nullptr, nullptr, nullptr};
      a.alpha = alpha;
      a.tol_sq = tol * tol;
      a.max_iters = max_iters;
      a.bwK = bwK;
      a.cap = cap;
      a.rl_cnt = cnt.as<int32_t>();
      a.rl_col = lcol.as<int32_t>();
      a.rl_val = lval.as<double>();
      a.col_lo = crange.as<int64_t>();
      a.col_hi = a.col_lo + nn;
      a.p = vec.as<double>();
      a.r = a.p + nn;
      a.d = a.r + nn;
      a.w = a.d + nn;
      a.residual = resid.as<double>();
      a.fail = fl.as<int>();
      a.fail_col = fcol.as<int64_t>();
      a.fail_iters = fit.as<int64_t>();
      a.fail_rn = frn.as<double>();
      if (n > 0)
      {
        mr_sequential<<<1, kSeqTB, 0, s>>>(a);
        check_launch(ctx, "mr_sequential");
      }
      int hf[2] = {0, 0};
      int64_t col = 0, it = 0;
      double rn = 0.0;
      MG_CUDA(cudaMemcpyAsync(hf, fl.ptr, sizeof hf, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaMemcpyAsync(&col, fcol.ptr, sizeof col, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaMemcpyAsync(&it, fit.ptr, sizeof it, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaMemcpyAsync(&rn, frn.ptr, sizeof rn, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      if (hf[0] == kSeqCapacity)
      {
        if (cap >= nn)
          throw Error(MGPU_ERR_CUDA, "spai: sequential row lists overflowed at full capacity");
        cap = std::min<int64_t>(nn, 2 * cap);
        continue;
      }
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
      if (n > 0)
      {
        rl_counts<<<blocks_for(n), kThreads, 0, s>>>(n, cnt.as<int32_t>(), P->row_ptr);
        check_launch(ctx, "rl_counts");
        size_t tmp = 0;
        MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, P->row_ptr + 1, P->row_ptr + 1, n, s));
        DBuf tb(tmp, s);
        MG_CUDA(cub::DeviceScan::InclusiveSum(tb.ptr, tmp, P->row_ptr + 1, P->row_ptr + 1, n, s));
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
        rl_fill<<<blocks_for(n), kThreads, 0, s>>>(n, cap, cnt.as<int32_t>(), lcol.as<int32_t>(), lval.as<double>(),
                                                   P->row_ptr, P->col_idx, P->values);
        check_launch(ctx, "rl_fill");
      }
      if (col_residual && n > 0)
        MG_CUDA(cudaMemcpyAsync(col_residual, resid.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      break;
    }
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
