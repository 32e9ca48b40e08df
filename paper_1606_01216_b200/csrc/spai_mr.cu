// K-mr / K-mr-upd: the reference's minimal-residual SPAI (Alg. 2 / Alg. 4,
// spai.cpp:113-350) in FROZEN mode (d = alpha r, columns independent,
// spai.hpp:35-42), one warp per column.
//
// The reference keeps four sparse accumulators per column (Spa(n), O(n) each).
// Here a column's vectors p, r, d, w live in a dense WINDOW of shared memory:
// with K of lower/upper bandwidth (bl, bu), r's support after k steps lies in
// [j - (k+1) bu, j + (k+1) bl], so a window of W = 512 slots covers 50 steps
// of a bandwidth-5 operator.  Wider operators (or slowly converging columns) get a wider window:
// the build starts at 512 slots with 4 columns per block and, when a column outgrows its
// window, reruns at 2048 slots (2 columns per block) and then 6144 (1 column per block, 192 KB).  Entries outside a Spa's support are exact zeros
// in the window, so every sum over a support equals the sum over the window
// (zero terms add exactly nothing).  Arithmetic per entry matches spai.cpp:
// w_i accumulates K_ik d_k in ascending k without FMA, p += a d, r += (-a) w.
// Reductions (||r||^2, (w,w), (w,r)) are fixed warp trees instead of the
// reference's serial sums -> differences at the 1e-16 level.
//
// Column lengths differ, so the factor is produced in two deterministic passes
// (count, then fill), assembled as P^T and transposed to CSR.
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace mgpu
{
mgpu_csr *transpose_csr(mgpu_ctx *ctx, const mgpu_csr *A);
mgpu_csr *mr_build_sequential(mgpu_ctx *ctx, const mgpu_csr *K, const mgpu_csr *rhs_src, double alpha, double tol,
                              int64_t max_iters, double *col_residual);
void trace_dev(mgpu_ctx *ctx, const mgpu_csr *A, double *out_dev);
void trace_inner_dev(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double *out_dev);

namespace
{

// window ladder: slots per column, columns (warps) per block
constexpr int kMrLevels = 3;
constexpr int kMrW[kMrLevels] = {512, 2048, 6144};
constexpr int kMrWpb[kMrLevels] = {4, 2, 1};

enum MrFail : int
{
  kStall = MGPU_ERR_STAGNATION,          // iteration budget (spai.cpp:129-135)
  kZeroCurv = 16 | MGPU_ERR_STAGNATION,  // (w,w) == 0 (spai.cpp:178)
  kNonFiniteW = MGPU_ERR_NUMERICAL,      // (w,w) not finite (spai.cpp:174-177)
  kNonFiniteA = 16 | MGPU_ERR_NUMERICAL, // step not finite (spai.cpp:181-184)
  kWindow = MGPU_ERR_UNSUPPORTED,
};

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__global__ void bandwidth_kernel(int64_t n, DCsr A, int *bw) // bw[0] = lower, bw[1] = upper
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  const int64_t b = A.rp[i], e = A.rp[i + 1];
  if (b == e)
    return;
  const int64_t lo = i - A.ci[b], hi = A.ci[e - 1] - i;
  atomicMax(&bw[0], static_cast<int>(lo > INT_MAX ? INT_MAX : (lo < 0 ? 0 : lo)));
  atomicMax(&bw[1], static_cast<int>(hi > INT_MAX ? INT_MAX : (hi < 0 ? 0 : hi)));
}

struct MrArgs
{
  int64_t n;
  DCsr K;   // operator rows (w = K d)
  DCsr Kt;  // operator columns (initial residual)
  DCsr Rt;  // rhs columns (update) -- rp == nullptr for the build
  double alpha, tol_sq;
  int64_t max_iters;
  int bl, bu; // K's lower / upper bandwidth
  int W;      // window slots per column
  int *bw;               // pass 1: bandwidth bound of the factor
  int64_t *count;        // pass 1: nonzeros of column j
  double *residual;      // pass 1: final ||r|| (or ||r|| at failure)
  int64_t *fail_iters;   // pass 1: iterations at failure
  unsigned long long *err;
  const int64_t *offset; // pass 2: P^T row_ptr
  int32_t *out_rows;     // pass 2
  double *out_vals;      // pass 2
};

template <bool kFill, int kMrWarps>
__global__ void __launch_bounds__(kMrWarps * 32) mr_columns(MrArgs a)
{
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kMrWarps + warp;
  if (j >= a.n)
    return;
  const int kW = a.W;
  double *p = smem + static_cast<size_t>(warp) * 4 * kW;
  double *r = p + kW, *d = r + kW, *w = d + kW;
  const int64_t base = j - kW / 2; // slot(i) = i - base
  for (int s = lane; s < kW; s += 32)
  {
    p[s] = 0.0;
    r[s] = 0.0;
    d[s] = 0.0;
    w[s] = 0.0;
  }
  __syncwarp();
  auto fail = [&](int code, double rn, int64_t it) {
    if (lane == 0)
    {
      if (!kFill)
      {
        a.residual[j] = rn;
        a.fail_iters[j] = it;
      }
      atomicMin(a.err, (static_cast<unsigned long long>(j) << 8) | static_cast<unsigned long long>(code));
    }
  };
  // ---- p = alpha e_j ; r = rhs - alpha K e_j   (spai.cpp:119-122)
  int64_t lo = j, hi = j;
  if (a.Rt.rp)
  {
    for (int64_t q = a.Rt.rp[j] + lane; q < a.Rt.rp[j + 1]; q += 32)
    {
      const int64_t i = a.Rt.ci[q];
      if (i - base < 0 || i - base >= kW)
        continue; // checked below through lo/hi
      r[i - base] = __dmul_rn(1.0, a.Rt.v[q]);
    }
    if (a.Rt.rp[j + 1] > a.Rt.rp[j])
    {
      lo = min(lo, static_cast<int64_t>(a.Rt.ci[a.Rt.rp[j]]));
      hi = max(hi, static_cast<int64_t>(a.Rt.ci[a.Rt.rp[j + 1] - 1]));
    }
  }
  else if (lane == 0)
  {
    r[j - base] = 1.0;
  }
  if (a.Kt.rp[j + 1] > a.Kt.rp[j])
  {
    lo = min(lo, static_cast<int64_t>(a.Kt.ci[a.Kt.rp[j]]));
    hi = max(hi, static_cast<int64_t>(a.Kt.ci[a.Kt.rp[j + 1] - 1]));
  }
  if (lo - base < 0 || hi - base >= kW)
  {
    fail(kWindow, 0.0, 0);
    return;
  }
  __syncwarp();
  for (int64_t q = a.Kt.rp[j] + lane; q < a.Kt.rp[j + 1]; q += 32)
  {
    const int64_t i = a.Kt.ci[q];
    r[i - base] = __dadd_rn(r[i - base], __dmul_rn(-a.alpha, a.Kt.v[q]));
  }
  if (lane == 0)
    p[j - base] = a.alpha;
  __syncwarp();
  auto norm_sq = [&](int64_t l0, int64_t h0) {
    double acc = 0.0;
    for (int64_t i = l0 + lane; i <= h0; i += 32)
      acc = __dadd_rn(acc, __dmul_rn(r[i - base], r[i - base]));
    return warp_sum(acc);
  };
  double rnorm_sq = norm_sq(lo, hi);
  int64_t iters = 0;
  while (rnorm_sq > a.tol_sq)
  {
    if (iters >= a.max_iters)
    {
      fail(kStall, sqrt(rnorm_sq), iters);
      return;
    }
    // d = alpha r (frozen mode, spai.cpp:138-158)
    for (int64_t i = lo + lane; i <= hi; i += 32)
    {
      const double ri = r[i - base];
      d[i - base] = ri == 0.0 ? 0.0 : __dmul_rn(a.alpha, ri);
    }
    const int64_t wlo = max(static_cast<int64_t>(0), lo - a.bu);
    const int64_t whi = min(a.n - 1, hi + a.bl);
    if (wlo - base < 0 || whi - base >= kW)
    {
      fail(kWindow, sqrt(rnorm_sq), iters);
      return;
    }
    __syncwarp();
    // w = K d, each row in ascending column order (spai.cpp:159-169)
    double ww = 0.0, rw = 0.0;
    for (int64_t i = wlo + lane; i <= whi; i += 32)
    {
      double acc = 0.0;
      for (int64_t q = a.K.rp[i]; q < a.K.rp[i + 1]; ++q)
      {
        const int64_t k = a.K.ci[q];
        if (k < lo || k > hi)
          continue;
        acc = __dadd_rn(acc, __dmul_rn(d[k - base], a.K.v[q]));
      }
      w[i - base] = acc;
      ww = __dadd_rn(ww, __dmul_rn(acc, acc));
      rw = __dadd_rn(rw, __dmul_rn(acc, r[i - base]));
    }
    ww = warp_sum(ww);
    rw = warp_sum(rw);
    if (!(ww > 0.0))
    {
      fail(isfinite(ww) ? kZeroCurv : kNonFiniteW, sqrt(rnorm_sq), iters);
      return;
    }
    const double step = rw / ww;
    if (!isfinite(step))
    {
      fail(kNonFiniteA, sqrt(rnorm_sq), iters);
      return;
    }
    __syncwarp();
    for (int64_t i = lo + lane; i <= hi; i += 32)
      p[i - base] = __dadd_rn(p[i - base], __dmul_rn(step, d[i - base]));
    for (int64_t i = wlo + lane; i <= whi; i += 32)
      r[i - base] = __dadd_rn(r[i - base], __dmul_rn(-step, w[i - base]));
    lo = min(lo, wlo);
    hi = max(hi, whi);
    __syncwarp();
    rnorm_sq = norm_sq(lo, hi);
    ++iters;
  }
  // ---- column j of P: nonzeros of p in ascending row (spai.cpp:197-206)
  const int64_t plo = min(lo, j), phi = max(hi, j);
  if (!kFill)
  {
    int64_t cnt = 0;
    for (int64_t i = plo + lane; i <= phi; i += 32)
      cnt += p[i - base] != 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (lane == 0)
    {
      a.count[j] = cnt;
      a.residual[j] = sqrt(rnorm_sq);
      atomicMax(a.bw, static_cast<int>(max(j - plo, phi - j)));
    }
    return;
  }
  int64_t out = a.offset[j];
  for (int64_t i0 = plo; i0 <= phi; i0 += 32)
  {
    const int64_t i = i0 + lane;
    const bool nz = i <= phi && p[i - base] != 0.0;
    const unsigned int mask = __ballot_sync(0xffffffffu, nz);
    if (nz)
    {
      const int64_t o = out + __popc(mask & ((1u << lane) - 1u));
      a.out_rows[o] = static_cast<int32_t>(i);
      a.out_vals[o] = p[i - base];
    }
    out += __popc(mask);
  }
}

std::string fmt_f(double v)
{
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v); // std::to_string(double) format
  return buf;
}

mgpu_csr *mr_build(mgpu_ctx *ctx, const mgpu_csr *K, const mgpu_csr *rhs_src, double alpha, double tol,
                   int64_t max_iters, double *col_residual)
{
  const int64_t n = K->nrows;
  cudaStream_t s = ctx->stream;
  mgpu_csr *Kt = transpose_csr(ctx, K);
  mgpu_csr *Rt = rhs_src ? transpose_csr(ctx, rhs_src) : nullptr;
  DBuf bw(2 * sizeof(int), s);
  MG_CUDA(cudaMemsetAsync(bw.ptr, 0, 2 * sizeof(int), s));
  int hbw[2] = {0, 0};
  if (n > 0)
  {
    bandwidth_kernel<<<blocks_for(n), kThreads, 0, s>>>(n, K->view(), bw.as<int>());
    check_launch(ctx, "bandwidth_kernel");
    MG_CUDA(cudaMemcpyAsync(hbw, bw.ptr, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  DBuf count(sizeof(int64_t) * (n + 1), s), resid(sizeof(double) * (n > 0 ? n : 1), s),
      fit(sizeof(int64_t) * (n > 0 ? n : 1), s), err(sizeof(unsigned long long), s), pbw(sizeof(int), s);
  MG_CUDA(cudaMemsetAsync(pbw.ptr, 0, sizeof(int), s));
  MG_CUDA(cudaMemsetAsync(err.ptr, 0xff, sizeof(unsigned long long), s));
  MG_CUDA(cudaMemsetAsync(count.ptr, 0, sizeof(int64_t) * (n + 1), s));
  MG_CUDA(cudaStreamSynchronize(s));
  MrArgs a{};
  a.n = n;
  a.K = K->view();
  a.Kt = Kt->view();
  a.Rt = Rt ? Rt->view() : DCsr{nullptr, nullptr, nullptr};
  a.alpha = alpha;
  a.tol_sq = tol * tol;
  a.max_iters = max_iters;
  a.bl = hbw[0];
  a.bu = hbw[1];
  a.count = count.as<int64_t>() + 1;
  a.bw = pbw.as<int>();
  a.residual = resid.as<double>();
  a.fail_iters = fit.as<int64_t>();
  a.err = err.as<unsigned long long>();
  // one pass (count or fill) at window level lv
  int lv = 0;
  auto launch = [&](bool fill) {
    a.W = kMrW[lv];
    const int wpb = kMrWpb[lv];
    const size_t smem = sizeof(double) * 4 * static_cast<size_t>(a.W) * wpb;
    const unsigned grid = static_cast<unsigned>((n + wpb - 1) / wpb);
    auto go = [&](auto kern) {
      MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, wpb * 32, smem, s>>>(a);
    };
    if (wpb == 4)
      fill ? go(mr_columns<true, 4>) : go(mr_columns<false, 4>);
    else if (wpb == 2)
      fill ? go(mr_columns<true, 2>) : go(mr_columns<false, 2>);
    else
      fill ? go(mr_columns<true, 1>) : go(mr_columns<false, 1>);
    check_launch(ctx, fill ? "mr_columns<fill>" : "mr_columns<count>");
  };
  mgpu_csr *P = nullptr;
  try
  {
    unsigned long long h = ULLONG_MAX;
    for (;; ++lv)
    {
      if (n > 0)
        launch(false);
      MG_CUDA(cudaMemcpyAsync(&h, err.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      // the lowest failing column outgrew its window: rerun the count pass with the next wider one
      // (any other failure at a lower column would have been reported instead of it)
      if (h == ULLONG_MAX || static_cast<int>(h & 0xff) != kWindow || lv + 1 >= kMrLevels)
        break;
      MG_CUDA(cudaMemsetAsync(err.ptr, 0xff, sizeof(unsigned long long), s));
      MG_CUDA(cudaMemsetAsync(count.ptr, 0, sizeof(int64_t) * (n + 1), s));
      MG_CUDA(cudaMemsetAsync(pbw.ptr, 0, sizeof(int), s));
    }
    if (h != ULLONG_MAX)
    {
      const int64_t col = static_cast<int64_t>(h >> 8);
      const int code = static_cast<int>(h & 0xff);
      double rn = 0.0;
      int64_t it = 0;
      MG_CUDA(cudaMemcpy(&rn, resid.as<double>() + col, sizeof(double), cudaMemcpyDeviceToHost));
      MG_CUDA(cudaMemcpy(&it, fit.as<int64_t>() + col, sizeof(int64_t), cudaMemcpyDeviceToHost));
      const std::string c = std::to_string(col);
      switch (code)
      {
      case kStall:
        throw Error(MGPU_ERR_STAGNATION,
                    "spai: column " + c + " stalled at ||r|| = " + fmt_f(rn) + " after " + std::to_string(it) +
                        " iterations (tol " + fmt_f(tol) + ")",
                    col);
      case kZeroCurv:
        throw Error(MGPU_ERR_STAGNATION, "spai: zero curvature in column " + c + " with ||r|| > tol", col);
      case kNonFiniteW:
        throw Error(MGPU_ERR_NUMERICAL, "spai: non-finite values in column " + c, col);
      case kNonFiniteA:
        throw Error(MGPU_ERR_NUMERICAL, "spai: non-finite step in column " + c, col);
      default:
        throw Error(MGPU_ERR_UNSUPPORTED,
                    "spai: column " + c + " outgrew the device window (" + std::to_string(kMrW[kMrLevels - 1]) +
                        " slots; operator bandwidth " + std::to_string(hbw[0]) + "/" + std::to_string(hbw[1]) + ")",
                    col);
      }
    }
    // P^T row_ptr = scan of column counts
    mgpu_csr *PT = new mgpu_csr;
    PT->ctx = ctx;
    PT->nrows = n;
    PT->ncols = n;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&PT->row_ptr), sizeof(int64_t) * (n + 1), s));
    MG_CUDA(cudaMemcpyAsync(PT->row_ptr, count.ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
    if (n > 0)
    {
      size_t tmp = 0;
      MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, PT->row_ptr + 1, PT->row_ptr + 1, n, s));
      DBuf t(tmp, s);
      MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, PT->row_ptr + 1, PT->row_ptr + 1, n, s));
      count_launch(ctx);
    }
    int64_t nnz = 0;
    int hpbw = 0;
    MG_CUDA(cudaMemcpyAsync(&nnz, PT->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(&hpbw, pbw.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    PT->nnz = nnz;
    PT->bw = hpbw;
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&PT->col_idx), sizeof(int32_t) * (nnz > 0 ? nnz : 1), s));
    MG_CUDA(mg_malloc(reinterpret_cast<void **>(&PT->values), sizeof(double) * (nnz > 0 ? nnz : 1), s));
    a.offset = PT->row_ptr;
    a.out_rows = PT->col_idx;
    a.out_vals = PT->values;
    if (n > 0)
      launch(true);
    if (col_residual && n > 0)
      MG_CUDA(cudaMemcpyAsync(col_residual, resid.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    P = transpose_csr(ctx, PT);
    mgpu_csr_free(PT);
    MG_CUDA(cudaStreamSynchronize(s));
  }
  catch (...)
  {
    mgpu_csr_free(Kt);
    mgpu_csr_free(Rt);
    throw;
  }
  mgpu_csr_free(Kt);
  mgpu_csr_free(Rt);
  return P;
}

double fetch(mgpu_ctx *ctx, const double *dev)
{
  double h = 0.0;
  MG_CUDA(cudaMemcpyAsync(&h, dev, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  MG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_spai_build(mgpu_ctx *ctx, const mgpu_csr *K, double tol, int64_t max_col_iters, int mode, mgpu_csr **P,
                    double *col_residual)
{
  return guard(ctx, [&] {
    MG_ARG(K && P, "spai_build: null argument");
    MG_ARG(K->nrows == K->ncols, "spai_build: K must be square"); // spai.cpp:316-319
    MG_ARG(tol > 0.0, "spai_build: tol must be positive");
    MG_ARG(mode == MGPU_SPAI_FROZEN || mode == MGPU_SPAI_SEQUENTIAL, "spai_build: unknown mode");
    DBuf sc(2 * sizeof(double), ctx->stream);
    trace_inner_dev(ctx, K, K, sc.as<double>());
    trace_dev(ctx, K, sc.as<double>() + 1);
    const double denom = fetch(ctx, sc.as<double>());
    if (!(denom > 0.0))
      throw Error(MGPU_ERR_NUMERICAL, "spai_build: trace(K K^T) is not positive");
    const double alpha = fetch(ctx, sc.as<double>() + 1) / denom; // spai.cpp:329
    *P = mode == MGPU_SPAI_SEQUENTIAL ? mr_build_sequential(ctx, K, nullptr, alpha, tol, max_col_iters, col_residual)
                                      : mr_build(ctx, K, nullptr, alpha, tol, max_col_iters, col_residual);
  });
}

int mgpu_spai_update(mgpu_ctx *ctx, const mgpu_csr *K_old, const mgpu_csr *K_new, double tol, int64_t max_col_iters,
                     int mode, mgpu_csr **Q, double *col_residual)
{
  return guard(ctx, [&] {
    MG_ARG(K_old && K_new && Q, "spai_update: null argument");
    MG_ARG(K_old->nrows == K_old->ncols && K_new->nrows == K_new->ncols && K_old->nrows == K_new->nrows,
           "spai_update: operands must be square with equal shape");
    MG_ARG(tol > 0.0, "spai_update: tol must be positive");
    MG_ARG(mode == MGPU_SPAI_FROZEN || mode == MGPU_SPAI_SEQUENTIAL, "spai_update: unknown mode");
    DBuf sc(3 * sizeof(double), ctx->stream);
    trace_inner_dev(ctx, K_new, K_new, sc.as<double>());
    trace_inner_dev(ctx, K_old, K_new, sc.as<double>() + 1);
    trace_inner_dev(ctx, K_new, K_old, sc.as<double>() + 2);
    const double denom = fetch(ctx, sc.as<double>());
    if (!(denom > 0.0))
      throw Error(MGPU_ERR_NUMERICAL, "spai_update: trace(K_new^T K_new) is not positive");
    const double alpha = 0.5 * (fetch(ctx, sc.as<double>() + 1) + fetch(ctx, sc.as<double>() + 2)) / denom;
    *Q = mode == MGPU_SPAI_SEQUENTIAL // spai.cpp:348-349
             ? mr_build_sequential(ctx, K_new, K_old, alpha, tol, max_col_iters, col_residual)
             : mr_build(ctx, K_new, K_old, alpha, tol, max_col_iters, col_residual);
  });
}

} // extern "C"
