// K-asm (shifted operators), K-tr (traces), transpose, SpMV and chain apply.
//
// Rounding rules follow the reference TUs, which are built without -mfma:
// every a*x + b*y is two products and one add, each rounded (__dmul_rn /
// __dadd_rn keep nvcc from contracting them into FMAs).  SpMV rows accumulate
// in ascending column order exactly like kernels_scalar.cpp:39-47, so a
// device SpMV is bitwise identical to the reference's scalar gather_dot.
#include <cub/cub.cuh>

#include <climits>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace mgpu
{
namespace
{

// Streaming merge of row i of (a*A + b*B) and, when `third`, of
// sp_add(that, C, 1, 1): the composition shifted_operator performs
// (system.cpp:64-68 -> sparse.cpp:167-218), including the exact-zero drop of
// the intermediate md row (sparse.cpp:209).  Emits when out_ci != nullptr.
template <bool kThird>
__device__ __forceinline__ int64_t merge_row(int64_t i, DCsr A, DCsr B, DCsr Cm, double a, double b, int32_t *out_ci,
                                             double *out_v, int32_t *lohi = nullptr)
{
  int64_t ka = A.rp[i], ea = A.rp[i + 1];
  int64_t kb = B.rp[i], eb = B.rp[i + 1];
  int64_t kc = 0, ec = 0;
  if (kThird)
  {
    kc = Cm.rp[i];
    ec = Cm.rp[i + 1];
  }
  int64_t cnt = 0;
  while (ka < ea || kb < eb || kc < ec)
  {
    const int32_t ca = ka < ea ? A.ci[ka] : INT_MAX;
    const int32_t cb = kb < eb ? B.ci[kb] : INT_MAX;
    const int32_t cc = kc < ec ? Cm.ci[kc] : INT_MAX;
    const int32_t col = min(ca, min(cb, cc));
    bool has1 = false;
    double v1 = 0.0;
    if (ca == col && cb == col)
    {
      v1 = __dadd_rn(__dmul_rn(a, A.v[ka]), __dmul_rn(b, B.v[kb]));
      ++ka;
      ++kb;
      has1 = true;
    }
    else if (ca == col)
    {
      v1 = __dmul_rn(a, A.v[ka]);
      ++ka;
      has1 = true;
    }
    else if (cb == col)
    {
      v1 = __dmul_rn(b, B.v[kb]);
      ++kb;
      has1 = true;
    }
    if (has1 && v1 == 0.0)
      has1 = false; // the intermediate CSR never stores it
    double v;
    bool emit;
    if (kThird)
    {
      const bool hasc = cc == col;
      // sp_add_scaled(md, C, 1.0, 1.0): 1.0 * x == x exactly
      if (has1 && hasc)
        v = __dadd_rn(v1, Cm.v[kc]);
      else if (has1)
        v = v1;
      else
        v = hasc ? Cm.v[kc] : 0.0;
      if (hasc)
        ++kc;
      emit = (has1 || hasc) && v != 0.0;
    }
    else
    {
      v = v1;
      emit = has1;
    }
    if (emit)
    {
      if (lohi)
      {
        lohi[0] = min(lohi[0], col);
        lohi[1] = max(lohi[1], col);
      }
      if (out_ci)
      {
        out_ci[cnt] = col;
        out_v[cnt] = v;
      }
      ++cnt;
    }
  }
  return cnt;
}

struct ShiftArgs
{
  int *bw; // [128]: bandwidth of each output, then its longest row (atomicMax in the count pass)
  double a[64];
  double b[64];
  int64_t *rp[64];
  int32_t *ci[64];
  double *v[64];
};

template <bool kThird>
__global__ void add_count_kernel(int l, int64_t n, DCsr A, DCsr B, DCsr Cm, ShiftArgs args)
{
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(l) * n)
    return;
  const int p = static_cast<int>(g / n);
  const int64_t i = g - static_cast<int64_t>(p) * n;
  int32_t lohi[2] = {INT_MAX, -1};
  const int64_t cnt = merge_row<kThird>(i, A, B, Cm, args.a[p], args.b[p], nullptr, nullptr, lohi);
  args.rp[p][i + 1] = cnt;
  if (i == 0)
    args.rp[p][0] = 0;
  // reduce over the lanes of the same point first: one atomic per warp and point
  int bwv = cnt > 0 ? static_cast<int>(max(i - lohi[0], static_cast<int64_t>(lohi[1]) - i)) : 0;
  int mr = static_cast<int>(cnt);
  const unsigned grp = __match_any_sync(__activemask(), p);
  bwv = __reduce_max_sync(grp, bwv);
  mr = __reduce_max_sync(grp, mr);
  if ((threadIdx.x & 31) == __ffs(grp) - 1)
  {
    atomicMax(&args.bw[p], bwv);
    atomicMax(&args.bw[64 + p], mr);
  }
}

template <bool kThird>
__global__ void add_fill_kernel(int l, int64_t n, DCsr A, DCsr B, DCsr Cm, ShiftArgs args)
{
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(l) * n)
    return;
  const int p = static_cast<int>(g / n);
  const int64_t i = g - static_cast<int64_t>(p) * n;
  const int64_t off = args.rp[p][i];
  merge_row<kThird>(i, A, B, Cm, args.a[p], args.b[p], args.ci[p] + off, args.v[p] + off);
}

// Inclusive scan of rp[1..n] in place (rp[0] = 0 already).
void scan_row_ptr(mgpu_ctx *ctx, int64_t *rp, int64_t n)
{
  if (n == 0)
    return;
  size_t tmp = 0;
  MG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, rp + 1, rp + 1, n, ctx->stream));
  DBuf t(tmp, ctx->stream);
  MG_CUDA(cub::DeviceScan::InclusiveSum(t.ptr, tmp, rp + 1, rp + 1, n, ctx->stream));
  count_launch(ctx);
}

struct RpBatch
{
  int64_t *rp[64];
};

// Inclusive scan of rp[1..n] for up to 64 row-pointer arrays, one block each
// (kScanItems consecutive entries per thread), totals[p] = rp[p][n].
constexpr int kScanTB = 512, kScanItems = 8;
__global__ void __launch_bounds__(kScanTB) scan_rows_batched(int64_t n, RpBatch rb, int64_t *__restrict__ totals)
{
  using BS = cub::BlockScan<int64_t, kScanTB>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  int64_t *rp = rb.rp[blockIdx.x];
  if (threadIdx.x == 0)
    carry = 0;
  __syncthreads();
  for (int64_t base = 1; base <= n; base += static_cast<int64_t>(kScanTB) * kScanItems)
  {
    const int64_t i0 = base + static_cast<int64_t>(threadIdx.x) * kScanItems;
    int64_t v[kScanItems];
    int64_t sum = 0;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u)
    {
      v[u] = i0 + u <= n ? rp[i0 + u] : 0;
      sum += v[u];
    }
    int64_t excl, agg;
    BS(tmp).ExclusiveSum(sum, excl, agg);
    int64_t run = carry + excl;
#pragma unroll
    for (int u = 0; u < kScanItems; ++u)
    {
      run += v[u];
      if (i0 + u <= n)
        rp[i0 + u] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0)
    totals[blockIdx.x] = carry;
}

// Batched sp_add over up to 64 (a_i, b_i) pairs, optionally + C.
template <bool kThird>
void batched_add(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, const mgpu_csr *Cm, int l, const double *as,
                 const double *bs, mgpu_csr **out)
{
  const int64_t n = A->nrows;
  for (int base = 0; base < l; base += 64)
  {
    const int cnt = l - base < 64 ? l - base : 64;
    ShiftArgs args{};
    std::vector<mgpu_csr *> made;
    try
    {
    for (int p = 0; p < cnt; ++p)
    {
      args.a[p] = as[base + p];
      args.b[p] = bs[base + p];
      mgpu_csr *o = new mgpu_csr;
      o->ctx = ctx;
      o->nrows = n;
      o->ncols = A->ncols;
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&o->row_ptr), sizeof(int64_t) * (n + 1), ctx->stream));
      made.push_back(o);
      args.rp[p] = o->row_ptr;
    }
    const DCsr cv = kThird ? Cm->view() : DCsr{nullptr, nullptr, nullptr};
    const int64_t total = static_cast<int64_t>(cnt) * n;
    DBuf bwbuf(sizeof(int) * 128, ctx->stream);
    MG_CUDA(cudaMemsetAsync(bwbuf.ptr, 0, sizeof(int) * 128, ctx->stream));
    args.bw = bwbuf.as<int>();
    if (n > 0)
    {
      add_count_kernel<kThird><<<blocks_for(total), kThreads, 0, ctx->stream>>>(cnt, n, A->view(), B->view(), cv, args);
      check_launch(ctx, "add_count_kernel");
    }
    else
    {
      for (int p = 0; p < cnt; ++p)
        MG_CUDA(cudaMemsetAsync(args.rp[p], 0, sizeof(int64_t), ctx->stream));
    }
    std::vector<int64_t> nnz(static_cast<size_t>(cnt), 0);
    int hbw[128] = {0};
    auto *hpin = static_cast<int64_t *>(pinned_scratch(ctx, sizeof(int64_t) * 64 + sizeof(int) * 128));
    if (n > 0 && n <= 262144)
    {
      // short operators: one launch scans every row pointer, one copy returns every nnz
      RpBatch rb{};
      for (int p = 0; p < cnt; ++p)
        rb.rp[p] = args.rp[p];
      DBuf tot(sizeof(int64_t) * 64, ctx->stream);
      scan_rows_batched<<<cnt, kScanTB, 0, ctx->stream>>>(n, rb, tot.as<int64_t>());
      check_launch(ctx, "scan_rows_batched");
      MG_CUDA(cudaMemcpyAsync(hpin, tot.ptr, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    }
    else
    {
      for (int p = 0; p < cnt; ++p)
      {
        scan_row_ptr(ctx, args.rp[p], n);
        MG_CUDA(cudaMemcpyAsync(hpin + p, args.rp[p] + n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
    // pinned staging: the copies stay asynchronous, one synchronisation for all of them
    MG_CUDA(cudaMemcpyAsync(hpin + 64, bwbuf.ptr, sizeof(int) * 128, cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(nnz.data(), hpin, sizeof(int64_t) * cnt);
    std::memcpy(hbw, hpin + 64, sizeof(int) * 128);
    for (int p = 0; p < cnt; ++p)
    {
      made[p]->bw = hbw[p];
      made[p]->maxrow = hbw[64 + p];
    }
    for (int p = 0; p < cnt; ++p)
    {
      mgpu_csr *o = made[p];
      o->nnz = nnz[p];
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&o->col_idx), sizeof(int32_t) * (nnz[p] > 0 ? nnz[p] : 1),
                              ctx->stream));
      MG_CUDA(mg_malloc(reinterpret_cast<void **>(&o->values), sizeof(double) * (nnz[p] > 0 ? nnz[p] : 1),
                              ctx->stream));
      args.ci[p] = o->col_idx;
      args.v[p] = o->values;
    }
    if (n > 0)
    {
      add_fill_kernel<kThird><<<blocks_for(total), kThreads, 0, ctx->stream>>>(cnt, n, A->view(), B->view(), cv, args);
      check_launch(ctx, "add_fill_kernel");
    }
    }
    catch (...)
    {
      // nothing is handed out on failure: this chunk's matrices and the earlier chunks' outputs
      for (auto *o : made)
        mgpu_csr_free(o);
      for (int q = 0; q < base; ++q)
      {
        mgpu_csr_free(out[q]);
        out[q] = nullptr;
      }
      throw;
    }
    for (int p = 0; p < cnt; ++p)
      out[base + p] = made[p];
  }
}

__global__ void diag_values(int64_t n, DCsr A, double *__restrict__ out)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int64_t lo = A.rp[i], hi = A.rp[i + 1];
  const int64_t end = hi;
  while (lo < hi) // sparse.cpp:92-106 at(i, i)
  {
    const int64_t mid = lo + (hi - lo) / 2;
    if (A.ci[mid] < i)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[i] = (lo < end && A.ci[lo] == i) ? A.v[lo] : 0.0;
}

// Per-row partial of trace_inner (sparse.cpp:262-296), row entries in order.
__global__ void row_inner(int64_t n, DCsr A, DCsr B, double *__restrict__ out)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  int64_t ka = A.rp[i], kb = B.rp[i];
  const int64_t ea = A.rp[i + 1], eb = B.rp[i + 1];
  double acc = 0.0;
  while (ka < ea && kb < eb)
  {
    const int32_t ca = A.ci[ka], cb = B.ci[kb];
    if (ca < cb)
      ++ka;
    else if (cb < ca)
      ++kb;
    else
    {
      acc = __dadd_rn(acc, __dmul_rn(A.v[ka], B.v[kb]));
      ++ka;
      ++kb;
    }
  }
  out[i] = acc;
}

__global__ void count_cols(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           int64_t *__restrict__ col_counts)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
    atomicAdd(reinterpret_cast<unsigned long long *>(&col_counts[static_cast<int64_t>(ci[k]) + 1]), 1ull);
}

// Bucket every entry into its column (arbitrary order inside a column).
__global__ void scatter_cols(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                             const int64_t *__restrict__ rpt, unsigned long long *__restrict__ cursor,
                             int64_t *__restrict__ perm, int32_t *__restrict__ trow)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
  {
    const int64_t j = ci[k];
    const int64_t pos = rpt[j] + static_cast<int64_t>(atomicAdd(&cursor[j], 1ull));
    perm[pos] = k;
    trow[pos] = static_cast<int32_t>(i);
  }
}

// Order each column by source position.  Source positions grow with the row
// (row-major CSR), so this is ascending original-row order (sparse.cpp:238-247);
// keys are unique, so the result does not depend on the bucketing order above.
__global__ void sort_cols(int64_t ncols, const int64_t *__restrict__ rpt, int64_t *__restrict__ perm,
                          int32_t *__restrict__ trow)
{
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= ncols)
    return;
  const int64_t b = rpt[j], len = rpt[j + 1] - b;
  int64_t *pk = perm + b;
  int32_t *pr = trow + b;
  // shell sort (gaps 3h+1): insertion sort for the short columns of banded operators,
  // bounded work for an occasional long one
  int64_t h = 1;
  while (h < len / 3)
    h = 3 * h + 1;
  for (; h >= 1; h /= 3)
    for (int64_t u = h; u < len; ++u)
    {
      const int64_t kv = pk[u];
      const int32_t rv = pr[u];
      int64_t v = u;
      while (v >= h && pk[v - h] > kv)
      {
        pk[v] = pk[v - h];
        pr[v] = pr[v - h];
        v -= h;
      }
      pk[v] = kv;
      pr[v] = rv;
    }
}

__global__ void gather_values(int64_t nnz, const int64_t *__restrict__ perm, const double *__restrict__ src,
                              double *__restrict__ dst)
{
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz)
    dst[k] = src[perm[k]];
}
} // namespace

// Transpose that also returns perm (T.values[k] = A.values[perm[k]]), so the
// same pattern can be re-transposed for new values with a gather.  Sort-free:
// column counts -> scan -> bucket -> per-column order by source position.
mgpu_csr *transpose_perm(mgpu_ctx *ctx, const mgpu_csr *A, DBuf &perm)
{
  mgpu_csr *T = new_csr(ctx, A->ncols, A->nrows, A->nnz);
  T->may_hold_zeros = A->may_hold_zeros;
  T->bw = A->bw; // max |i - j| is transpose invariant
  MG_CUDA(cudaMemsetAsync(T->row_ptr, 0, sizeof(int64_t) * (A->ncols + 1), ctx->stream));
  perm = DBuf(sizeof(int64_t) * (A->nnz > 0 ? A->nnz : 1), ctx->stream);
  if (A->nnz == 0)
    return T;
  count_cols<<<blocks_for(A->nrows), kThreads, 0, ctx->stream>>>(A->nrows, A->row_ptr, A->col_idx, T->row_ptr);
  check_launch(ctx, "count_cols");
  scan_row_ptr(ctx, T->row_ptr, A->ncols);
  DBuf cursor(sizeof(unsigned long long) * (A->ncols > 0 ? A->ncols : 1), ctx->stream);
  MG_CUDA(cudaMemsetAsync(cursor.ptr, 0, sizeof(unsigned long long) * A->ncols, ctx->stream));
  scatter_cols<<<blocks_for(A->nrows), kThreads, 0, ctx->stream>>>(
      A->nrows, A->row_ptr, A->col_idx, T->row_ptr, cursor.as<unsigned long long>(), perm.as<int64_t>(), T->col_idx);
  check_launch(ctx, "scatter_cols");
  sort_cols<<<blocks_for(A->ncols), kThreads, 0, ctx->stream>>>(A->ncols, T->row_ptr, perm.as<int64_t>(), T->col_idx);
  check_launch(ctx, "sort_cols");
  gather_values<<<blocks_for(A->nnz), kThreads, 0, ctx->stream>>>(A->nnz, perm.as<int64_t>(), A->values, T->values);
  check_launch(ctx, "gather_values");
  return T;
}

// Device CSR transpose, deterministic (each transposed row in ascending
// original-row order, sparse.cpp:238-247).
mgpu_csr *transpose_csr(mgpu_ctx *ctx, const mgpu_csr *A)
{
  DBuf perm;
  return transpose_perm(ctx, A, perm);
}

namespace
{
struct GatherBatch
{
  const double *src[64];
  double *dst[64];
};
__global__ void gather_batched_kernel(int l, int64_t nnz, const int64_t *__restrict__ perm, GatherBatch gb)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(l) * nnz)
    return;
  const int p = static_cast<int>(t / nnz);
  const int64_t k = t - static_cast<int64_t>(p) * nnz;
  gb.dst[p][k] = gb.src[p][perm[k]];
}
} // namespace

// dst[p][k] = src[p][perm[k]] for l value arrays sharing one permutation (one launch per 64).
void gather_batched(mgpu_ctx *ctx, int l, int64_t nnz, const int64_t *perm, const double *const *src,
                    double *const *dst)
{
  if (nnz == 0)
    return;
  for (int b = 0; b < l; b += 64)
  {
    const int c = l - b < 64 ? l - b : 64;
    GatherBatch gb{};
    for (int p = 0; p < c; ++p)
    {
      gb.src[p] = src[b + p];
      gb.dst[p] = dst[b + p];
    }
    gather_batched_kernel<<<blocks_for(static_cast<int64_t>(c) * nnz), kThreads, 0, ctx->stream>>>(c, nnz, perm, gb);
    check_launch(ctx, "gather_batched");
  }
}

void gather_dev(mgpu_ctx *ctx, int64_t nnz, const int64_t *perm, const double *src, double *dst)
{
  if (nnz == 0)
    return;
  gather_values<<<blocks_for(nnz), kThreads, 0, ctx->stream>>>(nnz, perm, src, dst);
  check_launch(ctx, "gather_values");
}

void trace_dev(mgpu_ctx *ctx, const mgpu_csr *A, double *out_dev)
{
  const int64_t n = A->nrows < A->ncols ? A->nrows : A->ncols;
  DBuf vals(sizeof(double) * (n > 0 ? n : 1), ctx->stream);
  if (n > 0)
  {
    diag_values<<<blocks_for(n), kThreads, 0, ctx->stream>>>(n, A->view(), vals.as<double>());
    check_launch(ctx, "diag_values");
  }
  det_sum(ctx, vals.as<double>(), n, out_dev);
}

void trace_inner_dev(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double *out_dev)
{
  MG_ARG(A->nrows == B->nrows && A->ncols == B->ncols, "trace_inner: shape mismatch");
  const int64_t n = A->nrows;
  DBuf vals(sizeof(double) * (n > 0 ? n : 1), ctx->stream);
  if (n > 0)
  {
    row_inner<<<blocks_for(n), kThreads, 0, ctx->stream>>>(n, A->view(), B->view(), vals.as<double>());
    check_launch(ctx, "row_inner");
  }
  det_sum(ctx, vals.as<double>(), n, out_dev);
}

namespace
{
__global__ void spmv_kernel(int64_t n, DCsr A, const double *__restrict__ x, double *__restrict__ y)
{
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n)
    return;
  double acc = 0.0;
  for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
    acc = __dadd_rn(acc, __dmul_rn(A.v[k], x[A.ci[k]]));
  y[i] = acc;
}
} // namespace

void spmv_dev(mgpu_ctx *ctx, const mgpu_csr *A, const double *x, double *y)
{
  if (A->nrows == 0)
    return;
  spmv_kernel<<<blocks_for(A->nrows), kThreads, 0, ctx->stream>>>(A->nrows, A->view(), x, y);
  check_launch(ctx, "spmv_kernel");
}

} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_sp_add_scaled(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double a, double b, mgpu_csr **out)
{
  return guard(ctx, [&] {
    MG_ARG(A && B && out, "sp_add_scaled: null argument");
    MG_ARG(A->nrows == B->nrows && A->ncols == B->ncols, "sp_add_scaled: shape mismatch");
    batched_add<false>(ctx, A, B, nullptr, 1, &a, &b, out);
  });
}

int mgpu_shifted_operators(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int l,
                           const double *shifts, mgpu_csr **out)
{
  return guard(ctx, [&] {
    MG_ARG(M && D && K && shifts && out && l >= 0, "shifted_operators: null argument");
    MG_ARG(M->nrows == D->nrows && M->nrows == K->nrows && M->ncols == D->ncols && M->ncols == K->ncols,
           "sp_add_scaled: shape mismatch");
    std::vector<double> a(static_cast<size_t>(l)), b(static_cast<size_t>(l));
    for (int i = 0; i < l; ++i)
    {
      a[i] = shifts[i] * shifts[i]; // system.cpp:66: s * s on the host, like the reference
      b[i] = shifts[i];
    }
    batched_add<true>(ctx, M, D, K, l, a.data(), b.data(), out);
  });
}

int mgpu_transpose(mgpu_ctx *ctx, const mgpu_csr *A, mgpu_csr **out)
{
  return guard(ctx, [&] {
    MG_ARG(A && out, "transpose: null argument");
    *out = transpose_csr(ctx, A);
  });
}

int mgpu_trace(mgpu_ctx *ctx, const mgpu_csr *A, double *out)
{
  return guard(ctx, [&] {
    MG_ARG(A && out, "trace: null argument");
    DBuf d(sizeof(double), ctx->stream);
    trace_dev(ctx, A, d.as<double>());
    MG_CUDA(cudaMemcpyAsync(out, d.ptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mgpu_trace_inner(mgpu_ctx *ctx, const mgpu_csr *A, const mgpu_csr *B, double *out)
{
  return guard(ctx, [&] {
    MG_ARG(A && B && out, "trace_inner: null argument");
    DBuf d(sizeof(double), ctx->stream);
    trace_inner_dev(ctx, A, B, d.as<double>());
    MG_CUDA(cudaMemcpyAsync(out, d.ptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int mgpu_spmv(mgpu_ctx *ctx, const mgpu_csr *A, const double *x, double *y)
{
  return guard(ctx, [&] {
    MG_ARG(A && x && y, "spmv: null argument");
    spmv_dev(ctx, A, x, y);
  });
}

int mgpu_chain_apply(mgpu_ctx *ctx, int z, const mgpu_csr *const *factors, const double *x, double *y,
                     mgpu_memkind where)
{
  return guard(ctx, [&] {
    MG_ARG(z >= 0 && x && y && (z == 0 || factors), "chain_apply: null argument");
    MG_ARG(z > 0 || where == MGPU_HOST || where == MGPU_DEVICE, "chain_apply: bad memory kind");
    if (z == 0)
    {
      // empty chain = identity (spai.hpp:77-78); dimension comes from the caller
      throw Error(MGPU_ERR_ARG, "chain_apply: empty chain needs the vector length; use a copy");
    }
    const int64_t n = factors[0]->nrows;
    for (int f = 0; f < z; ++f)
      MG_ARG(factors[f]->nrows == n && factors[f]->ncols == n, "chain_apply: dimension mismatch");
    DBuf a(sizeof(double) * (n > 0 ? n : 1), ctx->stream), b(sizeof(double) * (n > 0 ? n : 1), ctx->stream);
    MG_CUDA(cudaMemcpyAsync(a.ptr, x, sizeof(double) * n,
                            where == MGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
    double *src = a.as<double>(), *dst = b.as<double>();
    for (int f = z - 1; f >= 0; --f) // oldest (last) factor first, spai.cpp:368
    {
      spmv_dev(ctx, factors[f], src, dst);
      std::swap(src, dst);
    }
    MG_CUDA(cudaMemcpyAsync(y, src, sizeof(double) * n,
                            where == MGPU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
    MG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

} // extern "C"
