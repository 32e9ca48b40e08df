// Global Arnoldi + projection on the device:
//
//   thin_qr         dense.cpp:153-246   Householder QR of the n x k basis block
//   project_reduce  airga.cpp:485-500   Mh, Dh, Kh = V^T S V, Fh = V^T F, Cph/Cvh = C V
//   arnoldi_deflate airga.cpp:456-473   X -= <B_t, X> B_t over two sweeps
//
// thin_qr is one cooperative persistent kernel that follows the reference's
// column loop: per column k a tail norm (sigma^2 = x_k^2 + sum_{i>k} x_i^2),
// the Householder vector, the trailing dots tau <v, y_j> (warps split the
// columns, lanes the rows of a block's fixed row slab) and the rank-1 update,
// three grid barriers per column.  The rank test, the zeroed flushed columns,
// Q = H_0 ... H_{n-1} E applied per column in descending k, the sign fix and
// the rank count are the reference's; its serial dots become fixed-order
// trees (deterministic, ~1e-16 relative).  Every scalar update is an
// unfused multiply then add, like the scalar kernel table.
//
// project_reduce: V^T (S V) for M, D, K in one fused kernel (proj_fused below: the S V tiles are
// formed in shared memory in CSR row order, spmv_into's order, and never written to HBM); V^T F,
// Cp V, Cv V are hand-written FP64 GEMMs (dense_gemm.cu).  No cuBLAS.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
namespace
{

constexpr int kQrTB = 256;
constexpr int kQrMaxCols = 1024;

__device__ __forceinline__ double qr_warp_sum(double v)
{
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__device__ double qr_block_sum(double v, double *red)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = qr_warp_sum(v);
  if (lane == 0)
    red[warp] = v;
  __syncthreads();
  double t = lane < kQrTB / 32 ? red[lane] : 0.0;
  t = qr_warp_sum(t);
  __syncthreads();
  return t; // every thread
}

struct QrArgs
{
  int64_t m; // rows
  int n;     // columns
  double *W; // m x n column-major: A in, Householder vectors (rows >= k of column k) + R above out
  double *Q; // m x n
  double *diag, *tau;
  double tol;
  double *part; // [G][n + 1]
  int k0, k1;   // qr_factor: the panel [k0, k1); reflectors update columns < k1 only
};

// Factorisation: dense.cpp:165-190.
__global__ void __launch_bounds__(kQrTB) qr_factor(QrArgs a)
{
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double red[kQrTB / 32];
  __shared__ double sj[kQrMaxCols];
  const int64_t m = a.m;
  const int n = a.n;
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t r0 = m * b / G, r1 = m * (b + 1) / G; // this block's row slab
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *part = a.part + static_cast<int64_t>(b) * (n + 1);
  for (int k = a.k0; k < a.k1; ++k)
  {
    double *x = a.W + static_cast<int64_t>(k) * m;
    // ---- tail norm over rows > k
    double t = 0.0;
    for (int64_t i = max(r0, static_cast<int64_t>(k) + 1) + threadIdx.x; i < r1; i += kQrTB)
    {
      const double xi = x[i];
      t = __dadd_rn(t, __dmul_rn(xi, xi));
    }
    t = qr_block_sum(t, red);
    if (threadIdx.x == 0)
      part[0] = t;
    grid.sync();
    double tail = 0.0;
    for (int bb = 0; bb < G; ++bb) // fixed order, identical in every block
      tail = __dadd_rn(tail, __ldcg(a.part + static_cast<int64_t>(bb) * (n + 1)));
    const double x0 = __ldcg(x + k);
    const double sigma = sqrt(__dadd_rn(__dmul_rn(x0, x0), tail));
    if (sigma <= a.tol)
    {
      // rank-deficient direction (dense.cpp:168-174)
      for (int64_t i = max(r0, static_cast<int64_t>(k)) + threadIdx.x; i < r1; i += kQrTB)
        x[i] = 0.0;
      if (b == 0 && threadIdx.x == 0)
      {
        a.diag[k] = 0.0;
        a.tau[k] = 0.0;
      }
      grid.sync();
      continue;
    }
    const double alpha = x0 >= 0.0 ? -sigma : sigma;
    const double v0 = __dsub_rn(x0, alpha);
    const double vtv = __dadd_rn(__dmul_rn(v0, v0), tail);
    const double tk = vtv > 0.0 ? 2.0 / vtv : 0.0;
    if (b == 0 && threadIdx.x == 0)
    {
      a.diag[k] = alpha;
      a.tau[k] = tk;
    }
    // ---- dots <v, y_j> for j > k over this block's rows (v_k = v0)
    for (int j = k + 1 + warp; j < a.k1; j += kQrTB / 32)
    {
      const double *y = a.W + static_cast<int64_t>(j) * m;
      double d = 0.0;
      for (int64_t i = max(r0, static_cast<int64_t>(k)) + lane; i < r1; i += 32)
      {
        const double xi = i == k ? v0 : x[i];
        d = __dadd_rn(d, __dmul_rn(xi, y[i]));
      }
      d = qr_warp_sum(d);
      if (lane == 0)
        part[1 + j] = d;
    }
    grid.sync();
    for (int j = k + 1 + threadIdx.x; j < a.k1; j += kQrTB)
    {
      double d = 0.0;
      for (int bb = 0; bb < G; ++bb)
        d = __dadd_rn(d, __ldcg(a.part + static_cast<int64_t>(bb) * (n + 1) + 1 + j));
      sj[j] = __dmul_rn(tk, d); // s = tau * dot (dense.cpp:187)
    }
    __syncthreads();
    // ---- y_j -= s_j v over this block's rows (dense.cpp:188)
    const int64_t lo = max(r0, static_cast<int64_t>(k));
    for (int j = k + 1; j < a.k1; ++j) // column-outer: no per-element index division
    {
      double *y = a.W + static_cast<int64_t>(j) * m;
      const double ns = -sj[j];
      for (int64_t i = lo + threadIdx.x; i < r1; i += kQrTB)
      {
        const double xi = i == k ? v0 : x[i];
        y[i] = __dadd_rn(y[i], __dmul_rn(ns, xi));
      }
    }
    __syncthreads();
    if (k >= r0 && k < r1 && threadIdx.x == 0)
      x[k] = v0;
    grid.sync();
  }
}

// Q = H_0 ... H_{n-1} E_n (dense.cpp:205-224): column j gets H_j, ..., H_0 in
// that order; a descending k over all columns j >= k is the same sequence per column.
__global__ void __launch_bounds__(kQrTB) qr_form_q(QrArgs a)
{
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double sj[kQrMaxCols];
  const int64_t m = a.m;
  const int n = a.n;
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t r0 = m * b / G, r1 = m * (b + 1) / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *part = a.part + static_cast<int64_t>(b) * (n + 1);
  // Q = E on the kept columns, zero elsewhere
  for (int j = 0; j < n; ++j)
  {
    const bool keep = a.diag[j] != 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kQrTB)
      a.Q[static_cast<int64_t>(j) * m + i] = (i == j && keep) ? 1.0 : 0.0;
  }
  grid.sync();
  for (int k = n - 1; k >= 0; --k)
  {
    const double tk = a.tau[k];
    if (tk == 0.0)
      continue;
    const double *v = a.W + static_cast<int64_t>(k) * m;
    const int64_t lo = max(r0, static_cast<int64_t>(k));
    for (int j = k + warp; j < n; j += kQrTB / 32)
    {
      if (a.diag[j] == 0.0)
        continue;
      const double *q = a.Q + static_cast<int64_t>(j) * m;
      double d = 0.0;
      for (int64_t i = lo + lane; i < r1; i += 32)
        d = __dadd_rn(d, __dmul_rn(v[i], q[i]));
      d = qr_warp_sum(d);
      if (lane == 0)
        part[1 + j] = d;
    }
    grid.sync();
    for (int j = k + threadIdx.x; j < n; j += kQrTB)
    {
      double d = 0.0;
      if (a.diag[j] != 0.0)
        for (int bb = 0; bb < G; ++bb)
          d = __dadd_rn(d, __ldcg(a.part + static_cast<int64_t>(bb) * (n + 1) + 1 + j));
      sj[j] = __dmul_rn(tk, d);
    }
    __syncthreads();
    for (int j = k; j < n; ++j)
    {
      if (a.diag[j] == 0.0)
        continue;
      double *q = a.Q + static_cast<int64_t>(j) * m;
      const double ns = -sj[j];
      for (int64_t i = lo + threadIdx.x; i < r1; i += kQrTB)
        q[i] = __dadd_rn(q[i], __dmul_rn(ns, v[i]));
    }
    grid.sync();
  }
}

// R (n x n) from W and diag, with the sign fix of dense.cpp:227-239 (rows with a
// negative diagonal flip, and so do the matching Q columns).
__global__ void qr_form_r(int64_t m, int n, const double *__restrict__ W, const double *__restrict__ diag,
                          double *__restrict__ R)
{
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(n) * n)
    return;
  const int k = static_cast<int>(e / n), i = static_cast<int>(e % n); // column k, row i
  double v = i < k ? W[static_cast<int64_t>(k) * m + i] : (i == k ? diag[k] : 0.0);
  if (i <= k && diag[i] < 0.0)
    v = -v;
  R[e] = v;
}

__global__ void qr_sign_q(int64_t m, int n, const double *__restrict__ diag, double *__restrict__ Q)
{
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<int64_t>(n) * m)
    return;
  if (diag[e / m] < 0.0)
    Q[e] = __dmul_rn(-1.0, Q[e]);
}

// Panel p = columns [j0, j0 + jb): V (rows j0..m-1, jb columns, ld mv = m - j0) with the
// Householder vectors as qr_factor leaves them (v_k(k) = v0 stored, rows above k zeroed).
__global__ void qr_panel_v(int64_t m, int64_t j0, int jb, const double *__restrict__ W, double *__restrict__ V)
{
  const int64_t mv = m - j0;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= mv * jb)
    return;
  const int c = static_cast<int>(t / mv);
  const int64_t i = t - static_cast<int64_t>(c) * mv; // row j0 + i
  V[t] = i < c ? 0.0 : W[(j0 + c) * m + j0 + i];
}

// Compact WY (forward, columnwise): H_0 ... H_{jb-1} = I - V T V^T with T upper triangular,
// T_kk = tau_k, T(0:k, k) = -tau_k T(0:k, 0:k) G(0:k, k), G = V^T V.  One warp.
__global__ void qr_panel_t(int jb, const double *__restrict__ G, const double *__restrict__ tau, double *__restrict__ T)
{
  const int i = threadIdx.x;
  for (int e = i; e < jb * jb; e += 32)
    T[e] = 0.0;
  __syncwarp();
  for (int k = 0; k < jb; ++k)
  {
    const double tk = tau[k];
    if (i < k)
    {
      double acc = 0.0;
      for (int l = i; l < k; ++l)
        acc = __dadd_rn(acc, __dmul_rn(T[l * jb + i], G[k * jb + l]));
      T[k * jb + i] = __dmul_rn(-tk, acc);
    }
    if (i == 0)
      T[k * jb + k] = tk;
    __syncwarp();
  }
}

// Q = E on the kept columns (diag != 0), zero elsewhere (dense.cpp:207-212).
__global__ void qr_init_q(int64_t m, int n, const double *__restrict__ diag, double *__restrict__ Q)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= m * n)
    return;
  const int64_t j = t / m, i = t - j * m;
  Q[t] = (i == j && diag[j] != 0.0) ? 1.0 : 0.0;
}

__global__ void square_all(int64_t count, const double *__restrict__ x, double *__restrict__ out)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count)
    out[t] = __dmul_rn(x[t], x[t]);
}

__global__ void product_all(int64_t count, const double *__restrict__ x, const double *__restrict__ y,
                            double *__restrict__ out)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < count)
    out[t] = __dmul_rn(x[t], y[t]);
}

// X -= g B unless g == 0 (airga.cpp:464-467), g read from device memory.
__global__ void deflate_axpy(int64_t count, const double *__restrict__ g, const double *__restrict__ B,
                             double *__restrict__ X)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const double gv = *g;
  if (t < count && gv != 0.0)
    X[t] = __dadd_rn(X[t], __dmul_rn(-gv, B[t]));
}

// V_slab^T (S_o V) for the three operators at once, S_o V never leaving the SM (verdict: no
// intermediate in HBM).  Block (tile, split): a 64 x 64 tile (ta, tb) of the three r x r outputs
// over the slab rows of its split, 16 rows at a time:
//   Ya  = Y[rows, ta cols]                                   (shared memory)
//   W_o = S_o[rows, :] Vext[:, tb cols]  (each row in CSR order, spmv_into, no FMA)  (shared memory)
//   acc_o += Ya^T W_o                                        (4 x 4 per thread, DFMA)
// Partial tiles go to part[split][o][r][r]; proj_reduce sums the splits in order (deterministic).
constexpr int kPT = 64, kPR = 16; // 16-row chunks: 33 KB of static shared memory

__global__ void __launch_bounds__(256) proj_fused(int64_t p, int64_t r, DCsr S0, DCsr S1, DCsr S2,
                                                  const double *__restrict__ V, int64_t ext0, int64_t ldv,
                                                  int64_t y0, int64_t rows_per_split, double *__restrict__ part)
{
  __shared__ double Ya[kPR][kPT + 1];
  __shared__ double Wo[3][kPR][kPT + 1];
  const int64_t ntile = (r + kPT - 1) / kPT;
  const int64_t ta = blockIdx.x % ntile, tb = blockIdx.x / ntile;
  const int64_t a0 = ta * kPT, b0 = tb * kPT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t lo = static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t hi = p < lo + rows_per_split ? p : lo + rows_per_split;
  const DCsr S[3] = {S0, S1, S2};
  double acc[3][4][4] = {};
  for (int64_t i0 = lo; i0 < hi; i0 += kPR)
  {
    // Ya: slab rows i0 .. i0 + 31 of basis columns a0 .. a0 + 63 (threads along rows: coalesced)
    for (int t = threadIdx.x; t < kPR * kPT; t += 256)
    {
      const int i = t % kPR, a = t / kPR;
      const int64_t gi = i0 + i, ga = a0 + a;
      Ya[i][a] = (gi < hi && ga < r) ? V[ga * ldv + y0 + gi] : 0.0;
    }
    // W_o = S_o rows i0 .. i0 + 31 times basis columns b0 .. b0 + 63
    for (int t = threadIdx.x; t < 3 * kPR * kPT; t += 256)
    {
      const int o = t / (kPR * kPT), rem = t % (kPR * kPT);
      const int i = rem % kPR, b = rem / kPR;
      const int64_t gi = i0 + i, gb = b0 + b;
      double w = 0.0;
      if (gi < hi && gb < r)
      {
        const double *vb = V + gb * ldv - ext0;
        for (int64_t q = S[o].rp[gi]; q < S[o].rp[gi + 1]; ++q)
          w = __dadd_rn(w, __dmul_rn(S[o].v[q], vb[S[o].ci[q]]));
      }
      Wo[o][i][b] = w;
    }
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < kPR; ++i)
    {
      double ya[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        ya[u] = Ya[i][ty + 16 * u];
#pragma unroll
      for (int o = 0; o < 3; ++o)
      {
        double wb[4];
#pragma unroll
        for (int v = 0; v < 4; ++v)
          wb[v] = Wo[o][i][tx + 16 * v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            acc[o][u][v] = fma(ya[u], wb[v], acc[o][u][v]);
      }
    }
    __syncthreads();
  }
  const int64_t rr = r * r;
#pragma unroll
  for (int o = 0; o < 3; ++o)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
      {
        const int64_t ga = a0 + ty + 16 * u, gb = b0 + tx + 16 * v;
        if (ga < r && gb < r)
          part[(static_cast<int64_t>(blockIdx.y) * 3 + o) * rr + gb * r + ga] = acc[o][u][v];
      }
}

__global__ void proj_reduce(int64_t rr, int splits, const double *__restrict__ part, double *__restrict__ H)
{
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 3 * rr)
    return;
  const int64_t o = t / rr, e = t - o * rr;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) // split order: deterministic
    s += part[(static_cast<int64_t>(z) * 3 + o) * rr + e];
  H[t] = s;
}

// Device staging of a `where` buffer: device pointers pass through, host ones are copied.
struct Staged
{
  DBuf buf;
  const double *ptr = nullptr;
  Staged(mgpu_ctx *ctx, const double *src, int64_t count, mgpu_memkind where)
  {
    if (where == MGPU_DEVICE || count == 0)
    {
      ptr = src;
      return;
    }
    buf = DBuf(sizeof(double) * static_cast<size_t>(count), ctx->stream);
    MG_CUDA(cudaMemcpyAsync(buf.ptr, src, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    ptr = buf.as<double>();
  }
};

void deliver(mgpu_ctx *ctx, double *dst, const double *dev, int64_t count, mgpu_memkind where)
{
  if (count == 0)
    return;
  MG_CUDA(cudaMemcpyAsync(dst, dev, sizeof(double) * count,
                          where == MGPU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" {

int mgpu_thin_qr(mgpu_ctx *ctx, int64_t rows, int64_t cols, const double *A, double rank_tol, double *Q, double *R,
                 int64_t *rank, mgpu_memkind where)
{
  return guard(ctx, [&] {
    MG_ARG(A && Q && R && rank && rows >= 0 && cols >= 0, "thin_qr: null argument");
    MG_ARG(where == MGPU_HOST || where == MGPU_DEVICE, "thin_qr: bad memory kind");
    MG_ARG(rows >= cols, "thin_qr: requires nrows >= ncols"); // dense.cpp:155-158
    if (cols > kQrMaxCols)
      throw Error(MGPU_ERR_UNSUPPORTED,
                  "thin_qr: at most " + std::to_string(kQrMaxCols) + " columns on the device (got " +
                      std::to_string(cols) + ")");
    cudaStream_t s = ctx->stream;
    const int64_t total = rows * cols;
    const size_t bytes = sizeof(double) * static_cast<size_t>(total > 0 ? total : 1);
    DBuf W(bytes, s), Qd(bytes, s), Rd(sizeof(double) * static_cast<size_t>(cols > 0 ? cols * cols : 1), s);
    DBuf diag(sizeof(double) * (cols > 0 ? cols : 1), s), tau(sizeof(double) * (cols > 0 ? cols : 1), s);
    MG_CUDA(cudaMemcpyAsync(W.ptr, A, sizeof(double) * total,
                            where == MGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    int64_t rk = 0;
    if (cols > 0)
    {
      // tol = rank_tol * ||A||_F (dense.cpp:162-163)
      DBuf sq(bytes, s), nrm(sizeof(double), s);
      square_all<<<blocks_for(total), kThreads, 0, s>>>(total, W.as<double>(), sq.as<double>());
      check_launch(ctx, "square_all");
      det_sum(ctx, sq.as<double>(), total, nrm.as<double>());
      double an2 = 0.0;
      MG_CUDA(cudaMemcpyAsync(&an2, nrm.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      const double anorm = std::sqrt(an2);
      const int G = ctx->num_sms;
      DBuf part(sizeof(double) * static_cast<size_t>(G) * (cols + 1), s);
      QrArgs a{rows, static_cast<int>(cols), W.as<double>(), Qd.as<double>(), diag.as<double>(), tau.as<double>(),
               rank_tol * (anorm > 0.0 ? anorm : 1.0), part.as<double>(), 0, static_cast<int>(cols)};
      void *args[] = {&a};
      if (ctx->opt[MGPU_OPT_QR_UNBLOCKED]) // diagnostics: the column-by-column reference schedule
      {
        MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(qr_factor), dim3(static_cast<unsigned>(G)),
                                            dim3(kQrTB), args, 0, s));
        check_launch(ctx, "qr_factor");
        MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(qr_form_q), dim3(static_cast<unsigned>(G)),
                                            dim3(kQrTB), args, 0, s));
        check_launch(ctx, "qr_form_q");
      }
      else
      {
        // Blocked (compact WY): the panel [j0, j0 + jb) is factored column by column (same
        // rank test and reflectors as the reference), then the trailing block gets all jb
        // reflectors at once, C -= V (T^T (V^T C)); Q applies I - V T V^T panel by panel in
        // reverse.  Same H_k, applied as GEMMs: rounding differs from the reference's
        // reflector-at-a-time order at the 1e-15 level.
        constexpr int kPanel = 32;
        const int ncol = static_cast<int>(cols);
        const int npan = (ncol + kPanel - 1) / kPanel;
        DBuf Tall(sizeof(double) * static_cast<size_t>(npan) * kPanel * kPanel, s);
        DBuf Vp(sizeof(double) * static_cast<size_t>(rows) * kPanel, s);
        DBuf Gm(sizeof(double) * kPanel * kPanel, s);
        DBuf Wt(sizeof(double) * static_cast<size_t>(kPanel) * ncol, s), Wt2(sizeof(double) * static_cast<size_t>(kPanel) * ncol, s);
        double *Wm = W.as<double>();
        auto panel_vt = [&](int pi, bool build_t) {
          const int64_t j0 = static_cast<int64_t>(pi) * kPanel;
          const int jb = static_cast<int>(std::min<int64_t>(kPanel, cols - j0));
          const int64_t mv = rows - j0;
          qr_panel_v<<<blocks_for(mv * jb), kThreads, 0, s>>>(rows, j0, jb, Wm, Vp.as<double>());
          check_launch(ctx, "qr_panel_v");
          if (build_t)
          {
            gemm(ctx, true, jb, jb, mv, 1.0, Vp.as<double>(), mv, Vp.as<double>(), mv, 0.0, Gm.as<double>(), jb);
            qr_panel_t<<<1, 32, 0, s>>>(jb, Gm.as<double>(), tau.as<double>() + j0,
                                        Tall.as<double>() + static_cast<size_t>(pi) * kPanel * kPanel);
            check_launch(ctx, "qr_panel_t");
          }
        };
        for (int pi = 0; pi < npan; ++pi)
        {
          const int64_t j0 = static_cast<int64_t>(pi) * kPanel;
          const int jb = static_cast<int>(std::min<int64_t>(kPanel, cols - j0));
          a.k0 = static_cast<int>(j0);
          a.k1 = static_cast<int>(j0 + jb);
          MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(qr_factor), dim3(static_cast<unsigned>(G)),
                                              dim3(kQrTB), args, 0, s));
          check_launch(ctx, "qr_factor");
          const int64_t nc = cols - j0 - jb;
          if (nc <= 0)
            continue;
          panel_vt(pi, true);
          const int64_t mv = rows - j0;
          const double *T = Tall.as<double>() + static_cast<size_t>(pi) * kPanel * kPanel;
          double *C = Wm + (j0 + jb) * rows + j0;
          gemm(ctx, true, jb, nc, mv, 1.0, Vp.as<double>(), mv, C, rows, 0.0, Wt.as<double>(), jb);
          gemm(ctx, true, jb, nc, jb, 1.0, T, jb, Wt.as<double>(), jb, 0.0, Wt2.as<double>(), jb);
          gemm(ctx, false, mv, nc, jb, -1.0, Vp.as<double>(), mv, Wt2.as<double>(), jb, 1.0, C, rows);
        }
        // T of the last panel (not needed for a trailing update, needed for Q)
        panel_vt(npan - 1, true);
        qr_init_q<<<blocks_for(total), kThreads, 0, s>>>(rows, ncol, diag.as<double>(), Qd.as<double>());
        check_launch(ctx, "qr_init_q");
        for (int pi = npan - 1; pi >= 0; --pi)
        {
          const int64_t j0 = static_cast<int64_t>(pi) * kPanel;
          const int jb = static_cast<int>(std::min<int64_t>(kPanel, cols - j0));
          const int64_t mv = rows - j0, nq = cols - j0;
          if (pi != npan - 1)
            panel_vt(pi, false);
          const double *T = Tall.as<double>() + static_cast<size_t>(pi) * kPanel * kPanel;
          double *Cq = Qd.as<double>() + j0 * rows + j0;
          gemm(ctx, true, jb, nq, mv, 1.0, Vp.as<double>(), mv, Cq, rows, 0.0, Wt.as<double>(), jb);
          gemm(ctx, false, jb, nq, jb, 1.0, T, jb, Wt.as<double>(), jb, 0.0, Wt2.as<double>(), jb);
          gemm(ctx, false, mv, nq, jb, -1.0, Vp.as<double>(), mv, Wt2.as<double>(), jb, 1.0, Cq, rows);
        }
      }
      qr_form_r<<<blocks_for(cols * cols), kThreads, 0, s>>>(rows, static_cast<int>(cols), W.as<double>(),
                                                             diag.as<double>(), Rd.as<double>());
      check_launch(ctx, "qr_form_r");
      qr_sign_q<<<blocks_for(total), kThreads, 0, s>>>(rows, static_cast<int>(cols), diag.as<double>(),
                                                       Qd.as<double>());
      check_launch(ctx, "qr_sign_q");
      std::vector<double> hd(static_cast<size_t>(cols));
      MG_CUDA(cudaMemcpyAsync(hd.data(), diag.ptr, sizeof(double) * cols, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
      for (double d : hd)
        rk += d != 0.0; // |R_kk| > 0 after the sign fix (dense.cpp:236-239)
    }
    deliver(ctx, Q, Qd.as<double>(), total, where);
    deliver(ctx, R, Rd.as<double>(), cols * cols, where);
    MG_CUDA(cudaStreamSynchronize(s));
    *rank = rk;
  });
}

int mgpu_project_reduce_slab(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t row0,
                             int64_t ext0, int64_t next, int64_t r, const double *Vext, int64_t m, const double *F,
                             int64_t q, const double *Cp, const double *Cv, double *Mh, double *Dh, double *Kh,
                             double *Fh, double *Cph, double *Cvh, mgpu_memkind where)
{
  return guard(ctx, [&] {
    MG_ARG(M && D && K && Vext && Mh && Dh && Kh && r >= 0 && m >= 0 && q >= 0 && next >= 0,
           "project_reduce: null argument");
    MG_ARG(where == MGPU_HOST || where == MGPU_DEVICE, "project_reduce: bad memory kind");
    MG_ARG(m == 0 || (F && Fh), "project_reduce: F / Fh missing");
    MG_ARG(q == 0 || (Cp && Cv && Cph && Cvh), "project_reduce: Cp / Cv missing");
    const int64_t p = M->nrows;
    for (const mgpu_csr *S : {M, D, K})
      MG_ARG(S->nrows == p, "project_reduce: operator slab shape mismatch");
    MG_ARG(row0 >= ext0 && row0 + p <= ext0 + next, "project_reduce: slab rows outside the extended basis");
    // precondition (mgpu.h): every column the slab touches lies in [ext0, ext0 + next)
    cudaStream_t s = ctx->stream;
    Staged dV(ctx, Vext, next * r, where), dF(ctx, F, p * m, where), dCp(ctx, Cp, q * p, where),
        dCv(ctx, Cv, q * p, where);
    const double *Y = dV.ptr + (row0 - ext0); // this slab's own rows of the basis (ld = next)
    // airga.cpp:489-491 matmul_tn(V, sparse_times_dense(S, V)) for M, D, K in one fused pass
    // (proj_fused: S V formed tile by tile in shared memory, never written to HBM)
    DBuf H(sizeof(double) * static_cast<size_t>(3 * r * r > 0 ? 3 * r * r : 1), s);
    if (r > 0 && p == 0)
      MG_CUDA(cudaMemsetAsync(H.ptr, 0, sizeof(double) * 3 * r * r, s));
    else if (r > 0)
    {
      const int64_t nt = (r + kPT - 1) / kPT, tiles = nt * nt;
      int64_t splits = std::max<int64_t>(1, (4 * static_cast<int64_t>(ctx->num_sms) + tiles - 1) / tiles);
      splits = std::min<int64_t>(splits, (p + kPR - 1) / kPR);
      splits = std::min<int64_t>(splits, std::max<int64_t>(1, (int64_t{24} << 20) / (3 * r * r))); // partials <= 192 MB
      int64_t per = (p + splits - 1) / splits;
      per = (per + kPR - 1) / kPR * kPR;
      splits = (p + per - 1) / per;
      DBuf part(sizeof(double) * static_cast<size_t>(splits * 3 * r * r), s);
      proj_fused<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(splits)), 256, 0, s>>>(
          p, r, M->view(), D->view(), K->view(), dV.ptr, ext0, next, row0 - ext0, per, part.as<double>());
      check_launch(ctx, "proj_fused");
      proj_reduce<<<blocks_for(3 * r * r), kThreads, 0, s>>>(r * r, static_cast<int>(splits), part.as<double>(),
                                                            H.as<double>());
      check_launch(ctx, "proj_reduce");
    }
    double *outs[3] = {Mh, Dh, Kh};
    for (int o = 0; o < 3; ++o)
      deliver(ctx, outs[o], H.as<double>() + o * r * r, r * r, where);
    MG_CUDA(cudaStreamSynchronize(s));
    if (m > 0) // airga.cpp:492: matmul_tn(V, F)
    {
      DBuf T(sizeof(double) * static_cast<size_t>(r * m > 0 ? r * m : 1), s);
      if (p == 0)
        MG_CUDA(cudaMemsetAsync(T.ptr, 0, sizeof(double) * r * m, s));
      else
        gemm(ctx, true, r, m, p, 1.0, Y, next, dF.ptr, p, 0.0, T.as<double>(), r);
      deliver(ctx, Fh, T.as<double>(), r * m, where);
      MG_CUDA(cudaStreamSynchronize(s));
    }
    if (q > 0) // airga.cpp:493-494: matmul(Cp, V), matmul(Cv, V)
    {
      DBuf T(sizeof(double) * static_cast<size_t>(q * r > 0 ? q * r : 1), s);
      for (int o = 0; o < 2; ++o)
      {
        if (p == 0)
          MG_CUDA(cudaMemsetAsync(T.ptr, 0, sizeof(double) * q * r, s));
        else
          gemm(ctx, false, q, r, p, 1.0, o == 0 ? dCp.ptr : dCv.ptr, q, Y, next, 0.0, T.as<double>(), q);
        deliver(ctx, o == 0 ? Cph : Cvh, T.as<double>(), q * r, where);
        MG_CUDA(cudaStreamSynchronize(s));
      }
    }
    MG_CUDA(cudaStreamSynchronize(s));
  });
}

int mgpu_project_reduce(mgpu_ctx *ctx, const mgpu_csr *M, const mgpu_csr *D, const mgpu_csr *K, int64_t r,
                        const double *V, int64_t m, const double *F, int64_t q, const double *Cp, const double *Cv,
                        double *Mh, double *Dh, double *Kh, double *Fh, double *Cph, double *Cvh, mgpu_memkind where)
{
  if (M && D && K)
  {
    const int64_t n = M->nrows;
    for (const mgpu_csr *S : {M, D, K})
      if (S->nrows != n || S->ncols != n)
        return guard(ctx, [&] { throw Error(MGPU_ERR_ARG, "project_reduce: operator shape mismatch"); });
    return mgpu_project_reduce_slab(ctx, M, D, K, 0, 0, n, r, V, m, F, q, Cp, Cv, Mh, Dh, Kh, Fh, Cph, Cvh, where);
  }
  return guard(ctx, [&] { throw Error(MGPU_ERR_ARG, "project_reduce: null argument"); });
}

int mgpu_arnoldi_deflate(mgpu_ctx *ctx, int64_t len, double *X, int nblocks, const double *const *blocks,
                         double *gammas, mgpu_memkind where)
{
  return guard(ctx, [&] {
    MG_ARG(X && nblocks >= 0 && (nblocks == 0 || (blocks && gammas)) && len >= 0, "arnoldi_deflate: null argument");
    MG_ARG(where == MGPU_HOST || where == MGPU_DEVICE, "arnoldi_deflate: bad memory kind");
    cudaStream_t s = ctx->stream;
    const size_t bytes = sizeof(double) * static_cast<size_t>(len > 0 ? len : 1);
    DBuf Xd(bytes, s), prod(bytes, s), g(sizeof(double) * (2 * nblocks > 0 ? 2 * nblocks : 1), s);
    MG_CUDA(cudaMemcpyAsync(Xd.ptr, X, sizeof(double) * len,
                            where == MGPU_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    std::vector<Staged> B;
    B.reserve(static_cast<size_t>(nblocks));
    for (int t = 0; t < nblocks; ++t)
      B.emplace_back(ctx, blocks[t], len, where);
    for (int sweep = 0; sweep < 2; ++sweep) // airga.cpp:459-470
      for (int t = 0; t < nblocks; ++t)
      {
        double *gd = g.as<double>() + sweep * nblocks + t;
        if (len > 0)
        {
          product_all<<<blocks_for(len), kThreads, 0, s>>>(len, B[t].ptr, Xd.as<double>(), prod.as<double>());
          check_launch(ctx, "product_all");
          det_sum(ctx, prod.as<double>(), len, gd); // trace_inner(B_t, X)
          deflate_axpy<<<blocks_for(len), kThreads, 0, s>>>(len, gd, B[t].ptr, Xd.as<double>());
          check_launch(ctx, "deflate_axpy");
        }
        else
          MG_CUDA(cudaMemsetAsync(gd, 0, sizeof(double), s));
      }
    std::vector<double> hg(static_cast<size_t>(2 * nblocks));
    if (nblocks > 0)
      MG_CUDA(cudaMemcpyAsync(hg.data(), g.ptr, sizeof(double) * 2 * nblocks, cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaMemcpyAsync(X, Xd.ptr, sizeof(double) * len,
                            where == MGPU_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    MG_CUDA(cudaStreamSynchronize(s));
    for (int t = 0; t < nblocks; ++t)
      gammas[t] = (0.0 + hg[static_cast<size_t>(t)]) + hg[static_cast<size_t>(nblocks + t)]; // gammas[t] += g
  });
}

} // extern "C"
