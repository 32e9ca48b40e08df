// K-cg: right-preconditioned CG (krylov.cpp:28-174) for l shifted systems x m
// right-hand sides in ONE persistent cooperative kernel.
//
// Design (DESIGN.md section "K-cg"):
//   * every (point p, rhs column c) pair is an independent recurrence; all of
//     them advance in lock step, one grid-wide barrier per phase;
//   * vectors are interleaved [p][row][c] so a CSR row of A_p (or of a chain
//     factor) is read once for all m columns (SpMM access);
//   * the control flow of pcg_solve -- confirm-on-true-residual / restart,
//     breakdown guard, maxit, finish -- runs on the device: every block holds
//     the per-system scalars in shared memory and takes identical decisions
//     from identical totals, so no host round trip happens per iteration;
//   * dot products are deterministic: per-tile partials (tile size fixed by n
//     only) reduced by the last tile to arrive, in a fixed order.
//   * SpMV and axpy arithmetic match the reference scalar kernels bitwise
//     (in-order rows, no FMA); only the dot-product summation order differs.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <cmath>
#include <cstring>
#include <chrono>
#include <vector>

#include "cg_common.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
int cg_cluster_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains,
                      int64_t n, int m, const double *B_dev, int64_t ldb, const int *halo, double rtol,
                      int64_t maxit, double *X, double *REC, double *TR, int64_t *d_it, int *d_conv, int *d_st,
                      int64_t *d_bd, double *d_hist, int64_t hist_cap, unsigned long long *d_loop, const DCsr *dA,
                      const DCsr *dF);

// cg_stream.cu
bool stream_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains, int64_t n,
                  int m, const double *B_dev, int64_t ldb, const int *halo, int hmax, double rtol, int64_t maxit,
                  double *X_dev, double *REC_dev, double *TR_dev, int64_t *d_it, int *d_conv, int *d_st, int64_t *d_bd,
                  double *d_hist, int64_t hist_cap, int64_t *d_loop);

namespace
{

// (batch limits, SysState, Seg, BandShared and the reductions: cg_common.cuh)

struct CgParams
{
  int l, m, z, tiles, rpt; // rpt = rows per thread per tile
  int64_t n, rows_per_tile;
  const DCsr *A; // [l]
  const DCsr *F; // [l * z], newest first
  double rtol;
  int64_t maxit;
  const double *b;
  double *xt, *r, *d, *w, *t0, *t1;
  double *partial;        // [l][2][kMaxM][tiles]
  double *totals;         // [2 (parity)][l][2][kMaxM]
  unsigned int *counter;  // [l]
  double *X, *REC, *TR;   // outputs [p][c][row] (nullable)
  int64_t *iters;         // [l*m]
  int *conv, *status;     // [l*m]
  int64_t *bd_iter;       // [l*m]
  double *hist;           // [l*m][hist_cap] (nullable)
  int64_t hist_cap;
  int64_t *loop_iters;    // [1]
};

struct Shared
{
  double rho[kMaxSys], target[kMaxSys], alpha[kMaxSys], beta[kMaxSys], bnorm[kMaxSys];
  int state[kMaxSys];
  int64_t sit[kMaxSys];
  int pmask[kMaxPoints];
  double red[kWarps][2 * kMaxM];
  int flag;
  unsigned int ticket_last;
};

// Deterministic block reduction of nv values per thread (nv <= 2*kMaxM).
// Result in red[0][v] for thread 0's use; fixed shuffle tree + warp order.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], Shared &sh)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k)
  {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      v[k] = __dadd_rn(v[k], __shfl_down_sync(0xffffffffu, v[k], off));
  }
  __syncthreads(); // red[] reuse guard
  if (lane == 0)
  {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      sh.red[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < NV)
  {
    double s = sh.red[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < kWarps; ++w)
      s = __dadd_rn(s, sh.red[w][threadIdx.x]);
    sh.red[0][threadIdx.x] = s;
  }
  __syncthreads();
}

// Publishes a tile's partials for point p; the last tile of p reduces all of
// them (fixed order) into totals[par][p][k][c].
template <int NK, int MT>
__device__ void publish(const CgParams &P, Shared &sh, int p, int tb, double (&v)[NK * MT], int par)
{
  block_reduce<NK * MT>(v, sh);
  if (threadIdx.x < NK * MT)
  {
    const int k = threadIdx.x / MT, c = threadIdx.x % MT;
    P.partial[((static_cast<int64_t>(p) * 2 + k) * kMaxM + c) * P.tiles + tb] = sh.red[0][threadIdx.x];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
  {
    const unsigned int t = atomicAdd(&P.counter[p], 1u);
    sh.ticket_last = (t == static_cast<unsigned int>(P.tiles - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (sh.ticket_last == 0u)
    return;
  __threadfence();
  double acc[NK * MT];
#pragma unroll
  for (int q = 0; q < NK * MT; ++q)
  {
    const int k = q / MT, c = q % MT;
    const double *src = P.partial + ((static_cast<int64_t>(p) * 2 + k) * kMaxM + c) * P.tiles;
    double a = 0.0;
    for (int t = threadIdx.x; t < P.tiles; t += kCgThreads)
      a = __dadd_rn(a, __ldcg(src + t));
    acc[q] = a;
  }
  block_reduce<NK * MT>(acc, sh);
  if (threadIdx.x < NK * MT)
  {
    const int k = threadIdx.x / MT, c = threadIdx.x % MT;
    P.totals[((static_cast<int64_t>(par) * P.l + p) * 2 + k) * kMaxM + c] = sh.red[0][threadIdx.x];
  }
  if (threadIdx.x == 0)
    P.counter[p] = 0u;
  __threadfence();
}

__device__ __forceinline__ double total(const CgParams &P, int par, int p, int k, int c)
{
  return __ldcg(P.totals + ((static_cast<int64_t>(par) * P.l + p) * 2 + k) * kMaxM + c);
}

// y = Mat x over interleaved vectors for the points in pmask.
template <int MT>
__device__ void spmv_phase(const CgParams &P, Shared &sh, const DCsr *mats, int mstride, int moff, const double *x,
                           double *y)
{
  const int m = P.m;
  for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
  {
    const int p = static_cast<int>(tile / P.tiles);
    if (!sh.pmask[p])
      continue;
    const int tb = static_cast<int>(tile % P.tiles);
    const DCsr A = mats[p * mstride + moff];
    const double *xp = x + static_cast<int64_t>(p) * P.n * m;
    double *yp = y + static_cast<int64_t>(p) * P.n * m;
    for (int j = 0; j < P.rpt; ++j)
    {
      const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
      if (i >= P.n)
        break;
      double acc[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
        acc[c] = 0.0;
      const int64_t e = __ldg(A.rp + i + 1);
      for (int64_t k = __ldg(A.rp + i); k < e; ++k)
      {
        const double v = __ldg(A.v + k);
        const int64_t col = __ldg(A.ci + k);
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
            acc[c] = __dadd_rn(acc[c], __dmul_rn(v, __ldcg(xp + col * m + c)));
      }
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
          __stcg(yp + i * m + c, acc[c]);
    }
  }
}

// chain_apply on the device (spai.cpp:361-373): oldest factor first.
// Returns the buffer holding P x (x itself when z == 0).
template <int MT>
__device__ const double *chain_phase(const CgParams &P, Shared &sh, cgrp::grid_group &grid, const double *x)
{
  const double *src = x;
  for (int q = 0; q < P.z; ++q)
  {
    double *dst = (q & 1) ? P.t1 : P.t0;
    spmv_phase<MT>(P, sh, P.F, P.z, P.z - 1 - q, src, dst);
    grid.sync();
    src = dst;
  }
  return src;
}

// res (-> w buffer) = b - A sol, partial ||res||^2 per column; totals[par].
template <int MT>
__device__ void residual_phase(const CgParams &P, Shared &sh, const double *sol, int par)
{
  const int m = P.m;
  for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
  {
    const int p = static_cast<int>(tile / P.tiles);
    if (!sh.pmask[p])
      continue;
    const int tb = static_cast<int>(tile % P.tiles);
    const DCsr A = P.A[p];
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    double part[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
      part[c] = 0.0;
    for (int j = 0; j < P.rpt; ++j)
    {
      const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
      if (i >= P.n)
        break;
      double acc[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
        acc[c] = 0.0;
      const int64_t e = __ldg(A.rp + i + 1);
      for (int64_t k = __ldg(A.rp + i); k < e; ++k)
      {
        const double v = __ldg(A.v + k);
        const int64_t col = __ldg(A.ci + k);
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
            acc[c] = __dadd_rn(acc[c], __dmul_rn(v, __ldcg(sol + base + col * m + c)));
      }
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
        {
          const double res = __dsub_rn(__ldg(P.b + base + i * m + c), acc[c]);
          __stcg(P.w + base + i * m + c, res);
          part[c] = __dadd_rn(part[c], __dmul_rn(res, res));
        }
    }
    publish<1, MT>(P, sh, p, tb, part, par);
  }
}

template <int MT>
__global__ void __launch_bounds__(kCgThreads) cg_persistent(CgParams P)
{
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ Shared sh;
  const int m = P.m;
  const int S = P.l * m;
  int par = 0; // totals parity, advanced after every reduction phase

  // ---- phase 0: ||b||^2 per system (krylov.cpp:40)
  for (int p = threadIdx.x; p < P.l; p += kCgThreads)
    sh.pmask[p] = 1;
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
  {
    const int p = static_cast<int>(tile / P.tiles);
    const int tb = static_cast<int>(tile % P.tiles);
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    double part[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
      part[c] = 0.0;
    for (int j = 0; j < P.rpt; ++j)
    {
      const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
      if (i >= P.n)
        break;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
        {
          const double bv = __ldg(P.b + base + i * m + c);
          part[c] = __dadd_rn(part[c], __dmul_rn(bv, bv));
        }
    }
    publish<1, MT>(P, sh, p, tb, part, par);
  }
  grid.sync();
  for (int s = threadIdx.x; s < S; s += kCgThreads)
  {
    const double bb = total(P, par, s / m, 0, s % m);
    const double bn = sqrt(bb);
    sh.bnorm[s] = bn;
    sh.rho[s] = bb; // rho = (r, r) with r = b (krylov.cpp:57)
    sh.target[s] = P.rtol * bn;
    sh.state[s] = (bn == 0.0) ? kZeroRhs : kRun; // krylov.cpp:44-51
    sh.sit[s] = 0;
  }
  par ^= 1;
  __syncthreads();

  int64_t it = 0;
  for (;;)
  {
    if (it >= P.maxit)
      break;
    // ---- confirm-on-true-residual (krylov.cpp:77-103)
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += kCgThreads)
    {
      int need = 0;
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        if (sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s])
          need = 1;
      }
      sh.pmask[p] = need;
      if (need)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (sh.flag)
    {
      const double *sol = chain_phase<MT>(P, sh, grid, P.xt);
      residual_phase<MT>(P, sh, sol, par);
      grid.sync();
      for (int s = threadIdx.x; s < S; s += kCgThreads)
      {
        if (!(sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s]))
          continue;
        const double tt = total(P, par, s / m, 0, s % m);
        if (sqrt(tt) <= sh.target[s])
        {
          sh.state[s] = kPendingConv;
          sh.sit[s] = it;
        }
        else
        {
          sh.rho[s] = tt; // r = true residual, d = r, rho = (r, r)
          if (sqrt(tt) <= sh.target[s])
          {
            sh.state[s] = kPendingConv;
            sh.sit[s] = it;
          }
          else
            sh.state[s] = kPendingRestart;
        }
      }
      par ^= 1;
      __syncthreads();
      // finish converged systems now (their sol / res buffers are reused later),
      // restart the others from the true residual.
      for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
      {
        const int p = static_cast<int>(tile / P.tiles);
        if (!sh.pmask[p])
          continue;
        const int tb = static_cast<int>(tile % P.tiles);
        const int64_t base = static_cast<int64_t>(p) * P.n * m;
        for (int j = 0; j < P.rpt; ++j)
        {
          const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
          if (i >= P.n)
            break;
          for (int c = 0; c < m; ++c)
          {
            const int s = p * m + c;
            const int64_t v = base + i * m + c;
            if (sh.state[s] == kPendingConv)
            {
              const int64_t o = (static_cast<int64_t>(s)) * P.n + i;
              if (P.X)
                P.X[o] = __ldcg(sol + v);
              if (P.TR)
                P.TR[o] = __ldcg(P.w + v);
            }
            else if (sh.state[s] == kPendingRestart)
            {
              const double res = __ldcg(P.w + v);
              __stcg(P.r + v, res);
              __stcg(P.d + v, res);
            }
          }
        }
      }
      grid.sync();
      for (int s = threadIdx.x; s < S; s += kCgThreads)
      {
        if (sh.state[s] == kPendingConv)
          sh.state[s] = kConverged;
        else if (sh.state[s] == kPendingRestart)
          sh.state[s] = kRun;
      }
      __syncthreads();
    }

    // ---- live points
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += kCgThreads)
    {
      int live = 0;
      for (int c = 0; c < m; ++c)
        live |= sh.state[p * m + c] == kRun;
      sh.pmask[p] = live;
      if (live)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (!sh.flag)
      break;

    // ---- w = A (P d); (d, w), (d, d)   (krylov.cpp:105-107)
    const double *t = chain_phase<MT>(P, sh, grid, P.d);
    for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
    {
      const int p = static_cast<int>(tile / P.tiles);
      if (!sh.pmask[p])
        continue;
      const int tb = static_cast<int>(tile % P.tiles);
      const DCsr A = P.A[p];
      const int64_t base = static_cast<int64_t>(p) * P.n * m;
      double part[2 * MT];
#pragma unroll
      for (int q = 0; q < 2 * MT; ++q)
        part[q] = 0.0;
      for (int j = 0; j < P.rpt; ++j)
      {
        const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
        if (i >= P.n)
          break;
        double acc[MT];
#pragma unroll
        for (int c = 0; c < MT; ++c)
          acc[c] = 0.0;
        const int64_t e = __ldg(A.rp + i + 1);
        for (int64_t k = __ldg(A.rp + i); k < e; ++k)
        {
          const double v = __ldg(A.v + k);
          const int64_t col = __ldg(A.ci + k);
#pragma unroll
          for (int c = 0; c < MT; ++c)
            if (c < m)
              acc[c] = __dadd_rn(acc[c], __dmul_rn(v, __ldcg(t + base + col * m + c)));
        }
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
          {
            __stcg(P.w + base + i * m + c, acc[c]);
            const double dv = __ldcg(P.d + base + i * m + c);
            part[c] = __dadd_rn(part[c], __dmul_rn(dv, acc[c]));
            part[MT + c] = __dadd_rn(part[MT + c], __dmul_rn(dv, dv));
          }
      }
      publish<2, MT>(P, sh, p, tb, part, par);
    }
    grid.sync();
    for (int s = threadIdx.x; s < S; s += kCgThreads)
    {
      if (sh.state[s] != kRun)
        continue;
      const double curv = total(P, par, s / m, 0, s % m);
      const double dd = total(P, par, s / m, 1, s % m);
      if (!(curv > 1e-30 * dd)) // krylov.cpp:108
      {
        sh.state[s] = kBreakdown;
        sh.sit[s] = it;
      }
      else
        sh.alpha[s] = sh.rho[s] / curv;
    }
    par ^= 1;
    __syncthreads();

    // ---- x~ += alpha d; r -= alpha w; (r, r)   (krylov.cpp:112-116)
    for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
    {
      const int p = static_cast<int>(tile / P.tiles);
      if (!sh.pmask[p])
        continue;
      const int tb = static_cast<int>(tile % P.tiles);
      const int64_t base = static_cast<int64_t>(p) * P.n * m;
      double part[MT];
      bool run[MT];
      double al[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        part[c] = 0.0;
        run[c] = c < m && sh.state[p * m + c] == kRun;
        al[c] = run[c] ? sh.alpha[p * m + c] : 0.0;
      }
      for (int j = 0; j < P.rpt; ++j)
      {
        const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
        if (i >= P.n)
          break;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (run[c])
          {
            const int64_t v = base + i * m + c;
            const double xn = __dadd_rn(__ldcg(P.xt + v), __dmul_rn(al[c], __ldcg(P.d + v)));
            const double rn = __dadd_rn(__ldcg(P.r + v), __dmul_rn(-al[c], __ldcg(P.w + v)));
            __stcg(P.xt + v, xn);
            __stcg(P.r + v, rn);
            part[c] = __dadd_rn(part[c], __dmul_rn(rn, rn));
          }
      }
      publish<1, MT>(P, sh, p, tb, part, par);
    }
    grid.sync();
    ++it;
    for (int s = threadIdx.x; s < S; s += kCgThreads)
    {
      if (sh.state[s] != kRun)
        continue;
      const double rn = total(P, par, s / m, 0, s % m);
      if (P.hist && blockIdx.x == 0 && it - 1 < P.hist_cap)
        P.hist[static_cast<int64_t>(s) * P.hist_cap + (it - 1)] = sqrt(rn) / sh.bnorm[s];
      sh.beta[s] = rn / sh.rho[s]; // krylov.cpp:118-119
      sh.rho[s] = rn;
    }
    par ^= 1;
    __syncthreads();

    // ---- d = r + beta d   (krylov.cpp:120-123)
    for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
    {
      const int p = static_cast<int>(tile / P.tiles);
      if (!sh.pmask[p])
        continue;
      const int tb = static_cast<int>(tile % P.tiles);
      const int64_t base = static_cast<int64_t>(p) * P.n * m;
      bool run[MT];
      double be[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        run[c] = c < m && sh.state[p * m + c] == kRun;
        be[c] = run[c] ? sh.beta[p * m + c] : 0.0;
      }
      for (int j = 0; j < P.rpt; ++j)
      {
        const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
        if (i >= P.n)
          break;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (run[c])
          {
            const int64_t v = base + i * m + c;
            __stcg(P.d + v, __dadd_rn(__ldcg(P.r + v), __dmul_rn(be[c], __ldcg(P.d + v))));
          }
      }
    }
    grid.sync();
  }

  // ---- budget exhausted: final true-residual check (krylov.cpp:128-137)
  if (threadIdx.x == 0)
    sh.flag = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P.l; p += kCgThreads)
  {
    int need = 0;
    for (int c = 0; c < m; ++c)
      need |= sh.state[p * m + c] == kRun;
    sh.pmask[p] = need;
    if (need)
      atomicOr(&sh.flag, 1);
  }
  __syncthreads();
  if (sh.flag)
  {
    const double *sol = chain_phase<MT>(P, sh, grid, P.xt);
    residual_phase<MT>(P, sh, sol, par);
    grid.sync();
    for (int s = threadIdx.x; s < S; s += kCgThreads)
    {
      if (sh.state[s] != kRun)
        continue;
      const double tt = total(P, par, s / m, 0, s % m);
      sh.state[s] = sqrt(tt) <= sh.target[s] ? kPendingConv : kMaxed;
      sh.sit[s] = it;
    }
    __syncthreads();
    for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
    {
      const int p = static_cast<int>(tile / P.tiles);
      if (!sh.pmask[p])
        continue;
      const int tb = static_cast<int>(tile % P.tiles);
      const int64_t base = static_cast<int64_t>(p) * P.n * m;
      for (int j = 0; j < P.rpt; ++j)
      {
        const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
        if (i >= P.n)
          break;
        for (int c = 0; c < m; ++c)
        {
          const int s = p * m + c;
          if (sh.state[s] != kPendingConv && sh.state[s] != kMaxed)
            continue;
          const int64_t v = base + i * m + c, o = static_cast<int64_t>(s) * P.n + i;
          if (P.X)
            P.X[o] = __ldcg(sol + v);
          if (P.TR)
            P.TR[o] = __ldcg(P.w + v);
        }
      }
    }
    for (int s = threadIdx.x; s < S; s += kCgThreads)
      if (sh.state[s] == kPendingConv)
        sh.state[s] = kConverged;
    __syncthreads();
  }

  // ---- recurrence residual block, zero-rhs outputs, per-column scalars
  for (int64_t tile = blockIdx.x; tile < static_cast<int64_t>(P.l) * P.tiles; tile += gridDim.x)
  {
    const int p = static_cast<int>(tile / P.tiles);
    const int tb = static_cast<int>(tile % P.tiles);
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    for (int j = 0; j < P.rpt; ++j)
    {
      const int64_t i = tb * P.rows_per_tile + static_cast<int64_t>(j) * kCgThreads + threadIdx.x;
      if (i >= P.n)
        break;
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        const int64_t o = static_cast<int64_t>(s) * P.n + i;
        if (sh.state[s] == kZeroRhs)
        {
          if (P.X)
            P.X[o] = 0.0;
          if (P.TR)
            P.TR[o] = 0.0;
          if (P.REC)
            P.REC[o] = 0.0;
        }
        else if (sh.state[s] != kBreakdown && P.REC)
          P.REC[o] = __ldcg(P.r + base + i * m + c);
      }
    }
  }
  if (blockIdx.x == 0)
  {
    for (int s = threadIdx.x; s < S; s += kCgThreads)
    {
      const int st = sh.state[s];
      P.iters[s] = sh.sit[s];
      P.conv[s] = (st == kConverged || st == kZeroRhs) ? 1 : 0;
      P.status[s] = st == kBreakdown ? MGPU_ERR_BREAKDOWN : MGPU_OK;
      P.bd_iter[s] = st == kBreakdown ? sh.sit[s] : -1;
    }
    if (threadIdx.x == 0)
      *P.loop_iters = it;
  }
}

// =====================================================================
// Banded fast path (all operators of the batch have bandwidth <= kMaxHalo):
// TWO grid barriers per iteration.
//   phase A: d_new = r + beta d_old (halo rows recomputed in shared memory),
//            t = P_chain d_new on shrinking halos, w = A t on owned rows,
//            partials (d_new, w), (d_new, d_new);
//   phase B: x~ += alpha d_new, r -= alpha w, partial (r, r).
// Work split: the flattened rows of all points (each point padded to a
// multiple of 32) are cut into one balanced, 32-row aligned range per block;
// a block processes its range in chunks of TB * RPT rows (one chunk for the
// L2-resident configurations), RPT rows per thread for memory-level
// parallelism.  Dot products: per thread in row order, fixed warp butterfly,
// fixed warp-order combine, chunks in order -> one partial per (block, point);
// after the barrier every block sums the per-block partials in block order.
// Deterministic for a given grid (one block per SM), no atomics.
// =====================================================================

struct BandParams
{
  int l, m, z, rpt;
  int64_t n, npad;
  int halo[kMaxZ + 1]; // halo rows needed by stage q (q = 0 .. z); halo[z] = bw(A)
  int hmax;            // halo[0]
  const DCsr *A, *F;
  double rtol;
  int64_t maxit;
  const double *b;
  double *xt, *r, *dbuf0, *dbuf1, *w, *sol;
  double *partial; // [l][2*kMaxM][gridDim]
  const Seg *seg;  // [gridDim][kMaxSeg], p = -1 terminates
  const int2 *pblk; // [l]: blocks [x, y) that own rows of point p
  double *X, *REC, *TR;
  int64_t *iters;
  int *conv, *status;
  int64_t *bd_iter;
  double *hist;
  int64_t hist_cap;
  int64_t *loop_iters;
};


template <int TB>
__device__ __forceinline__ void end_point(const BandParams &P, BandShared<TB> &sh, int p, int nv)
{
  end_point(P.partial, sh, p, nv);
}


// Phase A.  kCheck: source = x~, outputs sol (own rows) and res = b - A sol (in w);
// otherwise source = d_new = fresh ? r : r + beta d_old, output w.
template <int TB, int MT, int RPT, bool kCheck>
__device__ void band_phase_a(const BandParams &P, BandShared<TB> &sh, double *smem, const double *d_old,
                             double *d_new)
{
  const int m = P.m;
  const int H0 = P.hmax;
  constexpr int CH = TB * RPT;
  const int stride = (CH + 2 * H0) * m;
  // buf0 keeps stage 0 (d_new) for the dot products; the chain stages ping-pong between
  // buf1 and buf2 (allocated when z >= 2)
  double *buf0 = smem, *buf1 = smem + stride, *buf2 = smem + 2 * stride;
  for_segments(P, sh, [&](int p, int64_t rs, int64_t re) {
    begin_point(sh);
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    double be[MT];
    bool fr[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
    {
      const int s = p * m + c;
      fr[c] = c < m && sh.fresh[s];
      be[c] = (c < m) ? sh.beta[s] : 0.0;
    }
    const DCsr A = P.A[p];
    for (int64_t c0 = rs; c0 < re; c0 += CH)
    {
      const int64_t c1 = min(re, c0 + CH);
      // ---- stage 0 on [c0 - H0, c1 + H0)
      const int span0 = static_cast<int>(c1 - c0) + 2 * H0;
      for (int q = threadIdx.x; q < span0; q += TB)
      {
        const int64_t i = c0 - H0 + q;
        if (i < 0 || i >= P.n)
          continue;
#pragma unroll
        for (int c = 0; c < MT; ++c)
        {
          if (c >= m)
            break;
          const int64_t v = base + i * m + c;
          double x;
          if (kCheck)
            x = __ldcg(P.xt + v);
          else
          {
            const double rv = __ldcg(P.r + v);
            x = fr[c] ? rv : __dadd_rn(rv, __dmul_rn(be[c], __ldcg(d_old + v)));
            if (i >= c0 && i < c1)
              __stcg(d_new + v, x);
          }
          buf0[q * m + c] = x;
        }
      }
      __syncthreads();
      // ---- chain stages (oldest factor first), shrinking halos
      double *src = buf0, *dst = buf1;
      double *other = buf2;
      int hs = H0;
      for (int st = 0; st < P.z; ++st)
      {
        const DCsr F = P.F[p * P.z + (P.z - 1 - st)];
        const int hd = P.halo[st + 1];
        const int span = static_cast<int>(c1 - c0) + 2 * hd;
        const int64_t shift = static_cast<int64_t>(hs) - c0; // col k -> src row k + shift
        for (int q = threadIdx.x; q < span; q += TB)
        {
          const int64_t i = c0 - hd + q;
          if (i < 0 || i >= P.n)
            continue;
          double acc[MT];
#pragma unroll
          for (int c = 0; c < MT; ++c)
            acc[c] = 0.0;
          const int64_t e = __ldg(F.rp + i + 1);
          for (int64_t k = __ldg(F.rp + i); k < e; ++k)
          {
            const double fv = __ldg(F.v + k);
            const int loc = static_cast<int>(__ldg(F.ci + k) + shift) * m;
#pragma unroll
            for (int c = 0; c < MT; ++c)
              if (c < m)
                acc[c] = __dadd_rn(acc[c], __dmul_rn(fv, src[loc + c]));
          }
#pragma unroll
          for (int c = 0; c < MT; ++c)
            if (c < m)
              dst[q * m + c] = acc[c];
        }
        __syncthreads();
        // next stage writes the buffer that is neither its source nor buf0
        double *tmp = src == buf0 ? other : src;
        src = dst;
        dst = tmp;
        hs = hd;
      }
      // ---- y = A t on own rows, RPT rows per thread
      double pk[2 * MT];
#pragma unroll
      for (int q = 0; q < 2 * MT; ++q)
        pk[q] = 0.0;
      const int64_t shiftA = static_cast<int64_t>(hs) - c0;
#pragma unroll
      for (int j = 0; j < RPT; ++j)
      {
        const int lr = threadIdx.x + j * TB; // local row
        const int64_t i = c0 + lr;
        if (i >= c1)
          break;
        double acc[MT];
#pragma unroll
        for (int c = 0; c < MT; ++c)
          acc[c] = 0.0;
        const int64_t e = __ldg(A.rp + i + 1);
        for (int64_t k = __ldg(A.rp + i); k < e; ++k)
        {
          const double av = __ldg(A.v + k);
          const int loc = static_cast<int>(__ldg(A.ci + k) + shiftA) * m;
#pragma unroll
          for (int c = 0; c < MT; ++c)
            if (c < m)
              acc[c] = __dadd_rn(acc[c], __dmul_rn(av, src[loc + c]));
        }
#pragma unroll
        for (int c = 0; c < MT; ++c)
        {
          if (c >= m)
            break;
          const int64_t v = base + i * m + c;
          if (kCheck)
          {
            const double res = __dsub_rn(__ldg(P.b + v), acc[c]);
            __stcg(P.w + v, res);
            __stcg(P.sol + v, src[(hs + lr) * m + c]);
            pk[c] = __dadd_rn(pk[c], __dmul_rn(res, res));
          }
          else
          {
            const double dn = buf0[(H0 + lr) * m + c];
            __stcg(P.w + v, acc[c]);
            pk[c] = __dadd_rn(pk[c], __dmul_rn(dn, acc[c]));
            pk[MT + c] = __dadd_rn(pk[MT + c], __dmul_rn(dn, dn));
          }
        }
      }
      // pack (k, c) -> k * m + c
      double pv[2 * MT];
#pragma unroll
      for (int q = 0; q < 2 * MT; ++q)
        pv[q] = 0.0;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
        {
          pv[c] = pk[c];
          pv[m + c] = pk[MT + c];
        }
      chunk_sum<TB, 2 * MT>(sh, pv, kCheck ? m : 2 * m); // its barriers also guard buf reuse
    }
    end_point(P, sh, p, kCheck ? m : 2 * m);
  });
}

// Phase B: x~ += alpha d_new; r -= alpha w; partial (r, r) for running columns.
template <int TB, int MT, int RPT>
__device__ void band_phase_b(const BandParams &P, BandShared<TB> &sh, const double *d_new)
{
  const int m = P.m;
  constexpr int CH = TB * RPT;
  for_segments(P, sh, [&](int p, int64_t rs, int64_t re) {
    begin_point(sh);
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    bool run[MT];
    double al[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
    {
      run[c] = c < m && sh.state[p * m + c] == kRun;
      al[c] = run[c] ? sh.alpha[p * m + c] : 0.0;
    }
    for (int64_t c0 = rs; c0 < re; c0 += CH)
    {
      const int64_t c1 = min(re, c0 + CH);
      double pk[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
        pk[c] = 0.0;
#pragma unroll
      for (int j = 0; j < RPT; ++j)
      {
        const int64_t i = c0 + threadIdx.x + j * TB;
        if (i >= c1)
          break;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (run[c])
          {
            const int64_t v = base + i * m + c;
            const double xn = __dadd_rn(__ldcg(P.xt + v), __dmul_rn(al[c], __ldcg(d_new + v)));
            const double rn = __dadd_rn(__ldcg(P.r + v), __dmul_rn(-al[c], __ldcg(P.w + v)));
            __stcg(P.xt + v, xn);
            __stcg(P.r + v, rn);
            pk[c] = __dadd_rn(pk[c], __dmul_rn(rn, rn));
          }
      }
      chunk_sum<TB, MT>(sh, pk, m);
    }
    end_point(P, sh, p, m);
  });
}

// Copy phase after a confirmation check (finish converged / restart others).
template <int TB>
__device__ void band_finish_copy(const BandParams &P, BandShared<TB> &sh)
{
  const int m = P.m;
  for_segments(P, sh, [&](int p, int64_t rs, int64_t re) {
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    for (int64_t i = rs + threadIdx.x; i < re; i += TB)
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        const int64_t v = base + i * m + c, o = static_cast<int64_t>(s) * P.n + i;
        if (sh.state[s] == kPendingConv || sh.state[s] == kMaxed)
        {
          if (P.X)
            P.X[o] = __ldcg(P.sol + v);
          if (P.TR)
            P.TR[o] = __ldcg(P.w + v);
        }
        else if (sh.state[s] == kPendingRestart)
          __stcg(P.r + v, __ldcg(P.w + v));
      }
  });
}

template <int TB, int MT, int RPT>
__global__ void __launch_bounds__(TB, 1) cg_banded(BandParams P)
{
  cgrp::grid_group grid = cgrp::this_grid();
  extern __shared__ double smem_dyn[];
  __shared__ BandShared<TB> sh;
  const int m = P.m;
  const int S = P.l * m;

  // ---- segment plan, phase 0: ||b||^2
  if (threadIdx.x == 0)
  {
    int q = 0;
    while (q < kMaxSeg && P.seg[blockIdx.x * kMaxSeg + q].p >= 0)
    {
      sh.seg[q] = P.seg[blockIdx.x * kMaxSeg + q];
      ++q;
    }
    sh.nseg = q;
  }
  for (int p = threadIdx.x; p < P.l; p += TB)
    sh.pmask[p] = 1;
  __syncthreads();
  for_segments(P, sh, [&](int p, int64_t rs, int64_t re) {
    begin_point(sh);
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    for (int64_t c0 = rs; c0 < re; c0 += TB * RPT)
    {
      const int64_t c1 = min(re, c0 + TB * RPT);
      double pk[MT];
#pragma unroll
      for (int c = 0; c < MT; ++c)
        pk[c] = 0.0;
#pragma unroll
      for (int j = 0; j < RPT; ++j)
      {
        const int64_t i = c0 + threadIdx.x + j * TB;
        if (i >= c1)
          break;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
          {
            const double bv = __ldg(P.b + base + i * m + c);
            pk[c] = __dadd_rn(pk[c], __dmul_rn(bv, bv));
          }
      }
      chunk_sum<TB, MT>(sh, pk, m);
    }
    end_point(P, sh, p, m);
  });
  grid.sync();
  reduce_blocks<TB, BandParams>(P, sh, m);
  for (int s = threadIdx.x; s < S; s += TB)
  {
    const double bb = sh.tot[s];
    const double bn = sqrt(bb);
    sh.bnorm[s] = bn;
    sh.rho[s] = bb;
    sh.target[s] = P.rtol * bn;
    sh.state[s] = bn == 0.0 ? kZeroRhs : kRun;
    sh.fresh[s] = 1;
    sh.beta[s] = 0.0;
    sh.sit[s] = 0;
  }
  __syncthreads();

  int cur = 0; // d_old = dbuf[cur], d_new = dbuf[cur ^ 1]
  int64_t it = 0;
  for (;;)
  {
    if (it >= P.maxit)
      break;
    // ---- confirm on the true residual (krylov.cpp:77-103)
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += TB)
    {
      int need = 0;
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        need |= sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s];
      }
      sh.pmask[p] = need;
      if (need)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (sh.flag)
    {
      band_phase_a<TB, MT, RPT, true>(P, sh, smem_dyn, nullptr, nullptr);
      grid.sync();
      reduce_blocks<TB, BandParams>(P, sh, m);
      for (int s = threadIdx.x; s < S; s += TB)
      {
        if (!(sh.state[s] == kRun && sqrt(sh.rho[s]) <= sh.target[s]))
          continue;
        const double tt = sh.tot[s];
        if (sqrt(tt) <= sh.target[s])
        {
          sh.state[s] = kPendingConv;
          sh.sit[s] = it;
        }
        else
        {
          sh.rho[s] = tt;
          if (sqrt(tt) <= sh.target[s])
          {
            sh.state[s] = kPendingConv;
            sh.sit[s] = it;
          }
          else
          {
            sh.state[s] = kPendingRestart;
            sh.fresh[s] = 1; // d = r (the true residual)
          }
        }
      }
      __syncthreads();
      band_finish_copy<TB>(P, sh);
      grid.sync();
      for (int s = threadIdx.x; s < S; s += TB)
      {
        if (sh.state[s] == kPendingConv)
          sh.state[s] = kConverged;
        else if (sh.state[s] == kPendingRestart)
          sh.state[s] = kRun;
      }
      __syncthreads();
    }
    // ---- live points
    if (threadIdx.x == 0)
      sh.flag = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P.l; p += TB)
    {
      int live = 0;
      for (int c = 0; c < m; ++c)
        live |= sh.state[p * m + c] == kRun;
      sh.pmask[p] = live;
      if (live)
        atomicOr(&sh.flag, 1);
    }
    __syncthreads();
    if (!sh.flag)
      break;
    double *d_old = cur ? P.dbuf1 : P.dbuf0;
    double *d_new = cur ? P.dbuf0 : P.dbuf1;
    // ---- phase A: d_new, w = A P d_new, (d, w), (d, d)
    band_phase_a<TB, MT, RPT, false>(P, sh, smem_dyn, d_old, d_new);
    grid.sync();
    reduce_blocks<TB, BandParams>(P, sh, 2 * m);
    for (int s = threadIdx.x; s < S; s += TB)
    {
      if (sh.state[s] != kRun)
        continue;
      const int p = s / m, c = s % m;
      const double curv = sh.tot[p * m + c];
      const double dd = sh.tot[S + p * m + c];
      if (!(curv > 1e-30 * dd))
      {
        sh.state[s] = kBreakdown;
        sh.sit[s] = it;
      }
      else
        sh.alpha[s] = sh.rho[s] / curv;
    }
    __syncthreads();
    // ---- phase B
    band_phase_b<TB, MT, RPT>(P, sh, d_new);
    grid.sync();
    reduce_blocks<TB, BandParams>(P, sh, m);
    ++it;
    for (int s = threadIdx.x; s < S; s += TB)
    {
      if (sh.state[s] != kRun)
        continue;
      const double rn = sh.tot[s];
      if (P.hist && blockIdx.x == 0 && it - 1 < P.hist_cap)
        P.hist[static_cast<int64_t>(s) * P.hist_cap + (it - 1)] = sqrt(rn) / sh.bnorm[s];
      sh.beta[s] = rn / sh.rho[s];
      sh.rho[s] = rn;
      sh.fresh[s] = 0;
    }
    __syncthreads();
    cur ^= 1;
  }

  // ---- budget exhausted: final true-residual check
  if (threadIdx.x == 0)
    sh.flag = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P.l; p += TB)
  {
    int need = 0;
    for (int c = 0; c < m; ++c)
      need |= sh.state[p * m + c] == kRun;
    sh.pmask[p] = need;
    if (need)
      atomicOr(&sh.flag, 1);
  }
  __syncthreads();
  if (sh.flag)
  {
    band_phase_a<TB, MT, RPT, true>(P, sh, smem_dyn, nullptr, nullptr);
    grid.sync();
    reduce_blocks<TB, BandParams>(P, sh, m);
    for (int s = threadIdx.x; s < S; s += TB)
    {
      if (sh.state[s] != kRun)
        continue;
      const double tt = sh.tot[s];
      sh.state[s] = sqrt(tt) <= sh.target[s] ? kPendingConv : kMaxed;
      sh.sit[s] = it;
    }
    __syncthreads();
    band_finish_copy<TB>(P, sh);
    for (int s = threadIdx.x; s < S; s += TB)
      if (sh.state[s] == kPendingConv)
        sh.state[s] = kConverged;
    __syncthreads();
  }
  // ---- recurrence residual block, zero-rhs outputs, per-column scalars
  for (int p = threadIdx.x; p < P.l; p += TB)
    sh.pmask[p] = 1;
  __syncthreads();
  for_segments(P, sh, [&](int p, int64_t rs, int64_t re) {
    const int64_t base = static_cast<int64_t>(p) * P.n * m;
    for (int64_t i = rs + threadIdx.x; i < re; i += TB)
      for (int c = 0; c < m; ++c)
      {
        const int s = p * m + c;
        const int64_t o = static_cast<int64_t>(s) * P.n + i;
        if (sh.state[s] == kZeroRhs)
        {
          if (P.X)
            P.X[o] = 0.0;
          if (P.TR)
            P.TR[o] = 0.0;
          if (P.REC)
            P.REC[o] = 0.0;
        }
        else if (sh.state[s] != kBreakdown && P.REC)
          P.REC[o] = __ldcg(P.r + base + i * m + c);
      }
  });
  if (blockIdx.x == 0)
  {
    for (int s = threadIdx.x; s < S; s += TB)
    {
      const int st = sh.state[s];
      P.iters[s] = sh.sit[s];
      P.conv[s] = (st == kConverged || st == kZeroRhs) ? 1 : 0;
      P.status[s] = st == kBreakdown ? MGPU_ERR_BREAKDOWN : MGPU_OK;
      P.bd_iter[s] = st == kBreakdown ? sh.sit[s] : -1;
    }
    if (threadIdx.x == 0)
      *P.loop_iters = it;
  }
}


// B [p][c][row] (column-major per point; ldb between points) -> interleaved
// b, r = b, d = b, x~ = 0.
__global__ void cg_init(int l, int m, int64_t n, const double *__restrict__ B, int64_t ldb, double *__restrict__ b,
                        double *__restrict__ r, double *__restrict__ d, double *__restrict__ xt)
{
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = n * m;
  if (g >= per * l)
    return;
  const int64_t p = g / per, rem = g - p * per, i = rem / m, c = rem - i * m;
  const double v = B[p * ldb + c * n + i];
  b[g] = v;
  r[g] = v;
  d[g] = v;
  xt[g] = 0.0;
}

template <int MT>
void launch_cg(mgpu_ctx *ctx, const CgParams &P)
{
  int per_sm = 0;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_persistent<MT>, kCgThreads, 0));
  if (per_sm < 1)
    throw Error(MGPU_ERR_CUDA, "cg_persistent: kernel does not fit on an SM");
  int64_t want = static_cast<int64_t>(P.l) * P.tiles;
  int64_t grid = static_cast<int64_t>(per_sm) * ctx->num_sms;
  if (grid > want)
    grid = want;
  if (grid < 1)
    grid = 1;
  CgParams local = P;
  void *args[] = {&local};
  MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(cg_persistent<MT>), dim3(static_cast<unsigned>(grid)),
                                      dim3(kCgThreads), args, 0, ctx->stream));
  check_launch(ctx, "cg_persistent");
}

template <int TB, int MT, int RPT>
void launch_banded_cfg(mgpu_ctx *ctx, const BandParams &P)
{
  // stage-0 buffer (d_new, read again by the dot products) + the chain's ping-pong pair
  const size_t dyn = sizeof(double) * (P.z >= 2 ? 3 : 2) * static_cast<size_t>(TB * RPT + 2 * P.hmax) * P.m;
  MG_CUDA(cudaFuncSetAttribute(cg_banded<TB, MT, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(dyn)));
  int per_sm = 0;
  MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_banded<TB, MT, RPT>, TB, dyn));
  if (per_sm < 1)
    throw Error(MGPU_ERR_CUDA, "cg_banded: kernel does not fit on an SM");
  BandParams local = P;
  void *args[] = {&local};
  MG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(cg_banded<TB, MT, RPT>),
                                      dim3(static_cast<unsigned>(ctx->num_sms)), dim3(TB), args, dyn, ctx->stream));
  check_launch(ctx, "cg_banded");
}

// Rows per thread: enough that one chunk covers a block's range when the
// problem is small; capped for register pressure.
template <int TB, int MT>
void launch_banded_rpt(mgpu_ctx *ctx, BandParams &P)
{
  const int64_t per_point = P.l <= ctx->num_sms ? (ctx->num_sms / P.l) : 1;
  const int64_t rows_per_block =
      P.l <= ctx->num_sms ? (P.npad + per_point - 1) / per_point : P.npad * ((P.l + ctx->num_sms - 1) / ctx->num_sms);
  int rpt = static_cast<int>((rows_per_block + TB - 1) / TB);
  rpt = rpt < 1 ? 1 : (rpt > kMaxRpt ? kMaxRpt : rpt);
  if (rpt == 3)
    rpt = 4;
  // shorter chunks when the stage buffers (2, or 3 with a chain of >= 2 factors) would not fit
  int optin = 0;
  MG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const auto dyn_of = [&](int r) {
    return sizeof(double) * (P.z >= 2 ? 3 : 2) * static_cast<size_t>(TB * r + 2 * P.hmax) * P.m + 4096;
  };
  while (rpt > 1 && dyn_of(rpt) + sizeof(BandShared<TB>) > static_cast<size_t>(optin))
    rpt /= 2;
  P.rpt = rpt;
  if (rpt == 1)
    launch_banded_cfg<TB, MT, 1>(ctx, P);
  else if (rpt == 2)
    launch_banded_cfg<TB, MT, 2>(ctx, P);
  else
    launch_banded_cfg<TB, MT, 4>(ctx, P);
}

// Halo plan of the banded path; false when an operator is too wide for it.
bool band_plan(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains, int m,
               int *halo, int *hmax)
{
  if (z > kMaxZ || static_cast<int64_t>(l) * m > kMaxSys || l > kMaxPoints)
    return false;
  int64_t bwA = 0;
  std::vector<int64_t> bwF(static_cast<size_t>(z > 0 ? z : 1), 0);
  for (int p = 0; p < l; ++p)
  {
    bwA = std::max(bwA, csr_bandwidth(ctx, const_cast<mgpu_csr *>(A[p])));
    for (int f = 0; f < z; ++f)
      bwF[f] = std::max(bwF[f], csr_bandwidth(ctx, const_cast<mgpu_csr *>(chains[static_cast<size_t>(p) * z + f])));
  }
  // stage st applies chains[z-1-st]; halo[st] = halo[st+1] + bw of that factor
  int64_t h = bwA;
  halo[z] = static_cast<int>(std::min<int64_t>(h, INT32_MAX));
  for (int st = z - 1; st >= 0; --st)
  {
    h += bwF[z - 1 - st];
    halo[st] = static_cast<int>(std::min<int64_t>(h, INT32_MAX));
  }
  *hmax = halo[0];
  return h <= kMaxHalo;
}


// One sub-batch: l points (all columns m <= kMaxM).
void cg_batch(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains, int64_t n,
              int m, const double *B_dev, int64_t ldb, double rtol, int64_t maxit, double *X_dev, double *REC_dev,
              double *TR_dev, int64_t *iters, int *conv, int *status, int64_t *bd, double *hist, int64_t hist_cap,
              double *ms_out, int64_t *loop_out)
{
  cudaStream_t s = ctx->stream;
  host_mark("cg_batch enter");
  int halo[kMaxZ + 1] = {0};
  int hmax = 0;
  const bool banded = ctx->cg_path != 1 && band_plan(ctx, l, A, z, chains, m, halo, &hmax);
  host_mark("band_plan done");
  const int64_t vec = static_cast<int64_t>(l) * n * m;
  const int64_t vbytes = sizeof(double) * (vec > 0 ? vec : 1);
  DBuf b, xt, r, d, w, t0, t1; // grid kernels' vectors, allocated only if those kernels run
  const int S = l * m;
  // per-system results in ONE device block (iterations, breakdown iteration, loop count,
  // converged, status), read back with one copy into the context's pinned staging buffer
  const size_t o_bd = sizeof(int64_t) * S, o_loop = 2 * sizeof(int64_t) * S, o_conv = o_loop + sizeof(int64_t),
               o_st = o_conv + sizeof(int) * S, res_bytes = o_st + sizeof(int) * S;
  DBuf res(res_bytes, s);
  auto *p_it = res.as<int64_t>();
  auto *p_bd = reinterpret_cast<int64_t *>(res.as<char>() + o_bd);
  auto *p_loop = reinterpret_cast<int64_t *>(res.as<char>() + o_loop);
  auto *p_conv = reinterpret_cast<int *>(res.as<char>() + o_conv);
  auto *p_st = reinterpret_cast<int *>(res.as<char>() + o_st);
  DBuf d_hist(hist ? sizeof(double) * static_cast<size_t>(S) * hist_cap : 8, s);
  std::vector<DCsr> hA(static_cast<size_t>(l)), hF(static_cast<size_t>(l) * (z > 0 ? z : 1));
  for (int p = 0; p < l; ++p)
  {
    hA[p] = A[p]->view();
    for (int f = 0; f < z; ++f)
      hF[static_cast<size_t>(p) * z + f] = chains[static_cast<size_t>(p) * z + f]->view();
  }
  DBuf dA(sizeof(DCsr) * hA.size(), s), dF(sizeof(DCsr) * hF.size(), s);
  MG_CUDA(cudaMemcpyAsync(dA.ptr, hA.data(), sizeof(DCsr) * hA.size(), cudaMemcpyHostToDevice, s));
  MG_CUDA(cudaMemcpyAsync(dF.ptr, hF.data(), sizeof(DCsr) * hF.size(), cudaMemcpyHostToDevice, s));

  host_mark("descriptors staged");
  DBuf partial, totals, counter, segs, pblk;
  int clustered = 0;
  if (banded && ctx->cg_path != 2 && ctx->cg_path != 4)
  {
    // systems small enough to live on chip: one cluster per point, no grid barrier
    MG_CUDA(cudaMemsetAsync(p_loop, 0, sizeof(int64_t), s));
    MG_CUDA(cudaEventRecord(ctx->ev0, s));
    clustered = cg_cluster_solve(ctx, l, A, z, chains, n, m, B_dev, ldb, halo, rtol, maxit, X_dev, REC_dev, TR_dev,
                                 p_it, p_conv, p_st, p_bd,
                                 hist ? d_hist.as<double>() : nullptr, hist_cap,
                                 reinterpret_cast<unsigned long long *>(p_loop), dA.as<DCsr>(), dF.as<DCsr>());
    if (clustered)
      MG_CUDA(cudaEventRecord(ctx->ev1, s));
    host_mark("cluster launched");
  }
  bool streamed = false;
  // streaming pays once a block's share of the batch (rows x columns) hides the
  // per-pass pipeline fill; below that the grid-banded kernel is as fast (measured
  // break-even ~1K elements per SM on B200)
  // and the chain is short: every chain stage adds factor buffers to each ring slot, so the
  // chunks shrink and the per-chunk cost wins -- measured on configs[2] (n = 1e5, 8 points,
  // LS update chain, 1000 iterations): stream 31 / 44 / 50 / 68 / 88 / 97 / 132 / 145 ms at
  // z = 1..8 against banded 45 / 56 / 67 / 77 / 89 / 99 / 110 / 121 ms, so z >= 7 goes to the
  // banded kernel
  const bool stream_pays = static_cast<int64_t>(l) * n * m >= static_cast<int64_t>(2048) * ctx->num_sms && z <= 6;
  if (banded && !clustered && (ctx->cg_path == 4 || (ctx->cg_path == 0 && stream_pays)))
  {
    MG_CUDA(cudaMemsetAsync(p_loop, 0, sizeof(int64_t), s));
    streamed = stream_solve(ctx, l, A, z, chains, n, m, B_dev, ldb, halo, hmax, rtol, maxit, X_dev, REC_dev, TR_dev,
                            p_it, p_conv, p_st, p_bd,
                            hist ? d_hist.as<double>() : nullptr, hist_cap, p_loop);
  }
  if (!clustered && !streamed)
  {
    b = DBuf(vbytes, s);
    xt = DBuf(vbytes, s);
    r = DBuf(vbytes, s);
    d = DBuf(vbytes, s);
    w = DBuf(vbytes, s);
    t0 = DBuf(banded || z >= 1 ? vbytes : 8, s);
    t1 = DBuf(banded || z >= 2 ? vbytes : 8, s);
    cg_init<<<blocks_for(vec), kThreads, 0, s>>>(l, m, n, B_dev, ldb, b.as<double>(), r.as<double>(), d.as<double>(),
                                                   xt.as<double>());
    check_launch(ctx, "cg_init");
  }
  if (clustered || streamed)
  {
  }
  else if (banded)
  {
    partial = DBuf(sizeof(double) * static_cast<size_t>(l) * 2 * kMaxM * ctx->num_sms, s);
    // Segment plan: with l <= #SMs every point gets its own run of blocks (no
    // block straddles two points, so no block runs two latency chains); else
    // blocks take whole points.  Rows split in 32-row aligned pieces.
    const int G = ctx->num_sms;
    std::vector<Seg> hseg(static_cast<size_t>(G) * kMaxSeg, Seg{-1, 0, 0, 0});
    std::vector<int2> hpb(static_cast<size_t>(l));
    if (l <= G)
    {
      for (int p = 0; p < l; ++p)
      {
        const int b0 = static_cast<int>(static_cast<int64_t>(p) * G / l);
        const int b1 = static_cast<int>(static_cast<int64_t>(p + 1) * G / l);
        const int64_t groups = (n + 31) / 32;
        const int nb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b1 - b0, groups))); // no row-less blocks
        for (int k = 0; k < nb; ++k)
        {
          const int64_t g0 = groups * k / nb, g1 = groups * (k + 1) / nb;
          hseg[static_cast<size_t>(b0 + k) * kMaxSeg] =
              Seg{p, static_cast<int>(g0 * 32), static_cast<int>(std::min<int64_t>(n, g1 * 32)), 0};
        }
        hpb[p] = make_int2(b0, b0 + nb);
      }
    }
    else
    {
      for (int b = 0; b < G; ++b)
      {
        const int p0 = static_cast<int>(static_cast<int64_t>(b) * l / G);
        const int p1 = static_cast<int>(static_cast<int64_t>(b + 1) * l / G);
        if (p1 - p0 > kMaxSeg)
          throw Error(MGPU_ERR_UNSUPPORTED, "cg: too many shifts per SM for the banded kernel");
        for (int p = p0; p < p1; ++p)
        {
          hseg[static_cast<size_t>(b) * kMaxSeg + (p - p0)] = Seg{p, 0, static_cast<int>(n), 0};
          hpb[p] = make_int2(b, b + 1);
        }
      }
    }
    segs = DBuf(sizeof(Seg) * hseg.size(), s);
    pblk = DBuf(sizeof(int2) * hpb.size(), s);
    MG_CUDA(cudaMemcpyAsync(segs.ptr, hseg.data(), sizeof(Seg) * hseg.size(), cudaMemcpyHostToDevice, s));
    MG_CUDA(cudaMemcpyAsync(pblk.ptr, hpb.data(), sizeof(int2) * hpb.size(), cudaMemcpyHostToDevice, s));
    BandParams P{};
    P.seg = segs.as<Seg>();
    P.pblk = pblk.as<int2>();
    P.l = l;
    P.m = m;
    P.z = z;
    P.n = n;
    P.npad = (n + 31) / 32 * 32;
    for (int q = 0; q <= z; ++q)
      P.halo[q] = halo[q];
    P.hmax = hmax;
    P.A = dA.as<DCsr>();
    P.F = dF.as<DCsr>();
    P.rtol = rtol;
    P.maxit = maxit;
    P.b = b.as<double>();
    P.xt = xt.as<double>();
    P.r = r.as<double>();
    P.dbuf0 = d.as<double>();
    P.dbuf1 = t0.as<double>();
    P.w = w.as<double>();
    P.sol = t1.as<double>();
    P.partial = partial.as<double>();
    P.X = X_dev;
    P.REC = REC_dev;
    P.TR = TR_dev;
    P.iters = p_it;
    P.conv = p_conv;
    P.status = p_st;
    P.bd_iter = p_bd;
    P.hist = hist ? d_hist.as<double>() : nullptr;
    P.hist_cap = hist_cap;
    P.loop_iters = p_loop;
    MG_CUDA(cudaEventRecord(ctx->ev0, s));
    if (m == 1)
      launch_banded_rpt<1024, 1>(ctx, P);
    else if (m == 2)
      launch_banded_rpt<1024, 2>(ctx, P);
    else if (m <= 4)
      launch_banded_rpt<512, 4>(ctx, P);
    else
      launch_banded_rpt<512, 8>(ctx, P);
    MG_CUDA(cudaEventRecord(ctx->ev1, s));
  }
  else
  {
    // tile geometry depends on n only -> reduction order independent of the GPU
    int rpt = static_cast<int>((n + static_cast<int64_t>(kCgThreads) * kMaxTiles - 1) /
                               (static_cast<int64_t>(kCgThreads) * kMaxTiles));
    if (rpt < 1)
      rpt = 1;
    const int64_t rows_per_tile = static_cast<int64_t>(rpt) * kCgThreads;
    const int tiles = static_cast<int>((n + rows_per_tile - 1) / rows_per_tile);
    partial = DBuf(sizeof(double) * static_cast<size_t>(l) * 2 * kMaxM * tiles, s);
    totals = DBuf(sizeof(double) * 2 * static_cast<size_t>(l) * 2 * kMaxM, s);
    counter = DBuf(sizeof(unsigned int) * l, s);
    MG_CUDA(cudaMemsetAsync(counter.ptr, 0, sizeof(unsigned int) * l, s));
    CgParams P{};
    P.l = l;
    P.m = m;
    P.z = z;
    P.tiles = tiles;
    P.rpt = rpt;
    P.n = n;
    P.rows_per_tile = rows_per_tile;
    P.A = dA.as<DCsr>();
    P.F = dF.as<DCsr>();
    P.rtol = rtol;
    P.maxit = maxit;
    P.b = b.as<double>();
    P.xt = xt.as<double>();
    P.r = r.as<double>();
    P.d = d.as<double>();
    P.w = w.as<double>();
    P.t0 = t0.as<double>();
    P.t1 = t1.as<double>();
    P.partial = partial.as<double>();
    P.totals = totals.as<double>();
    P.counter = counter.as<unsigned int>();
    P.X = X_dev;
    P.REC = REC_dev;
    P.TR = TR_dev;
    P.iters = p_it;
    P.conv = p_conv;
    P.status = p_st;
    P.bd_iter = p_bd;
    P.hist = hist ? d_hist.as<double>() : nullptr;
    P.hist_cap = hist_cap;
    P.loop_iters = p_loop;
    MG_CUDA(cudaEventRecord(ctx->ev0, s));
    if (m == 1)
      launch_cg<1>(ctx, P);
    else if (m == 2)
      launch_cg<2>(ctx, P);
    else if (m <= 4)
      launch_cg<4>(ctx, P);
    else
      launch_cg<8>(ctx, P);
    MG_CUDA(cudaEventRecord(ctx->ev1, s));
  }

  host_mark("results requested");
  char *hres = static_cast<char *>(pinned_scratch(ctx, res_bytes));
  MG_CUDA(cudaMemcpyAsync(hres, res.ptr, res_bytes, cudaMemcpyDeviceToHost, s));
  if (hist)
    MG_CUDA(cudaMemcpyAsync(hist, d_hist.ptr, sizeof(double) * static_cast<size_t>(S) * hist_cap,
                            cudaMemcpyDeviceToHost, s));
  MG_CUDA(cudaStreamSynchronize(s));
  std::memcpy(iters, hres, sizeof(int64_t) * S);
  std::memcpy(bd, hres + o_bd, sizeof(int64_t) * S);
  std::memcpy(conv, hres + o_conv, sizeof(int) * S);
  std::memcpy(status, hres + o_st, sizeof(int) * S);
  int64_t loop = 0;
  std::memcpy(&loop, hres + o_loop, sizeof(int64_t));
  host_mark("results read");
  float ms = 0.f;
  MG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  *ms_out += ms;
  *loop_out += loop;
  ctx->last_cg_path = clustered ? clustered : (streamed ? 4 : (banded ? 0 : 1));
}

} // namespace
} // namespace mgpu

using namespace mgpu;

extern "C" int mgpu_cg_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains,
                             int64_t n, int64_t m, const double *B, int64_t ldb_point, double rtol, int64_t maxit,
                             mgpu_memkind where, mgpu_cg_out *out)
{
  return guard(ctx, [&] {
    host_mark("mgpu_cg_solve enter");
    MG_ARG(l >= 1 && A != nullptr && B != nullptr && out != nullptr, "pcg_solve: null argument");
    MG_ARG(z >= 0 && (z == 0 || chains != nullptr), "pcg_solve: bad preconditioner chain");
    MG_ARG(m >= 1 && n >= 0, "block_solve: right-hand-side rows do not match the operator dimension");
    MG_ARG(where == MGPU_HOST || where == MGPU_DEVICE, "pcg_solve: bad memory kind");
    MG_ARG(out->iterations && out->converged && out->status && out->breakdown_iteration,
           "pcg_solve: per-column outputs are required");
    for (int p = 0; p < l; ++p)
    {
      MG_ARG(A[p] != nullptr && A[p]->nrows == n && A[p]->ncols == n,
             "block_solve: right-hand-side rows do not match the operator dimension");
      for (int f = 0; f < z; ++f)
      {
        const mgpu_csr *F = chains[static_cast<size_t>(p) * z + f];
        MG_ARG(F != nullptr && F->nrows == n && F->ncols == n, "pcg_solve: dimension mismatch");
      }
    }
    MG_ARG(rtol > 0.0, "pcg_solve: rtol must be positive"); // krylov.cpp:37-40
    cudaStream_t s = ctx->stream;
    const int64_t blk = n * m;
    const int64_t ldb = ldb_point;
    MG_ARG(ldb == 0 || ldb >= blk, "pcg_solve: ldb_point smaller than one n x m block");

    // stage host inputs/outputs through device buffers
    DBuf Bd, Xd, Rd, Td;
    const double *B_dev = B;
    double *X_dev = out->X, *REC_dev = out->recurrence, *TR_dev = out->true_res;
    const int64_t outer_elems = static_cast<int64_t>(l) * blk;
    if (where == MGPU_HOST)
    {
      const int64_t in_elems = ldb == 0 ? blk : static_cast<int64_t>(l - 1) * ldb + blk;
      Bd = DBuf(sizeof(double) * (in_elems > 0 ? in_elems : 1), s);
      if (in_elems > 0)
        MG_CUDA(cudaMemcpyAsync(Bd.ptr, B, sizeof(double) * in_elems, cudaMemcpyHostToDevice, s));
      B_dev = Bd.as<double>();
      if (out->X)
      {
        Xd = DBuf(sizeof(double) * (outer_elems > 0 ? outer_elems : 1), s);
        X_dev = Xd.as<double>();
      }
      if (out->recurrence)
      {
        Rd = DBuf(sizeof(double) * (outer_elems > 0 ? outer_elems : 1), s);
        REC_dev = Rd.as<double>();
      }
      if (out->true_res)
      {
        Td = DBuf(sizeof(double) * (outer_elems > 0 ? outer_elems : 1), s);
        TR_dev = Td.as<double>();
      }
    }

    double total_ms = 0.0;
    int64_t total_loop = 0;
    const int S = l * static_cast<int>(m);
    std::vector<int64_t> it(static_cast<size_t>(S)), bd(static_cast<size_t>(S));
    std::vector<int> cv(static_cast<size_t>(S)), st(static_cast<size_t>(S));
    std::vector<double> hist;
    if (out->history && out->history_cap > 0)
      hist.resize(static_cast<size_t>(S) * out->history_cap);

    if (n > 0)
    {
      // split into launches of <= kMaxM columns and <= kMaxSys systems
      for (int64_t c0 = 0; c0 < m; c0 += kMaxM)
      {
        const int mc = static_cast<int>(m - c0 < kMaxM ? m - c0 : kMaxM);
        const int pts = kMaxSys / mc < kMaxPoints ? kMaxSys / mc : kMaxPoints;
        for (int p0 = 0; p0 < l; p0 += pts)
        {
          const int lp = l - p0 < pts ? l - p0 : pts;
          if (mc == m)
          {
            // every column in one launch: the caller's [point][column][row] layout is the
            // kernel's, so B is read in place (point stride ldb, 0 = shared) and the
            // outputs are written in place
            const int Ss = lp * mc;
            std::vector<int64_t> sit(Ss), sbd(Ss);
            std::vector<int> scv(Ss), sst(Ss);
            std::vector<double> shist(hist.empty() ? 0 : static_cast<size_t>(Ss) * out->history_cap);
            const int64_t o = static_cast<int64_t>(p0) * blk;
            cg_batch(ctx, lp, A + p0, z, z > 0 ? chains + static_cast<size_t>(p0) * z : nullptr, n, mc,
                     B_dev + (ldb == 0 ? 0 : static_cast<int64_t>(p0) * ldb), ldb, rtol, maxit,
                     X_dev ? X_dev + o : nullptr, REC_dev ? REC_dev + o : nullptr, TR_dev ? TR_dev + o : nullptr,
                     sit.data(), scv.data(), sst.data(), sbd.data(), shist.empty() ? nullptr : shist.data(),
                     out->history_cap, &total_ms, &total_loop);
            for (int q = 0; q < Ss; ++q)
            {
              const int64_t dst = static_cast<int64_t>(p0) * m + q;
              it[dst] = sit[q];
              cv[dst] = scv[q];
              st[dst] = sst[q];
              bd[dst] = sbd[q];
              if (!hist.empty())
                std::copy(shist.begin() + static_cast<int64_t>(q) * out->history_cap,
                          shist.begin() + static_cast<int64_t>(q + 1) * out->history_cap,
                          hist.begin() + dst * out->history_cap);
            }
            continue;
          }
          // gather the column slice [c0, c0+mc) of every point into a compact block
          DBuf Bs(sizeof(double) * static_cast<size_t>(lp) * n * mc, s);
          for (int p = 0; p < lp; ++p)
          {
            const double *src = B_dev + (ldb == 0 ? 0 : static_cast<int64_t>(p0 + p) * ldb) + c0 * n;
            MG_CUDA(cudaMemcpyAsync(Bs.as<double>() + static_cast<int64_t>(p) * n * mc, src,
                                    sizeof(double) * n * mc, cudaMemcpyDeviceToDevice, s));
          }
          const int Ss = lp * mc;
          DBuf Xs(X_dev ? sizeof(double) * static_cast<size_t>(Ss) * n : 8, s);
          DBuf Rs(REC_dev ? sizeof(double) * static_cast<size_t>(Ss) * n : 8, s);
          DBuf Ts(TR_dev ? sizeof(double) * static_cast<size_t>(Ss) * n : 8, s);
          std::vector<int64_t> sit(Ss), sbd(Ss);
          std::vector<int> scv(Ss), sst(Ss);
          std::vector<double> shist(hist.empty() ? 0 : static_cast<size_t>(Ss) * out->history_cap);
          cg_batch(ctx, lp, A + p0, z, z > 0 ? chains + static_cast<size_t>(p0) * z : nullptr, n, mc, Bs.as<double>(),
                   static_cast<int64_t>(n) * mc, rtol, maxit, X_dev ? Xs.as<double>() : nullptr,
                   REC_dev ? Rs.as<double>() : nullptr, TR_dev ? Ts.as<double>() : nullptr, sit.data(), scv.data(),
                   sst.data(), sbd.data(), shist.empty() ? nullptr : shist.data(), out->history_cap, &total_ms,
                   &total_loop);
          for (int p = 0; p < lp; ++p)
            for (int c = 0; c < mc; ++c)
            {
              const int64_t dst = static_cast<int64_t>(p0 + p) * m + c0 + c;
              const int src = p * mc + c;
              it[dst] = sit[src];
              cv[dst] = scv[src];
              st[dst] = sst[src];
              bd[dst] = sbd[src];
              if (!hist.empty())
                std::copy(shist.begin() + static_cast<int64_t>(src) * out->history_cap,
                          shist.begin() + static_cast<int64_t>(src + 1) * out->history_cap,
                          hist.begin() + dst * out->history_cap);
              const int64_t o = dst * n, so = static_cast<int64_t>(src) * n;
              if (X_dev)
                MG_CUDA(cudaMemcpyAsync(X_dev + o, Xs.as<double>() + so, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                                        s));
              if (REC_dev)
                MG_CUDA(cudaMemcpyAsync(REC_dev + o, Rs.as<double>() + so, sizeof(double) * n,
                                        cudaMemcpyDeviceToDevice, s));
              if (TR_dev)
                MG_CUDA(cudaMemcpyAsync(TR_dev + o, Ts.as<double>() + so, sizeof(double) * n,
                                        cudaMemcpyDeviceToDevice, s));
            }
        }
      }
    }
    else
    {
      for (int q = 0; q < S; ++q)
      {
        it[q] = 0;
        cv[q] = 1; // empty system: ||b|| = 0 -> converged (krylov.cpp:44-51)
        st[q] = MGPU_OK;
        bd[q] = -1;
      }
    }
    if (where == MGPU_HOST && outer_elems > 0)
    {
      if (out->X)
        MG_CUDA(cudaMemcpyAsync(out->X, X_dev, sizeof(double) * outer_elems, cudaMemcpyDeviceToHost, s));
      if (out->recurrence)
        MG_CUDA(cudaMemcpyAsync(out->recurrence, REC_dev, sizeof(double) * outer_elems, cudaMemcpyDeviceToHost, s));
      if (out->true_res)
        MG_CUDA(cudaMemcpyAsync(out->true_res, TR_dev, sizeof(double) * outer_elems, cudaMemcpyDeviceToHost, s));
    }
    MG_CUDA(cudaStreamSynchronize(s));
    ctx->last_cg_ms = total_ms;
    ctx->last_cg_iters = total_loop;
    for (int q = 0; q < S; ++q)
    {
      out->iterations[q] = it[q];
      out->converged[q] = cv[q];
      out->status[q] = st[q];
      out->breakdown_iteration[q] = bd[q];
    }
    if (!hist.empty())
      std::copy(hist.begin(), hist.end(), out->history);
    // first breakdown in (point, column) order, with block_solve's payload
    for (int q = 0; q < S; ++q)
    {
      if (st[q] == MGPU_ERR_BREAKDOWN)
      {
        const int64_t col = q % m, pt = q / m;
        throw Error(MGPU_ERR_BREAKDOWN,
                    "block_solve: column " + std::to_string(col) +
                        ": pcg_solve: direction curvature breakdown at iteration " + std::to_string(bd[q]),
                    bd[q], col, pt);
      }
    }
  });
}
