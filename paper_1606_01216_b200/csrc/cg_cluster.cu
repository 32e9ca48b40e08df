// K-cg (cluster-resident): one thread-block CLUSTER per shifted system.
//
// The l shifted systems are independent, so a solve needs
// no grid-wide synchronisation at all: each point gets a cluster of CS <= 16
// CTAs (one per SM) that owns its rows for the whole solve.  Everything the
// CG loop touches lives on chip:
//   * A(s) and the SPAI chain factors, repacked once into ELL rows in shared
//     memory (values + int8 column offsets, bandwidth <= 64);
//   * x~, r, d (double-buffered) in shared memory, w in registers;
//   * halo rows of r / d / x~ are read from the neighbouring CTAs' shared
//     memory through DSMEM (cluster.map_shared_rank);
//   * dot products: per thread in row order -> fixed warp butterfly -> fixed
//     warp order -> per-CTA slot; after the cluster barrier every CTA sums
//     the CS slots in rank order, so all CTAs take identical decisions.
// Per iteration: 2 cluster barriers (hardware, ~0.2 us) instead of 2 grid
// barriers (~1.2 us), and no L2 round trips on the critical path.
// Semantics are those of krylov.cpp:28-139 (see cg.cu); SpMV / axpy
// arithmetic is bitwise that of the reference's scalar kernels.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "internal.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
int64_t csr_max_row(mgpu_ctx *ctx, mgpu_csr *A);

namespace
{

constexpr int kCMaxZ = 8;
constexpr int kCMaxM = 4;
constexpr int kCMaxCS = 16;

enum CState : int
{
  cRun = 0,
  cConverged = 1,
  cBreakdown = 2,
  cZeroRhs = 3,
  cMaxed = 4,
};

struct ClParams
{
  int l, m, z, cs, rb; // rb: rows per CTA (last CTA may own fewer)
  int ea;              // ELL width of A
  int ef[kCMaxZ];      // ELL width of chain factor used by stage st
  int halo[kCMaxZ + 1];
  int64_t n;
  const DCsr *A, *F;
  const double *B;
  int64_t ldb;
  double rtol;
  int64_t maxit;
  // shared-memory carve-up (bytes)
  size_t off_x, off_r, off_d0, off_d1, off_s0, off_s1, off_part, off_av, off_ao, off_fv[kCMaxZ], off_fo[kCMaxZ];
  double *X, *REC, *TR;
  int64_t *iters;
  int *conv, *status;
  int64_t *bd_iter;
  double *hist;
  int64_t hist_cap;
  unsigned long long *loop_iters;
};

struct ClShared
{
  double rho[kCMaxM], target[kCMaxM], alpha[kCMaxM], beta[kCMaxM], bnorm[kCMaxM];
  double tot[2 * kCMaxM];
  int state[kCMaxM], fresh[kCMaxM];
  int64_t sit[kCMaxM];
  double red[32][2 * kCMaxM];
};

// CTA-level deterministic sum of NV per-thread values into slot[k] (k < nv).
template <int TB, int NV>
__device__ __forceinline__ void cta_sum(ClShared &sh, double (&v)[NV], int nv, double *slot)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k)
  {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      v[k] = __dadd_rn(v[k], __shfl_xor_sync(0xffffffffu, v[k], off));
  }
  if (lane == 0)
  {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      sh.red[warp][k] = v[k];
  }
  __syncthreads();
  if (warp == 0)
  {
    for (int k = 0; k < nv; ++k)
    {
      double x = lane < TB / 32 ? sh.red[lane][k] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, off));
      if (lane == 0)
        slot[k] = x;
    }
  }
}

// After cluster.sync(): tot[k] = sum over ranks (fixed order) of slot[k].
__device__ __forceinline__ void cluster_total(cgrp::cluster_group &cl, ClShared &sh, double *slot, int nv, int cs)
{
  if (threadIdx.x < nv)
  {
    double vals[kCMaxCS];
#pragma unroll
    for (int q = 0; q < kCMaxCS; ++q)
      vals[q] = q < cs ? cl.map_shared_rank(slot, q)[threadIdx.x] : 0.0;
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kCMaxCS; ++q)
      if (q < cs)
        t = __dadd_rn(t, vals[q]);
    sh.tot[threadIdx.x] = t;
  }
  __syncthreads();
}

template <int TB, int MT, int RPT>
struct Cl
{
  const ClParams &P;
  cgrp::cluster_group &cl;
  ClShared &sh;
  unsigned char *raw;
  int rank, p, m, R;
  int64_t c0, c1;

  __device__ double *x() const { return reinterpret_cast<double *>(raw + P.off_x); }
  __device__ double *r() const { return reinterpret_cast<double *>(raw + P.off_r); }
  __device__ double *d(int k) const { return reinterpret_cast<double *>(raw + (k ? P.off_d1 : P.off_d0)); }
  __device__ double *s(int k) const { return reinterpret_cast<double *>(raw + (k ? P.off_s1 : P.off_s0)); }
  __device__ double *part(int k) const { return reinterpret_cast<double *>(raw + P.off_part) + k * 2 * kCMaxM; }

  // value of a cluster-owned vector (x / r / d buffer) at global row i
  __device__ __forceinline__ const double *remote(double *local, int64_t i, int c) const
  {
    const int owner = static_cast<int>(i / P.rb);
    const int64_t li = i - static_cast<int64_t>(owner) * P.rb;
    const double *base = owner == rank ? local : cl.map_shared_rank(local, owner);
    return base + li * m + c;
  }

  // stage 0 on [c0 - H0, c1 + H0): source x~ (check) or d_new = fresh ? r : r + beta d_old
  template <bool kCheck>
  __device__ void stage0(int cur)
  {
    const int H0 = P.halo[0];
    double *s0 = s(0);
    double *dold = d(cur), *dnew = d(cur ^ 1);
    const int span = R + 2 * H0;
    for (int q = threadIdx.x; q < span; q += TB)
    {
      const int64_t i = c0 - H0 + q;
      if (i < 0 || i >= P.n)
        continue;
      const bool own = i >= c0 && i < c1;
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        if (c >= m)
          break;
        double v;
        if (kCheck)
          v = *remote(x(), i, c);
        else
        {
          const double rv = *remote(r(), i, c);
          v = sh.fresh[c] ? rv : __dadd_rn(rv, __dmul_rn(sh.beta[c], *remote(dold, i, c)));
          if (own)
            dnew[(i - c0) * m + c] = v;
        }
        s0[q * m + c] = v;
      }
    }
    __syncthreads();
  }

  // chain stages on shared memory; returns the buffer index holding P source, and its halo
  __device__ int chain(int &hs_out)
  {
    int src = 0, hs = P.halo[0];
    for (int st = 0; st < P.z; ++st)
    {
      const int hd = P.halo[st + 1];
      const int E = P.ef[st];
      const double *fv = reinterpret_cast<const double *>(raw + P.off_fv[st]);
      const signed char *fo = reinterpret_cast<const signed char *>(raw + P.off_fo[st]);
      const double *in = s(src);
      double *out = s(src ^ 1);
      const int span = R + 2 * hd;
      for (int q = threadIdx.x; q < span; q += TB)
      {
        const int64_t i = c0 - hd + q;
        if (i < 0 || i >= P.n)
          continue;
        const int base_in = (q + hs - hd); // local row of i in the input buffer
        double acc[MT];
#pragma unroll
        for (int c = 0; c < MT; ++c)
          acc[c] = 0.0;
        for (int e = 0; e < E; ++e)
        {
          const double fvv = fv[q * E + e];
          const int loc = (base_in + fo[q * E + e]) * m;
#pragma unroll
          for (int c = 0; c < MT; ++c)
            if (c < m)
              acc[c] = __dadd_rn(acc[c], __dmul_rn(fvv, in[loc + c]));
        }
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
            out[q * m + c] = acc[c];
      }
      __syncthreads();
      src ^= 1;
      hs = hd;
    }
    hs_out = hs;
    return src;
  }

  // y = A t for own rows (thread-owned rows lr = threadIdx.x + j * TB)
  __device__ void apply_a(int src, int hs, double (&y)[RPT][MT])
  {
    const double *av = reinterpret_cast<const double *>(raw + P.off_av);
    const signed char *ao = reinterpret_cast<const signed char *>(raw + P.off_ao);
    const double *in = s(src);
    const int E = P.ea;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * TB;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        y[j][c] = 0.0;
      if (lr >= R)
        continue;
      for (int e = 0; e < E; ++e)
      {
        const double a = av[lr * E + e];
        const int loc = (lr + hs + ao[lr * E + e]) * m;
#pragma unroll
        for (int c = 0; c < MT; ++c)
          if (c < m)
            y[j][c] = __dadd_rn(y[j][c], __dmul_rn(a, in[loc + c]));
      }
    }
  }
};

// ELL repack of rows [r0, r1) of a CSR matrix (offsets relative to the row).
__device__ void load_ell(DCsr M, int64_t r0, int64_t r1, int64_t n, int E, double *v, signed char *o, int TBn)
{
  const int64_t rows = r1 - r0;
  for (int64_t q = threadIdx.x; q < rows; q += TBn)
  {
    const int64_t i = r0 + q;
    int64_t k = 0, e = 0;
    if (i >= 0 && i < n)
    {
      k = M.rp[i];
      e = M.rp[i + 1];
    }
    for (int t = 0; t < E; ++t)
    {
      if (k + t < e)
      {
        v[q * E + t] = M.v[k + t];
        o[q * E + t] = static_cast<signed char>(M.ci[k + t] - i);
      }
      else
      {
        v[q * E + t] = 0.0; // padding after the row's entries: adds +0 at the end
        o[q * E + t] = 0;
      }
    }
  }
}

template <int TB, int MT, int RPT>
__global__ void __launch_bounds__(TB, 1) cg_cluster(ClParams P)
{
  cgrp::cluster_group cl = cgrp::this_cluster();
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ ClShared sh;
  const int cs = P.cs;
  Cl<TB, MT, RPT> C{P, cl, sh, raw, static_cast<int>(cl.block_rank()), static_cast<int>(blockIdx.x / cs), P.m, 0, 0,
                    0};
  C.c0 = static_cast<int64_t>(C.rank) * P.rb;
  C.c1 = min(P.n, C.c0 + P.rb);
  C.R = C.c1 > C.c0 ? static_cast<int>(C.c1 - C.c0) : 0;
  const int m = P.m, p = C.p;
  const int64_t c0 = C.c0;
  const int R = C.R;

  // ---- load operators (ELL) and the rhs
  load_ell(P.A[p], c0, c0 + R, P.n, P.ea, reinterpret_cast<double *>(raw + P.off_av),
           reinterpret_cast<signed char *>(raw + P.off_ao), TB);
  for (int st = 0; st < P.z; ++st)
  {
    const int hd = P.halo[st + 1];
    load_ell(P.F[p * P.z + (P.z - 1 - st)], c0 - hd, c0 + R + hd, P.n, P.ef[st],
             reinterpret_cast<double *>(raw + P.off_fv[st]), reinterpret_cast<signed char *>(raw + P.off_fo[st]), TB);
  }
  double bv[RPT][MT];
  double w[RPT][MT];
  double part[2 * MT];
#pragma unroll
  for (int q = 0; q < 2 * MT; ++q)
    part[q] = 0.0;
#pragma unroll
  for (int j = 0; j < RPT; ++j)
  {
    const int lr = threadIdx.x + j * TB;
#pragma unroll
    for (int c = 0; c < MT; ++c)
    {
      bv[j][c] = 0.0;
      if (lr < R && c < m)
      {
        bv[j][c] = P.B[static_cast<int64_t>(p) * P.ldb + static_cast<int64_t>(c) * P.n + c0 + lr];
        C.x()[lr * m + c] = 0.0;
        C.r()[lr * m + c] = bv[j][c];
        C.d(0)[lr * m + c] = bv[j][c];
        part[c] = __dadd_rn(part[c], __dmul_rn(bv[j][c], bv[j][c]));
      }
    }
  }
  cta_sum<TB, 2 * MT>(sh, part, m, C.part(0));
  cl.sync();
  cluster_total(cl, sh, C.part(0), m, cs);
  if (threadIdx.x < m)
  {
    const int c = threadIdx.x;
    const double bb = sh.tot[c], bn = sqrt(bb);
    sh.bnorm[c] = bn;
    sh.rho[c] = bb;
    sh.target[c] = P.rtol * bn;
    sh.state[c] = bn == 0.0 ? cZeroRhs : cRun;
    sh.fresh[c] = 1;
    sh.beta[c] = 0.0;
    sh.sit[c] = 0;
  }
  __syncthreads();

  // true-residual check: sol = P x~, res = b - A sol, ||res||^2 -> decisions
  // kind 0: confirm (krylov.cpp:77-103), kind 1: budget exhausted (:128-137)
  auto check = [&](int kind, int64_t it) {
    C.template stage0<true>(0);
    int hs;
    const int src = C.chain(hs);
    double y[RPT][MT], sol[RPT][MT];
    C.apply_a(src, hs, y);
    double pk[2 * MT];
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
      pk[q] = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * TB;
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        sol[j][c] = 0.0;
        if (lr < R && c < m)
        {
          sol[j][c] = C.s(src)[(lr + hs) * m + c];
          y[j][c] = __dsub_rn(bv[j][c], y[j][c]); // res
          pk[c] = __dadd_rn(pk[c], __dmul_rn(y[j][c], y[j][c]));
        }
      }
    }
    cta_sum<TB, 2 * MT>(sh, pk, m, C.part(0));
    cl.sync();
    cluster_total(cl, sh, C.part(0), m, cs);
    // decisions (identical in every CTA)
    int fin[MT], rst[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
    {
      fin[c] = rst[c] = 0;
      if (c >= m || sh.state[c] != cRun)
        continue;
      if (kind == 0 && !(sqrt(sh.rho[c]) <= sh.target[c]))
        continue;
      const double tt = sh.tot[c];
      if (kind == 1)
        fin[c] = 1;
      else if (sqrt(tt) <= sh.target[c])
        fin[c] = 1;
      else if (sqrt(tt) <= sh.target[c]) // krylov.cpp:98-102 (rho = (r, r) of the same vector)
        fin[c] = 1;
      else
        rst[c] = 1;
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * TB;
      if (lr >= R)
        continue;
#pragma unroll
      for (int c = 0; c < MT; ++c)
      {
        if (c >= m)
          continue;
        const int64_t o = (static_cast<int64_t>(p) * m + c) * P.n + c0 + lr;
        if (fin[c])
        {
          if (P.X)
            P.X[o] = sol[j][c];
          if (P.TR)
            P.TR[o] = y[j][c];
        }
        else if (rst[c])
          C.r()[lr * m + c] = y[j][c];
      }
    }
    __syncthreads(); // all reads of sh.tot / sh.state done before the updates
    if (threadIdx.x < m)
    {
      const int c = threadIdx.x;
      if (fin[c])
      {
        sh.state[c] = (kind == 1 && !(sqrt(sh.tot[c]) <= sh.target[c])) ? cMaxed : cConverged;
        sh.sit[c] = it;
      }
      else if (rst[c])
      {
        sh.rho[c] = sh.tot[c];
        sh.fresh[c] = 1;
      }
    }
    cl.sync(); // restarted r visible to the neighbours; slots free again
  };

  int cur = 0;
  int64_t it = 0;
  for (;;)
  {
    if (it >= P.maxit)
      break;
    bool need = false, live = false;
    for (int c = 0; c < m; ++c)
    {
      need |= sh.state[c] == cRun && sqrt(sh.rho[c]) <= sh.target[c];
      live |= sh.state[c] == cRun;
    }
    if (need)
    {
      check(0, it);
      live = false;
      for (int c = 0; c < m; ++c)
        live |= sh.state[c] == cRun;
    }
    if (!live)
      break;
    // ---- phase A: d_new (own + halo), t = P_chain d_new, w = A t, (d,w), (d,d)
    C.template stage0<false>(cur);
    int hs;
    const int src = C.chain(hs);
    C.apply_a(src, hs, w);
    const double *dnew = C.d(cur ^ 1);
    double pk[2 * MT];
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
      pk[q] = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * TB;
      if (lr >= R)
        continue;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (c < m)
        {
          const double dn = dnew[lr * m + c];
          pk[c] = __dadd_rn(pk[c], __dmul_rn(dn, w[j][c]));
          pk[MT + c] = __dadd_rn(pk[MT + c], __dmul_rn(dn, dn));
        }
    }
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
    cta_sum<TB, 2 * MT>(sh, pv, 2 * m, C.part(0));
    cl.sync();
    cluster_total(cl, sh, C.part(0), 2 * m, cs);
    bool run[MT];
    double al[MT];
#pragma unroll
    for (int c = 0; c < MT; ++c)
    {
      run[c] = false;
      al[c] = 0.0;
      if (c < m && sh.state[c] == cRun)
      {
        const double curv = sh.tot[c], dd = sh.tot[m + c];
        if (!(curv > 1e-30 * dd)) // krylov.cpp:108
        {
          if (threadIdx.x == 0)
          {
            sh.state[c] = cBreakdown;
            sh.sit[c] = it;
          }
        }
        else
        {
          run[c] = true;
          al[c] = sh.rho[c] / curv;
        }
      }
    }
    // ---- phase B: x~ += alpha d_new, r -= alpha w, (r, r)
#pragma unroll
    for (int q = 0; q < 2 * MT; ++q)
      pk[q] = 0.0;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * TB;
      if (lr >= R)
        continue;
#pragma unroll
      for (int c = 0; c < MT; ++c)
        if (run[c])
        {
          double *xp = C.x() + lr * m + c, *rp = C.r() + lr * m + c;
          *xp = __dadd_rn(*xp, __dmul_rn(al[c], dnew[lr * m + c]));
          const double rn = __dadd_rn(*rp, __dmul_rn(-al[c], w[j][c]));
          *rp = rn;
          pk[c] = __dadd_rn(pk[c], __dmul_rn(rn, rn));
        }
    }
    cta_sum<TB, 2 * MT>(sh, pk, m, C.part(1));
    cl.sync();
    cluster_total(cl, sh, C.part(1), m, cs);
    ++it;
    if (threadIdx.x < m)
    {
      const int c = threadIdx.x;
      if (run[c])
      {
        const double rn = sh.tot[c];
        if (P.hist && C.rank == 0 && it - 1 < P.hist_cap)
          P.hist[(static_cast<int64_t>(p) * m + c) * P.hist_cap + (it - 1)] = sqrt(rn) / sh.bnorm[c];
        sh.beta[c] = rn / sh.rho[c];
        sh.rho[c] = rn;
        sh.fresh[c] = 0;
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  bool live = false;
  for (int c = 0; c < m; ++c)
    live |= sh.state[c] == cRun;
  if (live)
    check(1, it);
  // ---- outputs: recurrence residual block, zero-rhs blocks, scalars
  for (int q = threadIdx.x; q < R; q += TB)
    for (int c = 0; c < m; ++c)
    {
      const int64_t o = (static_cast<int64_t>(p) * m + c) * P.n + c0 + q;
      if (sh.state[c] == cZeroRhs)
      {
        if (P.X)
          P.X[o] = 0.0;
        if (P.TR)
          P.TR[o] = 0.0;
        if (P.REC)
          P.REC[o] = 0.0;
      }
      else if (sh.state[c] != cBreakdown && P.REC)
        P.REC[o] = C.r()[q * m + c];
    }
  if (C.rank == 0 && threadIdx.x < m)
  {
    const int c = threadIdx.x, s = p * m + c;
    const int st = sh.state[c];
    P.iters[s] = sh.sit[c];
    P.conv[s] = (st == cConverged || st == cZeroRhs) ? 1 : 0;
    P.status[s] = st == cBreakdown ? MGPU_ERR_BREAKDOWN : MGPU_OK;
    P.bd_iter[s] = st == cBreakdown ? sh.sit[c] : -1;
    if (c == 0)
      atomicMax(P.loop_iters, static_cast<unsigned long long>(it));
  }
  cl.sync(); // no CTA leaves while others may still read its shared memory
}

template <int TB, int MT, int RPT>
bool launch_cluster(mgpu_ctx *ctx, ClParams &P, size_t dyn)
{
  auto kern = cg_cluster<TB, MT, RPT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)) != cudaSuccess)
  {
    cudaGetLastError();
    return false;
  }
  if (P.cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
  {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(P.l * P.cs));
  cfg.blockDim = dim3(TB);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(P.cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1)
  {
    cudaGetLastError();
    return false;
  }
  MG_CUDA(cudaLaunchKernelEx(&cfg, kern, P));
  check_launch(ctx, "cg_cluster");
  return true;
}

} // namespace

// Tries the cluster-resident solve; false when the systems do not fit on chip
// (the caller then uses the grid-wide kernels).
bool cg_cluster_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains,
                      int64_t n, int m, const double *B_dev, int64_t ldb, const int *halo, double rtol,
                      int64_t maxit, double *X, double *REC, double *TR, int64_t *d_it, int *d_conv, int *d_st,
                      int64_t *d_bd, double *d_hist, int64_t hist_cap, unsigned long long *d_loop, const DCsr *dA,
                      const DCsr *dF)
{
  if (m > kCMaxM || z > kCMaxZ || n <= 0 || n > INT32_MAX)
    return false;
  int ea = 0;
  int ef[kCMaxZ] = {0};
  for (int p = 0; p < l; ++p)
  {
    ea = std::max<int>(ea, static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(A[p]))));
    for (int st = 0; st < z; ++st)
      ef[st] = std::max<int>(ef[st], static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(
                                                                       chains[static_cast<size_t>(p) * z + (z - 1 - st)]))));
  }
  const int TB = m <= 2 ? 1024 : 512;
  const int rpt_max = 2;
  int cdev = 0;
  MG_CUDA(cudaDeviceGetAttribute(&cdev, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const size_t budget = static_cast<size_t>(cdev) - sizeof(ClShared) - 1024;
  for (int cs = 1; cs <= kCMaxCS; cs *= 2)
  {
    const int64_t rb = (n + cs - 1) / cs;
    if (rb > static_cast<int64_t>(TB) * rpt_max)
      continue;
    if (rb < halo[0] && cs > 1)
      break; // halos would span several CTAs: not worth it at this size
    ClParams P{};
    P.l = l;
    P.m = m;
    P.z = z;
    P.cs = cs;
    P.rb = static_cast<int>(rb);
    P.ea = ea;
    for (int st = 0; st < z; ++st)
      P.ef[st] = ef[st];
    for (int q = 0; q <= z; ++q)
      P.halo[q] = halo[q];
    P.n = n;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 15) & ~static_cast<size_t>(15);
      return o;
    };
    const size_t vec = sizeof(double) * static_cast<size_t>(rb) * m;
    P.off_x = take(vec);
    P.off_r = take(vec);
    P.off_d0 = take(vec);
    P.off_d1 = take(vec);
    const size_t stg = sizeof(double) * static_cast<size_t>(rb + 2 * halo[0]) * m;
    P.off_s0 = take(stg);
    P.off_s1 = take(stg);
    P.off_part = take(sizeof(double) * 4 * kCMaxM);
    P.off_av = take(sizeof(double) * static_cast<size_t>(rb) * ea);
    P.off_ao = take(static_cast<size_t>(rb) * ea);
    for (int st = 0; st < z; ++st)
    {
      const size_t rows = static_cast<size_t>(rb + 2 * halo[st + 1]);
      P.off_fv[st] = take(sizeof(double) * rows * ef[st]);
      P.off_fo[st] = take(rows * ef[st]);
    }
    if (off > budget)
      continue;
    P.A = dA;
    P.F = dF;
    P.B = B_dev;
    P.ldb = ldb;
    P.rtol = rtol;
    P.maxit = maxit;
    P.X = X;
    P.REC = REC;
    P.TR = TR;
    P.iters = d_it;
    P.conv = d_conv;
    P.status = d_st;
    P.bd_iter = d_bd;
    P.hist = d_hist;
    P.hist_cap = hist_cap;
    P.loop_iters = d_loop;
    const int rpt = rb > TB ? 2 : 1;
    bool ok;
    if (TB == 1024)
    {
      if (m == 1)
        ok = rpt == 1 ? launch_cluster<1024, 1, 1>(ctx, P, off) : launch_cluster<1024, 1, 2>(ctx, P, off);
      else
        ok = rpt == 1 ? launch_cluster<1024, 2, 1>(ctx, P, off) : launch_cluster<1024, 2, 2>(ctx, P, off);
    }
    else
      ok = rpt == 1 ? launch_cluster<512, 4, 1>(ctx, P, off) : launch_cluster<512, 4, 2>(ctx, P, off);
    if (ok)
      return true;
  }
  return false;
}

} // namespace mgpu
