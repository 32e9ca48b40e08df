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
#include <cmath>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace cgrp = cooperative_groups;

namespace mgpu
{
int64_t csr_max_row(mgpu_ctx *ctx, mgpu_csr *A);

namespace
{

constexpr int kCMaxZ = 12; // chain factors (the AIRGA update chain grows by one per outer iteration)
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

// CTA sum of nv values, PUSHED into slot k * kCMaxCS + rank of every CTA's
// `inbox` (one remote store per destination, issued before the barrier):
// after the cluster barrier each CTA reduces its own, local inbox.
template <int TB, int NV>
__device__ __forceinline__ void cta_sum_push(ClShared &sh, double (&v)[NV], int nv, cgrp::cluster_group &cl,
                                             double *inbox, int cs, int rank)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
  {
#pragma unroll
    for (int k = 0; k < NV; ++k) // quantities interleaved: independent shuffle chains in flight
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
    double x[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k)
      x[k] = (k < nv && lane < TB / 32) ? sh.red[lane][k] : 0.0;
    // lanes >= TB / 32 hold exact zeros: the first butterfly level would add 0 (x + 0 == x)
#pragma unroll
    for (int off = TB / 32 >= 32 ? 16 : TB / 64; off > 0; off >>= 1)
    {
#pragma unroll
      for (int k = 0; k < NV; ++k)
        x[k] = __dadd_rn(x[k], __shfl_xor_sync(0xffffffffu, x[k], off));
    }
    if (lane < cs)
    {
      double *dst = cl.map_shared_rank(inbox, lane);
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (k < nv)
          dst[k * kCMaxCS + rank] = x[k];
    }
  }
}

template <int NV>
__device__ __forceinline__ void warp_inbox_total(const double *inbox, int nv, int cs, double (&out)[NV])
{
  // cs <= kCMaxCS = 16 slots: both half-warps load the same slots and reduce over 4 levels.
  // Bitwise what a 5-level butterfly over 16 values + 16 zeros gives (x + 0 == x).
  static_assert(kCMaxCS == 16, "half-warp inbox reduction");
  const int slot = threadIdx.x & (kCMaxCS - 1);
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k)
    v[k] = (k < nv && slot < cs) ? inbox[k * kCMaxCS + slot] : 0.0;
#pragma unroll
  for (int off = kCMaxCS / 2; off > 0; off >>= 1)
  {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      v[k] = __dadd_rn(v[k], __shfl_xor_sync(0xffffffffu, v[k], off));
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
    out[k] = v[k];
}

// ---- asynchronous cluster exchange (v2 main loop): remote stores that complete an
// mbarrier transaction on the receiving CTA, so a reduction waits only for its own data
// instead of a cluster-wide barrier (no release fence over every prior store, no L1 flush).
__device__ __forceinline__ uint32_t cl_map(const void *local, int rank)
{
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(local))), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar)
{
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cl_mbar_init(uint64_t *bar)
{
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void cl_mbar_arm(uint64_t *bar, uint32_t bytes)
{
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_mbar_wait(uint64_t *bar, uint32_t parity)
{
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\t"
               "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra W_%=;\n\t}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(parity)
               : "memory");
}

// cta_sum_push over the asynchronous exchange: the CTA total of nv values goes to slot
// k * kCMaxCS + rank of every CTA's inbox, completing `bar` (same offset) there.
template <int TB, int NV>
__device__ __forceinline__ void cta_sum_push_async(ClShared &sh, double (&v)[NV], int nv, double *inbox,
                                                   uint64_t *bar, int cs, int rank)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
  {
#pragma unroll
    for (int k = 0; k < NV; ++k)
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
    // every sending lane sums the TB/32 warp totals itself (broadcast reads, pairwise tree):
    // no shuffle round trips on the critical path
    static_assert((TB / 32 & (TB / 32 - 1)) == 0, "warp count must be a power of two");
    double x[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k)
    {
      double t[TB / 32];
#pragma unroll
      for (int w = 0; w < TB / 32; ++w)
        t[w] = k < nv ? sh.red[w][k] : 0.0;
#pragma unroll
      for (int h = TB / 64; h > 0; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w)
          t[w] = __dadd_rn(t[2 * w], t[2 * w + 1]);
      x[k] = t[0];
    }
    if (lane < cs)
    {
      const uint32_t rb = cl_map(bar, lane);
#pragma unroll
      for (int k = 0; k < NV; ++k)
        if (k < nv)
          st_async_f64(cl_map(inbox + k * kCMaxCS + rank, lane), x[k], rb);
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

// Entry-major ELL repack (v[t * rows + q]): consecutive rows -> consecutive shared-memory
// words, so a warp's SpMV loads are bank-conflict free; the row's int8 column offsets are
// packed into one 64-bit word (E <= 8): one offset load per row instead of E byte loads.
__device__ void load_ell_em_packed(DCsr M, int64_t r0, int64_t r1, int64_t n, int E, double *v,
                                   unsigned long long *o, int TBn)
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
    unsigned long long word = 0;
    for (int t = 0; t < E; ++t)
    {
      const bool has = k + t < e;
      v[t * rows + q] = has ? M.v[k + t] : 0.0;
      const unsigned long long b =
          has ? static_cast<unsigned long long>(static_cast<unsigned char>(static_cast<signed char>(M.ci[k + t] - i)))
              : 0ull;
      word |= b << (8 * t);
    }
    o[q] = word;
  }
}

__device__ __forceinline__ int off8(unsigned long long w, int t)
{
  return static_cast<int>(static_cast<signed char>((w >> (8 * t)) & 0xffull));
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

// =====================================================================
// v2 (single right-hand side): vectors in REGISTERS, d in a halo-padded
// shared buffer updated in place, neighbours exchange only boundary rows.
// Footprint ~110 B/row (A and P in ELL + d + t), so a 2e4-row system fits a
// 10-CTA cluster and 8 systems run in ONE wave (11 co-resident 10-CTA
// clusters on B200 vs 7 of 16).
//   exports (parity-double-buffered, read by the neighbours through DSMEM):
//     ex_r[q][side]: boundary rows of r_k  (written in phase B of k-1)
//     ex_d[q][side]: boundary rows of d_{k-1} (written in phase A of k-1)
//     ex_x[side]   : boundary rows of x~ (written before a residual check)
// =====================================================================
constexpr int kV2TB = 512;

struct V2Params
{
  int l, z, cs, rb, ea, H;
  int ef[kCMaxZ];
  int halo[kCMaxZ + 1];
  int64_t n;
  const DCsr *A, *F;
  const double *B;
  int64_t ldb;
  double rtol;
  int64_t maxit;
  size_t off_d, off_t0, off_t1, off_part, off_ex, off_av, off_ao, off_fv[kCMaxZ], off_fo[kCMaxZ];
  double *X, *REC, *TR;
  int64_t *iters;
  int *conv, *status;
  int64_t *bd_iter;
  double *hist;
  int64_t hist_cap;
  unsigned long long *loop_iters;
  long long *prof; // optional [16] accumulated clock64 deltas per phase (cluster 0, rank 0, thread 0)
  int async_x;     // 1: main-loop reductions and halos over st.async + mbarriers, 0: cluster barriers
};

// EC > 0: every operator row (A and each chain factor) holds exactly EC ELL entries, known at
// compile time, so the entry loops unroll with constant offsets; EC = 0: runtime widths.
// AX: asynchronous exchange (else cluster barriers); PR: per-phase clock64 profile (MGPU_PROFILE_PHASES)
// acc + a * b in cg_cluster_v2's SpMV, dot and axpy terms: two roundings (the reference's scalar
// kernel table, bitwise) by default; one DFMA with -DMGPU_CLUSTER_FMA (the reference's AVX2 table
// contracts these, kernels_avx2.cpp:34-35, 57, 88) -- the DESIGN.md 5 experiment (tools/fma_experiment.py).
#ifdef MGPU_CLUSTER_FMA
#define V2_MADD(acc, a, b) fma((a), (b), (acc))
#else
#define V2_MADD(acc, a, b) __dadd_rn((acc), __dmul_rn((a), (b)))
#endif

template <int RPT, int EC = 0, bool AX = true, bool PR = false>
__global__ void __launch_bounds__(kV2TB, 1) cg_cluster_v2(V2Params P)
{
  cgrp::cluster_group cl = cgrp::this_cluster();
  extern __shared__ __align__(16) unsigned char raw[];
  __shared__ ClShared sh;
  const int cs = P.cs, H = P.H;
  const int rank = static_cast<int>(cl.block_rank());
  const int p = static_cast<int>(blockIdx.x / cs);
  const int64_t c0 = static_cast<int64_t>(rank) * P.rb;
  const int64_t c1 = min(P.n, c0 + P.rb);
  const int R = c1 > c0 ? static_cast<int>(c1 - c0) : 0;
  double *dpad = reinterpret_cast<double *>(raw + P.off_d); // rows [c0 - H, c1 + H)
  double *tb[2] = {reinterpret_cast<double *>(raw + P.off_t0), reinterpret_cast<double *>(raw + P.off_t1)};
  double *part = reinterpret_cast<double *>(raw + P.off_part); // inboxes [2 phases][2 * kCMaxM][kCMaxCS]
  double *inboxA = part, *inboxB = part + 2 * kCMaxM * kCMaxCS;
  double *ex = reinterpret_cast<double *>(raw + P.off_ex);                    // exports
  auto ex_r = [&](double *base, int q, int side) { return base + ((0 * 2 + q) * 2 + side) * H; };
  auto ex_d = [&](double *base, int q, int side) { return base + ((1 * 2 + q) * 2 + side) * H; };
  auto ex_x = [&](double *base, int side) { return base + (4 * 2 + side) * H; };
  // boundary rows are PUSHED into the neighbours' import buffers (remote
  // stores before the barrier), so halos are read from local shared memory.
  double *left = rank > 0 ? cl.map_shared_rank(ex, rank - 1) : nullptr;       // left neighbour's imports
  double *right = rank + 1 < cs ? cl.map_shared_rank(ex, rank + 1) : nullptr; // right neighbour's imports
  // my row lr (boundary) -> the neighbour import slot that mirrors it
  auto push = [&](auto sel, int q, int lr, double v) {
    if (lr < H && left)
      sel(left, q, 1)[lr] = v;
    if (lr >= R - H && right)
      sel(right, q, 0)[lr - (R - H)] = v;
  };
  auto sel_r = [&](double *b, int q, int side) { return ex_r(b, q, side); };
  auto sel_d = [&](double *b, int q, int side) { return ex_d(b, q, side); };
  auto sel_x = [&](double *b, int, int side) { return ex_x(b, side); };
  // asynchronous exchange (P.async_x): xbar[0] completes when phase A's partials (every CTA)
  // and d boundary rows (neighbours) have landed, xbar[1] likewise for phase B and r
  __shared__ __align__(8) uint64_t xbar[2];
  const int nbrs = (rank > 0 ? 1 : 0) + (rank + 1 < cs ? 1 : 0);
  const uint32_t bytesA = static_cast<uint32_t>(8 * (2 * cs + H * nbrs));
  const uint32_t bytesB = static_cast<uint32_t>(8 * (cs + H * nbrs));
  uint32_t exL = 0, exR = 0, barL[2] = {0, 0}, barR[2] = {0, 0};
  if constexpr (AX)
  {
    if (threadIdx.x == 0)
    {
      cl_mbar_init(&xbar[0]);
      cl_mbar_init(&xbar[1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      cl_mbar_arm(&xbar[0], bytesA);
      cl_mbar_arm(&xbar[1], bytesB);
    }
    if (rank > 0)
    {
      exL = cl_map(ex, rank - 1);
      barL[0] = cl_map(&xbar[0], rank - 1);
      barL[1] = cl_map(&xbar[1], rank - 1);
    }
    if (rank + 1 < cs)
    {
      exR = cl_map(ex, rank + 1);
      barR[0] = cl_map(&xbar[0], rank + 1);
      barR[1] = cl_map(&xbar[1], rank + 1);
    }
  }
  // boundary row lr of r (which 0) or d (which 1), parity slot q -> the neighbours' imports,
  // completing their phase-B (r) or phase-A (d) barrier
  auto push_async = [&](int which, int q, int lr, double v) {
    if (lr < H && exL)
      st_async_f64(exL + 8u * static_cast<uint32_t>(((which * 2 + q) * 2 + 1) * H + lr), v, barL[which ^ 1]);
    if (lr >= R - H && exR)
      st_async_f64(exR + 8u * static_cast<uint32_t>(((which * 2 + q) * 2 + 0) * H + (lr - (R - H))), v,
                   barR[which ^ 1]);
  };

  load_ell_em_packed(P.A[p], c0, c0 + R, P.n, P.ea, reinterpret_cast<double *>(raw + P.off_av),
                     reinterpret_cast<unsigned long long *>(raw + P.off_ao), kV2TB);
  for (int st = 0; st < P.z; ++st)
  {
    const int hd = P.halo[st + 1];
    load_ell_em_packed(P.F[p * P.z + (P.z - 1 - st)], c0 - hd, c0 + R + hd, P.n, P.ef[st],
                       reinterpret_cast<double *>(raw + P.off_fv[st]),
                       reinterpret_cast<unsigned long long *>(raw + P.off_fo[st]), kV2TB);
  }
  double r[RPT], x[RPT], w[RPT];
  // b is re-read from global memory by the (rare) true-residual checks: not register-resident
  auto b_at = [&](int lr) { return P.B[static_cast<int64_t>(p) * P.ldb + c0 + lr]; };
  double bv[RPT];
  double pk[2] = {0.0, 0.0};
#pragma unroll
  for (int j = 0; j < RPT; ++j)
  {
    const int lr = threadIdx.x + j * kV2TB;
    bv[j] = lr < R ? P.B[static_cast<int64_t>(p) * P.ldb + c0 + lr] : 0.0;
    r[j] = bv[j];
    x[j] = 0.0;
    w[j] = 0.0;
    if (lr < R)
    {
      dpad[H + lr] = bv[j];
      pk[0] = __dadd_rn(pk[0], __dmul_rn(bv[j], bv[j]));
      push(sel_r, 0, lr, bv[j]);
      push(sel_d, 0, lr, bv[j]);
    }
  }
  cta_sum_push<kV2TB, 2>(sh, pk, 1, cl, inboxA, cs, rank);
  cl.sync();
  // per-system scalars live in registers; every thread derives identical values
  double tv[2];
  warp_inbox_total<2>(inboxA, 1, cs, tv);
  const double bnorm = sqrt(tv[0]);
  double rho = tv[0], beta = 0.0;
  const double target = P.rtol * bnorm;
  int state = bnorm == 0.0 ? cZeroRhs : cRun, fresh = 1;
  int64_t sit = 0;

  // chain on shared memory: stage 0 source = dpad (halo H = halo[0]); returns
  // the buffer holding P(source) and its halo.
  auto chain = [&](int &hs) -> const double * {
    const double *in = dpad;
    hs = P.halo[0];
    for (int st = 0; st < P.z; ++st)
    {
      const int hd = P.halo[st + 1];
      const int E = EC > 0 ? EC : P.ef[st];
      const double *fv = reinterpret_cast<const double *>(raw + P.off_fv[st]);
      const unsigned long long *fo = reinterpret_cast<const unsigned long long *>(raw + P.off_fo[st]);
      double *out = tb[st & 1];
      const int span = R + 2 * hd;
      // K rows per thread, entries outer / rows inner: independent accumulation chains in
      // flight (ILP); per-row order is unchanged.  K = RPT when the halo-extended span still
      // fits RPT slots (no dead, predicated-off slot in the unrolled body), else RPT + 1.
      auto rows_k = [&](auto kc) {
        constexpr int K = decltype(kc)::value;
        int q[K];
        bool ok[K];
        double acc[K];
        unsigned long long ow[K];
#pragma unroll
        for (int j = 0; j < K; ++j)
        {
          q[j] = threadIdx.x + j * kV2TB;
          const int64_t i = c0 - hd + q[j];
          ok[j] = q[j] < span && i >= 0 && i < P.n;
          acc[j] = 0.0;
          ow[j] = ok[j] ? fo[q[j]] : 0ull;
        }
#pragma unroll
        for (int e = 0; e < (EC > 0 ? EC : E); ++e)
        {
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (ok[j])
              acc[j] = V2_MADD(acc[j], fv[e * span + q[j]], in[q[j] + hs - hd + off8(ow[j], e)]);
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (ok[j])
            out[q[j]] = acc[j];
      };
      constexpr int K = RPT + 1;
      if (span <= RPT * kV2TB)
        rows_k(std::integral_constant<int, RPT>{});
      else
        rows_k(std::integral_constant<int, RPT + 1>{});
      for (int qq = threadIdx.x + K * kV2TB; qq < span; qq += kV2TB) // only if span > K * TB
      {
        const int64_t i = c0 - hd + qq;
        if (i < 0 || i >= P.n)
          continue;
        double a = 0.0;
        const unsigned long long w1 = fo[qq];
        for (int e = 0; e < E; ++e)
          a = V2_MADD(a, fv[e * span + qq], in[qq + hs - hd + off8(w1, e)]);
        out[qq] = a;
      }
      __syncthreads();
      in = out;
      hs = hd;
    }
    return in;
  };
  auto apply_a = [&](const double *in, int hs, double (&y)[RPT]) {
    const double *av = reinterpret_cast<const double *>(raw + P.off_av);
    const unsigned long long *ao = reinterpret_cast<const unsigned long long *>(raw + P.off_ao);
    const int E = EC > 0 ? EC : P.ea;
    bool ok[RPT];
    unsigned long long ow[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      y[j] = 0.0;
      ok[j] = threadIdx.x + j * kV2TB < R;
      ow[j] = ok[j] ? ao[threadIdx.x + j * kV2TB] : 0ull;
    }
#pragma unroll
    for (int e = 0; e < (EC > 0 ? EC : E); ++e)
    {
#pragma unroll
      for (int j = 0; j < RPT; ++j)
      {
        const int lr = threadIdx.x + j * kV2TB;
        if (ok[j])
          y[j] = V2_MADD(y[j], av[e * R + lr], in[lr + hs + off8(ow[j], e)]);
      }
    }
  };
  // halo rows of dpad from the neighbours' exports (mode 0: d_new = fresh ? r : r + beta d; 1: x~)
  auto fill_halo = [&](int mode, int q) {
    for (int t = threadIdx.x; t < 2 * H; t += kV2TB)
    {
      const int side = t / H, k = t % H; // side 0: rows c0 - H + k (left neighbour's right export)
      const int64_t i = side == 0 ? c0 - H + k : c1 + k;
      if (i < 0 || i >= P.n)
        continue;
      double v;
      if (mode == 1)
        v = ex_x(ex, side)[k];
      else
      {
        const double rv = ex_r(ex, q, side)[k];
        v = fresh ? rv : V2_MADD(rv, beta, ex_d(ex, q, side)[k]);
      }
      dpad[side == 0 ? k : H + R + k] = v;
    }
  };

  // true-residual check (kind 0 confirm, krylov.cpp:77-103; kind 1 budget exhausted, :128-137)
  auto check = [&](int kind, int64_t it) {
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      if (lr < R)
      {
        dpad[H + lr] = x[j]; // d_old is not needed afterwards: the single column finishes or restarts
        push(sel_x, 0, lr, x[j]);
      }
    }
    cl.sync();
    fill_halo(1, 0);
    __syncthreads();
    int hs;
    const double *t = chain(hs);
    double y[RPT], sol[RPT];
    apply_a(t, hs, y);
    double q2[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      sol[j] = 0.0;
      if (lr < R)
      {
        sol[j] = t[lr + hs];
        y[j] = __dsub_rn(b_at(lr), y[j]);
        q2[0] = V2_MADD(q2[0], y[j], y[j]);
      }
    }
    cta_sum_push<kV2TB, 2>(sh, q2, 1, cl, inboxA, cs, rank);
    cl.sync();
    double cv[2];
    warp_inbox_total<2>(inboxA, 1, cs, cv);
    const double tt = cv[0];
    bool fin = kind == 1 || sqrt(tt) <= target;
    const bool rst = !fin;
    if (kind == 0 && !fin && sqrt(tt) <= target) // krylov.cpp:98-102
      fin = true;
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      if (lr >= R)
        continue;
      const int64_t o = static_cast<int64_t>(p) * P.n + c0 + lr;
      if (fin)
      {
        if (P.X)
          P.X[o] = sol[j];
        if (P.TR)
          P.TR[o] = y[j];
      }
      else
      {
        r[j] = y[j]; // restart from the true residual, d = r
        push(sel_r, static_cast<int>(it & 1), lr, y[j]);
      }
    }
    if (fin)
    {
      state = (kind == 1 && !(sqrt(tt) <= target)) ? cMaxed : cConverged;
      sit = it;
    }
    else if (rst)
    {
      rho = tt;
      fresh = 1;
    }
    cl.sync(); // restarted r exports visible; the slots are free again
  };

  const bool prof = PR && P.prof && blockIdx.x == 0 && threadIdx.x == 0;
  long long pacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tmark = clock64();
  auto mark = [&](int k) {
    if (prof)
    {
      const long long now = clock64();
      pacc[k] += now - tmark;
      tmark = now;
    }
  };
  int64_t it = 0;
  for (;;)
  {
    if (it >= P.maxit)
      break;
    if (state == cRun && sqrt(rho) <= target)
      check(0, it);
    if (state != cRun)
      break;
    mark(0);
    const int q = static_cast<int>(it & 1);
    // ---- phase A: d_new in place (own rows) + halo from exports, t = P d, w = A t
    double pa[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      if (lr < R)
      {
        const double dn = fresh ? r[j] : V2_MADD(r[j], beta, dpad[H + lr]);
        dpad[H + lr] = dn;
        if constexpr (AX)
          push_async(1, q ^ 1, lr, dn);
        else
          push(sel_d, q ^ 1, lr, dn);
      }
    }
    fill_halo(0, q);
    __syncthreads();
    mark(1);
    int hs;
    const double *t = chain(hs);
    mark(2);
    apply_a(t, hs, w);
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      if (lr < R)
      {
        const double dn = dpad[H + lr];
        pa[0] = V2_MADD(pa[0], dn, w[j]);
        pa[1] = V2_MADD(pa[1], dn, dn);
      }
    }
    mark(3);
    if constexpr (AX)
    {
      cta_sum_push_async<kV2TB, 2>(sh, pa, 2, inboxA, &xbar[0], cs, rank);
      mark(4);
      cl_mbar_wait(&xbar[0], static_cast<uint32_t>(q));
      if (threadIdx.x == 0)
        cl_mbar_arm(&xbar[0], bytesA); // next phase; peers send into it only after our phase-B partial
    }
    else
    {
      cta_sum_push<kV2TB, 2>(sh, pa, 2, cl, inboxA, cs, rank);
      mark(4);
      cl.sync();
    }
    mark(5);
    double ta[2];
    warp_inbox_total<2>(inboxA, 2, cs, ta);
    mark(6);
    const double curv = ta[0], dd = ta[1];
    if (!(curv > 1e-30 * dd)) // krylov.cpp:108
    {
      state = cBreakdown;
      sit = it;
      break;
    }
    const double alpha = rho / curv;
    // ---- phase B: x~ += alpha d, r -= alpha w, (r, r); export boundary r_{k+1}
    double pb[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < RPT; ++j)
    {
      const int lr = threadIdx.x + j * kV2TB;
      if (lr < R)
      {
        x[j] = V2_MADD(x[j], alpha, dpad[H + lr]);
        r[j] = V2_MADD(r[j], -alpha, w[j]);
        pb[0] = V2_MADD(pb[0], r[j], r[j]);
        if constexpr (AX)
          push_async(0, q ^ 1, lr, r[j]);
        else
          push(sel_r, q ^ 1, lr, r[j]);
      }
    }
    mark(7);
    if constexpr (AX)
    {
      cta_sum_push_async<kV2TB, 2>(sh, pb, 1, inboxB, &xbar[1], cs, rank);
      cl_mbar_wait(&xbar[1], static_cast<uint32_t>(q));
      if (threadIdx.x == 0)
        cl_mbar_arm(&xbar[1], bytesB);
    }
    else
    {
      cta_sum_push<kV2TB, 2>(sh, pb, 1, cl, inboxB, cs, rank);
      cl.sync();
    }
    mark(8);
    double tb2[2];
    warp_inbox_total<2>(inboxB, 1, cs, tb2);
    mark(9);
    ++it;
    const double rn = tb2[0];
    if (P.hist && rank == 0 && threadIdx.x == 0 && it - 1 < P.hist_cap)
      P.hist[static_cast<int64_t>(p) * P.hist_cap + (it - 1)] = sqrt(rn) / bnorm;
    beta = rn / rho; // krylov.cpp:118-119
    rho = rn;
    fresh = 0;
  }
  if (prof)
    for (int k = 0; k < 10; ++k)
      P.prof[k] = pacc[k];
  if (state == cRun)
    check(1, it);
  for (int j = 0; j < RPT; ++j)
  {
    const int lr = threadIdx.x + j * kV2TB;
    if (lr >= R)
      continue;
    const int64_t o = static_cast<int64_t>(p) * P.n + c0 + lr;
    if (state == cZeroRhs)
    {
      if (P.X)
        P.X[o] = 0.0;
      if (P.TR)
        P.TR[o] = 0.0;
      if (P.REC)
        P.REC[o] = 0.0;
    }
    else if (state != cBreakdown && P.REC)
      P.REC[o] = r[j];
  }
  if (rank == 0 && threadIdx.x == 0)
  {
    P.iters[p] = sit;
    P.conv[p] = (state == cConverged || state == cZeroRhs) ? 1 : 0;
    P.status[p] = state == cBreakdown ? MGPU_ERR_BREAKDOWN : MGPU_OK;
    P.bd_iter[p] = state == cBreakdown ? sit : -1;
    atomicMax(P.loop_iters, static_cast<unsigned long long>(it));
  }
  cl.sync();
}

// cudaOccupancyMaxActiveClusters costs tens of microseconds and v2_solve asks it for every
// cluster size on every solve: the answer depends only on (device, kernel, cluster size,
// dynamic shared memory), so it is memoised.
int cached_active_clusters(int device, uintptr_t kernel_id, int cs, size_t dyn, const std::function<int(int, size_t)> &query)
{
  static std::mutex mu;
  static std::map<std::tuple<int, uintptr_t, int, size_t>, int> cache;
  const auto key = std::make_tuple(device, kernel_id, cs, dyn);
  {
    std::lock_guard<std::mutex> g(mu);
    const auto it = cache.find(key);
    if (it != cache.end())
      return it->second;
  }
  const int v = query(cs, dyn);
  std::lock_guard<std::mutex> g(mu);
  cache[key] = v;
  return v;
}

using V2Kernel = void (*)(V2Params);

template <int RPT, int EC>
V2Kernel v2_kernel_ec(const V2Params &P)
{
  return !P.async_x ? cg_cluster_v2<RPT, EC, false>
                    : (P.prof ? cg_cluster_v2<RPT, EC, true, true> : cg_cluster_v2<RPT, EC, true, false>);
}

// The exact instance v2_launch runs for these parameters (the uniform 5-entry-row variant for the
// Hermite operators and their A-pattern factors at 4 rows per thread).
template <int RPT>
V2Kernel v2_kernel(const V2Params &P)
{
  if constexpr (RPT == 4)
  {
    bool uniform5 = P.ea == 5;
    for (int st = 0; st < P.z; ++st)
      uniform5 = uniform5 && P.ef[st] == 5;
    if (uniform5)
      return v2_kernel_ec<4, 5>(P);
  }
  return v2_kernel_ec<RPT, 0>(P);
}

int v2_active_clusters_query(V2Kernel kern, int cs, size_t dyn)
{
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
  {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(cs));
  cfg.blockDim = dim3(kV2TB);
  cfg.dynamicSmemBytes = dyn;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess)
  {
    cudaGetLastError();
    return 0;
  }
  return clusters;
}

// Co-resident clusters of the instance that will actually launch (memoised per instance).
template <int RPT>
int v2_active_clusters(mgpu_ctx *ctx, const V2Params &P, size_t dyn)
{
  const V2Kernel kern = v2_kernel<RPT>(P);
  return cached_active_clusters(ctx->device, reinterpret_cast<uintptr_t>(kern), P.cs, dyn,
                                [kern](int cs, size_t d) { return v2_active_clusters_query(kern, cs, d); });
}

template <int RPT>
void v2_launch(mgpu_ctx *ctx, const V2Params &P, size_t dyn)
{
  const V2Kernel kern = v2_kernel<RPT>(P);
  MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  MG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(P.l * P.cs));
  cfg.blockDim = dim3(kV2TB);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(P.cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MG_CUDA(cudaLaunchKernelEx(&cfg, kern, P));
  check_launch(ctx, "cg_cluster_v2");
}

// Plans and launches v2; false when no cluster size fits.  Picks the size that
// minimises (waves x rows per CTA) given the co-residency the driver reports.
bool v2_solve(mgpu_ctx *ctx, V2Params P, size_t budget)
{
  int best_cs = 0, best_rpt = 0;
  size_t best_dyn = 0;
  double best_cost = 1e300;
  V2Params best{};
  const int only_cs = static_cast<int>(ctx->opt[MGPU_OPT_CLUSTER_CS]); // k > 0: cluster size k only (diagnostics)
  for (int cs = 1; cs <= kCMaxCS; ++cs)
  {
    if (only_cs > 0 && cs != only_cs)
      continue;
    const int64_t rb = (P.n + cs - 1) / cs;
    if (rb > static_cast<int64_t>(kV2TB) * 4)
      continue;
    const int64_t last = P.n - static_cast<int64_t>(cs - 1) * rb;
    if (cs > 1 && (rb < P.halo[0] || last < P.halo[0]))
      continue;
    V2Params Q = P;
    Q.cs = cs;
    Q.rb = static_cast<int>(rb);
    Q.H = P.halo[0];
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 15) & ~static_cast<size_t>(15);
      return o;
    };
    Q.off_d = take(sizeof(double) * static_cast<size_t>(rb + 2 * Q.H));
    Q.off_t0 = take(Q.z >= 1 ? sizeof(double) * static_cast<size_t>(rb + 2 * Q.halo[1]) : 16);
    Q.off_t1 = take(Q.z >= 2 ? sizeof(double) * static_cast<size_t>(rb + 2 * Q.halo[2]) : 16);
    Q.off_part = take(sizeof(double) * 4 * kCMaxM * kCMaxCS);
    Q.off_ex = take(sizeof(double) * 10 * static_cast<size_t>(std::max(Q.H, 1)));
    Q.off_av = take(sizeof(double) * static_cast<size_t>(rb) * Q.ea);
    Q.off_ao = take(sizeof(unsigned long long) * static_cast<size_t>(rb));
    for (int st = 0; st < Q.z; ++st)
    {
      const size_t rows = static_cast<size_t>(rb + 2 * Q.halo[st + 1]);
      Q.off_fv[st] = take(sizeof(double) * rows * Q.ef[st]);
      Q.off_fo[st] = take(sizeof(unsigned long long) * rows);
    }
    if (off > budget)
      continue;
    const int rpt = static_cast<int>((rb + kV2TB - 1) / kV2TB);
    const int r4 = rpt <= 1 ? 1 : (rpt == 2 ? 2 : 4);
    const int act = r4 == 1 ? v2_active_clusters<1>(ctx, Q, off)
                            : (r4 == 2 ? v2_active_clusters<2>(ctx, Q, off) : v2_active_clusters<4>(ctx, Q, off));
    if (act < 1)
      continue;
    const double waves = std::ceil(static_cast<double>(P.l) / act);
    const double cost = waves * static_cast<double>(rb) * (1.0 + 0.02 * cs); // larger clusters: costlier barriers
    if (cost < best_cost)
    {
      best_cost = cost;
      best_cs = cs;
      best_rpt = r4;
      best_dyn = off;
      best = Q;
    }
  }
  if (best_cs == 0)
    return false;
  if (best_rpt == 1)
    v2_launch<1>(ctx, best, best_dyn);
  else if (best_rpt == 2)
    v2_launch<2>(ctx, best, best_dyn);
  else
    v2_launch<4>(ctx, best, best_dyn);
  return true;
}

} // namespace

// Tries the cluster-resident solve; false when the systems do not fit on chip
// (the caller then uses the grid-wide kernels).
int cg_cluster_solve(mgpu_ctx *ctx, int l, const mgpu_csr *const *A, int z, const mgpu_csr *const *chains,
                     int64_t n, int m, const double *B_dev, int64_t ldb, const int *halo, double rtol,
                     int64_t maxit, double *X, double *REC, double *TR, int64_t *d_it, int *d_conv, int *d_st,
                     int64_t *d_bd, double *d_hist, int64_t hist_cap, unsigned long long *d_loop, const DCsr *dA,
                     const DCsr *dF)
{
  if (m > kCMaxM || z > kCMaxZ || n <= 0 || n > INT32_MAX)
    return 0;
  int ea = 0;
  int ef[kCMaxZ] = {0};
  for (int p = 0; p < l; ++p)
  {
    ea = std::max<int>(ea, static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(A[p]))));
    for (int st = 0; st < z; ++st)
      ef[st] = std::max<int>(ef[st], static_cast<int>(csr_max_row(ctx, const_cast<mgpu_csr *>(
                                                                       chains[static_cast<size_t>(p) * z + (z - 1 - st)]))));
  }
  int cdev0 = 0;
  MG_CUDA(cudaDeviceGetAttribute(&cdev0, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  bool narrow = ea <= 8;
  for (int st = 0; st < z; ++st)
    narrow = narrow && ef[st] <= 8;
  if (m == 1 && ctx->cg_path != 3 && narrow)
  {
    V2Params V{};
    V.l = l;
    V.z = z;
    V.ea = ea;
    for (int st = 0; st < z; ++st)
      V.ef[st] = ef[st];
    for (int q = 0; q <= z; ++q)
      V.halo[q] = halo[q];
    V.n = n;
    V.A = dA;
    V.F = dF;
    V.B = B_dev;
    V.ldb = ldb;
    V.rtol = rtol;
    V.maxit = maxit;
    V.X = X;
    V.REC = REC;
    V.TR = TR;
    V.iters = d_it;
    V.conv = d_conv;
    V.status = d_st;
    V.bd_iter = d_bd;
    V.hist = d_hist;
    V.hist_cap = hist_cap;
    V.loop_iters = d_loop;
    V.prof = ctx->prof_dev;
    V.async_x = ctx->opt[MGPU_OPT_CLUSTER_ASYNC] != 0; // 0: cluster-barrier exchange (diagnostics)
    if (v2_solve(ctx, V, static_cast<size_t>(cdev0) - sizeof(ClShared) - 1024))
      return 2;
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
      return 3;
  }
  return 0;
}

} // namespace mgpu
