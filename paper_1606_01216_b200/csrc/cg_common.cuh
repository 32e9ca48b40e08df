// Shared by cg.cu and cg_stream.cu: batch limits, the per-system state machine, the block
// plan (row segments) and the deterministic block / grid reductions of the banded kernels.
#pragma once
#include <cooperative_groups.h>

#include "internal.cuh"

namespace mgpu
{
namespace
{

constexpr int kCgThreads = 256;
constexpr int kWarps = kCgThreads / 32;
constexpr int kMaxSys = 128;   // systems (points x columns) per launch (mgpu_cg_solve splits larger batches)
constexpr int kMaxPoints = 128;
constexpr int kMaxTiles = 1024; // tiles per point (reduction fan-in)
constexpr int kMaxM = 8;        // rhs columns per launch

enum SysState : int
{
  kRun = 0,
  kConverged = 1,
  kBreakdown = 2,
  kZeroRhs = 3,
  kMaxed = 4,
  kPendingConv = 5,
  kPendingRestart = 6,
};

constexpr int kMaxZ = 12; // chain factors (the AIRGA update chain grows by one per outer iteration)
constexpr int kMaxHalo = 64;
constexpr int kMaxRpt = 4;
constexpr int kMaxSeg = 8; // row segments per block

struct Seg
{
  int p, rs, re, pad; // rows [rs, re) of point p
};

template <int TB>
struct BandShared
{
  double rho[kMaxSys], target[kMaxSys], alpha[kMaxSys], beta[kMaxSys], bnorm[kMaxSys];
  double tot[kMaxSys * 2];
  int state[kMaxSys];
  int fresh[kMaxSys];
  int pend[kMaxSys]; // cg_stream: x~ += alpha d_old still owed (deferred from phase B)
  int64_t sit[kMaxSys];
  int pmask[kMaxPoints];
  Seg seg[kMaxSeg];
  int nseg;
  double wsum[TB / 32][2 * kMaxM];
  double acc[2 * kMaxM];
  int flag;
};

// Iterate this block's row segments [rs, re) of point p (host plan in shared memory).
template <class PT, class S, class F>
__device__ __forceinline__ void for_segments(const PT &, const S &sh, F &&fn)
{
  for (int q = 0; q < sh.nseg; ++q)
  {
    const Seg g = sh.seg[q];
    if (sh.pmask[g.p])
      fn(g.p, static_cast<int64_t>(g.rs), static_cast<int64_t>(g.re));
  }
}

// Adds this chunk's per-thread values (NV of them, nv used) to the block's
// running partials in a fixed order.
template <int TB, int NV>
__device__ __forceinline__ void chunk_sum(BandShared<TB> &sh, double (&v)[NV], int nv)
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
      sh.wsum[warp][k] = v[k];
  }
  __syncthreads();
  if (warp == 0)
  {
    for (int k = 0; k < nv; ++k)
    {
      double x = lane < TB / 32 ? sh.wsum[lane][k] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
        x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, off));
      if (lane == 0)
        sh.acc[k] = __dadd_rn(sh.acc[k], x);
    }
  }
  __syncthreads();
}

template <int TB>
__device__ __forceinline__ void begin_point(BandShared<TB> &sh)
{
  if (threadIdx.x < 2 * kMaxM)
    sh.acc[threadIdx.x] = 0.0;
  __syncthreads();
}

template <int TB>
__device__ __forceinline__ void end_point(double *partial, BandShared<TB> &sh, int p, int nv)
{
  if (threadIdx.x < nv)
    partial[(static_cast<int64_t>(p) * 2 * kMaxM + threadIdx.x) * gridDim.x + blockIdx.x] = sh.acc[threadIdx.x];
  __syncthreads();
}

// After a barrier: tot = sum over blocks (fixed order) for live points; quantity k < m of
// system (p, c = k) at tot[p m + c], quantity k >= m at tot[l m + p m + (k - m)].
template <int TB, class PT>
__device__ void reduce_blocks(const PT &P, BandShared<TB> &sh, int nk)
{
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int npairs = P.l * nk;
  for (int q = warp; q < npairs; q += TB / 32)
  {
    const int p = q / nk, k = q % nk;
    if (!sh.pmask[p])
      continue;
    const double *src = P.partial + (static_cast<int64_t>(p) * 2 * kMaxM + k) * gridDim.x;
    const int2 br = P.pblk[p];
    double a = 0.0;
    for (int t = br.x + lane; t < br.y; t += 32)
      a = __dadd_rn(a, __ldcg(src + t));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
      a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, off));
    if (lane == 0)
      sh.tot[k < P.m ? p * P.m + k : P.l * P.m + p * P.m + (k - P.m)] = a;
  }
  __syncthreads();
}

} // namespace
} // namespace mgpu
