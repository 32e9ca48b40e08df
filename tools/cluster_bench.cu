// Per-operation latency inside a 10-CTA cluster of 512 threads (B200), to size
// the cluster-resident CG iteration: cluster barrier, CTA reduction, DSMEM total.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ double warp_sum(double v)
{
  for (int off = 16; off > 0; off >>= 1)
    v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(int iters, double *out)
{
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[16], slot[2];
  double v = threadIdx.x * 1e-3, acc = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cs = cl.num_blocks();
  for (int it = 0; it < iters; ++it)
  {
    if (MODE == 0)
    {
      cl.sync();
    }
    else if (MODE == 1)
    { // cta_sum only
      double w = warp_sum(v);
      if (lane == 0) red[warp] = w;
      __syncthreads();
      if (warp == 0) { double x = lane < 16 ? red[lane] : 0; x = warp_sum(x); if (lane == 0) slot[it & 1] = x; }
      __syncthreads();
      acc += slot[it & 1];
    }
    else if (MODE == 2)
    { // cta_sum + cluster barrier
      double w = warp_sum(v);
      if (lane == 0) red[warp] = w;
      __syncthreads();
      if (warp == 0) { double x = lane < 16 ? red[lane] : 0; x = warp_sum(x); if (lane == 0) slot[it & 1] = x; }
      cl.sync();
      acc += 1;
    }
    else
    { // full: cta_sum + cluster barrier + per-warp DSMEM total
      double w = warp_sum(v);
      if (lane == 0) red[warp] = w;
      __syncthreads();
      if (warp == 0) { double x = lane < 16 ? red[lane] : 0; x = warp_sum(x); if (lane == 0) slot[it & 1] = x; }
      cl.sync();
      double t = lane < cs ? cl.map_shared_rank(slot, lane)[it & 1] : 0.0;
      acc += warp_sum(t);
    }
    v = v * 1.0000001 + acc * 1e-30;
  }
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc + v;
}

template <int MODE>
float run(int cs, int clusters, int iters)
{
  double *o;
  cudaMalloc(&o, 8);
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs * clusters);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, kern<MODE>, iters, o);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern<MODE>, iters, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  cudaFree(o);
  return ms * 1e3f / iters;
}

int main()
{
  const int iters = 20000;
  for (int cs : {2, 4, 8, 10, 16})
    printf("cs=%2d  cluster.sync %.3f us | cta_sum %.3f us | cta_sum+sync %.3f us | +dsmem total %.3f us\n", cs,
           run<0>(cs, 8, iters), run<1>(cs, 8, iters), run<2>(cs, 8, iters), run<3>(cs, 8, iters));
}
