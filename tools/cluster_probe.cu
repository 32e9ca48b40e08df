// Max active clusters on this device for the cluster-resident CG shape.
#include <cstdio>
__global__ void k(double *p) { extern __shared__ double s[]; if (p) p[0] = s[0]; }
int main()
{
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int smems[] = {200 << 10};
  int threads[] = {1024};
  for (int t : threads)
    for (int sm : smems)
    {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      for (int cs = 1; cs <= 16; ++cs)
      {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 8);
        cfg.blockDim = dim3(t);
        cfg.dynamicSmemBytes = sm;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("threads %4d smem %3dKB cluster %2d -> max active clusters %3d (%s)\n", t, sm >> 10, cs, n,
               cudaGetErrorString(e));
      }
    }
}
