// Grid-barrier cost on B200: cooperative-groups grid.sync vs a flag barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_sync_loop(int iters, double *sink)
{
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i)
  {
    acc += i;
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *sink = acc;
}

// sense-reversal barrier: one arrive counter + generation word, acquire/release
__device__ __forceinline__ void flag_barrier(unsigned int *count, unsigned int *gen, unsigned int nb)
{
  __syncthreads();
  if (threadIdx.x == 0)
  {
    unsigned int g0;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g0) : "l"(gen));
    unsigned int arrived;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(count));
    if (arrived == nb - 1)
    {
      *count = 0;
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1));
    }
    else
    {
      unsigned int g1;
      do
      {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g1) : "l"(gen));
      } while (g1 == g0);
    }
  }
  __syncthreads();
}

__global__ void flag_sync_loop(int iters, unsigned int *count, unsigned int *gen, double *sink)
{
  double acc = 0;
  for (int i = 0; i < iters; ++i)
  {
    acc += i;
    flag_barrier(count, gen, gridDim.x);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *sink = acc;
}

int main()
{
  double *sink;
  unsigned int *cnt, *gen;
  cudaMalloc(&sink, 8);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4);
  cudaMemset(gen, 0, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  int grids[] = {sms, 2 * sms, 4 * sms};
  int threads[] = {256, 512};
  for (int t : threads)
    for (int gsz : grids)
    {
      for (int kind = 0; kind < 2; ++kind)
      {
        int it = iters;
        void *args_cg[] = {&it, &sink};
        void *args_f[] = {&it, &cnt, &gen, &sink};
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep)
        {
          cudaEventRecord(a);
          cudaError_t e = kind == 0 ? cudaLaunchCooperativeKernel((void *)cg_sync_loop, gsz, t, args_cg, 0, 0)
                                    : cudaLaunchCooperativeKernel((void *)flag_sync_loop, gsz, t, args_f, 0, 0);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          if (e != cudaSuccess)
          {
            printf("launch failed %s\n", cudaGetErrorString(e));
            break;
          }
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        printf("%s grid=%d threads=%d: %.3f us per barrier\n", kind == 0 ? "cg::grid.sync" : "flag barrier ", gsz, t,
               1e3 * best / iters);
      }
    }
  return 0;
}
