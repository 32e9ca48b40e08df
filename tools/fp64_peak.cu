// FP64 pipe peak on this B200: DFMA (2 flops each) and DADD (1 flop) throughput with 8 independent
// chains per thread, 4 warps per scheduler, every SM.  Usage: ./fp64_peak  -> one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA>
__global__ void __launch_bounds__(512) spin(double *out, int iters, double a, double b)
{
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it)
  {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        x[k] = FMA ? fma(x[k], a, b) : x[k] + b;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    s += x[k];
  if (s == 1234.5)
    out[0] = s;
}

int main()
{
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, tb = 512, blocks = sms * 2;
  double res[2];
  for (int f = 0; f < 2; ++f)
  {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep)
    {
      cudaEventRecord(e0);
      if (f)
        spin<true><<<blocks, tb>>>(out, iters, 0.9999999, 1e-9);
      else
        spin<false><<<blocks, tb>>>(out, iters, 0.9999999, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double ops = 1.0 * blocks * tb * iters * 16 * 8;
    res[f] = ops * (f ? 2.0 : 1.0) / (best * 1e-3) / 1e12;
  }
  std::printf("{\"dfma_tflops\": %.2f, \"dadd_tflops\": %.2f, \"dadd_gops\": %.1f, \"sms\": %d, "
              "\"how\": \"%d blocks x %d threads, 8 independent chains per thread, best of 5 (CUDA events); "
              "DFMA = 2 flops, DADD = 1\"}\n",
              res[1], res[0], res[0] * 1e3, sms, blocks, tb);
  return 0;
}
