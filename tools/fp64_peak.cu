// FP64 DFMA peak microbenchmark (B200, sm_100a). Measures the denominator for
// the assembly roofline: 8 independent DFMA chains per thread, grid = 148*k CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
  double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  int iters = 4000;
  for (int tpb : {128, 256, 512}) for (int bps : {4, 8, 16}) {
    int grid = p.multiProcessorCount * bps;
    dfma_loop<<<grid, tpb>>>(d, 10, 0.999999, 1e-7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) dfma_loop<<<grid, tpb>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 3.0 * grid * tpb * (double)iters * 16 * 8 * 2;
    printf("tpb %d ctas/SM %d : %.2f TFLOP/s fp64 (DFMA=2)\n", tpb, bps, flops / (ms * 1e-3) / 1e12);
  }
  cudaError_t e = cudaGetLastError(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
