// FP64 tensor-core (DMMA m8n8k4) throughput probe vs the DFMA peak (profiles/r01_fp64_peak.txt)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int tpb : {128, 256, 512})
    for (int cps : {2, 4, 8}) {
      const int iters = 4096;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k_dmma<<<sms * cps, tpb>>>(d, 16);
      cudaEventRecord(e0);
      k_dmma<<<sms * cps, tpb>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)(sms * cps) * (tpb / 32);
      printf("tpb %d ctas/SM %d : %.2f TFLOP/s fp64 DMMA\n", tpb, cps, flops / ms / 1e9);
    }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
