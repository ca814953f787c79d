// FP64 throughput probes on B200 (profiles/r01_dmma_peak.txt): DMMA m8n8k4 alone, DFMA alone, and
// both interleaved in one warp stream (do the DP tensor sub-pipe and the FP64 pipe overlap?)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>   // 0 DMMA, 1 DFMA, 2 both
__global__ void k_probe(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2], f[16];
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int j = 0; j < 16; ++j) f[j] = j * 1e-3;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    if (MODE != 0) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = fma(f[j], b, a);
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  for (int j = 0; j < 16; ++j) s += f[j];
  if (s == 12345.0) out[0] = s;
}
template <int MODE>
void run(const char* name, double* d, int sms) {
  for (int tpb : {256, 512})
    for (int cps : {2, 4}) {
      const int iters = 2048;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k_probe<MODE><<<sms * cps, tpb>>>(d, 16);
      cudaEventRecord(e0);
      k_probe<MODE><<<sms * cps, tpb>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double threads = (double)(sms * cps) * tpb;
      const double fl_mma = MODE != 1 ? 2.0 * 8 * 8 * 4 * 8.0 * iters * threads / 32 : 0.0;
      const double fl_fma = MODE != 0 ? 2.0 * 8 * 16 * (double)iters * threads : 0.0;
      printf("%-6s tpb %d ctas/SM %d : %.2f TFLOP/s (DMMA %.2f + DFMA %.2f)\n", name, tpb, cps,
             (fl_mma + fl_fma) / ms / 1e9, fl_mma / ms / 1e9, fl_fma / ms / 1e9);
    }
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("dmma", d, sms);
  run<1>("dfma", d, sms);
  run<2>("both", d, sms);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
