// dmma_warps.cu — DMMA (mma.sync.m8n8k4.f64) throughput against warps per SM and independent
// accumulators, registers only.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_warps tools/dmma_warps.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double d[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) d[i][0] = d[i][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 2e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
template <int NACC> void run(int sms, int threads, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  k_dmma<NACC><<<sms, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_dmma<NACC><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fm = 512.0 * NACC * iters * (double)(threads / 32) * sms;
  printf("acc %2d warps/SM %2d: %.2f TFLOP/s\n", NACC, threads / 32, fm / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int th : {32, 64, 128, 256, 512}) { run<4>(sms, th, out); run<8>(sms, th, out); run<16>(sms, th, out); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
