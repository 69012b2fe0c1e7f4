// fp64_pipes.cu — throughput of the two fp64 paths on this GPU: DFMA (CUDA
// cores) vs mma.sync.m8n8k4.f64 (DMMA).  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_pipes tools/fp64_pipes.cu && /tmp/fp64_pipes
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double x = 1.0000001, y = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 2e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      const int blocks = sms * 2;
      k_dfma<<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      k_dfma<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 8 * iters * (double)threads * blocks;
      if (rep) printf("DFMA  threads/CTA %4d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
      k_dmma<<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      k_dmma<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fm = 512.0 * 8 * iters * (double)(threads / 32) * blocks;
      if (rep) printf("DMMA  threads/CTA %4d: %.2f TFLOP/s\n", threads, fm / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
