// How many clusters of the C3 filter's CTA shape (768 threads, 200 KB dynamic shared memory, one CTA
// per SM) can be resident at once, per cluster size?  cudaOccupancyMaxActiveClusters on a stand-in
// kernel with the same launch footprint as k_filter_cl<16, 4, true>.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_slots tools/cluster_slots.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(768, 1) k_standin(double* out) {
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (out) out[blockIdx.x * blockDim.x + threadIdx.x] = sm[(threadIdx.x + 1) % blockDim.x];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  cudaFuncSetAttribute(k_standin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_standin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clusters\": {", p.name, p.multiProcessorCount);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(768, 1, 1);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int n = -1;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_standin, &cfg);
    printf("%s\"%d\": {\"max_active\": %d, \"sms_busy\": %d%s%s}", cs > 1 ? ", " : "", cs, n, n * cs,
           e == cudaSuccess ? "" : ", \"error\": ", e == cudaSuccess ? "" : "1");
    cudaGetLastError();
  }
  printf("}}\n");
  return 0;
}
