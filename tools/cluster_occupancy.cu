// How many thread-block clusters of the variant-stage shape can be resident
// at once (cudaOccupancyMaxActiveClusters): 256-thread CTAs, 64 KiB of
// dynamic shared memory (a 2^11-amplitude complex128 chunk + transpose
// scratch), cluster sizes 2..16.  nvcc -gencode arch=compute_100a,code=sm_100a
// -o /tmp/cocc tools/cluster_occupancy.cu && /tmp/cocc
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) probe(double* p) {
  extern __shared__ double s[];
  s[threadIdx.x] = p ? p[threadIdx.x] : 0.0;
  __syncthreads();
  if (p) p[threadIdx.x] = s[255 - threadIdx.x];
}

// where the CTAs of n_clusters 16-CTA clusters land (%smid), each CTA
// spinning ~20 us so they are co-resident
__global__ void __launch_bounds__(256, 1) where(int* smid_out, long long spin) {
  extern __shared__ double s[];
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  const long long t0 = clock64();
  while (clock64() - t0 < spin) s[threadIdx.x] += 1.0;
  if (threadIdx.x == 0) smid_out[blockIdx.x + gridDim.x * blockIdx.y] = int(id);
}

void placement(int n_clusters, int c, int smem_kb) {
  cudaFuncSetAttribute(where, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  cudaFuncSetAttribute(where, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int* d = nullptr;
  cudaMalloc(&d, sizeof(int) * 4096);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c, n_clusters, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = size_t(smem_kb) * 1024;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = c;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, where, d, 40000LL);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, where, d, 40000LL);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int h[4096];
  cudaMemcpy(h, d, sizeof(int) * size_t(n_clusters * c), cudaMemcpyDeviceToHost);
  int per_sm[256] = {0};
  int used = 0, dbl = 0;
  for (int i = 0; i < n_clusters * c; ++i) {
    if (per_sm[h[i] & 255]++ == 0) ++used;
    else ++dbl;
  }
  std::printf("%d clusters x %2d CTAs, %d KiB: %d SMs used, %d CTAs sharing an SM, %.1f us (spin ~20 us) %s\n",
              n_clusters, c, smem_kb, used, dbl, ms * 1e3, err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  for (int n : {4, 8}) placement(n, 16, 64);
  placement(8, 16, 96);
  placement(16, 8, 64);
  placement(32, 4, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem_kb : {32, 64, 96, 128}) {
    for (int c : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c * 64, 1, 1);
      cfg.blockDim = dim3(256, 1, 1);
      cfg.dynamicSmemBytes = size_t(smem_kb) * 1024;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = c;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
      std::printf("smem %3d KiB cluster %2d: max active clusters %d (%d CTAs)%s\n", smem_kb, c, n, n * c,
                  e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
