// TMEM read throughput on one SM per CTA (sm_100a): W warps each issue R
// rounds of tcgen05.ld of one shape + wait::ld over a 512-column
// allocation; prints bytes per SM-cycle for every (warps, shape). The
// int8 merge's epilogue reads 7-8 int32 diagonals per real output from
// TMEM (ozaki.cu), so this rate bounds it at K <= 32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_ld_bw tools/tmem_ld_bw.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int X>
__device__ __forceinline__ uint32_t ld_x(uint32_t taddr);


template <>
__device__ __forceinline__ uint32_t ld_x<8>(uint32_t t) {
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= v[i];
  return s;
}
template <>
__device__ __forceinline__ uint32_t ld_x<16>(uint32_t t) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  return s;
}
template <>
__device__ __forceinline__ uint32_t ld_x<32>(uint32_t t) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s ^= v[i];
  return s;
}
// 16x256b.x4: 16 lanes x 256 bit per repetition; 16 regs per thread
__device__ __forceinline__ uint32_t ld_16x256b_x4(uint32_t t) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  return s;
}

// two loads in flight before one wait (x8 each), as the merge epilogue does
__device__ __forceinline__ uint32_t ld_x8_pair(uint32_t t) {
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(t + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  return s;
}

// MODE: 8/16/32 = 32x32b.xMODE, 1 = 16x256b.x4, 2 = two x8 per wait
template <int MODE>
__global__ void tmem_bw(int rounds, uint32_t* sink, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int q = warp & 3;
  const int nw = blockDim.x >> 5;
  const uint32_t base = tmem + (uint32_t(q * 32) << 16) + uint32_t(((warp >> 2) * 64) & 511);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const uint32_t col = uint32_t((r * 64) & 255);
    if (MODE == 8) acc ^= ld_x<8>(base + col);
    else if (MODE == 16) acc ^= ld_x<16>(base + col);
    else if (MODE == 32) acc ^= ld_x<32>(base + col);
    else if (MODE == 1) acc ^= ld_16x256b_x4(base + col);
    else acc ^= ld_x8_pair(base + col);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  (void)nw;
}

template <int MODE>
void run(int warps, int sms) {
  const int rounds = 4096;
  uint32_t* sink;
  long long* cyc;
  CK(cudaMalloc(&sink, size_t(sms) * warps * 32 * 4));
  CK(cudaMalloc(&cyc, sms * 8));
  tmem_bw<MODE><<<sms, warps * 32, 100 * 1024>>>(rounds, sink, cyc);  // smem forces 1 CTA/SM
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  long long* h = (long long*)malloc(sms * 8);
  CK(cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += double(h[i]);
  avg /= sms;
  // 32x32b.xN: 32 lanes x N columns x 4 B per warp instruction; 16x256b.x4:
  // 16 lanes x 32 B x 4 = 2 KiB; mode 2: two 32x32b.x8 per wait
  const int bytes_per_ld = MODE == 1 ? 16 * 32 * 4 : (MODE == 2 ? 32 * 4 * 16 : 32 * 4 * MODE);
  const double bytes = double(bytes_per_ld) * rounds * warps;
  printf("mode %-3d warps %2d  %8.1f cycles  %7.1f B/cycle/SM\n", MODE, warps, avg, bytes / avg);
  free(h);
  CK(cudaFree(sink));
  CK(cudaFree(cyc));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(tmem_bw<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(tmem_bw<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(tmem_bw<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(tmem_bw<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  CK(cudaFuncSetAttribute(tmem_bw<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  for (int w : {4, 8, 16}) {
    run<8>(w, sms);
    run<2>(w, sms);
    run<16>(w, sms);
    run<32>(w, sms);
    run<1>(w, sms);
  }
  return 0;
}
