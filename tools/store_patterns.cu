// Write-bandwidth of output tilings for the merge's 16 GiB state (2^15 x 2^15
// complex128 rows): which store pattern does the HBM write stream want?
// Every variant writes the whole state once with 16-byte evict-first stores,
// 148 persistent CTAs x 512 threads.
//   P0: tile = 128 l x 16 h, contiguous tile range per CTA with h fastest; a warp writes 4 rows x 512 B
//   P1: same tiles dealt round-robin with l fastest; a warp writes 1 row x 2 KB
//   P2: tile = 1024 l x 2 h, round-robin; a warp writes 1 row x 2 KB
//   P3: tiles as P1; a warp writes 4 rows x 512 B
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_patterns tools/store_patterns.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int64_t W = 1 << 15, H = 1 << 15;

template <int P>
__global__ void __launch_bounds__(512, 1) stores(double2* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2 v = make_double2(1.0, 2.0);
  if (P == 0 || P == 1 || P == 3 || P == 11) {
    const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
    const int64_t c0 = blockIdx.x * tiles / gridDim.x, c1 = (blockIdx.x + 1) * tiles / gridDim.x;
    for (int64_t k = 0;; ++k) {
      int64_t t, lt, hb;
      if (P == 0) {  // contiguous tile range per CTA, h fastest (the first int8 merge schedule)
        t = c0 + k;
        if (t >= c1) break;
        lt = t / n_hb; hb = t % n_hb;
      } else if (P == 11) {  // contiguous tile range per CTA, l fastest
        t = c0 + k;
        if (t >= c1) break;
        hb = t / n_lt; lt = t % n_lt;
      } else {       // round robin, l tile fastest
        t = blockIdx.x + k * gridDim.x;
        if (t >= tiles) break;
        hb = t / n_lt; lt = t % n_lt;
      }
      double2* base = out + hb * 16 * W + lt * 128;
      if (P == 0 || P == 3 || P == 11) {
        const int q = warp & 3, r0 = (warp >> 2) * 4;  // 16 warps: 4 quarters x 4 row groups of 4
        for (int j = 0; j < 4; ++j) __stcs(base + (r0 + j) * W + q * 32 + lane, v);
      } else {
        const int r = warp;  // 16 warps = 16 rows; each writes its row's 2 KB as 4 x 512 B
        for (int j = 0; j < 4; ++j) __stcs(base + r * W + j * 32 + lane, v);
      }
    }
  } else if (P == 2) {
    const int64_t n_lt = W / 1024, n_hb = H / 2, tiles = n_lt * n_hb;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t lt = t % n_lt, hb = t / n_lt;
      double2* base = out + hb * 2 * W + lt * 1024;
      const int r = warp >> 3, c = (warp & 7) * 128;
      for (int j = 0; j < 4; ++j) __stcs(base + r * W + c + j * 32 + lane, v);
    }
  }
}

// P4: non-persistent grid, one 128 l x 16 h tile per CTA (512 threads)
// P5: persistent, 2 CTAs/SM x 256 threads, warp = 4 rows x 512 B per tile
// P6: persistent 148 x 512, 2 tiles per iteration (8 stores in flight per thread)
// P7: like P1 but 256-bit stores (a warp writes 1 KB contiguous per instruction)
template <int P, int THREADS, int BPSM>
__global__ void __launch_bounds__(THREADS, BPSM) stores2(double2* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2 v = make_double2(1.0, 2.0);
  const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
  const int nw = THREADS / 32;
  if (P == 4) {
    const int64_t t = blockIdx.x;
    const int64_t hb = t / n_lt, lt = t % n_lt;
    double2* base = out + hb * 16 * W + lt * 128;
    const int q = warp & 3, r0 = (warp >> 2) * 4;
    for (int j = 0; j < 4; ++j) __stcs(base + (r0 + j) * W + q * 32 + lane, v);
    return;
  }
  for (int64_t t = blockIdx.x * (P == 6 ? 2 : 1); t < tiles; t += gridDim.x * (P == 6 ? 2 : 1)) {
#pragma unroll
    for (int u = 0; u < (P == 6 ? 2 : 1); ++u) {
      const int64_t tt = t + u;
      const int64_t hb = tt / n_lt, lt = tt % n_lt;
      double2* base = out + hb * 16 * W + lt * 128;
      if (P == 7) {
        // 16 rows x 2 KB = 32 KB per tile; thread writes 32 B: warp = 1 KB contiguous
        for (int j = threadIdx.x; j < 16 * 64; j += THREADS) {
          const int r = j >> 6, c = (j & 63) * 2;
          double* d = reinterpret_cast<double*>(base + r * W + c);
          asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(d), "d"(1.0), "d"(2.0), "d"(1.0), "d"(2.0) : "memory");
        }
      } else {
        for (int j = warp; j < 64; j += nw) {  // 64 (row, quarter) pieces of 512 B
          const int r = j >> 2, q = j & 3;
          __stcs(base + r * W + q * 32 + lane, v);
        }
      }
    }
  }
}

// P8: persistent 148 x 512, tiles fetched from a global atomic counter (the
// active set stays a compact window of consecutive tiles, like the hardware
// block scheduler's)
__global__ void __launch_bounds__(512, 1) stores_dyn(double2* out, unsigned long long* ctr) {
  __shared__ long long tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2 v = make_double2(1.0, 2.0);
  const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
  for (;;) {
    if (threadIdx.x == 0) tile = (long long)atomicAdd(ctr, 1ull);
    __syncthreads();
    const int64_t t = tile;
    __syncthreads();
    if (t >= tiles) break;
    const int64_t hb = t / n_lt, lt = t % n_lt;
    double2* base = out + hb * 16 * W + lt * 128;
    const int q = warp & 3, r0 = (warp >> 2) * 4;
    for (int j = 0; j < 4; ++j) __stcs(base + (r0 + j) * W + q * 32 + lane, v);
  }
}

// P9: persistent 148 x 128, each tile's 16 rows x 2 KB leave through the TMA
// (cp.async.bulk.global.shared::cta, one 2 KB bulk store per row) from a
// 4-deep ring of 32 KB shared-memory tiles; NOFILL skips the st.shared fill
template <bool NOFILL>
__global__ void __launch_bounds__(128, 1) stores_tma(double2* out) {
  extern __shared__ __align__(128) double2 sm[];
  const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
  int k = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
    double2* buf = sm + (k & 3) * 2048;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    __syncthreads();
    if (!NOFILL)
      for (int i = threadIdx.x; i < 2048; i += 128) buf[i] = make_double2(1.0, double(i));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 16) {
      const int64_t hb = t / n_lt, lt = t % n_lt;
      double2* dst = out + (hb * 16 + threadIdx.x) * W + lt * 128;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], 2048, %2;"
                   :: "l"(dst), "r"((unsigned)__cvta_generic_to_shared(buf + threadIdx.x * 128)),
                      "l"(0x14F0000000000000ull) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x < 16) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <bool NOFILL>
static int run_tma(double2* out, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaFuncSetAttribute(stores_tma<NOFILL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
  stores_tma<NOFILL><<<148, 128, 4 * 32768>>>(out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stores_tma<NOFILL><<<148, 128, 4 * 32768>>>(out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%s: %.3f ms  %.0f GB/s\n", name, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

// P10: persistent round-robin (as P3) plus a software grid barrier every
// `every` tiles: keeps the CTAs' write fronts within a window of tiles
__global__ void __launch_bounds__(512, 1) stores_sync(double2* out, unsigned* bar, int every) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2 v = make_double2(1.0, 2.0);
  const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
  unsigned epoch = 0;
  int k = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
    if (k && k % every == 0) {
      __syncthreads();
      ++epoch;
      if (threadIdx.x == 0) {
        atomicAdd(bar, 1u);
        while (atomicAdd(bar, 0u) < epoch * gridDim.x) __nanosleep(64);
      }
      __syncthreads();
    }
    const int64_t hb = t / n_lt, lt = t % n_lt;
    double2* base = out + hb * 16 * W + lt * 128;
    const int q = warp & 3, r0 = (warp >> 2) * 4;
    for (int j = 0; j < 4; ++j) __stcs(base + (r0 + j) * W + q * 32 + lane, v);
  }
}

static int run_sync(double2* out, int every) {
  unsigned* bar;
  CK(cudaMalloc(&bar, 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float tot = 0;
  for (int i = 0; i < 6; ++i) {
    cudaMemset(bar, 0, 4);
    cudaEventRecord(a);
    stores_sync<<<148, 512>>>(out, bar, every);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i) tot += ms;
  }
  const float ms = tot / 5;
  printf("P10 persistent + grid barrier every %d tiles: %.3f ms  %.0f GB/s\n", every, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

// P12: non-persistent, NT consecutive tiles (l fastest) per CTA, one CTA per
// SM resident at a time (150 KB of dynamic shared memory)
template <int NT>
__global__ void __launch_bounds__(512, 1) stores_chunk(double2* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2 v = make_double2(1.0, 2.0);
  const int64_t n_lt = W / 128;
  for (int k = 0; k < NT; ++k) {
    const int64_t t = int64_t(blockIdx.x) * NT + k;
    const int64_t hb = t / n_lt, lt = t % n_lt;
    double2* base = out + hb * 16 * W + lt * 128;
    const int q = warp & 3, r0 = (warp >> 2) * 4;
    for (int j = 0; j < 4; ++j) __stcs(base + (r0 + j) * W + q * 32 + lane, v);
  }
}

template <int NT>
static int run_chunk(double2* out, int smem) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaFuncSetAttribute(stores_chunk<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = int((W / 128) * (H / 16) / NT);
  stores_chunk<NT><<<grid, 512, smem>>>(out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stores_chunk<NT><<<grid, 512, smem>>>(out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("P12 non-persistent, %d tiles per CTA, smem %d: %.3f ms  %.0f GB/s\n", NT, smem, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

// P13: persistent round-robin (as P3) with different store cache policies
template <int POL>
__global__ void __launch_bounds__(512, 1) stores_pol(double2* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_lt = W / 128, n_hb = H / 16, tiles = n_lt * n_hb;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t hb = t / n_lt, lt = t % n_lt;
    double2* base = out + hb * 16 * W + lt * 128;
    const int q = warp & 3, r0 = (warp >> 2) * 4;
    if (POL == 4) {  // 256-bit stores, L2::evict_first: a warp writes 1 KB of one row
      for (int j = threadIdx.x; j < 1024; j += 512) {
        const int r = j >> 6, c = (j & 63) * 2;
        double* d = reinterpret_cast<double*>(base + r * W + c);
        asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1, %2, %3, %4};"
                     :: "l"(d), "d"(1.0), "d"(2.0), "d"(1.0), "d"(2.0) : "memory");
      }
      continue;
    }
    for (int j = 0; j < 4; ++j) {
      double2* d = base + (r0 + j) * W + q * 32 + lane;
      if (POL == 0) __stcs(d, make_double2(1.0, 2.0));
      else if (POL == 1) *d = make_double2(1.0, 2.0);
      else if (POL == 2) __stwt(d, make_double2(1.0, 2.0));
      else if (POL == 3) asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" :: "l"(d), "d"(1.0), "d"(2.0) : "memory");
      else if (POL == 5) __stcg(d, make_double2(1.0, 2.0));
    }
  }
}

template <int POL>
static int run_pol(double2* out, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  stores_pol<POL><<<148, 512>>>(out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stores_pol<POL><<<148, 512>>>(out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("P13 persistent, %s: %.3f ms  %.0f GB/s\n", name, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

static int run_dyn(double2* out) {
  unsigned long long* ctr;
  CK(cudaMalloc(&ctr, 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaMemset(ctr, 0, 8);
  stores_dyn<<<148, 512>>>(out, ctr);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) {
    cudaMemsetAsync(ctr, 0, 8);
    stores_dyn<<<148, 512>>>(out, ctr);
  }
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("P8 persistent, atomic tile counter: %.3f ms  %.0f GB/s\n", ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

template <int P, int THREADS, int BPSM>
static int run2(double2* out, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = P == 4 ? int((W / 128) * (H / 16)) : 148 * BPSM;
  stores2<P, THREADS, BPSM><<<grid, THREADS>>>(out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stores2<P, THREADS, BPSM><<<grid, THREADS>>>(out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%s: %.3f ms  %.0f GB/s\n", name, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

template <int P>
static int run(double2* out, const char* name) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  stores<P><<<148, 512>>>(out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) stores<P><<<148, 512>>>(out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%s: %.3f ms  %.0f GB/s\n", name, ms, 16.0 * W * H / ms / 1e6);
  return 0;
}

int main() {
  double2* out;
  CK(cudaMalloc(&out, sizeof(double2) * W * H));
  run_pol<0>(out, "st.global.cs"); run_pol<1>(out, "st.global"); run_pol<2>(out, "st.global.wt");
  run_pol<3>(out, "L1::no_allocate"); run_pol<4>(out, "256-bit L1::no_allocate.L2::evict_first"); run_pol<5>(out, "st.global.cg");
  run2<4, 512, 1>(out, "P4 non-persistent, one tile per CTA");
  cudaFree(out);
  return 0;
}
