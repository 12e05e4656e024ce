// Probe for the tcgen05 kind::i8 path used by the Ozaki merge (sm_100a).
// (1) correctness: D[128 x N] = A[128 x K] . B[N x K]^T, int8 K-major operands
//     in the no-swizzle canonical layout (core matrix = 8 rows x 16 B), int32
//     accumulator in TMEM read back with tcgen05.ld.32x32b;
// (2) throughput: cycles per MMA at N = 16..256 (accumulating R times) and
//     cycles per tcgen05.ld of 32 columns per warp (4 warps).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_i8_probe tools/tc_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)              // D = s32
       | (1u << 7) | (1u << 10) // A, B signed 8-bit
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  uint32_t z = 0;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n"
               :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(z));
}

__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  uint32_t z = 0;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}\n"
               :: "r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc), "r"(z));
}

// whole-warp form: every lane executes, elect.sync picks the issuing lane
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// core-matrix layout offset of (row r, byte k) inside one k-step block of `rows` rows x 32 B
__host__ __device__ inline uint32_t cm_off(int r, int k) {
  return (uint32_t)((r >> 3) * 256 + ((k >> 4) * 128) + (r & 7) * 16 + (k & 15));
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(const int8_t* A, const int8_t* B, int nk, int reps,
                                                int32_t* D, long long* cyc, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  int8_t* sA = (int8_t*)smem;                  // nk blocks of 4096 B
  int8_t* sB = (int8_t*)(smem + nk * 4096);    // nk blocks of N*32 B
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < nk * 4096; i += 128) sA[i] = A[i];
  for (int i = tid; i < nk * N * 32; i += 128) sB[i] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  constexpr uint32_t NCOL = 512;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_slot)), "r"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // TS mode: A lives in TMEM columns [384, 384 + 8 nk): lane = row, column c = bytes 4c..4c+3
  const uint32_t tmem_a = tmem + 384;
  if (TS) {
    const int row = warp * 32 + lane;
    for (int k = 0; k < nk; ++k) {
      uint32_t w[8];
      for (int c = 0; c < 8; ++c) {
        uint32_t x = 0;
        for (int b = 0; b < 4; ++b) x |= (uint32_t)(uint8_t)sA[k * 4096 + cm_off(row, 4 * c + b)] << (8 * b);
        w[c] = x;
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   :: "r"(tmem_a + ((uint32_t)(warp * 32) << 16) + 8 * k),
                      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_i8(128, N);
    t0 = clock64();
    const uint64_t da0 = make_desc(smem_u32(sA), 128, 256);
    const uint64_t db0 = make_desc(smem_u32(sB), 128, 256);
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < nk; ++k)
        for (int a = 0; a < nacc; ++a)
          if (TS) mma_i8_ts(tmem + a * N, tmem_a + 8 * k, db0 + (uint64_t)(k * N * 2), idesc, (r | k) ? 1u : 0u);
          else mma_i8(tmem + a * N, da0 + (uint64_t)(k * 256), db0 + (uint64_t)(k * N * 2), idesc, (r | k) ? 1u : 0u);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  if (tid == 0) { t1 = clock64(); cyc[0] = t1 - t0; }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // read back: warp w owns lanes 32w..32w+31 (= rows), 8 columns per ld
  const int row = warp * 32 + lane;
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = (int32_t)v[j];
  }
  // tcgen05.ld throughput: 32 columns per ld, all 4 warps, `reps` rounds
  __syncthreads();
  long long l0 = clock64();
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    uint32_t v[32];
    uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + ((r * 32) % NCOL);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    #pragma unroll
    for (int j = 0; j < 32; ++j) acc += v[j];
  }
  __syncthreads();
  long long l1 = clock64();
  if (tid == 0) cyc[1] = l1 - l0;
  if (acc == 0x12345678u) cyc[2] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(NCOL));
}

template <int N, bool TS = false>
static int run(int nk, int reps, int nacc = 1) {
  const int K = nk * 32;
  std::vector<int8_t> a(128 * K), b(N * K);
  srand(1234 + N + nk);
  for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
  std::vector<int8_t> ga(nk * 4096), gb(nk * N * 32);
  for (int r = 0; r < 128; ++r) for (int k = 0; k < K; ++k) ga[(k / 32) * 4096 + cm_off(r, k % 32)] = a[r * K + k];
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) gb[(k / 32) * N * 32 + cm_off(n, k % 32)] = b[n * K + k];
  int8_t *dA, *dB; int32_t* dD; long long* dc;
  CK(cudaMalloc(&dA, ga.size())); CK(cudaMalloc(&dB, gb.size()));
  CK(cudaMalloc(&dD, 128 * N * 4)); CK(cudaMalloc(&dc, 3 * 8));
  CK(cudaMemcpy(dA, ga.data(), ga.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, gb.data(), gb.size(), cudaMemcpyHostToDevice));
  size_t sm = nk * 4096 + nk * N * 32 + 1024;
  CK(cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  // correctness (reps = 1)
  probe<N, TS><<<1, 128, sm>>>(dA, dB, nk, 1, dD, dc, 1);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<int32_t> d(128 * N);
  CK(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
  long long bad = 0, first = -1;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    int32_t s = 0;
    for (int k = 0; k < K; ++k) s += (int32_t)a[m * K + k] * (int32_t)b[n * K + k];
    if (s != d[m * N + n]) { if (first < 0) first = m * N + n; ++bad; }
  }
  // timing
  probe<N, TS><<<1, 128, sm>>>(dA, dB, nk, reps, dD, dc, nacc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  long long c[3]; CK(cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost));
  double per_mma = (double)c[0] / (reps * nk * nacc);
  double macs = 128.0 * N * 32;
  printf("%s N=%3d nk=%d nacc=%d: mismatches %lld/%d (first %lld) | %.1f cyc/MMA = %.0f MAC/cyc | tcgen05.ld x32 (4 warps): %.1f cyc/round = %.0f B/cyc\n",
         TS ? "TS" : "SS", N, nk, nacc, bad, 128 * N, first, per_mma, macs / per_mma, (double)c[1] / reps, 128.0 * 32 * 4 * reps / c[1]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  return bad ? 1 : 0;
}

// stacked-diagonal MMA sequences (the Ozaki merge's pattern): per "tile" 8
// MMAs i = 0..7 into columns [32i, 256) with N = 32 (8 - i); `ntile`
// independent 256-column accumulators interleaved; `nks` k-steps per tile
template <int ALLOC, bool MKDESC>
__global__ void __launch_bounds__(128, 1) stacked(int reps, int ntile, int nks, int nsplit, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8 * 4096 + 8 * 1024; i += 128) smem[i] = (uint8_t)(i * 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_slot)), "r"(ALLOC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint64_t da0 = make_desc(smem_u32(smem), 128, 256);
    const uint64_t db0 = make_desc(smem_u32(smem + 8 * 4096), 128, 256);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int ks = 0; ks < nks; ++ks)
        for (int i = 0; i < 8; ++i)
          for (int t = 0; t < ntile; ++t) {
            if (nsplit == 0) {
              if (MKDESC) mma_i8(tmem + t * 256, make_desc(smem_u32(smem + i * 4096), 128, 256), make_desc(smem_u32(smem + 8 * 4096), 128, 256), idesc_i8(128, 256), (r | ks | i) ? 1u : 0u);
              else mma_i8(tmem + t * 256, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 256), (r | ks | i) ? 1u : 0u);
            } else if (nsplit == 1) {
              if (MKDESC) mma_i8(tmem + t * 256 + 32 * i, make_desc(smem_u32(smem + i * 4096), 128, 256), make_desc(smem_u32(smem + 8 * 4096), 128, 256), idesc_i8(128, 32 * (8 - i)), (r | ks | i) ? 1u : 0u);
              else mma_i8(tmem + t * 256 + 32 * i, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 32 * (8 - i)), (r | ks | i) ? 1u : 0u);
            } else {  // split each MMA's N range in two halves issued separately
              const int n = 32 * (8 - i);
              const int n0 = (n / 2 + 15) / 16 * 16, n1 = n - n0;
              mma_i8(tmem + t * 256 + 32 * i, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, n0), 1u);
              if (n1) mma_i8(tmem + t * 256 + 32 * i + n0, da0 + (uint64_t)(i * 256), db0 + (uint64_t)(n0 * 2), idesc_i8(128, n1), 1u);
            }
          }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[0] = clock64() - t0;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(ALLOC));
}

template <int ALLOC = 512, bool MKDESC = false>
static void run_stacked(int ntile, int nks, int nsplit) {
  long long* dc; CK(cudaMalloc(&dc, 8));
  size_t sm = 8 * 4096 + 8 * 1024 + 1024;
  CK(cudaFuncSetAttribute(stacked<ALLOC, MKDESC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int reps = 64;
  stacked<ALLOC, MKDESC><<<1, 128, sm>>>(reps, ntile, nks, nsplit, dc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
  const double per_group = (double)c / (reps * nks * ntile);
  printf("stacked alloc=%d mkdesc=%d ntile=%d nks=%d split=%d: %.0f cyc per 8-MMA group (%.1f per MMA) = %.0f MAC/cyc\n", ALLOC, (int)MKDESC, ntile, nks, nsplit,
         per_group, per_group / (8 * nsplit), 128.0 * 32 * 1152 / per_group);
  cudaFree(dc);
}

template <int MODE>  // 0: pure N=256 chain, 1: stacked, 2: two stacked tiles interleaved
__global__ void __launch_bounds__(128, 1) chain_elect(int reps, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8 * 4096 + 8 * 1024; i += 128) smem[i] = (uint8_t)(i * 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (warp == 0) {
    const uint64_t da0 = make_desc(smem_u32(smem), 128, 256);
    const uint64_t db0 = make_desc(smem_u32(smem + 8 * 4096), 128, 256);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) mma_i8_elect(tmem, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 256), (r | i) ? 1u : 0u);
        if (MODE == 1) mma_i8_elect(tmem + 32 * i, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 32 * (8 - i)), (r | i) ? 1u : 0u);
        if (MODE == 2) {
          mma_i8_elect(tmem + 32 * i, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 32 * (8 - i)), (r | i) ? 1u : 0u);
          mma_i8_elect(tmem + 256 + 32 * i, da0 + (uint64_t)(i * 256), db0, idesc_i8(128, 32 * (8 - i)), (r | i) ? 1u : 0u);
        }
      }
    }
    mma_commit_elect(&bar);
    mbar_wait(&bar, 0);
    if (tid == 0) cyc[0] = clock64() - t0;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

template <int MODE>
static void run_elect() {
  long long* dc; CK(cudaMalloc(&dc, 8));
  size_t sm = 8 * 4096 + 8 * 1024 + 1024;
  CK(cudaFuncSetAttribute(chain_elect<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int reps = 64;
  chain_elect<MODE><<<1, 128, sm>>>(reps, dc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
  printf("elect-issued mode=%d: %.0f cyc per 8-MMA group\n", MODE, (double)c / (reps * (MODE == 2 ? 2 : 1)));
  cudaFree(dc);
}

int main() {
  int bad = 0;
  run_elect<0>(); run_elect<1>(); run_elect<2>();
  run_stacked<512, false>(1, 1, 0); run_stacked<512, false>(1, 1, 1); run_stacked<512, false>(2, 1, 1);
  run_elect<0>(); run_elect<1>(); run_elect<2>();
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad;
}
