// Tensor-core merge for K = 8..64 terms (used from K = 16 by default): the complex rank-K product of the n=2
// merge (merging.py:86-94 `_axpy_outer`, summed over m as in merging.py:178-185)
//   out[h][l] = sum_t (coef_t hi_t[h]) lo_t[l]
// computed exactly on the int8 tensor cores (tcgen05.mma kind::i8, TMEM
// accumulators) by error-free splitting of the FP64 operands (Ozaki scheme).
//
// Real GEMM form: D[l][(h,v)] = sum_k A[l][k] B[(h,v)][k], k = 2t+u,
//   A[l] = (lr_0, li_0, lr_1, li_1, ...),
//   B[(h,0)] = (Hr_0, -Hi_0, ...)  -> Re out,   B[(h,1)] = (Hi_0, Hr_0, ...) -> Im out.
// Every row of A (per l) and every pair of rows of B (per h) is scaled by a
// power of two 2^-e so its entries are <= 1/2 in magnitude, rounded to
// fixed point and split into S balanced int8 digits: by default S = 7
// base-256 digits (55-bit fixed point), or S = 8 base-128 digits (56-bit;
// option merge_ozaki_digits = 7). Digit products of equal weight i + j = p
// ("diagonal p") accumulate exactly in int32:
//   D_p = sum_{i+j=p} A_i B_j^T,   out = 2^(e_l + e_h) sum_p B^-(p+2) D_p
// keeping p <= S-1 (the dropped terms are ~2^-55 / 2^-56 relative to the
// row/column maxima: the rounding level of a K-term FP64 dot product;
// measured max|d| / max|out| 1.1e-15 / 5.7e-16 at K = 16).
//
// Diagonal stacking: the B digit slices of one h block are stacked along N
// (slice j = rows 32j..32j+31), so ONE MMA per A slice i,
//   D[:, 32i : 256] += A_i . [B_0; ...; B_{7-i}]^T      (N = 32 (8 - i)),
// adds A_i B_{p-i} into every diagonal p >= i at once: 8 MMAs per k-step
// instead of 36 (tools/tc_i8_probe.cu: 616 cycles per 8-MMA group against a
// 576-cycle tensor floor).
//
// Roles per CTA (persistent, one per SM): warp 0 streams digit blocks with
// cp.async.bulk (TMA bulk copies, mbarrier complete_tx), warp 1 issues the
// MMAs (one elected lane) into one of two 256-column TMEM accumulators, two
// groups of 8 epilogue warps (warps 2..17, alternate tiles) drain TMEM
// (tcgen05.ld), combine the diagonals pairwise in int32, convert to FP64,
// scale and write each output amplitude once (st.global.cs, 512 contiguous
// bytes per warp store). DESIGN.md §3 has the measurements.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <utility>
#include <cstdint>
#include <map>
#include <mutex>

#include "ops.hpp"

namespace cutsim {
namespace {

// Digit base 2^kDigitBits: 8 -> 7 balanced base-256 digits (|d| <= 128,
// top digit <= 65), 7 int32 diagonals per output; 7 -> 8 base-128 digits, 8
// diagonals. 7 diagonals cut the epilogue's TMEM reads and the digit-pair
// MMAs (28 instead of 36) by 1/8 and 2/9 at twice the truncation.
// Option "merge_ozaki_digits" selects DB (8 default). Truncation measured in
// a host emulation: max |error| / (max|a| max|b|) = 2.2e-15 (DB = 8) and
// 5.6e-16 (DB = 7) over K = 16 terms; on the B200 (tools/ozaki_ab.py, q=30,
// with the base-256 digit pairs combined in int32 for K <= 32): DB = 8 K=16
// 3.01 vs 3.27 ms, K=32 4.64 vs 4.89, K=64 7.54 vs 7.69, q=32 K=16 14.0 vs
// 14.75 ms.
template <int DB>
struct Digits {
  static constexpr int S = DB == 8 ? 7 : 8;  // slices
  // fixed-point bits of a row (|Y| < 2^Fix), chosen so the top digit fits int8
  static constexpr int Fix = DB == 8 ? 54 : 55;
  // sa[l] = 2^(e_l + SaShift): the epilogue's combined diagonals Q0 + 2^-Q1Shift
  // Q1 times sa * sb is the product (base 256: Q0 = D_0..D_3 with D_3 at
  // weight 1 = 2^72 of the 2^-110 fixed point -> 2^-38; base 128: 2^-35)
  static constexpr int SaShift = DB == 8 ? -38 : -35;
  static constexpr int Q1Shift = DB == 8 ? 24 : 28;
};
#define OZ_DIGIT_CONSTS                          \
  constexpr int kDigitBits = DB;                 \
  constexpr int kSlices = Digits<DB>::S;         \
  constexpr int kFix = Digits<DB>::Fix;          \
  constexpr int kSaShift = Digits<DB>::SaShift;  \
  (void)kDigitBits; (void)kSlices; (void)kFix; (void)kSaShift;
constexpr int kHB = 16;                      // h rows per tile (32 real B rows per slice)
constexpr int kLT = 128;                     // l rows per tile (MMA M)
constexpr int kEpiWarps = 16;                // two groups of 8 (alternate tiles)
constexpr int kABlock = kLT * 32;            // one (k-step, slice) block of A: 4 KiB
constexpr int kBBlock = 2 * kHB * 32;        // one (k-step, slice) block of B: 1 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}

// K-major, no-swizzle canonical layout: core matrix = 8 rows x 16 B (128 B
// contiguous), 16-byte K chunks 128 B apart (LBO), 8-row groups 256 B apart (SBO)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46);
}

__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kLT >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// whole-warp: one elected lane arms the barrier and issues the bulk copy
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// The tcgen05 issue helpers are executed by a whole warp; elect.sync inside
// the asm picks the issuing lane. (Issued from a single-lane branch instead,
// the compiler wraps each instruction in an ELECT loop and a chain of
// dependent MMAs runs at ~240 cycles per instruction instead of the
// 128 N / 256 floor: tools/tc_i8_probe.cu.)
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// power-of-two exponent e with max|x| * 2^-e < 1/2, from the double's bits
// (0 for an all-zero row)
__device__ __forceinline__ int row_exponent(double mx) {
  const int b = int((__double_as_longlong(mx) >> 52) & 0x7ff);
  return b ? b - 1021 : 0;  // mx in [2^(b-1023), 2^(b-1022))
}

// 2^(kFix + 1 - e): the fixed-point scale of a row (|y| < 1/2 -> |Y| <
// 2^kFix; clamped for rows below ~1e-290, whose digits then keep fewer bits)
template <int DB>
__device__ __forceinline__ double digit_scale(int e) {
  OZ_DIGIT_CONSTS
  const int b = min(max(kFix + 1 - e + 1023, 1), 2046);
  return __hiloint2double(b << 20, 0);
}

// kSlices balanced base-2^kDigitBits digits of y = x 2^-e (|y| < 1/2):
// Y = rint(y 2^(kFix+1)) (the rounding is the scheme's truncation level),
// then d_{S-1}..d_1 = ((Y + B/2) & (B-1)) - B/2 from the least significant
// end and d_0 = what remains (|d_0| <= 65); y ~ sum_i d_i B^-(i+1) 2^(...).
template <int DB>
__device__ __forceinline__ void digits_split(double x, double scale, int (&d)[Digits<DB>::S]) {
  OZ_DIGIT_CONSTS
  constexpr long long B = 1ll << kDigitBits;
  long long Y = __double2ll_rn(x * scale);
#pragma unroll
  for (int i = kSlices - 1; i > 0; --i) {
    const int di = int((Y + B / 2) & (B - 1)) - int(B / 2);
    d[i] = di;
    Y = (Y - di) >> kDigitBits;
  }
  d[0] = int(Y);
}

__device__ __forceinline__ uint32_t cm_row_off(int r) { return uint32_t((r >> 3) * 256 + (r & 7) * 16); }

__device__ __forceinline__ uint32_t pack2(int a, int b) {
  return uint32_t(uint8_t(int8_t(a))) | (uint32_t(uint8_t(int8_t(b))) << 8);
}

// the digit-preparation kernels' inputs (one slot, K <= 64 terms; a small
// parameter block keeps their launches cheap)
struct OzPrep {
  const double2* hi;
  const double2* lo;
  int64_t hi_len, lo_len, row_begin;
  int32_t K;
  int32_t hidx[64];
  int32_t lidx[64];
  double2 coef[64];
};

// ---------------------------------------------------------------------------
// digit preparation. Four adjacent lanes share one (row, k-step): the row
// maximum is reduced over the lanes with shuffles, and lane `sub` splits
// terms 4 sub .. 4 sub + 3 of the k-step (bytes 8 sub .. 8 sub + 7 of the
// row's 32-byte k-step: the first 16 at the block row, the last 16 one
// 128-byte K-chunk further). Four times the threads of one lane per row —
// at small q each side is only a few thousand rows and the single-lane form
// was latency bound (q=24 K=16: 8 + 12 us ahead of a 63 us merge kernel).
// ---------------------------------------------------------------------------
constexpr int kPrepLanes = 4;

__device__ __forceinline__ uint32_t lane_chunk_off(int sub) { return sub < 2 ? 8u * sub : 128u + 8u * (sub - 2); }

// A (the lo side). adig layout: [l_tile][ks][slice][4096 B canonical block];
// sa[l] = 2^(e_l + kSaShift)
template <int KS, int DB>
__device__ __forceinline__ void ozaki_prep_lo(const OzPrep& p, int64_t gidx, int8_t* adig, double* sa) {
  OZ_DIGIT_CONSTS
  const int sub = int(gidx & (kPrepLanes - 1));
  const int64_t idx = gidx / kPrepLanes;
  const bool live = idx < p.lo_len * KS;  // the 4 lanes of a group agree; no early exit before the shuffles
  const int ks = live ? int(idx / p.lo_len) : 0;
  const int64_t l = live ? idx - int64_t(ks) * p.lo_len : 0;
  const double2* lo = p.lo;
  const int K = p.K;
  double mx = 0.0;
  int finite = 1;
  if (live) {
    for (int t = sub; t < K; t += kPrepLanes) {
      const double2 v = __ldg(lo + int64_t(p.lidx[t]) * p.lo_len + l);
      finite &= isfinite(v.x) && isfinite(v.y);
      mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
    }
  }
#pragma unroll
  for (int o = 1; o < kPrepLanes; o <<= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    finite &= __shfl_xor_sync(0xffffffffu, finite, o);
  }
  if (!live) return;
  const int e = row_exponent(finite ? mx : 0.0);
  // a NaN/Inf operand makes the whole output column NaN (as the FP64 kernels
  // propagate it) instead of saturated digits turning it into a finite value
  if (ks == 0 && sub == 0) sa[l] = finite ? ldexp(1.0, e + kSaShift) : __longlong_as_double(0x7ff8000000000000ll);
  const double sc = digit_scale<DB>(e);
  uint32_t w[kSlices][2];
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    const int t = 16 * ks + 4 * sub + tt;
    double2 v = make_double2(0.0, 0.0);
    if (t < K) v = __ldg(lo + int64_t(p.lidx[t]) * p.lo_len + l);
    int dr[kSlices], di[kSlices];
    digits_split<DB>(v.x, sc, dr);
    digits_split<DB>(v.y, sc, di);
#pragma unroll
    for (int i = 0; i < kSlices; ++i) {
      // bytes 2tt, 2tt + 1 of this lane's 8 bytes: (re, im)
      const uint32_t pr = pack2(dr[i], di[i]) << (16 * (tt & 1));
      if (tt & 1) w[i][tt >> 1] |= pr;
      else w[i][tt >> 1] = pr;
    }
  }
  int8_t* base = adig + (l >> 7) * int64_t(KS * kSlices * kABlock) + cm_row_off(int(l & 127)) + lane_chunk_off(sub);
#pragma unroll
  for (int i = 0; i < kSlices; ++i)
    *reinterpret_cast<uint2*>(base + (ks * kSlices + i) * kABlock) = make_uint2(w[i][0], w[i][1]);
}

// B (the hi side with the coefficients). bdig layout: [h_block][ks][slice]
// [1024 B canonical block], row r = 2 (h % 16) + v; sb[h] = 2^e_h
template <int KS, int DB>
__device__ __forceinline__ void ozaki_prep_hi(const OzPrep& p, int64_t gidx, int64_t nrows, int8_t* bdig, double* sb) {
  OZ_DIGIT_CONSTS
  const int sub = int(gidx & (kPrepLanes - 1));
  const int64_t idx = gidx / kPrepLanes;
  const bool live = idx < nrows * KS;
  const int ks = live ? int(idx / nrows) : 0;
  const int64_t hr = live ? idx - int64_t(ks) * nrows : 0;
  const int64_t h = p.row_begin + hr;
  const double2* hi = p.hi;
  const int K = p.K;
  double mx = 0.0;
  int finite = 1;
  if (live) {
    for (int t = sub; t < K; t += kPrepLanes) {
      const double2 v = __ldg(hi + int64_t(p.hidx[t]) * p.hi_len + h);
      const double cr = p.coef[t].x, ci = p.coef[t].y;
      const double br = v.x * cr - v.y * ci, bi = v.x * ci + v.y * cr;
      finite &= isfinite(br) && isfinite(bi);
      mx = fmax(mx, fmax(fabs(br), fabs(bi)));
    }
  }
#pragma unroll
  for (int o = 1; o < kPrepLanes; o <<= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    finite &= __shfl_xor_sync(0xffffffffu, finite, o);
  }
  if (!live) return;
  const int e = row_exponent(finite ? mx : 0.0);
  if (ks == 0 && sub == 0) sb[hr] = finite ? ldexp(1.0, e) : __longlong_as_double(0x7ff8000000000000ll);
  const double sc = digit_scale<DB>(e);
  uint32_t w0[kSlices][2], w1[kSlices][2];
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    const int t = 16 * ks + 4 * sub + tt;
    double br = 0.0, bi = 0.0;
    if (t < K) {
      const double2 v = __ldg(hi + int64_t(p.hidx[t]) * p.hi_len + h);
      const double cr = p.coef[t].x, ci = p.coef[t].y;
      br = v.x * cr - v.y * ci;
      bi = v.x * ci + v.y * cr;
    }
    int dr[kSlices], di[kSlices], dn[kSlices];
    digits_split<DB>(br, sc, dr);
    digits_split<DB>(bi, sc, di);
    // -Hi split on its own: a balanced base-256 digit may be -128, whose
    // negation does not fit int8 (base 128: -d is a valid digit)
    if constexpr (DB == 8) {
      digits_split<DB>(-bi, sc, dn);
    } else {
#pragma unroll
      for (int i = 0; i < kSlices; ++i) dn[i] = -di[i];
    }
#pragma unroll
    for (int i = 0; i < kSlices; ++i) {
      // row (h, 0): (Hr, -Hi) -> real part; row (h, 1): (Hi, Hr) -> imaginary part
      const uint32_t p0 = pack2(dr[i], dn[i]) << (16 * (tt & 1));
      const uint32_t p1 = pack2(di[i], dr[i]) << (16 * (tt & 1));
      if (tt & 1) {
        w0[i][tt >> 1] |= p0;
        w1[i][tt >> 1] |= p1;
      } else {
        w0[i][tt >> 1] = p0;
        w1[i][tt >> 1] = p1;
      }
    }
  }
  const int hl = int(hr & (kHB - 1));
  int8_t* base = bdig + (hr / kHB) * int64_t(KS * kSlices * kBBlock) + lane_chunk_off(sub);
#pragma unroll
  for (int i = 0; i < kSlices; ++i) {
    int8_t* blk = base + (ks * kSlices + i) * kBBlock;
    *reinterpret_cast<uint2*>(blk + cm_row_off(2 * hl)) = make_uint2(w0[i][0], w0[i][1]);
    *reinterpret_cast<uint2*>(blk + cm_row_off(2 * hl + 1)) = make_uint2(w1[i][0], w1[i][1]);
  }
}

// both sides in one launch: blocks [0, lo_blocks) the lo rows, the rest the
// hi rows (independent work; one launch and no serialisation between them)
template <int KS, int DB>
__global__ void __launch_bounds__(128) ozaki_prep(const __grid_constant__ OzPrep p, int64_t nrows, int64_t lo_blocks,
                                                 int8_t* adig, double* sa, int8_t* bdig, double* sb) {
  if (int64_t(blockIdx.x) < lo_blocks)
    ozaki_prep_lo<KS, DB>(p, int64_t(blockIdx.x) * blockDim.x + threadIdx.x, adig, sa);
  else
    ozaki_prep_hi<KS, DB>(p, (int64_t(blockIdx.x) - lo_blocks) * blockDim.x + threadIdx.x, nrows, bdig, sb);
}

struct OzParams {
  const int8_t* adig;
  const int8_t* bdig;
  const double* sa;  // per l: 2^(e_l + kSaShift)
  const double* sb;  // per h: 2^e_h
  double2* out;  // row 0 of the range
  int64_t W;     // lo_len
  int64_t n_hb;  // h blocks in the range
  int64_t n_lt;   // l tiles (W / 128)
  int64_t n_hc;   // h chunks: work unit u = (h chunk u / n_lt, l tile u % n_lt)
  int64_t n_units;
};

// Work units = (h chunk, l tile), dealt round-robin to the persistent CTAs
// with the l tile fastest: at any moment the CTAs write the same h rows at
// consecutive l tiles (long contiguous row segments for the DRAM write
// stream; h-chunk-major per CTA instead gave 2 KB row pieces scattered over
// the state and ~5.5 TB/s). Inside a unit a CTA walks its h blocks with the
// unit's A digits resident in shared memory.
struct TileWalk {
  const OzParams& p;
  int64_t u, lt, hb, hb_end;
  __device__ explicit TileWalk(const OzParams& pp) : p(pp), u(blockIdx.x) { begin(); }
  __device__ void begin() {
    if (u >= p.n_units) return;
    const int64_t hc = u / p.n_lt;
    lt = u - hc * p.n_lt;
    hb = hc * p.n_hb / p.n_hc;
    hb_end = (hc + 1) * p.n_hb / p.n_hc;
  }
  __device__ bool valid() const { return u < p.n_units; }
  __device__ void next() {
    if (++hb == hb_end) {
      u += gridDim.x;
      begin();
    }
  }
};

// UNIT = false: persistent, one CTA per SM, two 256-column accumulators and
// two epilogue groups. UNIT = true: one work unit per CTA (a short-lived
// CTA, two per SM), one accumulator and one epilogue group: short-lived CTAs
// sustain a faster HBM write stream than persistent ones
// (tools/store_patterns.cu: 7.3 vs 6.2 TB/s).
template <bool UNIT>
constexpr int oz_threads() { return 64 + 32 * (UNIT ? kEpiWarps / 2 : kEpiWarps); }

// A digit buffers in shared memory: two (the next work unit's l-tile digits
// load while the current unit's MMAs run) where they fit next to the B ring
template <int KS, bool UNIT>
constexpr int oz_abufs() { return (!UNIT && KS <= 2) ? 2 : 1; }

template <int KS, int NST, bool ACC, bool UNIT, int DB>
__global__ void __launch_bounds__(oz_threads<UNIT>(), UNIT ? 2 : 1) ozaki_merge_kernel(const __grid_constant__ OzParams p) {
  OZ_DIGIT_CONSTS
  constexpr int NBUF = UNIT ? 1 : 2;  // TMEM accumulators (= epilogue groups)
  constexpr int NA = oz_abufs<KS, UNIT>();
  constexpr uint32_t TCOLS = 256 * NBUF;
  constexpr uint32_t A_BYTES = KS * kSlices * kABlock;
  constexpr uint32_t B_BYTES = KS * kSlices * kBBlock;
  extern __shared__ __align__(1024) uint8_t smem[];
  int8_t* sA = reinterpret_cast<int8_t*>(smem);  // [NA]
  int8_t* sB = reinterpret_cast<int8_t*>(smem + NA * A_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NA * A_BYTES + NST * B_BYTES);
  uint64_t* full = bars;             // [NST]
  uint64_t* empty = bars + NST;      // [NST]
  uint64_t* afull = bars + 2 * NST;  // [NA]
  uint64_t* aempty = afull + NA;     // [NA]
  uint64_t* tfull = aempty + NA;     // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // warp index through a shuffle so the compiler knows it is warp-uniform
  // (TMEM addresses derived from it then stay in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < NA; ++a) {
      mbar_init(afull + a, 1);
      mbar_init(aempty + a, 1);
    }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, kEpiWarps / 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {
      int64_t cur = -1;
      int uc = -1;  // work units (A loads) so far
      int it = 0;
      for (TileWalk w(p); w.valid(); w.next(), ++it) {
        const int64_t lt = w.lt, hb = w.hb;
        if (lt != cur) {
          ++uc;
          const int ab = uc % NA;
          // buffer ab was last filled for unit uc - NA: wait for its MMAs
          if (uc >= NA) mbar_wait(aempty + ab, ((uc / NA) - 1) & 1);
          bulk_load(sA + ab * A_BYTES, p.adig + lt * A_BYTES, A_BYTES, afull + ab);
          cur = lt;
        }
        const int st = it % NST;
        const uint32_t ph = (it / NST) & 1;
        mbar_wait(empty + st, ph ^ 1);
        bulk_load(sB + st * B_BYTES, p.bdig + hb * B_BYTES, B_BYTES, full + st);
      }
    }
  } else if (warp == 1) {
    {
      int64_t cur = -1;
      int uc = -1;
      int it = 0;
      uint32_t a0 = smem_u32(sA);
      const uint32_t b0 = smem_u32(sB);
      for (TileWalk w(p); w.valid(); w.next(), ++it) {
        const int64_t lt = w.lt;
        if (lt != cur) {
          // the previous unit's MMAs release its A buffer when they complete
          if (uc >= 0) mma_commit(aempty + (uc % NA));
          ++uc;
          mbar_wait(afull + (uc % NA), (uc / NA) & 1);
          a0 = smem_u32(sA + (uc % NA) * A_BYTES);
          cur = lt;
        }
        const int st = it % NST;
        mbar_wait(full + st, (it / NST) & 1);
        const int b = it % NBUF;
        mbar_wait(tempty + b, ((it / NBUF) & 1) ^ 1);
        tc_after_sync();
        const uint32_t dbase = tmem + uint32_t(b * 256);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint64_t db = smem_desc(b0 + st * B_BYTES + ks * kSlices * kBBlock);
#pragma unroll
          for (int i = 0; i < kSlices; ++i) {
            const uint64_t da = smem_desc(a0 + (ks * kSlices + i) * kABlock);
            mma_i8(dbase + uint32_t(32 * i), da, db, idesc_i8(32 * (kSlices - i)), (ks | i) ? 1u : 0u);
          }
        }
        mma_commit(empty + st);
        mma_commit(tfull + b);
      }
    }
  } else {
    // two groups of 8 warps take alternate tiles (= alternate TMEM buffers), so
    // one group's TMEM loads and barrier waits overlap the other's math and
    // stores; in a group every lane quarter q has two warps, one per 8 h rows
    const int g = (warp - 2) >> 3;
    const int wg = (warp - 2) & 7;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int hl_base = (wg >> 2) * 8;
    const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(g * 256);
    uint32_t n = 0;
    int it = 0;
    for (TileWalk w(p); w.valid(); w.next(), ++it) {
      if ((it % NBUF) != g) continue;
      const int64_t lt = w.lt, hb = w.hb;
      const int64_t l = lt * kLT + q * 32 + lane;
      const double sl = __ldg(p.sa + l);  // 2^(e_l + kSaShift)
      // accumulate (K > 64 in 64-term chunks): prefetch the 8 outputs being
      // added to into L2 before waiting for the accumulator, so their DRAM
      // reads overlap the MMA chain (held in registers instead, they spilled)
      if (ACC) {
        const double2* src = p.out + (hb * kHB + hl_base) * p.W + l;
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(src + j * p.W));
      }
      // the 8 row scales of this warp's h rows, fetched before the wait so
      // their load latency hides under the MMA instead of the epilogue
      double sbv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) sbv[j] = __ldg(p.sb + hb * kHB + hl_base + j);
      mbar_wait(tfull + g, n & 1);
      ++n;
      tc_after_sync();
      uint32_t d[2][kSlices][8];
#pragma unroll
      for (int pd = 0; pd < kSlices; ++pd) tmem_ld8(tbase + uint32_t(pd * 32 + 2 * hl_base), d[0][pd]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int pd = 0; pd < kSlices; ++pd) tmem_ld8(tbase + uint32_t(pd * 32 + 2 * (hl_base + 4)), d[1][pd]);
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
        if (hc == 1) {  // second chunk landed under the first one's math: hand the buffer back
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tc_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty + g);
        }
        const int hl0 = hl_base + 4 * hc;
        double2* dst = p.out + (hb * kHB + hl0) * p.W + l;
#pragma unroll
        for (int j = 0; j < 4; ++j, dst += p.W) {
          const double s = sl * sbv[4 * hc + j];
          double v2[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int c = 2 * j + v;
            // q0, q1 are produced with the int64 -> double bias 0x4338000000000000
            // (1.5 * 2^52) already folded into the 64-bit addend of the
            // IMAD.WIDE: bias_ext(x) = 2^32 (0x43380000 + (x >> 31)) + (uint32)x
            // = bias + sign-extended x, one IADD3 (+ SHF) for the high word
            // instead of a separate 64-bit add per value
            auto bias_ext = [](int x) {
              const unsigned hi = unsigned(x >> 31) + 0x43380000u;
              return static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | unsigned(x));
            };
            long long q0, q1;
            if constexpr (kDigitBits == 8) {
              // base 256, 7 diagonals (|D_p| < 2^24): Q0 = D_0 2^24 + D_1 2^16
              // + D_2 2^8 + D_3, Q1 = D_4 2^16 + D_5 2^8 + D_6 (|Q0| < 2^49,
              // |Q1| < 2^41: exact in int64 and in a double); product =
              // 2^-38 (Q0 + 2^-24 Q1) sa sb
              if constexpr (KS <= 2) {
                // K <= 32: |D_p| <= 7 * 64 * 2^14 < 2^22.9, so the digit
                // pairs D_2m 2^8 + D_2m+1 stay exact in int32 (one IMAD each)
                const int a0 = int(d[hc][0][c]) * 256 + int(d[hc][1][c]);
                const int a1 = int(d[hc][2][c]) * 256 + int(d[hc][3][c]);
                const int a2 = int(d[hc][4][c]) * 256 + int(d[hc][5][c]);
                q0 = static_cast<long long>(a0) * 65536 + bias_ext(a1);
                q1 = static_cast<long long>(a2) * 256 + bias_ext(int(d[hc][6][c]));
              } else {
                // K = 64: |D_p| < 2^23.7, a digit pair may overflow int32;
                // Horner chains of 32 x 32 -> 64-bit multiply-adds (one
                // IMAD.WIDE per diagonal) on the biased low diagonal
                auto wide = [](int x, int m, long long acc) { return static_cast<long long>(x) * m + acc; };
                q0 = wide(int(d[hc][0][c]), 1 << 24,
                          wide(int(d[hc][1][c]), 1 << 16, wide(int(d[hc][2][c]), 1 << 8, bias_ext(int(d[hc][3][c])))));
                q1 = wide(int(d[hc][4][c]), 1 << 16, wide(int(d[hc][5][c]), 1 << 8, bias_ext(int(d[hc][6][c]))));
              }
            } else {
              // base 128, 8 diagonals: P_m = 128 D_2m + D_2m+1 (|D_p| < 2^23:
              // exact in int32), Q0 = 2^14 P_0 + P_1, Q1 = 2^14 P_2 + P_3;
              // sum_p 2^-7(p+2) D_p = 2^-35 (Q0 + 2^-28 Q1)
              const int p0 = int(d[hc][0][c]) * 128 + int(d[hc][1][c]);
              const int p1 = int(d[hc][2][c]) * 128 + int(d[hc][3][c]);
              const int p2 = int(d[hc][4][c]) * 128 + int(d[hc][5][c]);
              const int p3 = int(d[hc][kSlices - 2][c]) * 128 + int(d[hc][kSlices - 1][c]);
              q0 = static_cast<long long>(p0) * 16384 + bias_ext(p1);
              q1 = static_cast<long long>(p2) * 16384 + bias_ext(p3);
            }
            // int64 -> double: the bias is in q already (|q - bias| < 2^51)
            const double f0 = __longlong_as_double(q0) - 0x1.8p52;
            const double f1 = __longlong_as_double(q1) - 0x1.8p52;
            v2[v] = fma(f1, kDigitBits == 8 ? 0x1p-24 : 0x1p-28, f0) * s;
          }
          double2 val = make_double2(v2[0], v2[1]);
          if (ACC) {
            const double2 prev = __ldcs(dst);
            val.x += prev.x;
            val.y += prev.y;
          }
          __stcs(dst, val);  // evict-first: the state is written once
        }
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
}

template <int KS, int NST, int DB, bool UNIT>
constexpr size_t oz_smem() {
  constexpr int kSlices = Digits<DB>::S;
  return size_t(oz_abufs<KS, UNIT>()) * KS * kSlices * kABlock + size_t(NST) * KS * kSlices * kBBlock + 256;
}

// digit workspace per stream (grow-only; merges on different streams may overlap)
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
};
// keyed by (device, stream): the legacy default stream (0) is shared by all
// devices, and a workspace allocated on one device must not serve another
std::map<std::pair<int, cudaStream_t>, Workspace> g_oz_ws;
std::mutex g_oz_mu;
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: one bit
// per (device, instantiation)
std::atomic<uint64_t> g_oz_configured[16];

template <int KS, int NST, bool UNIT, int DB>
cudaError_t run_ozaki(const MergeParams& mp, int64_t nrows, void* out, int accumulate, int sms,
                      cudaStream_t stream) {
  constexpr int kSlices = Digits<DB>::S;
  const int64_t W = mp.lo_len;
  const size_t a_bytes = size_t(W / kLT) * KS * kSlices * kABlock;
  const size_t b_bytes = size_t(nrows / kHB) * KS * kSlices * kBBlock;
  const size_t ea_bytes = size_t(W) * 8, eb_bytes = size_t(nrows) * 8;
  const size_t need = a_bytes + b_bytes + ea_bytes + eb_bytes + 1024;
  int dev = 0;
  {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
  }
  std::lock_guard<std::mutex> lk(g_oz_mu);
  Workspace& ws = g_oz_ws[{dev, stream}];
  if (ws.bytes < need) {
    if (ws.ptr) {
      cudaError_t e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return e;
      cudaFree(ws.ptr);
      ws = Workspace{};
    }
    cudaError_t e = cudaMalloc(&ws.ptr, need);
    if (e != cudaSuccess) return e;
    ws.bytes = need;
  }
  int8_t* adig = static_cast<int8_t*>(ws.ptr);
  int8_t* bdig = adig + a_bytes;
  double* sa = reinterpret_cast<double*>(bdig + b_bytes);
  double* sb = sa + W;
  OzPrep pp;
  pp.hi = static_cast<const double2*>(mp.hi);
  pp.lo = static_cast<const double2*>(mp.lo);
  pp.hi_len = mp.hi_len;
  pp.lo_len = mp.lo_len;
  pp.row_begin = mp.row_begin;
  pp.K = mp.K;
  for (int t = 0; t < mp.K; ++t) {
    pp.hidx[t] = mp.hidx[t];
    pp.lidx[t] = mp.lidx[t];
    pp.coef[t] = make_double2(mp.coef[2 * t], mp.coef[2 * t + 1]);
  }
  const int64_t lo_blocks = (W * KS * kPrepLanes + 127) / 128;
  const int64_t hi_blocks = (nrows * KS * kPrepLanes + 127) / 128;
  ozaki_prep<KS, DB><<<unsigned(lo_blocks + hi_blocks), 128, 0, stream>>>(pp, nrows, lo_blocks, adig, sa, bdig, sb);
  OzParams op;
  op.adig = adig;
  op.bdig = bdig;
  op.sa = sa;
  op.sb = sb;
  op.out = static_cast<double2*>(out);
  op.W = W;
  op.n_hb = nrows / kHB;
  op.n_lt = W / kLT;
  if (UNIT) {
    // one unit (l tile x 64 h blocks) per CTA (8 / 16 / 32 / 128 measured
    // slower or equal)
    op.n_hc = std::max<int64_t>(1, op.n_hb / 64);
  } else {
    // h chunks so that n_lt * n_hc is a multiple of the grid (equal work per CTA)
    int64_t a = sms, b = op.n_lt;
    while (b) {
      const int64_t r = a % b;
      a = b;
      b = r;
    }
    op.n_hc = std::max<int64_t>(1, std::min<int64_t>(op.n_hb, sms / a));
  }
  op.n_units = op.n_lt * op.n_hc;

  // persistent: at least ~116 KB of shared memory so that exactly one CTA
  // (and one 512-column TMEM allocation) lives on each SM; unit CTAs: two
  // per SM (256 TMEM columns each)
  const size_t smem = UNIT ? oz_smem<KS, NST, DB, UNIT>() : std::max<size_t>(oz_smem<KS, NST, DB, UNIT>(), 116 * 1024);
  constexpr int inst = ((KS == 1 ? 0 : KS == 2 ? 1 : 2) * 2 + (UNIT ? 1 : 0)) * 2 + (DB == 8 ? 1 : 0);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(g_oz_configured[inst].load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(ozaki_merge_kernel<KS, NST, false, UNIT, DB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ozaki_merge_kernel<KS, NST, true, UNIT, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem));
    if (e != cudaSuccess) return e;
    g_oz_configured[inst].fetch_or(bit);
  }
  const int64_t grid = UNIT ? op.n_units : std::min<int64_t>(sms, op.n_units);
  if (grid > 0x7fffffff) return cudaErrorInvalidValue;
  constexpr int threads = oz_threads<UNIT>();
  if (accumulate) ozaki_merge_kernel<KS, NST, true, UNIT, DB><<<unsigned(grid), threads, smem, stream>>>(op);
  else ozaki_merge_kernel<KS, NST, false, UNIT, DB><<<unsigned(grid), threads, smem, stream>>>(op);
  return cudaGetLastError();
}

}  // namespace

// K in {8, 16, 32, 64} terms (K = 8 pads the inner dimension to 32), complex128,
// one slot; lo_len % 128 == 0 and (row_end - row_begin) % 16 == 0.
bool merge_ozaki_supported(int K, int64_t lo_len, int64_t nrows) {
  return (K == 8 || K == 16 || K == 32 || K == 64) && lo_len >= kLT && lo_len % kLT == 0 && nrows >= kHB &&
         nrows % kHB == 0;
}

// mp: hi/lo/hidx/lidx/coef/K/row_begin/hi_len/lo_len as for the other merge
// kernels (slot 0); out = row row_begin of the output.
// unit: short-lived CTAs (two per SM) for K <= 32; K = 64 (128 KB of A
// digits per CTA) always runs persistent
cudaError_t launch_merge_ozaki(const MergeParams& mp, int64_t nrows, void* out, int accumulate, int sms, bool unit,
                               cudaStream_t stream, int digit_bits) {
  if (digit_bits == 7) {
    switch (mp.K) {
      case 8:
      case 16:
        return unit ? run_ozaki<1, 4, true, 7>(mp, nrows, out, accumulate, sms, stream)
                    : run_ozaki<1, 6, false, 7>(mp, nrows, out, accumulate, sms, stream);
      case 32:
        return unit ? run_ozaki<2, 2, true, 7>(mp, nrows, out, accumulate, sms, stream)
                    : run_ozaki<2, 4, false, 7>(mp, nrows, out, accumulate, sms, stream);
      case 64: return run_ozaki<4, 2, false, 7>(mp, nrows, out, accumulate, sms, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  // base 256 (7 slices: 7/8 of the A/B digit bytes): K = 64 fits a third B stage
  switch (mp.K) {
    case 8:
    case 16:
      return unit ? run_ozaki<1, 4, true, 8>(mp, nrows, out, accumulate, sms, stream)
                  : run_ozaki<1, 6, false, 8>(mp, nrows, out, accumulate, sms, stream);
    case 32:
      return unit ? run_ozaki<2, 2, true, 8>(mp, nrows, out, accumulate, sms, stream)
                  : run_ozaki<2, 4, false, 8>(mp, nrows, out, accumulate, sms, stream);
    case 64: return run_ozaki<4, 3, false, 8>(mp, nrows, out, accumulate, sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cutsim
