// sm_100a kernels of libcutsim: the gate-sweep kernel (subcircuit batches and
// the uncut simulator), the merge-terms kernel (full-state reconstruction, the
// HBM-write-bound hot op), basis init and deterministic device reductions.
//
// Reference seams replaced (paths under /root/reference/pkg/src/cutbench):
//   sweep_kernel  <- engine.py:62-139  (_k_h/_k_x/_k_phase/_k_cx/_k_cz, _run_gates)
//   merge_kernel  <- merging.py:86-110 (_axpy_outer/_outer_into/_iadd) and the
//                    per-term loop merging.py:161-186, as one write-once pass
//   init_basis    <- engine.py:47-51   (StateVec.zero_state)
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "ops.hpp"

namespace cutsim {

template <typename R>
using vec2_t = typename std::conditional<std::is_same<R, double>::value, double2, float2>::type;

template <typename R>
__device__ __forceinline__ vec2_t<R> cmul(vec2_t<R> a, R br, R bi) {
  vec2_t<R> r;
  r.x = a.x * br - a.y * bi;
  r.y = a.x * bi + a.y * br;
  return r;
}

// acc += a * b (complex), four fused multiply-adds
template <typename R>
__device__ __forceinline__ void cfma(vec2_t<R>& acc, vec2_t<R> a, vec2_t<R> b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// ---------------------------------------------------------------------------
// Gate sweep: one CTA owns one tile of 2^T amplitudes of one state (local
// bits [0,L) = qubits [0,L), bits [L,T) = qubits hq[], the tile id scattered
// over the remaining qubits oq[]). The tile is staged in shared memory, every
// op of the launch is applied there, and the tile is written back once.
//
// Dense ops come in register groups of up to 4 commuting ops on distinct
// qubits: each thread loads the 2^k amplitudes of one k-qubit cell into
// registers, applies all k 2x2 matrices, and stores once — k times less
// shared-memory traffic and k-1 fewer barriers than op-by-op. Shared memory
// is XOR-swizzled on 16-byte granules so the cell strides (2^t elements) do
// not collide on banks.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t swz(uint32_t e) {
  uint32_t x = e >> 3;
  x ^= (x >> 3) ^ (x >> 6) ^ (x >> 9);
  return e ^ (x & 7u);
}

template <typename R>
__device__ __forceinline__ void apply2x2(vec2_t<R>& a, vec2_t<R>& b, const double* m) {
  const R m00r = R(m[0]), m00i = R(m[1]), m01r = R(m[2]), m01i = R(m[3]);
  const R m10r = R(m[4]), m10i = R(m[5]), m11r = R(m[6]), m11i = R(m[7]);
  vec2_t<R> u, w;
  u.x = m00r * a.x - m00i * a.y + m01r * b.x - m01i * b.y;
  u.y = m00r * a.y + m00i * a.x + m01r * b.y + m01i * b.x;
  w.x = m10r * a.x - m10i * a.y + m11r * b.x - m11i * b.y;
  w.y = m10r * a.y + m10i * a.x + m11r * b.y + m11i * b.x;
  a = u;
  b = w;
}

// One register group of K commuting dense ops for the VB states this CTA
// holds (shared memory layout: element e of state b at swz(e) * VB + b).
template <typename R, int K, int VB>
__device__ __forceinline__ int apply_group(vec2_t<R>* s, const SweepOp* ops, int i0, uint64_t base,
                                           uint64_t variant0, int T, uint32_t tid, uint32_t bd) {
  using V = vec2_t<R>;
  int tgt[K];
  uint32_t lm[K];
  bool act[K];
  int first[K];
  int slot[K];
  int j = i0;
#pragma unroll
  for (int g = 0; g < K; ++g) {
    const SweepOp& o = ops[j];
    first[g] = j;
    slot[g] = o.slot;
    tgt[g] = o.target;
    lm[g] = o.lmask;
    act[g] = (base & o.omask) == o.omask;
    j += (o.slot >= 0) ? 2 : 1;
  }
  int srt[K];
#pragma unroll
  for (int g = 0; g < K; ++g) srt[g] = tgt[g];
#pragma unroll
  for (int a = 1; a < K; ++a)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (srt[b] < srt[b - 1]) {
        const int t = srt[b];
        srt[b] = srt[b - 1];
        srt[b - 1] = t;
      }
  uint32_t off[1 << K];
#pragma unroll
  for (int i = 0; i < (1 << K); ++i) {
    uint32_t o = 0;
#pragma unroll
    for (int g = 0; g < K; ++g)
      if ((i >> g) & 1) o |= 1u << tgt[g];
    off[i] = o;
  }
  const uint32_t cells = 1u << (T - K);
  for (uint32_t c = tid; c < cells; c += bd) {
    uint32_t e = c;
#pragma unroll
    for (int g = 0; g < K; ++g) {
      const uint32_t b = (1u << srt[g]) - 1u;
      e = ((e & ~b) << 1) | (e & b);
    }
    V v[1 << K][VB];
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) {
      const uint32_t a = swz(e | off[i]) * VB;
#pragma unroll
      for (int b = 0; b < VB; ++b) v[i][b] = s[a + b];
    }
#pragma unroll
    for (int g = 0; g < K; ++g) {
      if (!act[g] || (e & lm[g]) != lm[g]) continue;
      if (slot[g] < 0) {
        const double* m = ops[first[g]].m;
#pragma unroll
        for (int i = 0; i < (1 << K); ++i) {
          if ((i >> g) & 1) continue;
#pragma unroll
          for (int b = 0; b < VB; ++b) apply2x2<R>(v[i][b], v[i | (1 << g)][b], m);
        }
      } else {
#pragma unroll
        for (int b = 0; b < VB; ++b) {
          const double* m = ops[first[g] + int(((variant0 + b) >> slot[g]) & 1ull)].m;
#pragma unroll
          for (int i = 0; i < (1 << K); ++i) {
            if ((i >> g) & 1) continue;
            apply2x2<R>(v[i][b], v[i | (1 << g)][b], m);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < (1 << K); ++i) {
      const uint32_t a = swz(e | off[i]) * VB;
#pragma unroll
      for (int b = 0; b < VB; ++b) s[a + b] = v[i][b];
    }
  }
  return j;
}

// A run of diagonal ops [i0, i1): each thread keeps a chunk of its elements
// (all VB states) in registers, walks the ops once (uniform loads, the
// tile-constant outside-mask test hoisted), multiplies matching elements (a
// sign flip for CZ-type -1 phases), and stores once.
template <typename R, int VB>
__device__ __forceinline__ void apply_phase_run(vec2_t<R>* s, const SweepOp* ops, int i0, int i1, uint64_t base,
                                                uint64_t variant0, uint32_t n, uint32_t tid, uint32_t bd) {
  using V = vec2_t<R>;
  constexpr int CH = VB >= 4 ? 2 : (VB == 2 ? 4 : 8);
  for (uint32_t e0 = tid; e0 < n; e0 += bd * CH) {
    V v[CH][VB];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t e = e0 + uint32_t(c) * bd;
      if (e < n) {
#pragma unroll
        for (int b = 0; b < VB; ++b) v[c][b] = s[swz(e) * VB + b];
      }
    }
    for (int k = i0; k < i1;) {
      const SweepOp& o = ops[k];
      const int sl = o.slot;
      const int here = k;
      k += (sl >= 0) ? 2 : 1;
      if ((base & o.omask) != o.omask) continue;
      const uint32_t lm = o.lmask;
      if (sl < 0) {
        const double qr = o.m[0], qi = o.m[1];
        if (qi == 0.0 && qr == -1.0) {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint32_t e = e0 + uint32_t(c) * bd;
            if ((e & lm) == lm) {
#pragma unroll
              for (int b = 0; b < VB; ++b) {
                v[c][b].x = -v[c][b].x;
                v[c][b].y = -v[c][b].y;
              }
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint32_t e = e0 + uint32_t(c) * bd;
            if ((e & lm) == lm) {
#pragma unroll
              for (int b = 0; b < VB; ++b) v[c][b] = cmul<R>(v[c][b], R(qr), R(qi));
            }
          }
        }
      } else {
#pragma unroll
        for (int b = 0; b < VB; ++b) {
          const double* q = ops[here + int(((variant0 + b) >> sl) & 1ull)].m;
          const R qr = R(q[0]), qi = R(q[1]);
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const uint32_t e = e0 + uint32_t(c) * bd;
            if ((e & lm) == lm) v[c][b] = cmul<R>(v[c][b], qr, qi);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint32_t e = e0 + uint32_t(c) * bd;
      if (e < n) {
#pragma unroll
        for (int b = 0; b < VB; ++b) s[swz(e) * VB + b] = v[c][b];
      }
    }
  }
}

// One CTA = one tile of VB consecutive states of the batch.
template <typename R, int CAP, int VB, int MINB>
__global__ void __launch_bounds__(256, MINB) sweep_kernel(const __grid_constant__ SweepParamsT<CAP> p) {
  using V = vec2_t<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* s = reinterpret_cast<V*>(smem_raw);
  const int T = p.tile_bits;
  const int L = p.low_bits;
  const uint32_t n = 1u << T;
  const uint32_t nchunks = 1u << (T - L);
  const uint32_t lowmask = (1u << L) - 1u;
  int64_t* chunkoff = reinterpret_cast<int64_t*>(smem_raw + sizeof(V) * size_t(n) * VB);
  SweepOp* ops = reinterpret_cast<SweepOp*>(smem_raw + sizeof(V) * size_t(n) * VB + sizeof(int64_t) * size_t(nchunks));
  const uint32_t tid = threadIdx.x;
  const uint32_t bd = blockDim.x;
  const int n_ops = p.n_ops;

  // stage the op list in shared memory once (uniform reads from the 31 KiB
  // parameter bank would miss the constant cache at every step)
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(&p.ops[0]);
    uint64_t* dst = reinterpret_cast<uint64_t*>(ops);
    const uint32_t words = uint32_t(n_ops) * uint32_t(sizeof(SweepOp) / 8);
    for (uint32_t w = tid; w < words; w += bd) dst[w] = src[w];
  }

  uint64_t base = 0;
  {
    const uint64_t tile = blockIdx.x;
    for (int j = 0; j < p.n_out; ++j)
      if ((tile >> j) & 1ull) base |= 1ull << p.oq[j];
  }
  const int v0 = int(blockIdx.y) * VB;
  const uint64_t variant0 = p.variant_base + uint64_t(v0);
  V* st = reinterpret_cast<V*>(p.states) + int64_t(v0) * p.stride;
  const int nvalid = min(VB, p.n_states - v0);

  for (uint32_t c = tid; c < nchunks; c += bd) {
    int64_t off = 0;
    for (int j = 0; j < p.n_high; ++j)
      if ((c >> j) & 1u) off |= int64_t(1) << p.hq[j];
    chunkoff[c] = off;
  }
  __syncthreads();

  if (p.init_basis) {
    for (uint32_t e = tid; e < n; e += bd) {
      V z;
      z.x = (base == 0 && e == 0) ? R(1) : R(0);
      z.y = R(0);
#pragma unroll
      for (int b = 0; b < VB; ++b) s[swz(e) * VB + b] = z;
    }
  } else {
    for (uint32_t e = tid; e < n; e += bd) {
      const int64_t g = int64_t(base) + chunkoff[e >> L] + (e & lowmask);
#pragma unroll
      for (int b = 0; b < VB; ++b) {
        V z;
        z.x = R(0);
        z.y = R(0);
        if (b < nvalid) z = st[int64_t(b) * p.stride + g];
        s[swz(e) * VB + b] = z;
      }
    }
  }
  __syncthreads();

  int i = 0;
  while (i < n_ops) {
    const SweepOp& op = ops[i];
    if (op.type == OP_PHASE) {
      int j = i;
      while (j < n_ops && ops[j].type == OP_PHASE) j += (ops[j].slot >= 0) ? 2 : 1;
      apply_phase_run<R, VB>(s, ops, i, j, base, variant0, n, tid, bd);
      __syncthreads();
      i = j;
      continue;
    }
    // register budget: 8 (double) / 16 (float) complex values per thread
    constexpr int kBudget = (std::is_same<R, double>::value ? 8 : 16) * 2 / MINB;
    constexpr int KMAX = (kBudget / VB) >= 16 ? 4 : (kBudget / VB) >= 8 ? 3 : (kBudget / VB) >= 4 ? 2 : 1;
    int left = op.gsize > 0 ? op.gsize : 1;
    while (left > 0) {
      const int k = left < KMAX ? left : KMAX;
      if constexpr (KMAX >= 4) {
        if (k == 4) i = apply_group<R, 4, VB>(s, ops, i, base, variant0, T, tid, bd);
      }
      if constexpr (KMAX >= 3) {
        if (k == 3) i = apply_group<R, 3, VB>(s, ops, i, base, variant0, T, tid, bd);
      }
      if constexpr (KMAX >= 2) {
        if (k == 2) i = apply_group<R, 2, VB>(s, ops, i, base, variant0, T, tid, bd);
      }
      if (k == 1) i = apply_group<R, 1, VB>(s, ops, i, base, variant0, T, tid, bd);
      left -= k;
      if (left > 0) __syncthreads();
    }
    __syncthreads();
  }

  for (uint32_t e = tid; e < n; e += bd) {
    const int64_t g = int64_t(base) + chunkoff[e >> L] + (e & lowmask);
#pragma unroll
    for (int b = 0; b < VB; ++b)
      if (b < nvalid) st[int64_t(b) * p.stride + g] = s[swz(e) * VB + b];
  }
}

// ---------------------------------------------------------------------------
// Register-tile sweep: the same tile geometry as sweep_kernel, but the tile
// lives in registers (2^RB amplitudes per thread). Dense gates on register
// bits run entirely in registers — no shared-memory traffic, no barrier;
// diagonal gates test thread/register masks; a REMAP (two barriers, one
// swizzled shared-memory transpose) brings the next gates' targets into the
// register bits. The host chooses the remaps (plan.cpp: reg_program).
// ---------------------------------------------------------------------------
template <typename R, int RB>
__device__ __forceinline__ void reg_dense(vec2_t<R> (&v)[1 << RB], int k, uint32_t rmask, const double2 (&q)[4]) {
  const double mm[8] = {q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y, q[3].x, q[3].y};
#pragma unroll
  for (int kk = 0; kk < RB; ++kk) {
    if (kk != k) continue;
    if (rmask == 0) {
#pragma unroll
      for (int j = 0; j < (1 << RB); ++j)
        if (!((j >> kk) & 1)) apply2x2<R>(v[j], v[j | (1 << kk)], mm);
    } else {
#pragma unroll
      for (int j = 0; j < (1 << RB); ++j) {
        if ((j >> kk) & 1) continue;
        if ((uint32_t(j) & rmask) != rmask) continue;
        apply2x2<R>(v[j], v[j | (1 << kk)], mm);
      }
    }
  }
}

__device__ __forceinline__ void load_op(const RegOp* ops, int i, uint4& hdr, uint64_t& om, double2 (&mat)[4]) {
  hdr = *reinterpret_cast<const uint4*>(&ops[i]);
  om = ops[i].omask;
  const double2* mp = reinterpret_cast<const double2*>(ops[i].m);
  mat[0] = mp[0];
  mat[1] = mp[1];
  mat[2] = mp[2];
  mat[3] = mp[3];
}

template <typename R, int RB, int CAP>
__global__ void __launch_bounds__(512) rsweep_kernel(const __grid_constant__ RegParamsT<CAP> p) {
  using V = vec2_t<R>;
  constexpr int NR = 1 << RB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* s = reinterpret_cast<V*>(smem_raw);
  const int T = p.tile_bits;
  const int L = p.low_bits;
  const uint32_t n = 1u << T;
  const uint32_t nchunks = 1u << (T - L);
  const uint32_t lowmask = (1u << L) - 1u;
  int64_t* chunkoff = reinterpret_cast<int64_t*>(smem_raw + sizeof(V) * size_t(n));
  RegOp* ops = reinterpret_cast<RegOp*>(smem_raw + ((sizeof(V) * size_t(n) + sizeof(int64_t) * size_t(nchunks) + 15) & ~size_t(15)));
  const uint32_t tid = threadIdx.x;
  const uint32_t bd = blockDim.x;  // = 2^(T - RB)
  const int n_ops = p.n_ops;
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(&p.ops[0]);
    uint64_t* dst = reinterpret_cast<uint64_t*>(ops);
    const uint32_t words = uint32_t(n_ops) * uint32_t(sizeof(RegOp) / 8);
    for (uint32_t w = tid; w < words; w += bd) dst[w] = src[w];
  }
  uint64_t base = 0;
  {
    const uint64_t tile = blockIdx.x;
    for (int j = 0; j < p.n_out; ++j)
      if ((tile >> j) & 1ull) base |= 1ull << p.oq[j];
  }
  const uint64_t variant = p.variant_base + blockIdx.y;
  V* st = reinterpret_cast<V*>(p.states) + int64_t(blockIdx.y) * p.stride;
  for (uint32_t c = tid; c < nchunks; c += bd) {
    int64_t off = 0;
    for (int j = 0; j < p.n_high; ++j)
      if ((c >> j) & 1u) off |= int64_t(1) << p.hq[j];
    chunkoff[c] = off;
  }
  __syncthreads();

  // canonical mapping: register bits = top RB tile bits, so element
  // e = tid + j * bd and consecutive threads touch consecutive addresses
  V v[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const uint32_t e = tid + uint32_t(j) * bd;
    if (p.init_basis) {
      v[j].x = (base == 0 && e == 0) ? R(1) : R(0);
      v[j].y = R(0);
    } else if (e & p.zmask) {
      v[j].x = R(0);
      v[j].y = R(0);
    } else {
      v[j] = st[int64_t(base) + chunkoff[e >> L] + (e & lowmask)];
    }
  }
  // current mapping: thread part of the element index and register offsets
  uint32_t tpart = tid;
  uint32_t roff[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) roff[j] = uint32_t(j) * bd;

  // software-pipelined op loop: the next op's 16-byte header, outside mask and
  // matrix are loaded while the current op computes
  uint4 hdr = make_uint4(0, 0, 0, 0);
  uint64_t om = 0;
  double2 mat[4];
  if (n_ops > 0) load_op(ops, 0, hdr, om, mat);
  for (int i = 0; i < n_ops;) {
    const int kind = int(hdr.x & 0xffu);
    const int slot = int(int16_t(hdr.x >> 16));
    const int next = i + ((kind != ROP_REMAP && slot >= 0) ? 2 : 1);
    uint4 hdr_n = hdr;
    uint64_t om_n = 0;
    double2 mat_n[4];
    // RB = 4 keeps 16 amplitudes live: prefetch only the header there
    constexpr bool kPrefetchMatrix = RB <= 3;
    if (next < n_ops) {
      if (kPrefetchMatrix) {
        load_op(ops, next, hdr_n, om_n, mat_n);
      } else {
        hdr_n = *reinterpret_cast<const uint4*>(&ops[next]);
        om_n = ops[next].omask;
      }
    }
    if (kind == ROP_REMAP) {
      const uint32_t rp = hdr.w;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NR; ++j) s[swz(tpart | roff[j])] = v[j];
      // thread bits fill the non-register tile bits in ascending order:
      // insert a zero at each (ascending) register position
      uint32_t tp = tid;
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const uint32_t pos = (rp >> (8 * k)) & 0xffu;
        const uint32_t below = (1u << pos) - 1u;
        tp = ((tp & ~below) << 1) | (tp & below);
      }
      tpart = tp;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        uint32_t o = 0;
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if ((j >> k) & 1) o |= 1u << ((rp >> (8 * k)) & 0xffu);
        roff[j] = o;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NR; ++j) v[j] = s[swz(tpart | roff[j])];
    } else if ((base & om) == om && (tid & hdr.y) == hdr.y) {
      double2 cur[4] = {mat[0], mat[1], mat[2], mat[3]};
      if (!kPrefetchMatrix) {
        const double2* mp = reinterpret_cast<const double2*>(ops[i].m);
        cur[0] = mp[0];
        cur[1] = mp[1];
        cur[2] = mp[2];
        cur[3] = mp[3];
      }
      if (slot >= 0 && ((variant >> slot) & 1ull)) {
        const double2* mp = reinterpret_cast<const double2*>(ops[i + 1].m);
        cur[0] = mp[0];
        cur[1] = mp[1];
        cur[2] = mp[2];
        cur[3] = mp[3];
      }
      const uint32_t rm = hdr.z;
      if (kind == ROP_DENSE) {
        reg_dense<R, RB>(v, int((hdr.x >> 8) & 0xffu), rm, cur);
      } else {
        const double qr = cur[0].x, qi = cur[0].y;
        if (qi == 0.0 && qr == -1.0) {
#pragma unroll
          for (int j = 0; j < NR; ++j)
            if ((uint32_t(j) & rm) == rm) {
              v[j].x = -v[j].x;
              v[j].y = -v[j].y;
            }
        } else {
#pragma unroll
          for (int j = 0; j < NR; ++j)
            if ((uint32_t(j) & rm) == rm) v[j] = cmul<R>(v[j], R(qr), R(qi));
        }
      }
    }
    hdr = hdr_n;
    om = om_n;
    if (kPrefetchMatrix) {
      mat[0] = mat_n[0];
      mat[1] = mat_n[1];
      mat[2] = mat_n[2];
      mat[3] = mat_n[3];
    }
    i = next;
  }

#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const uint32_t e = tid + uint32_t(j) * bd;
    st[int64_t(base) + chunkoff[e >> L] + (e & lowmask)] = v[j];
  }
}

// ---------------------------------------------------------------------------
// merge_terms: out[s][h][l] (+)= sum_t coef[s,t] * hi[hidx[s,t]][h] * lo[lidx[s,t]][l]
// A CTA owns `iters` row groups x C columns; each thread keeps its CC columns
// of every lo term in registers (read once), the CTA's rows of coef*hi are
// staged in shared memory, and every output amplitude is written exactly once
// with a warp-contiguous 16-byte streaming store — no zero-fill, no
// read-modify-write (the reference zero-fills and then does one RMW pass per
// term, merging.py:117,94).
// ---------------------------------------------------------------------------
template <typename R, int K, int CC, bool WIDE>
__global__ void __launch_bounds__(256, 2) merge_kernel(const __grid_constant__ MergeParams p) {
  using V = vec2_t<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* bs = reinterpret_cast<V*>(smem_raw);
  const int sl = blockIdx.z;
  const int bd = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t W = p.lo_len;
  const int64_t rows_cta = int64_t(p.iters) * p.rows_per_iter;
  const int64_t row0 = p.row_begin + int64_t(blockIdx.y) * rows_cta;
  const int32_t* hidx = p.hidx + sl * K;
  const int32_t* lidx = p.lidx + sl * K;
  const double* coef = p.coef + 2 * sl * K;
  const V* hi = reinterpret_cast<const V*>(p.hi);
  const V* lo = reinterpret_cast<const V*>(p.lo);

  // stage coef * hi for this CTA's rows
  for (int idx = tid; idx < rows_cta * K; idx += bd) {
    const int r = idx / K;
    const int t = idx - r * K;
    const int64_t h = row0 + r;
    V b;
    b.x = R(0);
    b.y = R(0);
    if (h < p.row_end) {
      const V hv = __ldg(hi + int64_t(hidx[t]) * p.hi_len + h);
      b = cmul<R>(hv, R(coef[2 * t]), R(coef[2 * t + 1]));
    }
    bs[idx] = b;
  }

  V a[K][CC];
  int64_t col[CC];
  int rsub[CC];
#pragma unroll
  for (int j = 0; j < CC; ++j) {
    const int flat = tid + j * bd;
    if (WIDE) {
      col[j] = int64_t(blockIdx.x) * (int64_t(bd) * CC) + flat;
      rsub[j] = 0;
    } else {
      col[j] = flat & (p.cols - 1);
      rsub[j] = flat >> p.log_cols;
    }
#pragma unroll
    for (int t = 0; t < K; ++t) a[t][j] = __ldg(lo + int64_t(lidx[t]) * W + col[j]);
  }
  __syncthreads();

  V* out = reinterpret_cast<V*>(p.out) + int64_t(sl) * p.out_slot_stride;
  for (int i = 0; i < p.iters; ++i) {
    if (WIDE) {
      // RR rows at a time share the register-resident lo columns; each output
      // sums its K terms in two interleaved accumulators (even / odd t) so the
      // FP64 dependency chains are K long instead of 2K
      constexpr int RR = K == 8 ? 2 : 1;
      const int r0 = i;
      i += RR - 1;
      V b[RR][K];
#pragma unroll
      for (int rr = 0; rr < RR; ++rr)
#pragma unroll
        for (int t = 0; t < K; ++t) {
          const int r = r0 + rr < rows_cta ? r0 + rr : r0;
          b[rr][t] = bs[r * K + t];
        }
#pragma unroll
      for (int rr = 0; rr < RR; ++rr) {
        const int64_t h = row0 + r0 + rr;
        if (r0 + rr >= p.iters || h >= p.row_end) break;
        const int64_t obase = (h - p.row_begin) * W;
#pragma unroll
        for (int j = 0; j < CC; ++j) {
          V acc0, acc1;
          acc0.x = R(0);
          acc0.y = R(0);
          acc1.x = R(0);
          acc1.y = R(0);
#pragma unroll
          for (int t = 0; t < K; t += 2) {
            cfma<R>(acc0, b[rr][t], a[t][j]);
            if (t + 1 < K) cfma<R>(acc1, b[rr][t + 1], a[t + 1][j]);
          }
          V acc;
          acc.x = acc0.x + acc1.x;
          acc.y = acc0.y + acc1.y;
          V* dst = out + obase + col[j];
          if (p.accumulate) {
            const V prev = *dst;
            acc.x += prev.x;
            acc.y += prev.y;
          }
          if (p.streaming) __stcs(dst, acc);
          else *dst = acc;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < CC; ++j) {
        const int r = i * p.rows_per_iter + rsub[j];
        const int64_t h = row0 + r;
        if (h >= p.row_end) continue;
        V acc;
        acc.x = R(0);
        acc.y = R(0);
#pragma unroll
        for (int t = 0; t < K; ++t) cfma<R>(acc, bs[r * K + t], a[t][j]);
        V* dst = out + (h - p.row_begin) * W + col[j];
        if (p.accumulate) {
          const V prev = *dst;
          acc.x += prev.x;
          acc.y += prev.y;
        }
        if (p.streaming) __stcs(dst, acc);
        else *dst = acc;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// merge_dmma_kernel: the same product for complex128 with K = 8 or 16 terms,
// where 4 FMA per term per amplitude make the DFMA version FP64-issue-bound.
// Written as a real GEMM on the FP64 tensor path (mma.sync m8n8k4 f64):
//   out[h][2l+v] = sum_k Bc[h][k] * Ac[k][2l+v],  k = 2t+u (2K real terms)
//   Bc[h][2t+u]   = (re, im)[u] of coef_t * hi_t[h]   (the staged rows)
//   Ac[2t][2l+v]  = (re, im)[v] of lo_t[l];  Ac[2t+1][2l] = -im, [2l+1] = re
// so an accumulator fragment (row, real cols 2c, 2c+1) is exactly one complex
// output and is stored as one 16-byte evict-first store. Each warp owns 8 rows
// x 4*NT complex columns per row block; its Ac fragments stay in registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KT, int NT>
__global__ void __launch_bounds__(256, 2) merge_dmma_kernel(const __grid_constant__ MergeParams p) {
  constexpr int KR = 2 * KT;          // real inner dimension
  constexpr int KS = KR / 4;          // mma k-steps
  constexpr int RS = KR + 4;          // padded smem row stride (doubles): conflict-free A fragments
  constexpr int COLS_W = 4 * NT;      // complex columns per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* bsd = reinterpret_cast<double*>(smem_raw);
  const int sl = blockIdx.z;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t W = p.lo_len;
  const int rows_cta = p.iters * 8;
  const int64_t row0 = p.row_begin + int64_t(blockIdx.y) * rows_cta;
  const int32_t* hidx = p.hidx + sl * KT;
  const int32_t* lidx = p.lidx + sl * KT;
  const double* coef = p.coef + 2 * sl * KT;
  const double2* hi = reinterpret_cast<const double2*>(p.hi);
  const double2* lo = reinterpret_cast<const double2*>(p.lo);

  constexpr int SU = 8;  // staging loads in flight per thread
  const int nst = rows_cta * KT;
  for (int base = tid; base < nst; base += SU * int(blockDim.x)) {
    double2 hv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int idx = base + u * int(blockDim.x);
      const int r = idx / KT;
      const int64_t h = row0 + r;
      hv[u] = make_double2(0.0, 0.0);
      if (idx < nst && h < p.row_end) hv[u] = __ldg(hi + int64_t(hidx[idx - r * KT]) * p.hi_len + h);
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int idx = base + u * int(blockDim.x);
      if (idx >= nst) break;
      const int r = idx / KT;
      const int t = idx - r * KT;
      const double cr = coef[2 * t], ci = coef[2 * t + 1];
      bsd[r * RS + 2 * t] = hv[u].x * cr - hv[u].y * ci;
      bsd[r * RS + 2 * t + 1] = hv[u].x * ci + hv[u].y * cr;
    }
  }

  __syncthreads();
  double2* out = reinterpret_cast<double2*>(p.out) + int64_t(sl) * p.out_slot_stride;
  const int arow = lane >> 2;
  const int acol = lane & 3;
  // RB row blocks at once: NT * RB independent accumulator chains per warp
  // hide the latency of the dependent m8n8k4 accumulation
  constexpr int RB = 8 / NT;
  // the CTA spans p.cols column groups of COLS_W complex columns; warps take
  // them round-robin and reuse the staged rows for each
  const int ncg = p.cols;
  for (int cg = warp; cg < ncg; cg += nwarps) {
    const int64_t col_w = (int64_t(blockIdx.x) * ncg + cg) * COLS_W;
    // B-operand fragments: lane holds Ac[k = s*4 + (lane&3)][n = lane>>2] of n-tile j
    double bop[NT][KS];
    {
      const int n = lane >> 2;
      const int v = n & 1;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int64_t l = col_w + j * 4 + (n >> 1);
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
          const int k = s2 * 4 + (lane & 3);
          const int t = k >> 1;
          const int u = k & 1;
          const double2 a = __ldg(lo + int64_t(lidx[t]) * W + l);
          bop[j][s2] = u == 0 ? (v == 0 ? a.x : a.y) : (v == 0 ? -a.y : a.x);
        }
      }
    }
    for (int rb0 = 0; rb0 < p.iters; rb0 += RB) {
      double acc[RB][NT][2];
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[r][j][0] = acc[r][j][1] = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const double a = bsd[((rb0 + r) * 8 + arow) * RS + s2 * 4 + acol];
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[r][j][0], acc[r][j][1], a, bop[j][s2]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int64_t h = row0 + (rb0 + r) * 8 + arow;
        if (rb0 + r >= p.iters || h >= p.row_end) continue;
        double2* dst = out + (h - p.row_begin) * W + col_w + acol;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          double2 v = make_double2(acc[r][j][0], acc[r][j][1]);
          if (p.accumulate) {
            const double2 prev = dst[j * 4];
            v.x += prev.x;
            v.y += prev.y;
          }
          if (p.streaming) __stcs(dst + j * 4, v);
          else dst[j * 4] = v;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// merge_dmma3_kernel: the complex product with three real GEMMs instead of
// four (Gauss / "3M"): with B_t = coef_t * hi_t[h] = (br, bi) and
// A_t = lo_t[l] = (ar, ai),
//   P1 = sum_t (br + bi) ar,  P2 = sum_t br (ai - ar),  P3 = sum_t bi (ar + ai)
//   re = P1 - P3,  im = P1 + P2
// so a complex output costs 3K real FMA on the FP64 tensor path instead of 4K
// (the merge is FP64-bound for K >= 16). Each m8n8k4 tile is 8 rows x 8
// complex columns of one of P1..P3; a lane's accumulator pair covers complex
// columns acol and acol + 4 of the tile (whole-sector stores). The three A
// operands per term are staged in shared memory ((br+bi) | br | bi row
// segments, stride 3K+4 doubles: two wavefronts per fragment load), the
// three B operands per column stay in registers for all of the CTA's rows.
// Rounding: |error| <= ~K eps (|br|+|bi|)(|ar|+|ai|) per output, far inside
// the 1e-10 parity bound.
// ---------------------------------------------------------------------------
template <int KT, int NT, int RB, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) merge_dmma3_kernel(const __grid_constant__ MergeParams p) {
  constexpr int KS = KT / 4;       // mma k-steps per GEMM
  constexpr int RS = 3 * KT + 4;   // smem row stride (doubles)
  constexpr int COLS_W = 8 * NT;   // complex columns per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* bsd = reinterpret_cast<double*>(smem_raw);
  const int sl = blockIdx.z;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t W = p.lo_len;
  const int rows_cta = p.iters * 8;
  const int64_t row0 = p.row_begin + int64_t(blockIdx.y) * rows_cta;
  const int32_t* hidx = p.hidx + sl * KT;
  const int32_t* lidx = p.lidx + sl * KT;
  const double* coef = p.coef + 2 * sl * KT;
  const double2* hi = reinterpret_cast<const double2*>(p.hi);
  const double2* lo = reinterpret_cast<const double2*>(p.lo);

  // staging: SU independent loads in flight per thread before any use
  constexpr int SU = 8;
  const int nst = rows_cta * KT;
  for (int base = tid; base < nst; base += SU * int(blockDim.x)) {
    double2 hv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int idx = base + u * int(blockDim.x);
      const int r = idx / KT;
      const int64_t h = row0 + r;
      hv[u] = make_double2(0.0, 0.0);
      if (idx < nst && h < p.row_end) hv[u] = __ldg(hi + int64_t(hidx[idx - r * KT]) * p.hi_len + h);
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int idx = base + u * int(blockDim.x);
      if (idx >= nst) break;
      const int r = idx / KT;
      const int t = idx - r * KT;
      const double cr = coef[2 * t], ci = coef[2 * t + 1];
      const double br = hv[u].x * cr - hv[u].y * ci;
      const double bi = hv[u].x * ci + hv[u].y * cr;
      double* row = bsd + r * RS;
      row[t] = br + bi;
      row[KT + t] = br;
      row[2 * KT + t] = bi;
    }
  }
  __syncthreads();

  double2* out = reinterpret_cast<double2*>(p.out) + int64_t(sl) * p.out_slot_stride;
  const int arow = lane >> 2;
  const int acol = lane & 3;
  const int ncg = p.cols;
  for (int cg = warp; cg < ncg; cg += nwarps) {
    const int64_t col_w = (int64_t(blockIdx.x) * ncg + cg) * COLS_W;
    // B fragments: lane holds X[t = 4s + (lane&3)][n = lane>>2], GEMM column n
    // being complex column (n>>1) + 4(n&1) of the tile, so that a lane's two
    // accumulator columns (n = 2 acol + c) are columns acol and acol + 4 and
    // each store instruction writes 64 contiguous bytes per row (whole sectors)
    double x0[NT][KS], x1[NT][KS], x2[NT][KS];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n = lane >> 2;
      const int64_t l = col_w + 8 * j + (n >> 1) + 4 * (n & 1);
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const double2 a = __ldg(lo + int64_t(lidx[4 * s + acol]) * W + l);
        x0[j][s] = a.x;
        x1[j][s] = a.y - a.x;
        x2[j][s] = a.x + a.y;
      }
    }
    for (int rb0 = 0; rb0 < p.iters; rb0 += RB) {
      double acc[RB][NT][3][2];
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int g = 0; g < 3; ++g) acc[r][j][g][0] = acc[r][j][g][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const double* row = bsd + ((rb0 + r) * 8 + arow) * RS + 4 * s + acol;
          const double a0 = row[0], a1 = row[KT], a2 = row[2 * KT];
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma884(acc[r][j][0][0], acc[r][j][0][1], a0, x0[j][s]);
            dmma884(acc[r][j][1][0], acc[r][j][1][1], a1, x1[j][s]);
            dmma884(acc[r][j][2][0], acc[r][j][2][1], a2, x2[j][s]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int64_t h = row0 + (rb0 + r) * 8 + arow;
        if (rb0 + r >= p.iters || h >= p.row_end) continue;
        double2* dst = out + (h - p.row_begin) * W + col_w + acol;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double p1 = acc[r][j][0][c];
            double2 v = make_double2(p1 - acc[r][j][2][c], p1 + acc[r][j][1][c]);
            double2* d = dst + 8 * j + 4 * c;
            if (p.accumulate) {
              const double2 prev = *d;
              v.x += prev.x;
              v.y += prev.y;
            }
            if (p.streaming) __stcs(d, v);
            else *d = v;
          }
        }
      }
    }
  }
}

template <int KT, int NT, int RB, int WARPS, int MINB = 16 / WARPS>
static cudaError_t launch_dmma3_kt(const MergeParams& p, dim3 grid, size_t smem, cudaStream_t stream) {
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(merge_dmma3_kernel<KT, NT, RB, WARPS, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  merge_dmma3_kernel<KT, NT, RB, WARPS, MINB><<<grid, WARPS * 32, smem, stream>>>(p);
  return cudaGetLastError();
}

// 3M kernel geometry per K: complex columns per warp and row blocks per pass
// (K = 64 keeps 48 B-operand doubles per thread in registers: one CTA per SM)
int merge_dmma3_cols_per_warp(int K) { return K <= 16 ? 16 : 8; }
int merge_dmma3_row_blocks(int K) { return K <= 16 ? 2 : (K == 32 ? 4 : 2); }

// warps = 8 (2 CTAs per SM) or 4 (4 CTAs per SM: staging of one CTA overlaps
// three others' math)
cudaError_t launch_merge_dmma3(const MergeParams& p, int K, int warps, dim3 grid, size_t smem,
                               cudaStream_t stream) {
  if (warps == 4) {
    switch (K) {
      case 8: return launch_dmma3_kt<8, 2, 2, 4>(p, grid, smem, stream);
      case 16: return launch_dmma3_kt<16, 2, 2, 4>(p, grid, smem, stream);
      case 32: return launch_dmma3_kt<32, 1, 4, 4>(p, grid, smem, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (K) {
    case 8: return launch_dmma3_kt<8, 2, 2, 8>(p, grid, smem, stream);
    case 16: return launch_dmma3_kt<16, 2, 2, 8>(p, grid, smem, stream);
    case 32: return launch_dmma3_kt<32, 1, 4, 8>(p, grid, smem, stream);
    case 64: return launch_dmma3_kt<64, 1, 2, 8, 1>(p, grid, smem, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int KT, int NT>
static cudaError_t launch_dmma_kt(const MergeParams& p, dim3 grid, int threads, size_t smem, cudaStream_t stream) {
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(merge_dmma_kernel<KT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  merge_dmma_kernel<KT, NT><<<grid, threads, smem, stream>>>(p);
  return cudaGetLastError();
}

// complex columns per warp for each instantiated K (register budget of the
// B-operand fragments: NT * K / 2 doubles per thread)
int merge_dmma_cols_per_warp(int K) { return K <= 16 ? 16 : (K == 32 ? 8 : 4); }

cudaError_t launch_merge_dmma(const MergeParams& p, int K, dim3 grid, int threads, size_t smem,
                              cudaStream_t stream) {
  switch (K) {
    case 8: return launch_dmma_kt<8, 4>(p, grid, threads, smem, stream);
    case 16: return launch_dmma_kt<16, 4>(p, grid, threads, smem, stream);
    case 32: return launch_dmma_kt<32, 2>(p, grid, threads, smem, stream);
    case 64: return launch_dmma_kt<64, 1>(p, grid, threads, smem, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// small utilities
// ---------------------------------------------------------------------------
template <typename R>
__global__ void init_basis_kernel(vec2_t<R>* states, int64_t len, int64_t n_states, int64_t index) {
  const int64_t total = len * n_states;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    vec2_t<R> z;
    z.x = ((i % len) == index) ? R(1) : R(0);
    z.y = R(0);
    states[i] = z;
  }
}

// Deterministic two-pass reductions: per-block partials, then one block.
// mode 0: max |a - b|; mode 1: sum conj(a) * b (re, im); mode 2: max |a|
template <typename R>
__global__ void reduce_pass1(const vec2_t<R>* a, const vec2_t<R>* b, int64_t n, int mode,
                             double2* partial) {
  __shared__ double sx[256], sy[256];
  double x = 0.0, y = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double ar = a[i].x, ai = a[i].y;
    if (mode == 0) {
      const double dr = ar - double(b[i].x), di = ai - double(b[i].y);
      x = fmax(x, sqrt(dr * dr + di * di));
    } else if (mode == 1) {
      const double br = b[i].x, bi = b[i].y;
      x += ar * br + ai * bi;
      y += ar * bi - ai * br;
    } else {
      x = fmax(x, sqrt(ar * ar + ai * ai));
    }
  }
  sx[threadIdx.x] = x;
  sy[threadIdx.x] = y;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      if (mode == 1) {
        sx[threadIdx.x] += sx[threadIdx.x + w];
        sy[threadIdx.x] += sy[threadIdx.x + w];
      } else {
        sx[threadIdx.x] = fmax(sx[threadIdx.x], sx[threadIdx.x + w]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(sx[0], sy[0]);
}

__global__ void reduce_pass2(const double2* partial, int n, int mode, double2* result) {
  __shared__ double sx[256], sy[256];
  double x = 0.0, y = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (mode == 1) {
      x += partial[i].x;
      y += partial[i].y;
    } else {
      x = fmax(x, partial[i].x);
    }
  }
  sx[threadIdx.x] = x;
  sy[threadIdx.x] = y;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      if (mode == 1) {
        sx[threadIdx.x] += sx[threadIdx.x + w];
        sy[threadIdx.x] += sy[threadIdx.x + w];
      } else {
        sx[threadIdx.x] = fmax(sx[threadIdx.x], sx[threadIdx.x + w]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *result = make_double2(sx[0], sy[0]);
}

template <typename R>
__global__ void gather_kernel(const vec2_t<R>* state, const int64_t* idx, int64_t m, vec2_t<R>* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = state[idx[i]];
}

// ---------------------------------------------------------------------------
// launchers (host)
// ---------------------------------------------------------------------------
size_t sweep_smem_bytes(int tile_bits, int low_bits, int dtype, int n_ops, int vb) {
  const size_t elem = dtype == 0 ? sizeof(double2) : sizeof(float2);
  return (size_t(1) << tile_bits) * elem * size_t(vb) + (size_t(1) << (tile_bits - low_bits)) * sizeof(int64_t) +
         size_t(n_ops) * sizeof(SweepOp);
}

template <typename R, int CAP, int VB, int MINB>
static cudaError_t launch_sweep_cap(const SweepParamsT<CAP>& p, uint32_t n_tiles, uint32_t n_groups, int threads,
                                    size_t smem, cudaStream_t stream) {
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<R, CAP, VB, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid(n_tiles, n_groups, 1);
  sweep_kernel<R, CAP, VB, MINB><<<grid, threads, smem, stream>>>(p);
  return cudaGetLastError();
}

int g_sweep_minb = 2;  // CTAs per SM the big-grid (uncut) sweep kernel is compiled for

template <typename R, int CAP>
static cudaError_t launch_sweep_vb(const SweepParamsT<CAP>& p, uint32_t n_tiles, int vb, int threads,
                                   cudaStream_t stream) {
  const int dt = std::is_same<R, double>::value ? 0 : 1;
  const size_t smem = sweep_smem_bytes(p.tile_bits, p.low_bits, dt, p.n_ops, vb);
  const uint32_t groups = uint32_t((p.n_states + vb - 1) / vb);
  switch (vb) {
    case 4: return launch_sweep_cap<R, CAP, 4, 2>(p, n_tiles, groups, threads, smem, stream);
    case 2: return launch_sweep_cap<R, CAP, 2, 2>(p, n_tiles, groups, threads, smem, stream);
    default:
      if (g_sweep_minb >= 4) return launch_sweep_cap<R, CAP, 1, 4>(p, n_tiles, groups, threads, smem, stream);
      if (g_sweep_minb == 3) return launch_sweep_cap<R, CAP, 1, 3>(p, n_tiles, groups, threads, smem, stream);
      return launch_sweep_cap<R, CAP, 1, 2>(p, n_tiles, groups, threads, smem, stream);
  }
}

template <typename R>
static cudaError_t launch_sweep_t(const SweepParams& p, uint32_t n_tiles, int vb, int threads, cudaStream_t stream) {
  if (p.n_ops <= kSmallOps) {
    static SweepParamsSmall ps;  // launch copies it; callers hold capi's lock
    std::memcpy(&ps, &p, offsetof(SweepParams, ops));
    std::memcpy(ps.ops, p.ops, sizeof(SweepOp) * size_t(p.n_ops));
    return launch_sweep_vb<R, kSmallOps>(ps, n_tiles, vb, threads, stream);
  }
  return launch_sweep_vb<R, kMaxOpsPerLaunch>(p, n_tiles, vb, threads, stream);
}

cudaError_t launch_sweep(const SweepParams& p, uint32_t n_tiles, int vb, int threads, cudaStream_t stream,
                         int dtype) {
  return dtype == 0 ? launch_sweep_t<double>(p, n_tiles, vb, threads, stream)
                    : launch_sweep_t<float>(p, n_tiles, vb, threads, stream);
}

size_t rsweep_smem_bytes(int tile_bits, int low_bits, int dtype, int n_ops) {
  const size_t elem = dtype == 0 ? sizeof(double2) : sizeof(float2);
  const size_t head = (size_t(1) << tile_bits) * elem + (size_t(1) << (tile_bits - low_bits)) * sizeof(int64_t);
  return ((head + 15) & ~size_t(15)) + size_t(n_ops) * sizeof(RegOp);
}

template <typename R, int RB, int CAP>
static cudaError_t launch_rsweep_rb(const RegParamsT<CAP>& p, uint32_t n_tiles, uint32_t n_states,
                                    cudaStream_t stream) {
  const int dt = std::is_same<R, double>::value ? 0 : 1;
  const size_t smem = rsweep_smem_bytes(p.tile_bits, p.low_bits, dt, p.n_ops);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(rsweep_kernel<R, RB, CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int threads = 1 << (p.tile_bits - RB);
  dim3 grid(n_tiles, n_states, 1);
  rsweep_kernel<R, RB, CAP><<<grid, threads, smem, stream>>>(p);
  return cudaGetLastError();
}

template <typename R, int CAP>
static cudaError_t launch_rsweep_cap(const RegParamsT<CAP>& p, int rb, uint32_t n_tiles, uint32_t n_states,
                                     cudaStream_t stream) {
  switch (rb) {
    case 1: return launch_rsweep_rb<R, 1, CAP>(p, n_tiles, n_states, stream);
    case 2: return launch_rsweep_rb<R, 2, CAP>(p, n_tiles, n_states, stream);
    case 3: return launch_rsweep_rb<R, 3, CAP>(p, n_tiles, n_states, stream);
    default: return launch_rsweep_rb<R, 4, CAP>(p, n_tiles, n_states, stream);
  }
}

// The launch copies the whole parameter block, so its host cost grows with
// the capacity (32 KiB at kMaxRegOps: ~15 us more per launch than 4 KiB,
// tools/sub_host_split.py): launch through the smallest capacity tier that
// holds the program.
template <typename R, int CAP>
static cudaError_t launch_rsweep_tier(const RegParams& p, int rb, uint32_t n_tiles, uint32_t n_states,
                                      cudaStream_t stream) {
  static RegParamsT<CAP> ps;  // launch copies it; callers hold capi's lock
  std::memcpy(&ps, &p, offsetof(RegParams, ops));
  std::memcpy(ps.ops, p.ops, sizeof(RegOp) * size_t(p.n_ops));
  return launch_rsweep_cap<R, CAP>(ps, rb, n_tiles, n_states, stream);
}

template <typename R>
static cudaError_t launch_rsweep_t(const RegParams& p, int rb, uint32_t n_tiles, uint32_t n_states,
                                   cudaStream_t stream) {
  if (p.n_ops <= kSmallOps) return launch_rsweep_tier<R, kSmallOps>(p, rb, n_tiles, n_states, stream);
  if (p.n_ops <= kMidRegOps) return launch_rsweep_tier<R, kMidRegOps>(p, rb, n_tiles, n_states, stream);
  if (p.n_ops <= kLargeRegOps) return launch_rsweep_tier<R, kLargeRegOps>(p, rb, n_tiles, n_states, stream);
  return launch_rsweep_cap<R, kMaxRegOps>(p, rb, n_tiles, n_states, stream);
}

cudaError_t launch_rsweep(const RegParams& p, int rb, uint32_t n_tiles, uint32_t n_states, cudaStream_t stream,
                          int dtype) {
  return dtype == 0 ? launch_rsweep_t<double>(p, rb, n_tiles, n_states, stream)
                    : launch_rsweep_t<float>(p, rb, n_tiles, n_states, stream);
}

template <typename R, int K, int CC>
static cudaError_t launch_merge_kc(const MergeParams& p, dim3 grid, int threads, size_t smem,
                                   bool wide, cudaStream_t stream) {
  if (wide) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(merge_kernel<R, K, CC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem));
    merge_kernel<R, K, CC, true><<<grid, threads, smem, stream>>>(p);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(merge_kernel<R, K, CC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(smem));
    merge_kernel<R, K, CC, false><<<grid, threads, smem, stream>>>(p);
  }
  return cudaGetLastError();
}

int merge_cols_per_thread(int K) { return K <= 4 ? 4 : (K == 8 ? 2 : 1); }

template <typename R>
static cudaError_t launch_merge_t(const MergeParams& p, int K, dim3 grid, int threads, size_t smem,
                                  bool wide, cudaStream_t stream) {
  switch (K) {
    case 1: return launch_merge_kc<R, 1, 4>(p, grid, threads, smem, wide, stream);
    case 2: return launch_merge_kc<R, 2, 4>(p, grid, threads, smem, wide, stream);
    case 4: return launch_merge_kc<R, 4, 4>(p, grid, threads, smem, wide, stream);
    case 8: return launch_merge_kc<R, 8, 2>(p, grid, threads, smem, wide, stream);
    case 16: return launch_merge_kc<R, 16, 1>(p, grid, threads, smem, wide, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_merge(const MergeParams& p, int K, dim3 grid, int threads, size_t smem, bool wide,
                         cudaStream_t stream, int dtype) {
  return dtype == 0 ? launch_merge_t<double>(p, K, grid, threads, smem, wide, stream)
                    : launch_merge_t<float>(p, K, grid, threads, smem, wide, stream);
}

cudaError_t launch_init_basis(void* states, int64_t len, int64_t n_states, int64_t index, int dtype,
                              cudaStream_t stream) {
  const int64_t total = len * n_states;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  if (dtype == 0)
    init_basis_kernel<double><<<unsigned(blocks), 256, 0, stream>>>(static_cast<double2*>(states), len,
                                                                    n_states, index);
  else
    init_basis_kernel<float><<<unsigned(blocks), 256, 0, stream>>>(static_cast<float2*>(states), len,
                                                                   n_states, index);
  return cudaGetLastError();
}

constexpr int kReduceBlocks = 148 * 4;

cudaError_t launch_reduce(const void* a, const void* b, int64_t n, int mode, int dtype, double2* scratch,
                          cudaStream_t stream) {
  // scratch: kReduceBlocks partials followed by one result
  if (dtype == 0)
    reduce_pass1<double><<<kReduceBlocks, 256, 0, stream>>>(static_cast<const double2*>(a),
                                                            static_cast<const double2*>(b), n, mode,
                                                            scratch);
  else
    reduce_pass1<float><<<kReduceBlocks, 256, 0, stream>>>(static_cast<const float2*>(a),
                                                           static_cast<const float2*>(b), n, mode,
                                                           scratch);
  reduce_pass2<<<1, 256, 0, stream>>>(scratch, kReduceBlocks, mode, scratch + kReduceBlocks);
  return cudaGetLastError();
}

int reduce_scratch_elems() { return kReduceBlocks + 1; }

cudaError_t launch_gather(const void* state, const int64_t* idx, int64_t m, void* out, int dtype,
                          cudaStream_t stream) {
  int64_t blocks = (m + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  if (dtype == 0)
    gather_kernel<double><<<unsigned(blocks), 256, 0, stream>>>(static_cast<const double2*>(state), idx, m,
                                                                static_cast<double2*>(out));
  else
    gather_kernel<float><<<unsigned(blocks), 256, 0, stream>>>(static_cast<const float2*>(state), idx, m,
                                                               static_cast<float2*>(out));
  return cudaGetLastError();
}

}  // namespace cutsim
