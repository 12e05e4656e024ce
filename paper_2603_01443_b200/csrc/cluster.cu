// Cluster-resident variant batches, compiled ahead of time (sm_100a).
//
// The subcircuit variant stage (reference engine.py:122-139 run once per
// variant by harness.py:136-139) simulates a batch of 2^12..2^16-amplitude
// states. Each state lives in the shared memory of one thread-block cluster
// (CTA r holds amplitudes [r 2^T, (r+1) 2^T)), 2^RB amplitudes per thread in
// registers, and the schedule's sweeps are phases separated by one cluster
// barrier (DSMEM exchange), as in the NVRTC form (jit.cpp
// jit_cluster_source). The NVRTC form bakes the register program into
// straight-line code: ~7000 instructions (109 KB) that every warp executes
// once, and ncu puts its warps on "no instruction" more than on anything
// else (profiles/x02_cluster_variant_cfg4a_ncu_full.json: 3.7 stall cycles
// per issue, issue active 20 %). Here the program is DATA — an 8-byte op
// stream plus coefficient sets read through the L1 — and the loop body is a
// few KB of code specialised per register bit, so the instruction stream
// stays resident and the FP64 pipe, not the fetch, sets the pace. One
// compiled kernel serves every circuit: no NVRTC compile on the cold path.
//
// Op semantics are those of rsweep_kernel (kernels.cu) / the NVRTC
// emitter: DENSE on register bit k (pairs j, j | 2^k whose register index
// has all rmask bits), PHASE / NEG on registers with all rmask bits, each
// gated by (base & omask) == omask && (tid & tmask) == tmask; REMAP is the
// swizzled shared-memory transpose; a slotted op takes its alternative
// coefficients when bit `slot` of the variant id is set.
#include "cluster.hpp"

#include <atomic>
#include <cstring>
#include <type_traits>

namespace cutsim {

namespace {

template <typename R>
using vec2_t = typename std::conditional<std::is_same<R, double>::value, double2, float2>::type;

enum : uint32_t { CK_DENSE_U = 0, CK_DENSE_G = 1, CK_PHASE = 2, CK_NEG = 3, CK_REMAP = 4, CK_NEXT = 5, CK_END = 6 };

// a: kind (3 bits) | k << 3 (2) | rmask << 5 (4) | (slot + 1) << 9 (7) | set << 16 (16)
// b: DENSE/PHASE/NEG: tmask (16) | omask << 16 (16); REMAP: rpos[k] in byte k;
//    NEXT: the next phase
struct CpOp {
  uint32_t a, b;
};
static_assert(sizeof(CpOp) == 8, "CpOp layout");
constexpr int kPhaseRec = 32;  // pos[16] (tile bit -> qubit), oq[8] (cluster rank bit -> qubit), n_oq

__device__ __forceinline__ uint32_t swz(uint32_t e) {
  uint32_t x = e >> 3;
  x ^= (x >> 3) ^ (x >> 6) ^ (x >> 9);
  return e ^ (x & 7u);
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

__device__ __forceinline__ void st_dsm(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_dsm(uint32_t a, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void ld_dsm(uint32_t a, double2& v) {
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void ld_dsm(uint32_t a, float2& v) {
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
}

// unit-diagonal 2x2 (the normalised form of plan.cpp normalize_dense):
// [[1, c0], [c1, 1]]; same expression order as the NVRTC emitter
template <typename V, int NR, int K>
__device__ __forceinline__ void dense_u(V (&v)[NR], uint32_t rm, V c0, V c1) {
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if ((j >> K) & 1) continue;
    if ((uint32_t(j) & rm) != rm) continue;
    const int jb = j | (1 << K);
    const V a = v[j], b = v[jb];
    v[j].x = a.x + c0.x * b.x - c0.y * b.y;
    v[j].y = a.y + c0.x * b.y + c0.y * b.x;
    v[jb].x = b.x + c1.x * a.x - c1.y * a.y;
    v[jb].y = b.y + c1.x * a.y + c1.y * a.x;
  }
}

// general 2x2 [[c0, c1], [c2, c3]]
template <typename V, int NR, int K>
__device__ __forceinline__ void dense_g(V (&v)[NR], uint32_t rm, const V (&c)[4]) {
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if ((j >> K) & 1) continue;
    if ((uint32_t(j) & rm) != rm) continue;
    const int jb = j | (1 << K);
    const V a = v[j], b = v[jb];
    V u, w;
    u.x = c[0].x * a.x - c[0].y * a.y + c[1].x * b.x - c[1].y * b.y;
    u.y = c[0].x * a.y + c[0].y * a.x + c[1].x * b.y + c[1].y * b.x;
    w.x = c[2].x * a.x - c[2].y * a.y + c[3].x * b.x - c[3].y * b.y;
    w.y = c[2].x * a.y + c[2].y * a.x + c[3].x * b.y + c[3].y * b.x;
    v[j] = u;
    v[jb] = w;
  }
}

// The packed program travels in the kernel-parameter block (constant bank:
// uniform LDC loads with a register offset, no upload, no device state);
// three capacities keep the per-launch parameter copy small.
template <int CAP>
struct alignas(16) ClusterParams {
  uint32_t ops_off, coef_off;
  int32_t T, pad;
  unsigned char data[CAP];
};
constexpr int kCaps[3] = {4096, 12288, 32000};

template <typename R, int RB, int CAP>
__global__ void __launch_bounds__(256, 1)
    cluster_prog_kernel(vec2_t<R>* __restrict__ states, long long stride, unsigned long long vbase,
                        const __grid_constant__ ClusterParams<CAP> P) {
  using V = vec2_t<R>;
  const unsigned char* prog = P.data;
  const int T = P.T;
  const uint32_t ops_off = P.ops_off, coef_off = P.coef_off;
  constexpr int NR = 1 << RB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* chunk = reinterpret_cast<V*>(smem_raw);
  V* sm = chunk + (1u << T);
  const uint32_t tid = threadIdx.x;
  const uint32_t bd = blockDim.x;  // 2^(T - RB)
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const CpOp* ops = reinterpret_cast<const CpOp*>(prog + ops_off);
  const V* cf = reinterpret_cast<const V*>(prog + coef_off);  // coefficient sets, in V units
  const uint64_t variant = vbase + blockIdx.y;
  V* st = states + (long long)blockIdx.y * stride;
  const uint32_t csa = static_cast<uint32_t>(__cvta_generic_to_shared(chunk));
  const uint32_t chunk_mask = (1u << T) - 1u;

  // phase geometry: global index of register j = base | dep_tid | sum_k bit_k(j) M[k]
  uint32_t base = 0, dep_tid = 0, M[RB];
  auto geometry = [&](uint32_t ph) {
    const unsigned char* g = prog + size_t(ph) * kPhaseRec;
    base = 0;
    const int n_oq = g[24];
    for (int j = 0; j < n_oq; ++j)
      if ((rank >> j) & 1u) base |= 1u << g[16 + j];
    dep_tid = 0;
    for (int p = 0; p < T - RB; ++p)
      if ((tid >> p) & 1u) dep_tid |= 1u << g[p];
#pragma unroll
    for (int k = 0; k < RB; ++k) M[k] = 1u << g[T - RB + k];
  };
  auto gidx = [&](int j) {
    uint32_t x = base | dep_tid;
#pragma unroll
    for (int k = 0; k < RB; ++k)
      if ((j >> k) & 1) x |= M[k];
    return x;
  };

  geometry(0);
  V v[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    v[j].x = gidx(j) == 0u ? R(1) : R(0);
    v[j].y = R(0);
  }
  uint32_t tpart = tid;
  uint32_t roff[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) roff[j] = uint32_t(j) * bd;
  // every CTA of the cluster runs before any DSMEM access
  cluster_sync();

  // a set holds 1 (PHASE), 2 (DENSE_U) or 4 (DENSE_G) complex coefficients;
  // a slotted op's alternative set follows its own; the first two are
  // prefetched, DENSE_G (rare) loads the other two when it runs
  auto set_of = [&](CpOp d) {
    uint32_t set = d.a >> 16;
    const int slot = int((d.a >> 9) & 127u) - 1;
    const uint32_t kind = d.a & 7u;
    if (slot >= 0 && ((variant >> slot) & 1ull)) set += kind == CK_DENSE_G ? 4u : (kind == CK_DENSE_U ? 2u : 1u);
    return set;
  };
  auto coef = [&](CpOp d, V (&c)[2]) {
    const V* p = cf + set_of(d);
    c[0] = p[0];
    c[1] = p[1];
  };
  auto ldop = [&](int i) { return ops[i]; };

  // software pipeline: op i+1's coefficients and op i+2's header load while
  // op i computes (the stream ends in two END ops, so the reads stay in range)
  CpOp d = ldop(0), dn = ldop(1);
  V c[2];
  coef(d, c);
  for (int i = 0;; ++i) {
    const uint32_t kind = d.a & 7u;
    if (kind == CK_END) break;
    const CpOp dnn = ldop(i + 2);
    V cn[2];
    coef(dn, cn);
    if (kind <= CK_NEG) {
      const uint32_t tm = d.b & 0xffffu, om = d.b >> 16;
      if ((base & om) == om && (tid & tm) == tm) {
        const uint32_t rm = (d.a >> 5) & 15u;
        const int k = int((d.a >> 3) & 3u);
        if (kind == CK_DENSE_U) {
          if (k == 0) dense_u<V, NR, 0>(v, rm, c[0], c[1]);
          else if (k == 1) dense_u<V, NR, 1>(v, rm, c[0], c[1]);
          else if (RB > 2 && k == 2) dense_u<V, NR, (RB > 2 ? 2 : 0)>(v, rm, c[0], c[1]);
          else if (RB > 3) dense_u<V, NR, (RB > 3 ? 3 : 0)>(v, rm, c[0], c[1]);
        } else if (kind == CK_DENSE_G) {
          const V* p = cf + set_of(d);
          const V cg[4] = {c[0], c[1], p[2], p[3]};
          if (k == 0) dense_g<V, NR, 0>(v, rm, cg);
          else if (k == 1) dense_g<V, NR, 1>(v, rm, cg);
          else if (RB > 2 && k == 2) dense_g<V, NR, (RB > 2 ? 2 : 0)>(v, rm, cg);
          else if (RB > 3) dense_g<V, NR, (RB > 3 ? 3 : 0)>(v, rm, cg);
        } else if (kind == CK_PHASE) {
          const R pr = c[0].x, pi = c[0].y;
#pragma unroll
          for (int j = 0; j < NR; ++j)
            if ((uint32_t(j) & rm) == rm) {
              const R x = v[j].x * pr - v[j].y * pi;
              v[j].y = v[j].x * pi + v[j].y * pr;
              v[j].x = x;
            }
        } else {
#pragma unroll
          for (int j = 0; j < NR; ++j)
            if ((uint32_t(j) & rm) == rm) {
              v[j].x = -v[j].x;
              v[j].y = -v[j].y;
            }
        }
      }
    } else if (kind == CK_REMAP) {
      const uint32_t rp = d.b;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NR; ++j) sm[swz(tpart | roff[j])] = v[j];
      // thread bits fill the non-register tile bits in ascending order
      uint32_t tp = tid;
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const uint32_t below = (1u << ((rp >> (8 * k)) & 0xffu)) - 1u;
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
      for (int j = 0; j < NR; ++j) v[j] = sm[swz(tpart | roff[j])];
    } else {  // CK_NEXT: hand the state to the next phase's tiling through DSMEM
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const uint32_t g = gidx(j);
        st_dsm(mapa(csa + (g & chunk_mask) * uint32_t(sizeof(V)), g >> T), v[j]);
      }
      cluster_sync();
      geometry(d.b);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const uint32_t g = gidx(j);
        ld_dsm(mapa(csa + (g & chunk_mask) * uint32_t(sizeof(V)), g >> T), v[j]);
      }
      tpart = tid;
#pragma unroll
      for (int j = 0; j < NR; ++j) roff[j] = uint32_t(j) * bd;
    }
    d = dn;
    dn = dnn;
    c[0] = cn[0];
    c[1] = cn[1];
  }
  // the last phase writes the state (canonical index order) to global memory
#pragma unroll
  for (int j = 0; j < NR; ++j) st[gidx(j)] = v[j];
  // no CTA leaves while another may still read its chunk
  cluster_sync();
}

template <typename R, int RB, int CAP>
cudaError_t launch_cap(const ClusterBlob& b, void* states, int64_t stride, uint64_t vbase, uint32_t n_states,
                       cudaStream_t st) {
  using V = vec2_t<R>;
  auto kern = cluster_prog_kernel<R, RB, CAP>;
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(configured.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 16);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  // the launch copies the parameter block; callers serialise (capi's lock)
  static ClusterParams<CAP> P;
  P.ops_off = b.ops_off;
  P.coef_off = b.coef_off;
  P.T = b.T;
  P.pad = 0;
  std::memcpy(P.data, b.bytes.data(), b.bytes.size());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(b.cluster), n_states, 1);
  cfg.blockDim = dim3(1u << (b.T - b.RB), 1, 1);
  cfg.dynamicSmemBytes = 2 * (size_t(1) << b.T) * sizeof(V);  // canonical chunk + transpose scratch
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(b.cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<V*>(states), (long long)stride, (unsigned long long)vbase, P);
}

template <typename R, int RB>
cudaError_t launch_rb(const ClusterBlob& b, void* states, int64_t stride, uint64_t vbase, uint32_t n_states,
                      cudaStream_t st) {
  const size_t n = b.bytes.size();
  if (n <= size_t(kCaps[0])) return launch_cap<R, RB, kCaps[0]>(b, states, stride, vbase, n_states, st);
  if (n <= size_t(kCaps[1])) return launch_cap<R, RB, kCaps[1]>(b, states, stride, vbase, n_states, st);
  if (n <= size_t(kCaps[2])) return launch_cap<R, RB, kCaps[2]>(b, states, stride, vbase, n_states, st);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_cluster_prog(const ClusterBlob& b, void* states, int64_t stride, uint64_t vbase,
                                uint32_t n_states, cudaStream_t st) {
  if (b.dtype == 0) {
    switch (b.RB) {
      case 2: return launch_rb<double, 2>(b, states, stride, vbase, n_states, st);
      case 3: return launch_rb<double, 3>(b, states, stride, vbase, n_states, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (b.RB) {
    case 2: return launch_rb<float, 2>(b, states, stride, vbase, n_states, st);
    case 3: return launch_rb<float, 3>(b, states, stride, vbase, n_states, st);
    case 4: return launch_rb<float, 4>(b, states, stride, vbase, n_states, st);
    default: return cudaErrorInvalidValue;
  }
}

bool cluster_blob_build(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
                        int T, int dtype, ClusterBlob* out, std::string* err) {
  const int RB = reg_bits_for(T);
  const size_t P = sweeps.size();
  auto bad = [&](const char* why) {
    *err = why;
    return false;
  };
  if (P == 0 || progs.size() != P) return bad("empty program");
  if (RB < 2 || RB > (dtype == 0 ? 3 : 4) || T > 12 || T - RB > 8) return bad("tile geometry not instantiated");
  std::vector<unsigned char> tab(P * kPhaseRec, 0);
  const size_t n_oq = sweeps[0]->oq.size();
  if (n_oq == 0 || n_oq > 4) return bad("cluster size");
  for (size_t ph = 0; ph < P; ++ph) {
    const Sweep& sw = *sweeps[ph];
    if (sw.tile_bits != T || sw.oq.size() != n_oq || int(sw.hq.size()) != T - sw.low_bits)
      return bad("phase geometry");
    unsigned char* g = &tab[ph * kPhaseRec];
    for (int p = 0; p < T; ++p) {
      const int q = p < sw.low_bits ? p : sw.hq[size_t(p - sw.low_bits)];
      if (q < 0 || q > 15) return bad("qubit index");
      g[p] = static_cast<unsigned char>(q);
    }
    for (size_t j = 0; j < n_oq; ++j) {
      if (sw.oq[j] < 0 || sw.oq[j] > 15) return bad("qubit index");
      g[16 + j] = static_cast<unsigned char>(sw.oq[j]);
    }
    g[24] = static_cast<unsigned char>(n_oq);
  }
  std::vector<CpOp> ops;
  std::vector<double> coef;  // (re, im) pairs: one V each
  auto push_set = [&](const double* m, int kind) {
    if (kind == CK_DENSE_U) coef.insert(coef.end(), m + 2, m + 6);
    else if (kind == CK_DENSE_G) coef.insert(coef.end(), m, m + 8);
    else coef.insert(coef.end(), m, m + 2);
  };
  auto unit = [](const RegOp& o) { return o.m[0] == 1.0 && o.m[1] == 0.0 && o.m[6] == 1.0 && o.m[7] == 0.0; };
  for (size_t ph = 0; ph < P; ++ph) {
    const std::vector<RegOp>& prog = *progs[ph];
    for (size_t i = 0; i < prog.size();) {
      const RegOp& op = prog[i];
      if (op.kind == ROP_REMAP) {
        uint32_t b = 0;
        for (int k = 0; k < RB; ++k) b |= uint32_t(op.rpos[k]) << (8 * k);
        ops.push_back(CpOp{CK_REMAP, b});
        ++i;
        continue;
      }
      const bool slotted = op.slot >= 0;
      if (slotted && i + 1 >= prog.size()) return bad("slotted op without its alternative");
      const RegOp* alt = slotted ? &prog[i + 1] : nullptr;
      uint32_t kind;
      if (op.kind == ROP_DENSE) {
        kind = (unit(op) && (!alt || unit(*alt))) ? CK_DENSE_U : CK_DENSE_G;
        if (op.k >= RB) return bad("register bit");
      } else {
        kind = (!slotted && op.m[0] == -1.0 && op.m[1] == 0.0) ? CK_NEG : CK_PHASE;
      }
      if (op.rmask >> RB || op.tmask >> 16 || op.omask >> 16 || op.slot > 125) return bad("mask range");
      const size_t set = coef.size() / 2;
      if (set + 8 > 65535) return bad("too many coefficients");
      push_set(op.m, int(kind));
      if (alt) push_set(alt->m, int(kind));
      const uint32_t a = kind | (uint32_t(op.k) << 3) | (op.rmask << 5) | (uint32_t(op.slot + 1) << 9) |
                         (uint32_t(set) << 16);
      ops.push_back(CpOp{a, op.tmask | uint32_t(op.omask << 16)});
      i += slotted ? 2 : 1;
    }
    ops.push_back(ph + 1 < P ? CpOp{CK_NEXT, uint32_t(ph + 1)} : CpOp{CK_END, 0});
  }
  ops.push_back(CpOp{CK_END, 0});
  ops.push_back(CpOp{CK_END, 0});
  coef.insert(coef.end(), 8, 0.0);  // the prefetch of the stream's END ops and DENSE_G's tail stay in range
  const size_t eb = dtype == 0 ? 8 : 4;
  const size_t ops_off = tab.size();
  const size_t coef_off = (ops_off + ops.size() * sizeof(CpOp) + 15) & ~size_t(15);
  out->bytes.assign(coef_off + coef.size() * eb, 0);
  std::memcpy(out->bytes.data(), tab.data(), tab.size());
  std::memcpy(out->bytes.data() + ops_off, ops.data(), ops.size() * sizeof(CpOp));
  if (dtype == 0) {
    std::memcpy(out->bytes.data() + coef_off, coef.data(), coef.size() * 8);
  } else {
    std::vector<float> f(coef.begin(), coef.end());
    std::memcpy(out->bytes.data() + coef_off, f.data(), f.size() * 4);
  }
  out->ops_off = uint32_t(ops_off);
  out->coef_off = uint32_t(coef_off);
  out->T = T;
  out->RB = RB;
  out->cluster = 1 << int(n_oq);
  out->dtype = dtype;
  out->n_ops = int64_t(ops.size());
  if (out->bytes.size() > size_t(kCaps[2])) return bad("program exceeds the kernel-parameter block");
  return true;
}

}  // namespace cutsim
