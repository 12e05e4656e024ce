// NVRTC specialisation of register-tile sweep programs.
//
// The interpreter kernel (rsweep_kernel) spends ~90 of ~120 instructions per
// gate on decoding the op record, branching on its masks and moving the
// matrix into registers; the 32 FP64 instructions of a 2-pair update are the
// minority. Here each launch of a (hot) program is emitted as straight-line
// CUDA with the tile geometry, masks, remap index maps and matrices baked in
// as literals, compiled once to an sm_100a CUBIN with NVRTC and loaded with
// cudaLibraryLoadData. Semantics are identical to rsweep_kernel (same
// register mapping, same swizzled transposes, same canonical load/store).
#include "jit.hpp"

#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <functional>
#include <thread>
#include <unordered_map>
#include <cstring>

namespace cutsim {

namespace {

struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
};

Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      r.why = "libnvrtc.so.12 not found";
      return r;
    }
    r.create = reinterpret_cast<decltype(r.create)>(dlsym(h, "nvrtcCreateProgram"));
    r.compile = reinterpret_cast<decltype(r.compile)>(dlsym(h, "nvrtcCompileProgram"));
    r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    r.cubin = reinterpret_cast<decltype(r.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    r.log_size = reinterpret_cast<decltype(r.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    r.log = reinterpret_cast<decltype(r.log)>(dlsym(h, "nvrtcGetProgramLog"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    r.ok = r.create && r.compile && r.cubin_size && r.cubin && r.log_size && r.log && r.destroy;
    if (!r.ok) r.why = "libnvrtc lacks the CUBIN entry points";
    return r;
  }();
  return n;
}

std::string lit(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return std::string("R(") + b + ")";
}

const char* kPrelude = R"(
#define DEV __device__ __forceinline__
DEV unsigned swz(unsigned e) { unsigned x = e >> 3; x ^= (x >> 3) ^ (x >> 6) ^ (x >> 9); return e ^ (x & 7u); }
DEV void ap(V& a, V& b, R m0r, R m0i, R m1r, R m1i, R m2r, R m2i, R m3r, R m3i) {
  V u, w;
  u.x = m0r * a.x - m0i * a.y + m1r * b.x - m1i * b.y;
  u.y = m0r * a.y + m0i * a.x + m1r * b.y + m1i * b.x;
  w.x = m2r * a.x - m2i * a.y + m3r * b.x - m3i * b.y;
  w.y = m2r * a.y + m2i * a.x + m3r * b.y + m3i * b.x;
  a = u; b = w;
}
DEV void ph(V& a, R pr, R pi) { const R x = a.x * pr - a.y * pi; a.y = a.x * pi + a.y * pr; a.x = x; }
DEV void ng(V& a) { a.x = -a.x; a.y = -a.y; }
DEV void cpa(V* dst, const V* src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if (sizeof(V) == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa), "l"(src) : "memory");
}
DEV void cpc() { asm volatile("cp.async.commit_group;" ::: "memory"); }
DEV void cpw() { asm volatile("cp.async.wait_all;" ::: "memory"); }
)";

}  // namespace

int64_t jit_cost(const std::vector<RegOp>& prog, int RB) {
  const int NR = 1 << RB;
  int64_t c = 0;
  for (const RegOp& r : prog) {
    if (r.kind == ROP_DENSE) {
      for (int j = 0; j < NR; ++j)
        if (!((j >> r.k) & 1) && (uint32_t(j) & r.rmask) == r.rmask) c += 16;
    } else if (r.kind == ROP_PHASE) {
      for (int j = 0; j < NR; ++j)
        if ((uint32_t(j) & r.rmask) == r.rmask) c += 4;
    } else {
      c += 4 * NR;
    }
  }
  return c;
}

// Straight-line code of one register program (dense / phase / remap ops)
// on registers v0..v{2^RB-1}: starts and ends in the canonical register
// mapping (register bit k = tile bit T - RB + k); uses tid, tp, base,
// variant and the shared-memory transpose buffer sm of the enclosing kernel.
static void emit_register_program(std::ostringstream& o, const std::vector<RegOp>& prog, int T, int RB,
                                  const std::function<std::string(double)>& val) {
  const int NR = 1 << RB;
  auto trivial = [](double v) { return v == 0.0 || v == 1.0 || v == -1.0; };
  int rpos[4];
  for (int k = 0; k < RB; ++k) rpos[k] = T - RB + k;
  auto roff = [&](int j) {
    uint32_t r = 0;
    for (int k = 0; k < RB; ++k)
      if ((j >> k) & 1) r |= 1u << rpos[k];
    return r;
  };
  for (size_t i = 0; i < prog.size();) {
    const RegOp& op = prog[i];
    if (op.kind == ROP_REMAP) {
      o << "  __syncthreads();\n";
      for (int j = 0; j < NR; ++j) o << "  sm[swz(tp | " << roff(j) << "u)] = v" << j << ";\n";
      for (int k = 0; k < RB; ++k) rpos[k] = op.rpos[k];
      o << "  tp = tid;";
      for (int k = 0; k < RB; ++k)
        o << " tp = ((tp >> " << rpos[k] << ") << " << (rpos[k] + 1) << ") | (tp & " << ((1u << rpos[k]) - 1u)
          << "u);";
      o << "\n  __syncthreads();\n";
      for (int j = 0; j < NR; ++j) o << "  v" << j << " = sm[swz(tp | " << roff(j) << "u)];\n";
      ++i;
      continue;
    }
    const bool slotted = op.slot >= 0;
    const RegOp* alt = slotted ? &prog[i + 1] : nullptr;
    o << "  {";
    std::string cond;
    if (op.omask) cond += "(base & " + std::to_string(op.omask) + "ull) == " + std::to_string(op.omask) + "ull";
    if (op.tmask) {
      if (!cond.empty()) cond += " && ";
      cond += "(tid & " + std::to_string(op.tmask) + "u) == " + std::to_string(op.tmask) + "u";
    }
    if (!cond.empty()) o << " if (" << cond << ")";
    o << " {";
    std::string m[8];
    const int nval = op.kind == ROP_DENSE ? 8 : 2;
    if (slotted) {
      o << " const bool sb = ((variant >> " << op.slot << ") & 1ull) != 0ull;";
      for (int q = 0; q < nval; ++q) {
        const std::string a = val(alt->m[q]);
        const std::string b = val(op.m[q]);
        o << " const R m" << q << " = sb ? " << a << " : " << b << ";";
        m[q] = "m" + std::to_string(q);
      }
    } else {
      for (int q = 0; q < nval; ++q) m[q] = trivial(op.m[q]) ? lit(op.m[q]) : val(op.m[q]);
    }
    if (op.kind == ROP_DENSE) {
      for (int j = 0; j < NR; ++j) {
        if ((j >> op.k) & 1) continue;
        if ((uint32_t(j) & op.rmask) != op.rmask) continue;
        const int jb = j | (1 << op.k);
        if (slotted) {
          o << " ap(v" << j << ", v" << jb << ", " << m[0] << ", " << m[1] << ", " << m[2] << ", " << m[3] << ", "
            << m[4] << ", " << m[5] << ", " << m[6] << ", " << m[7] << ");";
          continue;
        }
        // literal matrix: drop the terms whose coefficient is exactly zero
        // (U3 has a real m00, H/X are real) — fewer FP64 instructions
        auto comp = [&](int re, int im, const char* ax, const char* ay, const char* bx, const char* by, bool imag) {
          // imag == false: real part  = m[re]*ax - m[im]*ay + m[re+2]*bx - m[im+2]*by
          // imag == true : imag part  = m[re]*ay + m[im]*ax + m[re+2]*by + m[im+2]*bx
          // unit-coefficient terms (normalised matrices) go first, without a
          // multiply: left-to-right evaluation then makes them the FMA
          // accumulator (u + c1*x - c2*y = 2 DFMA; c1*x - c2*y + u = 3 ops)
          std::string e, unit;
          auto add = [&](double c, const std::string& cs, const char* v, bool neg) {
            if (c == 0.0) return;
            if (c == 1.0 || c == -1.0) {
              const bool minus = neg != (c < 0);
              if (!unit.empty() || minus) unit += minus ? " - " : " + ";
              unit += v;
              return;
            }
            e += neg ? " - " : " + ";
            e += cs + " * " + v;
          };
          if (!imag) {
            add(op.m[re], m[re], ax, false);
            add(op.m[im], m[im], ay, true);
            add(op.m[re + 2], m[re + 2], bx, false);
            add(op.m[im + 2], m[im + 2], by, true);
          } else {
            add(op.m[re], m[re], ay, false);
            add(op.m[im], m[im], ax, false);
            add(op.m[re + 2], m[re + 2], by, false);
            add(op.m[im + 2], m[im + 2], bx, false);
          }
          if (unit.empty() && e.empty()) return std::string("R(0)");
          if (unit.empty()) return e.compare(0, 3, " + ") == 0 ? e.substr(3) : "R(0)" + e;
          return (unit[0] == ' ' ? "R(0)" + unit : unit) + e;
        };
        o << " { const V a = v" << j << ", b = v" << jb << ";";
        o << " v" << j << ".x = " << comp(0, 1, "a.x", "a.y", "b.x", "b.y", false) << ";";
        o << " v" << j << ".y = " << comp(0, 1, "a.x", "a.y", "b.x", "b.y", true) << ";";
        o << " v" << jb << ".x = " << comp(4, 5, "a.x", "a.y", "b.x", "b.y", false) << ";";
        o << " v" << jb << ".y = " << comp(4, 5, "a.x", "a.y", "b.x", "b.y", true) << "; }";
      }
    } else {
      const bool neg = !slotted && op.m[0] == -1.0 && op.m[1] == 0.0;
      for (int j = 0; j < NR; ++j) {
        if ((uint32_t(j) & op.rmask) != op.rmask) continue;
        if (neg) o << " ng(v" << j << ");";
        else o << " ph(v" << j << ", " << m[0] << ", " << m[1] << ");";
      }
    }
    o << " } }\n";
    i += slotted ? 2 : 1;
  }
}

std::string jit_source(const Sweep& sw, const std::vector<RegOp>& prog, int RB, int dtype, const std::string& name,
                       int minb, bool persistent, std::vector<double>* pvals) {
  const int T = sw.tile_bits;
  const int L = sw.low_bits;
  const int NR = 1 << RB;
  const int BD = 1 << (T - RB);
  bool remap = false;
  for (const RegOp& r : prog) remap |= r.kind == ROP_REMAP;
  // value mode (pvals == null): matrices and phases as hex-float literals;
  // param mode: every coefficient that is not exactly 0 or +-1 is read from
  // the kernel-parameter block P (constant bank: DFMA takes it as an operand),
  // so the source — and the compiled module — depends only on the circuit's
  // structure (gate positions, tile sets, masks, slots), not on its angles
  auto val = [&](double v) -> std::string {
    if (!pvals) return lit(v);
    pvals->push_back(v);
    return "P.m[" + std::to_string(pvals->size() - 1) + "]";
  };
  std::ostringstream o;
  o << "  extern __shared__ __align__(16) unsigned char smraw[];\n";
  o << "  V* sm = reinterpret_cast<V*>(smraw); (void)sm;\n";
  o << "  const unsigned tid = threadIdx.x;\n";
  o << "  const unsigned long long variant = vbase + blockIdx.y; (void)variant;\n";
  o << "  V* st = states + (long long)blockIdx.y * stride;\n";
  auto base_of = [&](const char* dst, const char* tile) {
    std::ostringstream b;
    b << dst << " = 0ull;";
    for (size_t j = 0; j < sw.oq.size(); ++j)
      b << " " << dst << " |= ((" << tile << " >> " << j << ") & 1ull) << " << sw.oq[j] << ";";
    return b.str();
  };
  auto gidx = [&](int j, const char* basev) {
    std::ostringstream g;
    g << "{ const unsigned e = tid + " << (j * BD) << "u; const unsigned c = e >> " << L
      << "; unsigned long long g = " << basev << " + (e & " << ((1u << L) - 1u) << "u);";
    for (size_t i = 0; i < sw.hq.size(); ++i)
      g << " g |= (unsigned long long)((c >> " << i << ") & 1u) << " << sw.hq[i] << ";";
    return g.str();
  };
  for (int j = 0; j < NR; ++j) o << "  V v" << j << ";\n";
  if (persistent) {
    // one CTA per SM walks the tiles; each thread prefetches the amplitudes it
    // will own in the next tile into its own shared-memory slots with
    // cp.async while the current tile's gates run (no barrier needed: a
    // thread only ever reads the slots it filled itself)
    o << "  V* pf = sm + " << (remap ? (1u << T) : 0u) << "u;\n";
    o << "  unsigned long long tile = blockIdx.x, base;\n";
    o << "  if (!init && tile < n_tiles) { unsigned long long nb; " << base_of("nb", "tile") << "\n";
    for (int j = 0; j < NR; ++j)
      o << "    " << gidx(j, "nb") << " if (!(e & zmask)) cpa(pf + e, st + g); }\n";
    o << "  }\n  cpc();\n";
    o << "  for (; tile < n_tiles; tile += gridDim.x) {\n";
    o << "  " << base_of("base", "tile") << "\n";
    o << "  if (init) {\n";
    for (int j = 0; j < NR; ++j)
      o << "    { const unsigned e = tid + " << (j * BD) << "u; v" << j
        << ".x = (base == 0ull && e == 0u) ? R(1) : R(0); v" << j << ".y = R(0); }\n";
    o << "  } else {\n    cpw();\n";
    for (int j = 0; j < NR; ++j)
      o << "    v" << j << " = ((tid + " << (j * BD) << "u) & zmask) ? V{R(0), R(0)} : pf[tid + " << (j * BD)
        << "u];\n";
    o << "    const unsigned long long nt = tile + gridDim.x;\n";
    o << "    if (nt < n_tiles) { unsigned long long nb; " << base_of("nb", "nt") << "\n";
    for (int j = 0; j < NR; ++j)
      o << "      " << gidx(j, "nb") << " if (!(e & zmask)) cpa(pf + e, st + g); }\n";
    o << "    }\n    cpc();\n  }\n";
  } else {
    o << "  const unsigned long long tile = blockIdx.x; (void)n_tiles;\n";
    o << "  unsigned long long " << base_of("base", "tile") << "\n";
    // started from |0..0>, every tile but the one holding index 0 is all
    // zero and stays zero under the tile's gates: store zeros, skip the math
    // (base is uniform across the CTA, so the early return skips no barrier
    // another thread waits on)
    o << "  if (init && base != 0ull) {\n";
    for (int j = 0; j < NR; ++j) o << "    " << gidx(j, "base") << " st[g] = V{R(0), R(0)}; }\n";
    o << "    return;\n  }\n";
    for (int j = 0; j < NR; ++j)
      o << "  " << gidx(j, "base") << " if (init) { v" << j << ".x = (base == 0ull && e == 0u) ? R(1) : R(0); v" << j
        << ".y = R(0); } else v" << j << " = (e & zmask) ? V{R(0), R(0)} : st[g]; }\n";
  }
  o << "  unsigned tp = tid; (void)tp;\n";
  emit_register_program(o, prog, T, RB, val);
  for (int j = 0; j < NR; ++j) o << "  " << gidx(j, "base") << " st[g] = v" << j << "; }\n";
  if (persistent) o << "  }\n";
  o << "}\n";
  (void)dtype;
  std::ostringstream head;
  const bool params = pvals && !pvals->empty();
  if (params) head << "struct JP_" << name << " { R m[" << pvals->size() << "]; };\n";
  // zmask: tile-local bits whose amplitudes are known 0 in a start from
  // |0..0> (Sweep::zero_local_mask; 0 otherwise): not loaded
  head << "extern \"C\" __global__ void __launch_bounds__(" << BD << ", " << minb << ") " << name
       << "(V* __restrict__ states, long long stride, unsigned long long vbase, int init, unsigned long long n_tiles"
       << ", unsigned zmask";
  if (params) head << ", const JP_" << name << " P";
  head << ") {\n";
  return head.str() + o.str();
}

// Cluster-resident form of a whole program (north_star (1): states resident
// in cluster DSMEM when small). A state of nq qubits lives in the shared
// memory of a cluster of C = 2^(nq - T) CTAs: CTA r holds amplitudes
// [r 2^T, (r+1) 2^T) ("canonical chunk"). Every launch of the program (a
// sweep tile set, or part of one) becomes a phase of ONE kernel: CTA r takes
// tile r of that phase's geometry — loaded from the owning CTAs' chunks
// with ld.shared::cluster — runs the phase's register program, and writes it
// back with st.shared::cluster; one cluster barrier separates phases (every
// index belongs to exactly one tile per phase, so there is no other hazard).
// The first phase starts from |0..0> in registers; the last one stores to
// the state in global memory. The variant id is blockIdx.y (one cluster per
// variant state), as in the per-launch kernels.
std::string jit_cluster_source(const std::vector<const Sweep*>& sweeps,
                               const std::vector<const std::vector<RegOp>*>& progs, int T, int RB, int dtype,
                               const std::string& name, std::vector<double>* pvals) {
  const int NR = 1 << RB;
  const int BD = 1 << (T - RB);
  const int C = 1 << sweeps[0]->oq.size();
  bool remap = false;
  for (const auto* pr : progs)
    for (const RegOp& r : *pr) remap |= r.kind == ROP_REMAP;
  auto val = [&](double v) -> std::string {
    if (!pvals) return lit(v);
    pvals->push_back(v);
    return "P.m[" + std::to_string(pvals->size() - 1) + "]";
  };
  const char* vreg = dtype == 0 ? "d" : "f";
  const char* vty = dtype == 0 ? "f64" : "f32";
  std::ostringstream o;
  o << "  extern __shared__ __align__(16) unsigned char smraw[];\n";
  o << "  V* chunk = reinterpret_cast<V*>(smraw);\n";
  o << "  V* sm = chunk + " << (1u << T) << "u; (void)sm;\n";
  o << "  const unsigned tid = threadIdx.x;\n";
  o << "  unsigned rank; asm volatile(\"mov.u32 %0, %%cluster_ctarank;\" : \"=r\"(rank));\n";
  o << "  const unsigned long long variant = vbase + blockIdx.y; (void)variant;\n";
  o << "  V* st = states + (long long)blockIdx.y * stride; (void)n_tiles; (void)init;\n";
  o << "  const unsigned csa = (unsigned)__cvta_generic_to_shared(chunk);\n";
  o << "  unsigned long long base; unsigned tp;\n";
  for (int j = 0; j < NR; ++j) o << "  V v" << j << ";\n";
  // every CTA of the cluster is running before any DSMEM access
  o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n\\tbarrier.cluster.wait.acquire.aligned;\" ::: \"memory\");\n";
  auto base_of = [&](const Sweep& sw) {
    std::ostringstream b;
    b << "  base = 0ull;";
    for (size_t j = 0; j < sw.oq.size(); ++j)
      b << " base |= (unsigned long long)((rank >> " << j << ") & 1u) << " << sw.oq[j] << ";";
    return b.str();
  };
  auto gidx = [&](const Sweep& sw, int j) {
    const int L = sw.low_bits;
    std::ostringstream g;
    g << "{ const unsigned e = tid + " << (j * BD) << "u; const unsigned c = e >> " << L
      << "; unsigned long long g = base + (e & " << ((1u << L) - 1u) << "u);";
    for (size_t i = 0; i < sw.hq.size(); ++i)
      g << " g |= (unsigned long long)((c >> " << i << ") & 1u) << " << sw.hq[i] << ";";
    g << " unsigned ra; asm(\"mapa.shared::cluster.u32 %0, %1, %2;\" : \"=r\"(ra) : \"r\"(csa + (unsigned)(g & "
      << ((1u << T) - 1u) << "ull) * (unsigned)sizeof(V)), \"r\"((unsigned)(g >> " << T << ")));";
    return g.str();
  };
  for (size_t ph = 0; ph < sweeps.size(); ++ph) {
    const Sweep& sw = *sweeps[ph];
    o << "  // phase " << ph << "\n" << base_of(sw) << "\n";
    if (ph == 0) {
      for (int j = 0; j < NR; ++j)
        o << "  { const unsigned e = tid + " << (j * BD) << "u; v" << j
          << ".x = (base == 0ull && e == 0u) ? R(1) : R(0); v" << j << ".y = R(0); }\n";
    } else {
      for (int j = 0; j < NR; ++j)
        o << "  " << gidx(sw, j) << " asm volatile(\"ld.shared::cluster.v2." << vty << " {%0, %1}, [%2];\" : \"="
          << vreg << "\"(v" << j << ".x), \"=" << vreg << "\"(v" << j << ".y) : \"r\"(ra) : \"memory\"); }\n";
    }
    o << "  tp = tid;\n";
    emit_register_program(o, *progs[ph], T, RB, val);
    if (ph + 1 < sweeps.size()) {
      for (int j = 0; j < NR; ++j)
        o << "  " << gidx(sw, j) << " asm volatile(\"st.shared::cluster.v2." << vty << " [%0], {%1, %2};\" :: \"r\"(ra), \""
          << vreg << "\"(v" << j << ".x), \"" << vreg << "\"(v" << j << ".y) : \"memory\"); }\n";
      o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n\\tbarrier.cluster.wait.acquire.aligned;\" ::: \"memory\");\n";
    } else {
      // the last phase writes the state (canonical index order) to global memory
      for (int j = 0; j < NR; ++j) {
        const int L = sw.low_bits;
        o << "  { const unsigned e = tid + " << (j * BD) << "u; const unsigned c = e >> " << L
          << "; unsigned long long g = base + (e & " << ((1u << L) - 1u) << "u);";
        for (size_t i = 0; i < sw.hq.size(); ++i)
          o << " g |= (unsigned long long)((c >> " << i << ") & 1u) << " << sw.hq[i] << ";";
        o << " st[g] = v" << j << "; }\n";
      }
      // no CTA leaves while another may still read its chunk
      o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n\\tbarrier.cluster.wait.acquire.aligned;\" ::: \"memory\");\n";
    }
  }
  o << "}\n";
  (void)remap;
  std::ostringstream head;
  const bool params = pvals && !pvals->empty();
  if (params) head << "struct JP_" << name << " { R m[" << pvals->size() << "]; };\n";
  head << "extern \"C\" __global__ void __cluster_dims__(" << C << ", 1, 1) __launch_bounds__(" << BD << ", 1) "
       << name
       << "(V* __restrict__ states, long long stride, unsigned long long vbase, int init, unsigned long long n_tiles";
  if (params) head << ", const JP_" << name << " P";
  head << ") {\n";
  return head.str() + o.str();
}

namespace {

std::string header(int dtype) {
  std::string h = dtype == 0 ? "typedef double R; typedef double2 V;\n" : "typedef float R; typedef float2 V;\n";
  return h + kPrelude;
}

bool compile_source(const std::string& code, std::vector<char>* cubin, std::string* err) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    *err = nv.why;
    return false;
  }
  nvrtcProgram prog = nullptr;
  if (nv.create(&prog, code.c_str(), "cutsim_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    *err = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "--extra-device-vectorization"};
  const nvrtcResult rc = nv.compile(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) nv.log(prog, &log[0]);
    *err = "NVRTC compile failed: " + log.substr(0, 2000);
    nv.destroy(&prog);
    return false;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  cubin->assign(n, 0);
  nv.cubin(prog, cubin->data());
  nv.destroy(&prog);
  return true;
}

}  // namespace

// CUTSIM_JIT_DUMP=<dir>: also write each generated source and CUBIN there
// (SASS inspection with cuobjdump; no effect otherwise)
static void dump_artifact(const std::string& name, const std::string& code, const std::vector<char>& cubin) {
  const char* dir = std::getenv("CUTSIM_JIT_DUMP");
  if (!dir || !*dir) return;
  const std::string base = std::string(dir) + "/" + name;
  if (FILE* f = std::fopen((base + ".cu").c_str(), "wb")) {
    std::fwrite(code.data(), 1, code.size(), f);
    std::fclose(f);
  }
  if (FILE* f = std::fopen((base + ".cubin").c_str(), "wb")) {
    std::fwrite(cubin.data(), 1, cubin.size(), f);
    std::fclose(f);
  }
}

// Load NVRTC and run one trivial compile (which loads its builtins library)
// on the calling thread. The tiered compiler calls it before registering its
// exit-time drain, so that drain runs before the destructors of every library
// a compile uses (exit handlers run in reverse registration order).
bool jit_warm_nvrtc() {
  static const bool ok = [] {
    std::vector<char> cubin;
    std::string err;
    return compile_source("extern \"C\" __global__ void cs_warm() {}\n", &cubin, &err);
  }();
  return ok;
}

int g_jit_persistent = 0;  // prefetching persistent kernels for streaming sweeps (measured slower: opt-in)
int g_jit_minb = 2;  // __launch_bounds__ min blocks per SM of the streaming (many-tile) kernels

bool jit_cubin(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
               int dtype, std::vector<char>* cubin, std::vector<std::string>* names, std::string* err,
               bool param_mode) {
  std::string code = header(dtype);
  names->clear();
  for (size_t i = 0; i < sweeps.size(); ++i) {
    if (!progs[i]) {
      names->emplace_back();
      continue;
    }
    names->push_back("cs_jit_" + std::to_string(i));
    std::vector<double> vals;
    code += jit_source(*sweeps[i], *progs[i], reg_bits_for(sweeps[i]->tile_bits), dtype, names->back(),
                       g_jit_minb, g_jit_persistent != 0, param_mode ? &vals : nullptr);
  }
  const bool ok = compile_source(code, cubin, err);
  if (ok) dump_artifact("selftest", code, *cubin);
  return ok;
}

// Compiled units (one NVRTC program = one kernel) keyed by their full source:
// two launches with the same source share the module (in param mode the
// source is the launch's structure, so circuits that differ only in their
// angles reuse every kernel). Units stay loaded; the cache is bounded by
// evicting the least recently used unit no program references.
namespace {
std::mutex g_units_mu;
struct UnitEntry {
  std::shared_ptr<JitUnit> unit;
  uint64_t last_use = 0;
};
std::unordered_map<std::string, UnitEntry> g_units;
uint64_t g_units_clock = 0;
constexpr size_t kUnitCacheCap = 4096;
std::atomic<int64_t> g_units_compiled{0}, g_units_reused{0};
}  // namespace

JitUnit::~JitUnit() {
  if (lib) {
    cudaDeviceSynchronize();  // queued launches of this kernel must finish first
    cudaLibraryUnload(lib);
  }
}

int64_t jit_units_compiled() { return g_units_compiled.load(); }
int64_t jit_units_reused() { return g_units_reused.load(); }

// One NVRTC program per distinct launch source, compiled on parallel host
// threads (NVRTC is thread-safe), so a 12-sweep program costs about one
// sweep's compile time; sources already in the unit cache are not compiled.
std::shared_ptr<JitModule> jit_compile(const std::vector<const Sweep*>& sweeps,
                                       const std::vector<const std::vector<RegOp>*>& progs, int dtype,
                                       std::string* err, const std::vector<int>* minb,
                                       const std::vector<char>* persistent, bool param_mode) {
  const size_t n = sweeps.size();
  auto mod = std::make_shared<JitModule>();
  mod->units.assign(n, nullptr);
  mod->blobs.assign(n, {});
  std::vector<std::string> codes(n);
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_units_mu);
    for (size_t i = 0; i < n; ++i) {
      if (!progs[i]) continue;
      std::vector<double> vals;
      codes[i] = header(dtype) + jit_source(*sweeps[i], *progs[i], reg_bits_for(sweeps[i]->tile_bits), dtype,
                                            "cs_jit_k", minb ? (*minb)[i] : 1, persistent && (*persistent)[i],
                                            param_mode ? &vals : nullptr);
      if (!vals.empty()) {
        std::vector<unsigned char>& b = mod->blobs[i];
        if (dtype == 0) {
          b.resize(vals.size() * sizeof(double));
          std::memcpy(b.data(), vals.data(), b.size());
        } else {
          std::vector<float> f(vals.begin(), vals.end());
          b.resize(f.size() * sizeof(float));
          std::memcpy(b.data(), f.data(), b.size());
        }
      }
      auto it = g_units.find(codes[i]);
      if (it != g_units.end()) {
        it->second.last_use = ++g_units_clock;
        mod->units[i] = it->second.unit;
        ++g_units_reused;
      } else {
        bool dup = false;  // the same source twice in one program: compile once
        for (size_t j : todo) dup |= codes[j] == codes[i];
        if (!dup) todo.push_back(i);
      }
    }
  }
  std::vector<std::vector<char>> cubins(todo.size());
  std::vector<std::string> errs(todo.size());
  std::vector<char> ok(todo.size(), 0);
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t t = next++; t < todo.size(); t = next++) {
      const size_t i = todo[t];
      ok[t] = compile_source(codes[i], &cubins[t], &errs[t]) ? 1 : 0;
      if (ok[t]) dump_artifact("cs_jit_" + std::to_string(i), codes[i], cubins[t]);
    }
  };
  const size_t nt =
      std::max<size_t>(1, std::min<size_t>(todo.size(), std::max(1u, std::thread::hardware_concurrency())));
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  for (size_t t = 0; t < todo.size(); ++t) {
    if (!ok[t]) {
      *err = errs[t];
      return nullptr;
    }
    const size_t i = todo[t];
    auto u = std::make_shared<JitUnit>();
    cudaError_t e = cudaLibraryLoadData(&u->lib, cubins[t].data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
      u->lib = nullptr;
      *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
      return nullptr;
    }
    e = cudaLibraryGetKernel(&u->kernel, u->lib, "cs_jit_k");
    if (e != cudaSuccess) {
      *err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
      return nullptr;
    }
    const int T = sweeps[i]->tile_bits;
    const int RB = reg_bits_for(T);
    u->threads = 1 << (T - RB);
    bool remap = false;
    for (const RegOp& r : *progs[i]) remap |= r.kind == ROP_REMAP;
    u->persistent = persistent && (*persistent)[i];
    const size_t tile_bytes = (size_t(1) << T) * (dtype == 0 ? 16 : 8);
    u->smem = (remap ? tile_bytes : 0) + (u->persistent ? tile_bytes : 0);
    ++g_units_compiled;
    std::lock_guard<std::mutex> lk(g_units_mu);
    if (g_units.size() >= kUnitCacheCap) {
      auto lru = g_units.end();
      for (auto it = g_units.begin(); it != g_units.end(); ++it)
        if (it->second.unit.use_count() == 1 && (lru == g_units.end() || it->second.last_use < lru->second.last_use))
          lru = it;
      if (lru != g_units.end()) g_units.erase(lru);
    }
    g_units[codes[i]] = UnitEntry{u, ++g_units_clock};
    for (size_t j = 0; j < n; ++j)
      if (progs[j] && !mod->units[j] && codes[j] == codes[i]) mod->units[j] = u;
  }
  return mod;
}

// The cluster-resident program (jit_cluster_source) as one unit; cached by
// source like every other unit.
std::shared_ptr<JitModule> jit_compile_cluster(const std::vector<const Sweep*>& sweeps,
                                               const std::vector<const std::vector<RegOp>*>& progs, int T,
                                               int dtype, std::string* err, bool param_mode) {
  const int RB = reg_bits_for(T);
  std::vector<double> vals;
  const std::string code =
      header(dtype) + jit_cluster_source(sweeps, progs, T, RB, dtype, "cs_jit_k", param_mode ? &vals : nullptr);
  auto mod = std::make_shared<JitModule>();
  mod->cluster = 1 << sweeps[0]->oq.size();
  mod->units.assign(1, nullptr);
  mod->blobs.assign(1, {});
  if (!vals.empty()) {
    std::vector<unsigned char>& b = mod->blobs[0];
    if (dtype == 0) {
      b.resize(vals.size() * sizeof(double));
      std::memcpy(b.data(), vals.data(), b.size());
    } else {
      std::vector<float> f(vals.begin(), vals.end());
      b.resize(f.size() * sizeof(float));
      std::memcpy(b.data(), f.data(), b.size());
    }
    if (b.size() > 30000) {  // the kernel-parameter limit (32764 B minus the other arguments)
      *err = "cluster program has too many coefficients for the parameter block";
      return nullptr;
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_units_mu);
    auto it = g_units.find(code);
    if (it != g_units.end()) {
      it->second.last_use = ++g_units_clock;
      mod->units[0] = it->second.unit;
      ++g_units_reused;
      return mod;
    }
  }
  std::vector<char> cubin;
  if (!compile_source(code, &cubin, err)) return nullptr;
  dump_artifact("cs_jit_cluster", code, cubin);
  auto u = std::make_shared<JitUnit>();
  cudaError_t e = cudaLibraryLoadData(&u->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    u->lib = nullptr;
    *err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
    return nullptr;
  }
  e = cudaLibraryGetKernel(&u->kernel, u->lib, "cs_jit_k");
  if (e != cudaSuccess) {
    *err = std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
    return nullptr;
  }
  u->threads = 1 << (T - RB);
  u->smem = 2 * (size_t(1) << T) * (dtype == 0 ? 16 : 8);  // canonical chunk + transpose scratch
  ++g_units_compiled;
  std::lock_guard<std::mutex> lk(g_units_mu);
  g_units[code] = UnitEntry{u, ++g_units_clock};
  mod->units[0] = u;
  return mod;
}

// NVRTC step only of the cluster form (host self-test)
bool jit_cluster_cubin(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
                       int T, int dtype, std::vector<char>* cubin, std::string* err, bool param_mode) {
  std::vector<double> vals;
  const std::string code = header(dtype) + jit_cluster_source(sweeps, progs, T, reg_bits_for(T), dtype, "cs_jit_k",
                                                              param_mode ? &vals : nullptr);
  const bool ok = compile_source(code, cubin, err);
  if (ok) dump_artifact("cluster_selftest", code, *cubin);
  return ok;
}

}  // namespace cutsim
