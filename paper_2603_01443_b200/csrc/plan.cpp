// Host-side planning for libcutsim. See plan.hpp.
//
// lower_gates   <- reference engine.py:122-139 (kind dispatch) + engine.py:26-27
//                  (H constant, T phase) + this build's U3 and cut slots
// schedule_*    <- no reference analogue (the reference applies one gate per
//                  full pass, engine.py:142-155); this is the B200 tiling
// plan_chain    <- reference merging.py:156-186 + cutting.py:251-272, refactored
//                  as a chain tensor-network contraction
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>

#include "capi_codes.hpp"

namespace cutsim {

namespace {

constexpr double kSqrtHalf = 0.7071067811865475244;

inline int popcount64(uint64_t v) { return __builtin_popcountll(v); }
inline int ctz64(uint64_t v) { return __builtin_ctzll(v); }

void set2(double* m, double a, double b, double c, double d, double e, double f, double g, double h) {
  m[0] = a; m[1] = b; m[2] = c; m[3] = d; m[4] = e; m[5] = f; m[6] = g; m[7] = h;
}

// C = A * B for 2x2 complex matrices stored as (re, im) row-major
void matmul2(const double* A, const double* B, double* C) {
  double out[8];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      double re = 0, im = 0;
      for (int k = 0; k < 2; ++k) {
        const double ar = A[2 * (2 * r + k)], ai = A[2 * (2 * r + k) + 1];
        const double br = B[2 * (2 * k + c)], bi = B[2 * (2 * k + c) + 1];
        re += ar * br - ai * bi;
        im += ar * bi + ai * br;
      }
      out[2 * (2 * r + c)] = re;
      out[2 * (2 * r + c) + 1] = im;
    }
  for (int i = 0; i < 8; ++i) C[i] = out[i];
}

bool is_single(const LOp& o) {
  return (o.type == OP_DENSE && o.mask == 0) || (o.type == OP_PHASE && popcount64(o.mask) == 1);
}

int single_qubit(const LOp& o) { return o.type == OP_DENSE ? o.target : ctz64(o.mask); }

void as_matrix(const LOp& o, int bit, double* M) {
  const double* src = (o.slot >= 0 && bit) ? o.alt : o.m;
  if (o.type == OP_DENSE) {
    for (int i = 0; i < 8; ++i) M[i] = src[i];
  } else {
    set2(M, 1, 0, 0, 0, 0, 0, src[0], src[1]);
  }
}

uint64_t qubit_mask(const LOp& o) {
  return o.type == OP_DENSE ? (o.mask | (1ull << o.target)) : o.mask;
}

}  // namespace

std::vector<LOp> lower_gates(int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                             const double* params, const int32_t* slots, int64_t n_gates, bool split_u3) {
  std::vector<LOp> ops;
  ops.reserve(size_t(n_gates));
  for (int64_t g = 0; g < n_gates; ++g) {
    const int k = kinds[g];
    const int64_t a = qa[g];
    LOp o;
    const bool two = (k == 5 || k == 6);
    if (k > 7) throw PlanError{CS_ERR_INVALID, "unknown gate kind code " + std::to_string(k) +
                                                   " at position " + std::to_string(g)};
    if (a < 0 || a >= nq)
      throw PlanError{CS_ERR_INVALID, "gate at position " + std::to_string(g) + " acts on qubit " +
                                          std::to_string(a) + " outside [0, " + std::to_string(nq) + ")"};
    if (two) {
      const int64_t b = qb[g];
      if (b < 0 || b >= nq || b == a)
        throw PlanError{CS_ERR_INVALID, "two-qubit gate at position " + std::to_string(g) +
                                            " has invalid second qubit " + std::to_string(b)};
    }
    const int slot = slots ? slots[g] : -1;
    if (slot >= 0 && k != 3 && k != 4)
      throw PlanError{CS_ERR_INVALID, "cut slot on a gate that is not S/Sdg at position " + std::to_string(g)};
    if (slot > 62) throw PlanError{CS_ERR_INVALID, "cut slot index too large"};
    switch (k) {
      case 0:  // H (engine.py:62-70)
        o.type = OP_DENSE;
        o.target = int(a);
        set2(o.m, kSqrtHalf, 0, kSqrtHalf, 0, kSqrtHalf, 0, -kSqrtHalf, 0);
        break;
      case 1:  // X (engine.py:73-80)
        o.type = OP_DENSE;
        o.target = int(a);
        set2(o.m, 0, 0, 1, 0, 1, 0, 0, 0);
        break;
      case 2:  // T: diag(1, (sqrt(1/2), sqrt(1/2))) (engine.py:27,131)
        o.type = OP_PHASE;
        o.mask = 1ull << a;
        o.m[0] = kSqrtHalf;
        o.m[1] = kSqrtHalf;
        break;
      case 3:  // S = diag(1, +i); slot bit 1 -> Sdg (cutting.py:237-247)
      case 4:  // Sdg = diag(1, -i)
        o.type = OP_PHASE;
        o.mask = 1ull << a;
        if (slot >= 0) {
          o.slot = slot;
          o.m[0] = 0; o.m[1] = 1;
          o.alt[0] = 0; o.alt[1] = -1;
        } else {
          o.m[0] = 0;
          o.m[1] = (k == 3) ? 1.0 : -1.0;
        }
        break;
      case 5:  // CX: X on target where control = 1 (engine.py:92-107)
        o.type = OP_DENSE;
        o.target = int(qb[g]);
        o.mask = 1ull << a;
        set2(o.m, 0, 0, 1, 0, 1, 0, 0, 0);
        break;
      case 6:  // CZ: negate |11> (engine.py:110-119)
        o.type = OP_PHASE;
        o.mask = (1ull << a) | (1ull << qb[g]);
        o.m[0] = -1;
        o.m[1] = 0;
        break;
      case 7: {  // U3 (OpenQASM-2 u3)
        const double th = params[3 * g], ph = params[3 * g + 1], la = params[3 * g + 2];
        if (!std::isfinite(th) || !std::isfinite(ph) || !std::isfinite(la))
          throw PlanError{CS_ERR_INVALID, "non-finite U3 parameter at position " + std::to_string(g)};
        const double c = std::cos(th / 2), s = std::sin(th / 2);
        if (split_u3) {
          LOp pl;  // diag(1, e^{i la}) first, then Ry(th), then diag(1, e^{i ph})
          pl.type = OP_PHASE;
          pl.mask = 1ull << a;
          pl.m[0] = std::cos(la);
          pl.m[1] = std::sin(la);
          if (la != 0.0) ops.push_back(pl);
          LOp ry;
          ry.type = OP_DENSE;
          ry.target = int(a);
          set2(ry.m, c, 0, -s, 0, s, 0, c, 0);
          ops.push_back(ry);
          o.type = OP_PHASE;
          o.mask = 1ull << a;
          o.m[0] = std::cos(ph);
          o.m[1] = std::sin(ph);
          if (ph == 0.0) continue;
          break;
        }
        o.type = OP_DENSE;
        o.target = int(a);
        set2(o.m, c, 0, -std::cos(la) * s, -std::sin(la) * s, std::cos(ph) * s, std::sin(ph) * s,
             std::cos(ph + la) * c, std::sin(ph + la) * c);
        break;
      }
      default:
        break;
    }
    ops.push_back(o);
  }
  return ops;
}

std::vector<LOp> fuse_ops(const std::vector<LOp>& ops, bool same_type_only) {
  std::vector<LOp> out;
  out.reserve(ops.size());
  int last[64];
  for (int i = 0; i < 64; ++i) last[i] = -1;
  for (const LOp& op : ops) {
    if (is_single(op)) {
      const int q = single_qubit(op);
      if (last[q] >= 0) {
        LOp& prev = out[size_t(last[q])];
        const bool types_ok = !same_type_only || prev.type == op.type;
        if (types_ok && (prev.slot < 0 || op.slot < 0 || prev.slot == op.slot)) {
          LOp f;
          f.slot = std::max(prev.slot, op.slot);
          double A[8], B[8];
          as_matrix(op, 0, A);
          as_matrix(prev, 0, B);
          double M0[8], M1[8];
          matmul2(A, B, M0);
          as_matrix(op, 1, A);
          as_matrix(prev, 1, B);
          matmul2(A, B, M1);
          if (prev.type == OP_PHASE && op.type == OP_PHASE) {
            f.type = OP_PHASE;
            f.mask = 1ull << q;
            f.m[0] = M0[6]; f.m[1] = M0[7];
            f.alt[0] = M1[6]; f.alt[1] = M1[7];
          } else {
            f.type = OP_DENSE;
            f.target = q;
            f.mask = 0;
            for (int i = 0; i < 8; ++i) { f.m[i] = M0[i]; f.alt[i] = M1[i]; }
          }
          if (f.slot < 0)
            for (int i = 0; i < 8; ++i) f.alt[i] = 0;
          prev = f;
          continue;
        }
      }
      out.push_back(op);
      last[q] = int(out.size()) - 1;
    } else {
      out.push_back(op);
      uint64_t qm = qubit_mask(op);
      while (qm) {
        last[ctz64(qm)] = -1;
        qm &= qm - 1;
      }
    }
  }
  return out;
}

namespace {

struct Cx {
  double r = 1, i = 0;
};
inline Cx cmulx(Cx a, Cx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
inline Cx cdivx(Cx a, Cx b) {
  const double n = b.r * b.r + b.i * b.i;
  return {(a.r * b.r + a.i * b.i) / n, (a.i * b.r - a.r * b.i) / n};
}
inline double cabs2(Cx a) { return a.r * a.r + a.i * a.i; }
inline bool is_one(Cx a) { return a.r == 1.0 && a.i == 0.0; }

LOp phase_op(int q, Cx v) {
  LOp o;
  o.type = OP_PHASE;
  o.mask = 1ull << q;
  o.m[0] = v.r;
  o.m[1] = v.i;
  return o;
}

}  // namespace

std::vector<LOp> normalize_dense(const std::vector<LOp>& ops, int nq, double max_growth_bits, bool fixed_pivot) {
  std::vector<LOp> out;
  out.reserve(ops.size() + size_t(nq) + 1);
  std::vector<Cx> d0(static_cast<size_t>(nq)), d1(static_cast<size_t>(nq));
  // amplification of the executed state over the true one: each qubit's
  // pending D contributes -log2 min(|d0|, |d1|) bits, the deferred global
  // scalar -log2 |scale|; kept under max_growth_bits (each normalised op adds
  // up to 1/2 bit, so deep circuits would otherwise overflow / underflow)
  std::vector<double> grow(static_cast<size_t>(nq), 0.0);
  double grow_sum = 0.0, grow_scale = 0.0;
  Cx scale;
  auto bits_of = [](Cx a, Cx b) { return -0.5 * std::log2(std::min(cabs2(a), cabs2(b))); };
  auto flush = [&](int q) {
    const size_t k = size_t(q);
    if (is_one(d0[k]) && is_one(d1[k])) return;
    scale = cmulx(scale, d0[k]);  // D = d0 . diag(1, d1/d0)
    grow_scale = -0.5 * std::log2(cabs2(scale));
    const Cx r = cdivx(d1[k], d0[k]);
    if (!is_one(r)) out.push_back(phase_op(q, r));
    d0[k] = Cx{};
    d1[k] = Cx{};
    grow_sum -= grow[k];
    grow[k] = 0.0;
  };
  long last_dense = -1;
  for (const LOp& op : ops) {
    if (op.type == OP_PHASE) {  // diagonal: commutes with every pending D
      out.push_back(op);
      continue;
    }
    const int q = op.target;
    if (op.mask != 0 || op.slot >= 0) {  // controlled (or variant-switched) dense: apply D first
      flush(q);
      out.push_back(op);
      continue;
    }
    // M . D_q, then rows normalised by their pivot
    LOp n = op;
    const size_t k = size_t(q);
    Cx m[2][2];
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) m[r][c] = Cx{op.m[2 * (2 * r + c)], op.m[2 * (2 * r + c) + 1]};
    for (int r = 0; r < 2; ++r) {
      m[r][0] = cmulx(m[r][0], d0[k]);
      m[r][1] = cmulx(m[r][1], d1[k]);
    }
    Cx dn[2];
    int piv[2];
    for (int r = 0; r < 2; ++r) {
      if (fixed_pivot && cabs2(m[r][r]) >= 1e-24 * cabs2(m[r][1 - r]) && cabs2(m[r][r]) > 0.0)
        piv[r] = r;
      else
        piv[r] = cabs2(m[r][0]) >= cabs2(m[r][1]) ? 0 : 1;
      dn[r] = m[r][piv[r]];
    }
    const double g = bits_of(dn[0], dn[1]);
    if (grow_sum - grow[k] + g + grow_scale > max_growth_bits) {
      // over budget: execute M . D_q (times the deferred scalar) as it is,
      // which brings the executed state back to the true scale
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
          const Cx v = cmulx(m[r][c], scale);
          n.m[2 * (2 * r + c)] = v.r;
          n.m[2 * (2 * r + c) + 1] = v.i;
        }
      scale = Cx{};
      grow_scale = 0.0;
      d0[k] = Cx{};
      d1[k] = Cx{};
      grow_sum -= grow[k];
      grow[k] = 0.0;
    } else {
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) {
          const Cx v = c == piv[r] ? Cx{} : cdivx(m[r][c], dn[r]);
          n.m[2 * (2 * r + c)] = v.r;
          n.m[2 * (2 * r + c) + 1] = v.i;
        }
      d0[k] = dn[0];
      d1[k] = dn[1];
      grow_sum += g - grow[k];
      grow[k] = g;
    }
    last_dense = long(out.size());
    out.push_back(n);
  }
  for (int q = 0; q < nq; ++q) flush(q);
  // the scalar only arises from diagonals some uncontrolled dense op created
  if (!is_one(scale) && last_dense >= 0) {
    LOp& l = out[size_t(last_dense)];
    for (int e = 0; e < 4; ++e) {
      const Cx v = cmulx(Cx{l.m[2 * e], l.m[2 * e + 1]}, scale);
      l.m[2 * e] = v.r;
      l.m[2 * e + 1] = v.i;
    }
  }
  return out;
}

std::vector<LOp> commute_phases(const std::vector<LOp>& ops) {
  std::vector<LOp> out;
  out.reserve(ops.size());
  LOp pend[64];
  bool has[64] = {false};
  uint64_t pending = 0;
  auto flush_all = [&]() {
    uint64_t m = pending;
    while (m) {
      const int q = ctz64(m);
      m &= m - 1;
      out.push_back(pend[q]);
      has[q] = false;
    }
    pending = 0;
  };
  for (const LOp& op : ops) {
    if (op.type == OP_PHASE && popcount64(op.mask) == 1) {
      const int q = ctz64(op.mask);
      if (!has[q]) {
        pend[q] = op;
        has[q] = true;
        pending |= 1ull << q;
        continue;
      }
      LOp& prev = pend[q];
      if (prev.slot < 0 || op.slot < 0 || prev.slot == op.slot) {
        // diag(1, a) . diag(1, b) = diag(1, ab), per variant alternative
        LOp f;
        f.type = OP_PHASE;
        f.mask = op.mask;
        f.slot = std::max(prev.slot, op.slot);
        const double* a0 = prev.m;
        const double* a1 = prev.slot >= 0 ? prev.alt : prev.m;
        const double* b0 = op.m;
        const double* b1 = op.slot >= 0 ? op.alt : op.m;
        f.m[0] = a0[0] * b0[0] - a0[1] * b0[1];
        f.m[1] = a0[0] * b0[1] + a0[1] * b0[0];
        if (f.slot >= 0) {
          f.alt[0] = a1[0] * b1[0] - a1[1] * b1[1];
          f.alt[1] = a1[0] * b1[1] + a1[1] * b1[0];
        }
        prev = f;
        continue;
      }
      // two different cut slots on one qubit: emit the older one here
      out.push_back(prev);
      prev = op;
      continue;
    }
    if (op.type == OP_PHASE) {  // multi-qubit diagonal: commutes with every pending phase
      out.push_back(op);
      continue;
    }
    if (pending & (1ull << op.target)) {  // the phase must precede this op
      out.push_back(pend[op.target]);
      has[op.target] = false;
      pending &= ~(1ull << op.target);
    }
    out.push_back(op);
  }
  flush_all();
  return out;
}

static void emit_entries(const LOp& op, const int* local_pos, Sweep& sw, int gsize) {
  SweepOp e{};
  e.type = op.type;
  e.slot = op.slot;
  e.gsize = gsize;
  uint64_t mm = op.mask;
  while (mm) {
    const int q = ctz64(mm);
    mm &= mm - 1;
    if (local_pos[q] >= 0) e.lmask |= 1u << local_pos[q];
    else e.omask |= 1ull << q;
  }
  e.target = op.type == OP_DENSE ? int16_t(local_pos[op.target]) : int16_t(-1);
  for (int i = 0; i < 8; ++i) e.m[i] = op.m[i];
  sw.entries.push_back(e);
  if (op.slot >= 0) {
    for (int i = 0; i < 8; ++i) e.m[i] = op.alt[i];
    e.gsize = 0;
    sw.entries.push_back(e);
  }
}

// Emit a sweep's ops in order, packing runs of consecutive dense ops with
// pairwise-disjoint qubits (they commute) into register groups of <= kMaxGroup.
static void emit_run(const std::vector<LOp>& ops, const std::vector<int>& run, const int* local_pos, Sweep& sw,
                     int max_group) {
  size_t a = 0;
  while (a < run.size()) {
    const LOp& op = ops[size_t(run[a])];
    if (op.type != OP_DENSE) {
      emit_entries(op, local_pos, sw, 0);
      ++a;
      continue;
    }
    size_t b = a + 1;
    uint64_t used = qubit_mask(op);
    while (b < run.size() && int(b - a) < max_group) {
      const LOp& o2 = ops[size_t(run[b])];
      if (o2.type != OP_DENSE || (qubit_mask(o2) & used)) break;
      used |= qubit_mask(o2);
      ++b;
    }
    for (size_t k = a; k < b; ++k)
      emit_entries(ops[size_t(run[k])], local_pos, sw, k == a ? int(b - a) : 0);
    a = b;
  }
}

int sweep_threads(int tile_bits) { return std::max(32, std::min(256, 1 << std::max(0, tile_bits - 2))); }

int sweep_max_group(int tile_bits) {
  int lg = 0;
  while ((1 << lg) < sweep_threads(tile_bits)) ++lg;
  return std::max(1, std::min(kMaxGroup, tile_bits - lg));
}

int g_sweep_windows = 3;  // cost-aware tile sets (zero-start tiles); 1 = most absorbed ops per sweep

// Order each sweep's tile-id qubits so that, for a start from |0..0>, the
// tiles that can be non-zero are exactly t < 2^zero_tiles_log2: the qubits
// already held by an earlier sweep's tile (the support) come first.
static void order_tiles_for_zero_start(std::vector<Sweep>& sweeps) {
  uint64_t support = 0;
  for (Sweep& sw : sweeps) {
    std::stable_partition(sw.oq.begin(), sw.oq.end(), [&](int q) { return (support >> q) & 1ull; });
    int m = 0;
    for (int q : sw.oq) m += int((support >> q) & 1ull);
    sw.zero_tiles_log2 = m;
    uint32_t zm = 0;
    for (int q = 0; q < sw.low_bits; ++q) zm |= uint32_t(!((support >> q) & 1ull)) << q;
    for (size_t j = 0; j < sw.hq.size(); ++j) zm |= uint32_t(!((support >> sw.hq[j]) & 1ull)) << (sw.low_bits + int(j));
    sw.zero_local_mask = zm;
    for (int q = 0; q < sw.low_bits; ++q) support |= 1ull << q;
    for (int q : sw.hq) support |= 1ull << q;
  }
}

static std::vector<Sweep> schedule_sweeps_impl(const std::vector<LOp>& ops, int nq, int tile_bits, int low_bits,
                                               int max_group, int windows);

std::vector<Sweep> schedule_sweeps(const std::vector<LOp>& ops, int nq, int tile_bits, int low_bits,
                                   int max_group, int windows) {
  std::vector<Sweep> sweeps =
      schedule_sweeps_impl(ops, nq, tile_bits, low_bits, max_group, windows < 0 ? g_sweep_windows : windows);
  order_tiles_for_zero_start(sweeps);
  return sweeps;
}

static std::vector<Sweep> schedule_sweeps_impl(const std::vector<LOp>& ops, int nq, int tile_bits, int low_bits,
                                               int max_group, int windows) {
  std::vector<Sweep> sweeps;
  if (nq <= tile_bits) {
    Sweep sw;
    sw.tile_bits = nq;
    sw.low_bits = nq;
    int local_pos[64];
    for (int q = 0; q < 64; ++q) local_pos[q] = q < nq ? q : -1;
    std::vector<int> all(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) all[i] = int(i);
    emit_run(ops, all, local_pos, sw, max_group);
    sweeps.push_back(std::move(sw));
    return sweeps;
  }
  const int T = tile_bits;
  const int L = std::max(1, std::min(low_bits, T - 1));
  std::vector<int> pending(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) pending[i] = int(i);
  // dense ops a fixed tile set would absorb from `pending` (same rules as the
  // greedy pass below, without growing the set)
  auto absorbed_from = [&](const std::vector<int>& list, const bool* fixed, std::vector<int>* rest) {
    uint64_t bd = 0, bp = 0;
    int count = 0;
    for (int idx : list) {
      const LOp& op = ops[size_t(idx)];
      const uint64_t qm = qubit_mask(op);
      if (op.type == OP_PHASE) {
        if (qm & bd) {
          bp |= qm;
          if (rest) rest->push_back(idx);
        }
        continue;
      }
      if ((qm & (bd | bp)) || !fixed[op.target]) {
        bd |= qm;
        if (rest) rest->push_back(idx);
      } else {
        ++count;
      }
    }
    return count;
  };
  auto absorbed = [&](const bool* fixed) { return absorbed_from(pending, fixed, nullptr); };
  // best single-window count over a list (for the two-step look-ahead)
  auto best_window = [&](const std::vector<int>& list) {
    int best = 0;
    for (int a = L; a + (T - L) <= nq; ++a) {
      bool cand[64] = {false};
      for (int q = 0; q < L; ++q) cand[q] = true;
      for (int q = a; q < a + (T - L); ++q) cand[q] = true;
      best = std::max(best, absorbed_from(list, cand, nullptr));
    }
    return best;
  };
  // sweep_windows = 3: cost-aware choice for a start from |0..0> (zero-start
  // tiles): a candidate tile set costs the fraction of tiles it launches,
  // 2^(support qubits outside the set) / 2^(nq - T), times a dense-op term,
  // plus a per-launch constant; the set with the most absorbed dense ops per
  // unit cost wins. Once the support is complete every set costs the same
  // and this is the plain most-absorbed choice.
  uint64_t support = 0;
  const uint64_t high_mask = (nq >= 64 ? ~0ull : ((1ull << nq) - 1)) & ~((1ull << L) - 1);
  auto set_cost = [&](const bool* cand, int absorbed_ops) {
    uint64_t m = 0;
    for (int q = 0; q < nq; ++q)
      if (cand[q]) m |= 1ull << q;
    const int z = __builtin_popcountll(support & high_mask & ~m);
    const double frac = std::ldexp(1.0, z - (nq - T));
    // (weights from the measured full-sweep times t ~ 4.8 ms + 0.19 ms per
    // dense op at q=30; the schedule is insensitive to them within 2x)
    return frac * (1.0 + 0.04 * absorbed_ops) + 0.002;
  };
  bool first = true;
  while (!pending.empty() || first) {
    first = false;
    bool inset[64] = {false};
    for (int q = 0; q < L; ++q) inset[q] = true;
    int room = T - L;
    if (windows == 3 && nq - L > T - L) {
      double best_score = -1.0;
      int best_a = -1;
      for (int a = L; a + (T - L) <= nq; ++a) {
        bool cand[64] = {false};
        for (int q = 0; q < L; ++q) cand[q] = true;
        for (int q = a; q < a + (T - L); ++q) cand[q] = true;
        const int c = absorbed(cand);
        if (c <= 0) continue;
        const double sc = c / set_cost(cand, c);
        if (sc > best_score) {
          best_score = sc;
          best_a = a;
        }
      }
      // the greedy first-need set, for comparison (same rules as below)
      bool g[64] = {false};
      for (int q = 0; q < L; ++q) g[q] = true;
      {
        int r = T - L;
        uint64_t bd = 0, bp = 0;
        for (int idx : pending) {
          const LOp& op = ops[size_t(idx)];
          const uint64_t qm = qubit_mask(op);
          if (op.type == OP_PHASE) {
            if (qm & bd) bp |= qm;
            continue;
          }
          if (qm & (bd | bp)) bd |= qm;
          else if (!g[op.target]) {
            if (r > 0) {
              g[op.target] = true;
              --r;
            } else {
              bd |= qm;
            }
          }
        }
      }
      const int gc = absorbed(g);
      const double gscore = gc > 0 ? gc / set_cost(g, gc) : -1.0;
      if (best_a >= 0 && best_score > gscore) {
        for (int q = best_a; q < best_a + (T - L); ++q) inset[q] = true;
        room = 0;
      }
    } else if (windows && nq - L > T - L) {
      // candidate tile sets: the greedy first-need set (room filled below) vs
      // every contiguous window of T - L high qubits; take the window when it
      // absorbs more dense ops
      int best = -1, best_a = -1;
      for (int a = L; a + (T - L) <= nq; ++a) {
        bool cand[64] = {false};
        for (int q = 0; q < L; ++q) cand[q] = true;
        for (int q = a; q < a + (T - L); ++q) cand[q] = true;
        int c;
        if (windows >= 2) {  // score = this sweep + the best next window
          std::vector<int> rest;
          c = absorbed_from(pending, cand, &rest);
          c += best_window(rest);
        } else {
          c = absorbed(cand);
        }
        if (c > best) {
          best = c;
          best_a = a;
        }
      }
      // the greedy set, for comparison
      bool g[64] = {false};
      for (int q = 0; q < L; ++q) g[q] = true;
      {
        int r = T - L;
        uint64_t bd = 0, bp = 0;
        for (int idx : pending) {
          const LOp& op = ops[size_t(idx)];
          const uint64_t qm = qubit_mask(op);
          if (op.type == OP_PHASE) {
            if (qm & bd) bp |= qm;
            continue;
          }
          if (qm & (bd | bp)) bd |= qm;
          else if (!g[op.target]) {
            if (r > 0) {
              g[op.target] = true;
              --r;
            } else {
              bd |= qm;
            }
          }
        }
      }
      int greedy_score;
      if (windows >= 2) {
        std::vector<int> rest;
        greedy_score = absorbed_from(pending, g, &rest);
        greedy_score += best_window(rest);
      } else {
        greedy_score = absorbed(g);
      }
      if (best > greedy_score) {
        for (int q = best_a; q < best_a + (T - L); ++q) inset[q] = true;
        room = 0;
      }
    }
    uint64_t blocked_dense = 0, blocked_phase = 0;
    std::vector<int> run, deferred;
    for (int idx : pending) {
      const LOp& op = ops[size_t(idx)];
      const uint64_t qm = qubit_mask(op);
      if (op.type == OP_PHASE) {
        if (qm & blocked_dense) {
          blocked_phase |= qm;
          deferred.push_back(idx);
        } else {
          run.push_back(idx);
        }
        continue;
      }
      if (qm & (blocked_dense | blocked_phase)) {
        blocked_dense |= qm;
        deferred.push_back(idx);
      } else if (inset[op.target]) {
        run.push_back(idx);
      } else if (room > 0) {
        inset[op.target] = true;
        --room;
        run.push_back(idx);
      } else {
        blocked_dense |= qm;
        deferred.push_back(idx);
      }
    }
    Sweep sw;
    sw.tile_bits = T;
    sw.low_bits = L;
    for (int q = L; q < nq; ++q)
      if (inset[q]) sw.hq.push_back(q);
    for (int q = L; q < nq && int(sw.hq.size()) < T - L; ++q)
      if (!inset[q]) {
        inset[q] = true;
        sw.hq.push_back(q);
      }
    std::sort(sw.hq.begin(), sw.hq.end());
    for (int q = L; q < nq; ++q)
      if (!inset[q]) sw.oq.push_back(q);
    for (int q = 0; q < nq; ++q)
      if (inset[q]) support |= 1ull << q;
    int local_pos[64];
    for (int q = 0; q < 64; ++q) local_pos[q] = -1;
    for (int q = 0; q < L; ++q) local_pos[q] = q;
    for (size_t j = 0; j < sw.hq.size(); ++j) local_pos[sw.hq[j]] = L + int(j);
    emit_run(ops, run, local_pos, sw, max_group);
    sweeps.push_back(std::move(sw));
    pending.swap(deferred);
  }
  return sweeps;
}

std::string sweeps_to_json(const std::vector<Sweep>& sweeps, int nq) {
  std::ostringstream os;
  os.precision(17);
  os << "{\"nq\":" << nq << ",\"sweeps\":[";
  for (size_t s = 0; s < sweeps.size(); ++s) {
    const Sweep& sw = sweeps[s];
    if (s) os << ",";
    os << "{\"T\":" << sw.tile_bits << ",\"L\":" << sw.low_bits << ",\"hq\":[";
    for (size_t i = 0; i < sw.hq.size(); ++i) os << (i ? "," : "") << sw.hq[i];
    os << "],\"oq\":[";
    for (size_t i = 0; i < sw.oq.size(); ++i) os << (i ? "," : "") << sw.oq[i];
    os << "],\"z\":" << sw.zero_tiles_log2 << ",\"zl\":" << sw.zero_local_mask << ",\"entries\":[";
    for (size_t i = 0; i < sw.entries.size(); ++i) {
      const SweepOp& e = sw.entries[i];
      os << (i ? "," : "") << "{\"type\":" << e.type << ",\"target\":" << e.target
         << ",\"lmask\":" << e.lmask << ",\"omask\":" << e.omask << ",\"slot\":" << e.slot
         << ",\"gsize\":" << e.gsize << ",\"m\":[";
      for (int k = 0; k < 8; ++k) os << (k ? "," : "") << e.m[k];
      os << "]}";
    }
    os << "]}";
  }
  os << "]}";
  return os.str();
}

// ---------------------------------------------------------------------------
// register-tile lowering
// ---------------------------------------------------------------------------
int g_reg_bits = 0;

int reg_bits_for(int tile_bits) {
  if (tile_bits <= 2) return std::max(1, tile_bits);
  // override (tuning): only where it keeps 32..512 threads per tile
  if (g_reg_bits >= 2 && tile_bits - g_reg_bits >= 5 && tile_bits - g_reg_bits <= 9) return g_reg_bits;
  return std::max(2, std::min(4, tile_bits - 8));
}

namespace {

struct Mapping {
  int T = 0, RB = 0;
  int rpos[4] = {0, 0, 0, 0};
  int reg_of[32];     // tile bit -> register bit or -1
  int thread_of[32];  // tile bit -> thread bit or -1
  void build() {
    for (int b = 0; b < 32; ++b) reg_of[b] = thread_of[b] = -1;
    for (int k = 0; k < RB; ++k) reg_of[rpos[k]] = k;
    int m = 0;
    for (int b = 0; b < T; ++b)
      if (reg_of[b] < 0) thread_of[b] = m++;
  }
  void split(uint32_t lmask, uint32_t* tmask, uint32_t* rmask) const {
    *tmask = 0;
    *rmask = 0;
    for (int b = 0; b < T; ++b)
      if ((lmask >> b) & 1u) {
        if (reg_of[b] >= 0) *rmask |= 1u << reg_of[b];
        else *tmask |= 1u << thread_of[b];
      }
  }
  bool canonical() const {
    for (int k = 0; k < RB; ++k)
      if (rpos[k] != T - RB + k) return false;
    return true;
  }
};

void push_remap(std::vector<RegOp>& out, Mapping& map, const int* want) {
  RegOp r{};
  r.kind = ROP_REMAP;
  r.slot = -1;
  for (int k = 0; k < map.RB; ++k) {
    map.rpos[k] = want[k];
    r.rpos[k] = uint8_t(want[k]);
  }
  map.build();
  out.push_back(r);
}

}  // namespace

int g_reg_reorder = 1;

namespace {

// Ops i < j of one sweep commute when reordering them cannot change the
// result: two diagonal ops always; a dense op and a diagonal op when the
// diagonal does not touch the dense target; two dense ops when neither
// target is a qubit (target or control) of the other. Tile-local masks
// only: outside-tile bits are constants within a tile.
// The sweep's ops (a slotted op = two consecutive entries) in an order that
// needs fewer register remaps: list scheduling over the commutation DAG that
// prefers any ready op whose dense target is already a register bit, and on
// a miss loads the targets of the ready ops first, then the next ones in
// program order. Returns entry-index starts of the units in the new order.
std::vector<size_t> reorder_for_registers(const std::vector<SweepOp>& E, int RB, const int* rpos0, int T) {
  std::vector<size_t> start;
  start.reserve(E.size());
  for (size_t i = 0; i < E.size(); i += (E[i].slot >= 0 ? 2 : 1)) start.push_back(i);
  const size_t n = start.size();
  // Dependence edges with the same transitive closure as "i < j do not
  // commute" (commutes() above), found per tile bit instead of over all
  // pairs: a dense op acts as X on its target and Z on its controls, a
  // diagonal op as Z on its bits; two ops conflict iff one's X bit is the
  // other's X or Z bit. Per bit, an op depends on the bit's last X op and,
  // if it is X there, on the Z ops since. Readiness under list scheduling
  // is that of the full relation (every dropped edge is implied by a chain).
  std::vector<uint64_t> pairs;
  pairs.reserve(n * 4);
  std::vector<int> npred(n, 0), soff(n + 1, 0);
  int last_x[32];
  std::vector<int> zs[32];
  for (int b = 0; b < 32; ++b) last_x[b] = -1;
  auto edge = [&](int i, size_t j) {
    pairs.push_back(uint64_t(i) << 32 | uint64_t(j));
    ++soff[size_t(i) + 1];
    ++npred[j];
  };
  for (size_t j = 0; j < n; ++j) {
    const SweepOp& e = E[start[j]];
    const bool dense = e.type == OP_DENSE;
    uint32_t zmask = e.lmask & 0xffffffffu;
    if (dense) {
      const int t = e.target;
      if (last_x[t] >= 0) edge(last_x[t], j);
      for (int i : zs[t]) edge(i, j);
      zmask &= ~(1u << t);
    }
    for (uint32_t m = zmask; m; m &= m - 1) {
      const int b = __builtin_ctz(m);
      if (last_x[b] >= 0) edge(last_x[b], j);
    }
    if (dense) {
      last_x[e.target] = int(j);
      zs[e.target].clear();
    }
    for (uint32_t m = zmask; m; m &= m - 1) zs[__builtin_ctz(m)].push_back(int(j));
  }
  for (size_t i = 0; i < n; ++i) soff[i + 1] += soff[i];
  std::vector<int> succ(pairs.size()), fill(soff.begin(), soff.end() - 1);
  for (uint64_t pr : pairs) succ[size_t(fill[size_t(pr >> 32)]++)] = int(pr & 0xffffffffu);
  std::vector<char> done(n, 0);
  std::vector<size_t> order;
  order.reserve(n);
  bool inreg[32] = {false};
  for (int k = 0; k < RB; ++k) inreg[rpos0[k]] = true;
  auto take = [&](size_t u) {
    done[u] = 1;
    order.push_back(start[u]);
    for (int s = soff[u]; s < soff[u + 1]; ++s) --npred[size_t(succ[size_t(s)])];
  };
  while (order.size() < n) {
    bool progress = true;
    while (progress) {  // everything runnable without a remap, in program order
      progress = false;
      for (size_t u = 0; u < n; ++u) {
        if (done[u] || npred[u] > 0) continue;
        const SweepOp& e = E[start[u]];
        if (e.type != OP_DENSE || inreg[e.target]) {
          take(u);
          progress = true;
        }
      }
    }
    if (order.size() == n) break;
    // miss: new register set = targets of ready dense ops (program order),
    // then targets of the following dense ops, then current register bits
    int want[4];
    int m = 0;
    auto add = [&](int t) {
      for (int a = 0; a < m; ++a)
        if (want[a] == t) return;
      if (m < RB) want[m++] = t;
    };
    for (size_t u = 0; u < n && m < RB; ++u)
      if (!done[u] && npred[u] == 0 && E[start[u]].type == OP_DENSE) add(E[start[u]].target);
    for (size_t u = 0; u < n && m < RB; ++u)
      if (!done[u] && E[start[u]].type == OP_DENSE) add(E[start[u]].target);
    for (int b = 0; b < T && m < RB; ++b)
      if (inreg[b]) add(b);
    for (int b = 0; b < T && m < RB; ++b) add(b);
    for (int b = 0; b < 32; ++b) inreg[b] = false;
    for (int a = 0; a < m; ++a) inreg[want[a]] = true;
  }
  return order;
}

}  // namespace

std::vector<RegOp> reg_program(const Sweep& sw, int RB) {
  RB = std::max(1, std::min(RB, 4));
  const int T = sw.tile_bits;
  Mapping map;
  map.T = T;
  map.RB = RB;
  for (int k = 0; k < RB; ++k) map.rpos[k] = T - RB + k;
  map.build();
  std::vector<RegOp> out;
  out.reserve(sw.entries.size() + 16);
  // optionally reorder the sweep's commuting ops so fewer remaps are needed
  std::vector<SweepOp> reordered;
  if (g_reg_reorder) {
    reordered.reserve(sw.entries.size());
    const std::vector<size_t> order = reorder_for_registers(sw.entries, RB, map.rpos, T);
    for (size_t st : order) {
      reordered.push_back(sw.entries[st]);
      if (sw.entries[st].slot >= 0) reordered.push_back(sw.entries[st + 1]);
    }
  }
  const auto& E = g_reg_reorder ? reordered : sw.entries;
  for (size_t i = 0; i < E.size();) {
    const SweepOp& e = E[i];
    const size_t w = e.slot >= 0 ? 2 : 1;
    if (e.type == OP_DENSE && map.reg_of[e.target] < 0) {
      // new register set: this target and the next distinct dense targets
      int want[4];
      int n = 0;
      for (size_t j = i; j < E.size() && n < RB; j += (E[j].slot >= 0 ? 2 : 1)) {
        if (E[j].type != OP_DENSE) continue;
        bool dup = false;
        for (int a = 0; a < n; ++a) dup |= want[a] == E[j].target;
        if (!dup) want[n++] = E[j].target;
      }
      for (int k = 0; k < RB && n < RB; ++k) {  // keep current register bits
        bool dup = false;
        for (int a = 0; a < n; ++a) dup |= want[a] == map.rpos[k];
        if (!dup) want[n++] = map.rpos[k];
      }
      for (int b = 0; b < T && n < RB; ++b) {
        bool dup = false;
        for (int a = 0; a < n; ++a) dup |= want[a] == b;
        if (!dup) want[n++] = b;
      }
      for (int a = 1; a < RB; ++a)  // insertion sort (RB <= 4)
        for (int b = a; b > 0 && want[b] < want[b - 1]; --b) std::swap(want[b], want[b - 1]);
      push_remap(out, map, want);
    }
    for (size_t j = 0; j < w; ++j) {
      const SweepOp& x = E[i + j];
      RegOp r{};
      r.kind = x.type == OP_DENSE ? ROP_DENSE : ROP_PHASE;
      r.slot = int16_t(x.slot);
      r.k = x.type == OP_DENSE ? uint8_t(map.reg_of[x.target]) : 0;
      map.split(x.lmask, &r.tmask, &r.rmask);
      r.omask = x.omask;
      for (int q = 0; q < 8; ++q) r.m[q] = x.m[q];
      out.push_back(r);
    }
    i += w;
  }
  if (!map.canonical()) {
    int want[4];
    for (int k = 0; k < RB; ++k) want[k] = T - RB + k;
    push_remap(out, map, want);
  }
  return out;
}

std::string reg_programs_to_json(const std::vector<Sweep>& sweeps, int nq) {
  std::ostringstream os;
  os.precision(17);
  os << "{\"nq\":" << nq << ",\"sweeps\":[";
  for (size_t s = 0; s < sweeps.size(); ++s) {
    const Sweep& sw = sweeps[s];
    const int RB = reg_bits_for(sw.tile_bits);
    const std::vector<RegOp> prog = reg_program(sw, RB);
    if (s) os << ",";
    os << "{\"T\":" << sw.tile_bits << ",\"L\":" << sw.low_bits << ",\"RB\":" << RB << ",\"hq\":[";
    for (size_t i = 0; i < sw.hq.size(); ++i) os << (i ? "," : "") << sw.hq[i];
    os << "],\"oq\":[";
    for (size_t i = 0; i < sw.oq.size(); ++i) os << (i ? "," : "") << sw.oq[i];
    os << "],\"ops\":[";
    for (size_t i = 0; i < prog.size(); ++i) {
      const RegOp& r = prog[i];
      os << (i ? "," : "") << "{\"kind\":" << int(r.kind) << ",\"k\":" << int(r.k) << ",\"slot\":" << r.slot
         << ",\"tmask\":" << r.tmask << ",\"rmask\":" << r.rmask << ",\"omask\":" << r.omask << ",\"rpos\":["
         << int(r.rpos[0]) << "," << int(r.rpos[1]) << "," << int(r.rpos[2]) << "," << int(r.rpos[3]) << "],\"m\":[";
      for (int k = 0; k < 8; ++k) os << (k ? "," : "") << r.m[k];
      os << "]}";
    }
    os << "]}";
  }
  os << "]}";
  return os.str();
}

// ---------------------------------------------------------------------------
// cut preprocess
// ---------------------------------------------------------------------------
CutPrep cut_prepare(int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                    int64_t G, int n, const int32_t* sizes) {
  if (n < 2) throw PlanError{CS_ERR_INVALID, "segment count must be >= 2, got " + std::to_string(n)};
  CutPrep prep;
  prep.n = n;
  std::vector<int> seg_of;
  int total = 0;
  for (int s = 0; s < n; ++s) {
    if (sizes[s] < 1) throw PlanError{CS_ERR_INVALID, "segment sizes must be >= 1"};
    prep.sizes.push_back(sizes[s]);
    for (int k = 0; k < sizes[s]; ++k) seg_of.push_back(s);
    total += sizes[s];
  }
  if (total != nq)
    throw PlanError{CS_ERR_INVALID, "segment sizes must sum to q=" + std::to_string(nq)};
  std::vector<int> cut_at(size_t(G), -1);
  for (int64_t g = 0; g < G; ++g) {
    const int k = kinds[g];
    if (k > 7) throw PlanError{CS_ERR_INVALID, "unknown gate kind code " + std::to_string(k)};
    if (qa[g] < 0 || qa[g] >= nq) throw PlanError{CS_ERR_INVALID, "gate qubit outside the circuit"};
    if (k != 5 && k != 6) continue;
    if (qb[g] < 0 || qb[g] >= nq || qb[g] == qa[g]) throw PlanError{CS_ERR_INVALID, "bad two-qubit gate"};
    const int sa = seg_of[size_t(qa[g])], sb = seg_of[size_t(qb[g])];
    if (sa == sb) continue;
    if (std::abs(sa - sb) != 1)
      throw PlanError{CS_ERR_TOPOLOGY, "gate at position " + std::to_string(g) + " spans non-adjacent segments " +
                                           std::to_string(sa) + " and " + std::to_string(sb)};
    cut_at[size_t(g)] = int(prep.cut_pos.size());
    prep.cut_pos.push_back(g);
    prep.cut_boundary.push_back(std::min(sa, sb));
    prep.cut_ctrl.push_back(sa);
    prep.cut_tgt.push_back(sb);
  }
  int first = 0;
  for (int s = 0; s < n; ++s) {
    SegmentPlan sp;
    sp.nq = sizes[s];
    sp.first = first;
    {
      // upper bound of this segment's rows: its share of the gates plus 3 per cut
      const size_t cap = size_t(G) * size_t(sizes[s]) / size_t(nq) + size_t(G) / 8 + 3 * prep.cut_pos.size() + 16;
      sp.kinds.reserve(cap);
      sp.qa.reserve(cap);
      sp.qb.reserve(cap);
      sp.params.reserve(3 * cap);
      sp.slots.reserve(cap);
    }
    auto put = [&](uint8_t k, int64_t a, int64_t b, const double* p, int32_t slot) {
      sp.kinds.push_back(k);
      sp.qa.push_back(a);
      sp.qb.push_back(b);
      sp.params.push_back(p ? p[0] : 0.0);
      sp.params.push_back(p ? p[1] : 0.0);
      sp.params.push_back(p ? p[2] : 0.0);
      sp.slots.push_back(slot);
    };
    for (int64_t g = 0; g < G; ++g) {
      const int c = cut_at[size_t(g)];
      if (c >= 0) {
        // cut: control side gets S/Sdg, target side S/Sdg (CZ) or H,S/Sdg,H (CX)
        const int32_t bit = int32_t(sp.cut_ids.size());
        if (prep.cut_ctrl[size_t(c)] == s) {
          sp.cut_ids.push_back(c);
          put(3, qa[g] - first, -1, nullptr, bit);
        } else if (prep.cut_tgt[size_t(c)] == s) {
          sp.cut_ids.push_back(c);
          const int64_t lq = qb[g] - first;
          if (kinds[g] == 5) {
            put(0, lq, -1, nullptr, -1);
            put(3, lq, -1, nullptr, bit);
            put(0, lq, -1, nullptr, -1);
          } else {
            put(3, lq, -1, nullptr, bit);
          }
        }
        continue;
      }
      if (seg_of[size_t(qa[g])] != s) continue;
      const bool two = kinds[g] == 5 || kinds[g] == 6;
      put(kinds[g], qa[g] - first, two ? qb[g] - first : -1, params ? params + 3 * g : nullptr, -1);
    }
    first += sizes[s];
    prep.segs.push_back(std::move(sp));
  }
  return prep;
}

std::string cut_prep_to_json(const CutPrep& prep) {
  std::ostringstream o;
  o.precision(17);
  o << "{\"n\":" << prep.n << ",\"cuts\":[";
  for (size_t c = 0; c < prep.cut_pos.size(); ++c)
    o << (c ? "," : "") << "[" << prep.cut_pos[c] << "," << prep.cut_boundary[c] << "," << prep.cut_ctrl[c] << ","
      << prep.cut_tgt[c] << "]";
  o << "],\"segments\":[";
  for (size_t s = 0; s < prep.segs.size(); ++s) {
    const SegmentPlan& sp = prep.segs[s];
    o << (s ? "," : "") << "{\"nq\":" << sp.nq << ",\"first\":" << sp.first << ",\"cut_ids\":[";
    for (size_t i = 0; i < sp.cut_ids.size(); ++i) o << (i ? "," : "") << sp.cut_ids[i];
    o << "],\"kinds\":[";
    for (size_t i = 0; i < sp.kinds.size(); ++i) o << (i ? "," : "") << int(sp.kinds[i]);
    o << "],\"qa\":[";
    for (size_t i = 0; i < sp.qa.size(); ++i) o << (i ? "," : "") << sp.qa[i];
    o << "],\"qb\":[";
    for (size_t i = 0; i < sp.qb.size(); ++i) o << (i ? "," : "") << sp.qb[i];
    o << "],\"slots\":[";
    for (size_t i = 0; i < sp.slots.size(); ++i) o << (i ? "," : "") << sp.slots[i];
    o << "],\"params\":[";
    for (size_t i = 0; i < sp.params.size(); ++i) o << (i ? "," : "") << sp.params[i];
    o << "]}";
  }
  o << "]}";
  return o.str();
}

// ---------------------------------------------------------------------------
// chain contraction plan
// ---------------------------------------------------------------------------
bool plan_chain(int n, const int32_t* seg_nq, const int32_t* seg_ncuts, const int32_t* seg_cut_ids,
                int c_total, const int32_t* cut_boundary, const double* term_coef, int force_bond,
                ChainPlan* out, PlanError* err) {
  if (n < 2) {
    *err = {CS_ERR_INVALID, "merging needs at least 2 segments"};
    return false;
  }
  if (c_total < 0 || c_total > 40) {
    *err = {CS_ERR_INVALID, "c_total out of range"};
    return false;
  }
  // cuts per boundary, and each cut's index within its boundary
  std::vector<std::vector<int>> bcuts(size_t(n - 1));
  std::vector<int> index_in_boundary(size_t(c_total), -1);
  for (int c = 0; c < c_total; ++c) {
    const int b = cut_boundary[c];
    if (b < 0 || b >= n - 1) {
      *err = {CS_ERR_INVALID, "cut " + std::to_string(c) + " on invalid boundary " + std::to_string(b)};
      return false;
    }
    index_in_boundary[size_t(c)] = int(bcuts[size_t(b)].size());
    bcuts[size_t(b)].push_back(c);
  }
  int total_q = 0;
  std::vector<int> offs(size_t(n) + 1, 0);
  for (int j = 0; j < n; ++j) {
    if (seg_nq[j] < 1 || seg_nq[j] > 40) {
      *err = {CS_ERR_INVALID, "segment qubit count out of range"};
      return false;
    }
    total_q += seg_nq[j];
    offs[size_t(j) + 1] = offs[size_t(j)] + seg_ncuts[j];
    const int expect = (j > 0 ? int(bcuts[size_t(j - 1)].size()) : 0) + (j < n - 1 ? int(bcuts[size_t(j)].size()) : 0);
    if (seg_ncuts[j] != expect) {
      *err = {CS_ERR_INVALID, "segment " + std::to_string(j) + " lists " + std::to_string(seg_ncuts[j]) +
                                  " adjacent cuts, boundaries imply " + std::to_string(expect)};
      return false;
    }
    for (int lb = 0; lb < seg_ncuts[j]; ++lb) {
      const int c = seg_cut_ids[offs[size_t(j)] + lb];
      if (c < 0 || c >= c_total || (cut_boundary[c] != j - 1 && cut_boundary[c] != j)) {
        *err = {CS_ERR_INVALID, "segment " + std::to_string(j) + " lists a non-adjacent cut"};
        return false;
      }
    }
  }
  if (total_q > 62) {
    *err = {CS_ERR_CAPACITY, "total qubit count exceeds 62"};
    return false;
  }
  auto cb = [&](int b) { return int(bcuts[size_t(b)].size()); };
  // r_j(x, y): local variant index of segment j for bond bits x (boundary j-1), y (boundary j)
  auto variant_of = [&](int j, int64_t x, int64_t y) {
    int64_t r = 0;
    for (int lb = 0; lb < seg_ncuts[j]; ++lb) {
      const int c = seg_cut_ids[offs[size_t(j)] + lb];
      const int pos = index_in_boundary[size_t(c)];
      const int64_t bit = (cut_boundary[c] == j - 1) ? ((x >> pos) & 1) : ((y >> pos) & 1);
      r |= bit << lb;
    }
    return int32_t(r);
  };
  auto alpha = [&](int64_t bits, int count, double* re, double* im) {
    double ar = 1, ai = 0;
    for (int a = 0; a < count; ++a) {
      const double* t = term_coef + 2 * ((bits >> a) & 1);
      const double nr = ar * t[0] - ai * t[1];
      ai = ar * t[1] + ai * t[0];
      ar = nr;
    }
    *re = ar;
    *im = ai;
  };
  // bond choice: minimise modelled time of the final product + intermediates
  const double bw = 6.5e12, f64 = 3.5e13;
  auto step_cost = [&](double out_amps, double terms) {
    return std::max(out_amps * 16.0 / bw, out_amps * terms * 8.0 / f64);
  };
  int best = 0;
  double best_cost = 1e300;
  for (int k = 0; k < n - 1; ++k) {
    double cost = step_cost(std::ldexp(1.0, total_q), std::ldexp(1.0, cb(k)));
    int ql = 0;
    for (int j = 0; j <= k; ++j) {
      ql += seg_nq[j];
      if (j >= 1) cost += step_cost(std::ldexp(1.0, ql + cb(j)), std::ldexp(1.0, cb(j - 1)));
    }
    int qr = 0;
    for (int j = n - 1; j > k; --j) {
      qr += seg_nq[j];
      if (j <= n - 2) cost += step_cost(std::ldexp(1.0, qr + cb(j - 1)), std::ldexp(1.0, cb(j)));
    }
    if (cost < best_cost * (1 - 1e-9)) {
      best_cost = cost;
      best = k;
    }
  }
  if (force_bond >= 0) {
    if (force_bond > n - 2) {
      *err = {CS_ERR_INVALID, "forced bond out of range"};
      return false;
    }
    best = force_bond;
  }
  const int k = best;
  ChainPlan plan;
  plan.bond = k;
  auto new_buf = [&](int64_t amps) {
    plan.buf_amps.push_back(amps);
    return n + int(plan.buf_amps.size()) - 1;
  };
  // left side: L_0 = segment 0, L_j = sum_x alpha(x) psi_j[r_j(x,y)] (x) L_{j-1}[x]
  int lbuf = 0;
  int64_t llen = int64_t(1) << seg_nq[0];
  for (int j = 1; j <= k; ++j) {
    MergeStep st;
    st.S = 1 << cb(j);
    st.K = 1 << cb(j - 1);
    st.hi_buf = j;
    st.lo_buf = lbuf;
    st.hi_len = int64_t(1) << seg_nq[j];
    st.lo_len = llen;
    st.out_buf = new_buf(int64_t(st.S) * st.hi_len * st.lo_len);
    for (int64_t y = 0; y < st.S; ++y)
      for (int64_t x = 0; x < st.K; ++x) {
        st.hidx.push_back(variant_of(j, x, y));
        st.lidx.push_back(int32_t(x));
        double re, im;
        alpha(x, cb(j - 1), &re, &im);
        st.coef.push_back(re);
        st.coef.push_back(im);
      }
    lbuf = st.out_buf;
    llen = st.hi_len * st.lo_len;
    plan.steps.push_back(std::move(st));
  }
  // right side: R_{n-1} = segment n-1, R_j[x] = sum_y alpha(y) R_{j+1}[y] (x) psi_j[r_j(x,y)]
  int rbuf = n - 1;
  int64_t rlen = int64_t(1) << seg_nq[n - 1];
  for (int j = n - 2; j > k; --j) {
    MergeStep st;
    st.S = 1 << cb(j - 1);
    st.K = 1 << cb(j);
    st.hi_buf = rbuf;
    st.lo_buf = j;
    st.hi_len = rlen;
    st.lo_len = int64_t(1) << seg_nq[j];
    st.out_buf = new_buf(int64_t(st.S) * st.hi_len * st.lo_len);
    for (int64_t x = 0; x < st.S; ++x)
      for (int64_t y = 0; y < st.K; ++y) {
        st.hidx.push_back(int32_t(y));
        st.lidx.push_back(variant_of(j, x, y));
        double re, im;
        alpha(y, cb(j), &re, &im);
        st.coef.push_back(re);
        st.coef.push_back(im);
      }
    rbuf = st.out_buf;
    rlen = st.hi_len * st.lo_len;
    plan.steps.push_back(std::move(st));
  }
  // final product across bond k
  MergeStep fin;
  fin.final_step = true;
  fin.S = 1;
  fin.K = 1 << cb(k);
  fin.hi_buf = rbuf;
  fin.lo_buf = lbuf;
  fin.hi_len = rlen;
  fin.lo_len = llen;
  fin.out_buf = -1;
  for (int64_t z = 0; z < fin.K; ++z) {
    fin.hidx.push_back(int32_t(z));
    fin.lidx.push_back(int32_t(z));
    double re, im;
    alpha(z, cb(k), &re, &im);
    fin.coef.push_back(re);
    fin.coef.push_back(im);
  }
  plan.steps.push_back(std::move(fin));
  int ql = 0;
  for (int j = 0; j <= k; ++j) ql += seg_nq[j];
  plan.q_low = ql;
  *out = std::move(plan);
  return true;
}

}  // namespace cutsim
