// Host-side planning of libcutsim (pure C++, no CUDA): gate lowering and
// fusion, sweep scheduling for tiled state vectors, and the chain-contraction
// plan of the merge.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "ops.hpp"

namespace cutsim {

struct PlanError {
  int code;  // CS_ERR_*
  std::string msg;
};

// One lowered op on global qubits. Slotted ops carry both alternatives.
struct LOp {
  int16_t type = OP_DENSE;
  int target = -1;        // DENSE target qubit
  uint64_t mask = 0;      // DENSE: control qubits; PHASE: phase qubits
  int slot = -1;
  double m[8] = {0};      // bit-0 alternative (or the only one)
  double alt[8] = {0};    // bit-1 alternative when slot >= 0
};

// Lower the packed table (reference kinds 0..6, U3 = 7) into ops.
// slots may be null; slots[g] >= 0 marks an S gate that becomes Sdg for
// variant bit slots[g] = 1.
// split_u3: U3(th, ph, la) = diag(1, e^{i ph}) . Ry(th) . diag(1, e^{i la})
// (a real rotation between two phases) instead of one dense complex matrix.
std::vector<LOp> lower_gates(int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                             const double* params, const int32_t* slots, int64_t n_gates,
                             bool split_u3 = false);

// Merge runs of single-qubit ops on the same qubit (no intervening op on it).
// same_type_only: never fold a phase into a dense op (keeps real rotations
// real for the specialised kernels, where a phase costs 2 and a real 2x2
// 4 FP64 instructions per amplitude against 7 for a complex 2x2).
std::vector<LOp> fuse_ops(const std::vector<LOp>& ops, bool same_type_only = false);

// Rewrite every uncontrolled dense 2x2 M as D . M' with M' having a 1 in
// each row (pivot = the row's larger entry, so the other |entry| <= 1) and
// push the diagonal D into the next dense op on that qubit (M_next . D):
// a normalised complex 2x2 costs 4 FP64 instructions per amplitude in the
// specialised kernels (the 1-coefficient term is the FMA accumulator)
// instead of 7. Pending diagonals are emitted as phase ops (times a global
// scalar) before an op that does not commute with them (a controlled dense
// op on that target) and at the end; the global scalar is folded into the
// last dense op, which stays un-normalised. Normalising inflates the executed
// state by up to 1/2 bit per op; whenever the total would exceed
// max_growth_bits an op is emitted un-normalised (with the pending diagonal
// and scalar applied), restoring the true scale.
// fixed_pivot: every row is divided by its DIAGONAL entry (unless that is
// below 1e-12 of the other one: the growth budget bounds the inflation a
// small pivot causes; the precision of a + x b does not depend on |x|), so
// which coefficients become 1 depends on the gate structure, not on the
// angles (param-mode kernels, jit_struct)
std::vector<LOp> normalize_dense(const std::vector<LOp>& ops, int nq, double max_growth_bits,
                                 bool fixed_pivot = false);

// Defer single-qubit phases past everything they commute with (diagonal
// ops, dense ops controlled by or not touching their qubit) and merge the
// phases of one qubit; a qubit's pending phase is emitted right before the
// next dense op that targets it (or at the end).
std::vector<LOp> commute_phases(const std::vector<LOp>& ops);

struct Sweep {
  int tile_bits = 0, low_bits = 0;
  std::vector<int> hq;           // qubits of local bits [L, T)
  std::vector<int> oq;           // qubits selected by the tile id
  // started from |0..0>, only the tiles t < 2^zero_tiles_log2 can hold a
  // non-zero amplitude when this sweep runs: oq lists the qubits some earlier
  // sweep held in its tile first (a dense op never moves amplitude across
  // tiles, so a qubit no earlier sweep held is still 0 everywhere)
  int zero_tiles_log2 = 0;
  // tile-local index bits ([0, L): qubit q; L + j: hq[j]) whose qubit no
  // earlier sweep held: started from |0..0>, every amplitude with one of them
  // set is still 0 when this sweep runs, so its load can be skipped (and the
  // state need not be zeroed first when the sweeps together hold every qubit)
  uint32_t zero_local_mask = 0;
  std::vector<SweepOp> entries;  // slotted ops take two consecutive entries
};

// Greedy tiling: every sweep holds the low qubits [0, L) plus up to T - L
// more qubits chosen in order of first need; it absorbs every op whose
// non-diagonal target is in the tile and that commutes with all deferred ops.
// windows: tile-set policy (-1 = the sweep_windows option; 3 = cost-aware
// for a start from |0..0>)
std::vector<Sweep> schedule_sweeps(const std::vector<LOp>& ops, int nq, int tile_bits, int low_bits,
                                  int max_group = kMaxGroup, int windows = -1);

// Threads per CTA of the sweep kernel for a tile of 2^T amplitudes, and the
// largest register group that still gives every thread a cell.
int sweep_threads(int tile_bits);
int sweep_max_group(int tile_bits);

std::string sweeps_to_json(const std::vector<Sweep>& sweeps, int nq);

// Register-tile lowering of one sweep: register bits per thread for a tile of
// 2^T amplitudes, and the op list translated to register coordinates with the
// REMAPs it needs (ends in the canonical mapping, register bits = top bits).
int reg_bits_for(int tile_bits);
extern int g_reg_bits;
extern int g_reg_reorder;
extern int g_sweep_windows;  // option "sweep_windows": also try contiguous qubit windows as tile sets  // option "reg_reorder": list-schedule commuting ops to save remaps  // option "reg_bits": 0 = automatic, 2..4 = override where valid
std::vector<RegOp> reg_program(const Sweep& sw, int reg_bits);
std::string reg_programs_to_json(const std::vector<Sweep>& sweeps, int nq);

// ---- merge chain -----------------------------------------------------------
struct MergeStep {
  int hi_buf, lo_buf, out_buf;  // buffer ids: 0..n-1 segment states, n.. workspace
  int64_t hi_len, lo_len;
  int S, K;
  std::vector<int32_t> hidx, lidx;  // S*K
  std::vector<double> coef;         // 2*S*K
  bool final_step = false;
};

struct ChainPlan {
  int bond = 0;
  int q_low = 0;                      // qubits of the low (L) side of the final product
  std::vector<int64_t> buf_amps;      // workspace buffers (amplitudes), ids n..
  std::vector<MergeStep> steps;
};

// ---- cut preprocess (reference cutting.py:82-136, 190-248) -----------------
struct SegmentPlan {
  int nq = 0;
  int first = 0;
  std::vector<uint8_t> kinds;
  std::vector<int64_t> qa, qb;
  std::vector<double> params;   // 3 per gate
  std::vector<int32_t> slots;   // cut bit patching the gate, or -1
  std::vector<int32_t> cut_ids; // adjacent cuts in circuit order (local variant bit = index)
};

struct CutPrep {
  int n = 0;
  std::vector<int32_t> sizes;
  std::vector<int64_t> cut_pos;
  std::vector<int32_t> cut_boundary, cut_ctrl, cut_tgt;
  std::vector<SegmentPlan> segs;
  int c_total() const { return int(cut_pos.size()); }
};

// Throws PlanError: CS_ERR_INVALID (bad sizes / table), CS_ERR_TOPOLOGY
// (a two-qubit gate spans non-adjacent segments).
CutPrep cut_prepare(int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                    int64_t n_gates, int n_seg, const int32_t* sizes);
std::string cut_prep_to_json(const CutPrep& prep);

bool plan_chain(int n, const int32_t* seg_nq, const int32_t* seg_ncuts, const int32_t* seg_cut_ids,
                int c_total, const int32_t* cut_boundary, const double* term_coef, int force_bond,
                ChainPlan* out, PlanError* err);

}  // namespace cutsim
