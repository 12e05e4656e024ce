// Shared host/device structures of libcutsim (sm_100a).
//
// The gate program the kernels execute is a list of two op types, lowered on
// the host from the reference's packed gate table (kinds/qa/qb, reference
// engine.py:122-139) plus this build's U3 params and cut-slot column:
//   OP_DENSE : 2x2 complex matrix on one target qubit, optionally controlled
//              (H, X, U3, CX, and fused runs of 1q gates);
//   OP_PHASE : multiply every amplitude whose index has all `mask` bits set by
//              a complex phase (T, S, Sdg, CZ and fused diagonal runs).
// An op with slot >= 0 is a *cut slot*: the variant id's bit `slot` selects
// between this entry (bit 0 -> S side) and the next entry (bit 1 -> Sdg side),
// which is how one template table serves every subcircuit variant
// (reference cutting.py:237-247 patches a kind byte; we select a matrix).
#pragma once
#include <cstdint>

namespace cutsim {

enum : int16_t { OP_DENSE = 0, OP_PHASE = 1 };

// One op as seen by a sweep kernel. Masks are split into the bits that live
// inside the tile (lmask, tile-local positions) and the bits that select the
// tile (omask, global qubit positions, constant over a tile).
struct SweepOp {
  uint32_t lmask;     // DENSE: local control bits; PHASE: local phase bits
  int16_t type;
  int16_t target;     // DENSE: tile-local target bit
  uint64_t omask;     // outside-tile qubits that must be 1 for the op to act
  int32_t slot;       // -1, or cut bit choosing this entry (0) / next entry (1)
  int32_t gsize;      // DENSE, first op of a register group: ops in the group (1..4)
  double m[8];        // DENSE: m00 m01 m10 m11 as (re,im); PHASE: m[0..1]
};
static_assert(sizeof(SweepOp) == 88, "SweepOp layout");

constexpr int kMaxTileBits = 14;
constexpr int kMaxGroup = 4;           // dense ops applied together in registers
constexpr int kMaxOpsPerLaunch = 352;  // keeps SweepParams under the 32 KiB param limit
constexpr int kSmallOps = 40;          // small-program launch (about 4 KiB of params)

template <int CAP>
struct SweepParamsT {
  void* states;             // batch of states, state v at states + v * stride
  int64_t stride;           // amplitudes between consecutive states
  uint64_t variant_base;    // variant id of state 0 of this launch
  int32_t nq;               // qubits per state
  int32_t tile_bits;        // T
  int32_t low_bits;         // L: local bits [0, L) are qubits [0, L)
  int32_t n_high;           // T - L local bits mapped to qubits hq[]
  int32_t n_out;            // nq - T outside qubits, tile id bit j -> oq[j]
  int32_t n_ops;
  int32_t init_basis;       // 1: ignore memory, start from |0..0>
  int32_t n_states;         // states in this launch (CTA group y holds VB of them)
  int8_t hq[kMaxTileBits];
  int8_t oq[64];
  SweepOp ops[CAP];
};
using SweepParams = SweepParamsT<kMaxOpsPerLaunch>;
using SweepParamsSmall = SweepParamsT<kSmallOps>;
static_assert(sizeof(SweepParams) <= 32760, "kernel parameter limit");

// Register-tile program (rsweep_kernel): the tile's 2^T amplitudes live in
// registers, 2^RB per thread; register bit k of a thread's amplitude index is
// tile bit rpos[k] of the current mapping, the thread index bits are the other
// tile bits in ascending order. Gates act on register bits only; REMAP
// changes which tile bits are register bits (one shared-memory transpose).
enum : uint8_t { ROP_DENSE = 0, ROP_PHASE = 1, ROP_REMAP = 2 };

struct alignas(16) RegOp {
  uint8_t kind;
  uint8_t k;          // DENSE: target register bit
  int16_t slot;       // -1, or cut bit choosing this entry (0) / next entry (1)
  uint32_t tmask;     // thread-index bits that must be 1 (controls / phase bits)
  uint32_t rmask;     // register-index bits that must be 1
  uint8_t rpos[4];    // REMAP: tile bit of each register bit
  uint64_t omask;     // outside-tile qubits that must be 1
  uint64_t pad;
  double m[8];        // 16-byte aligned: four 128-bit shared-memory loads
};
static_assert(sizeof(RegOp) == 96, "RegOp layout");
constexpr int kMaxRegOps = 320;        // RegParams under the 32 KiB param limit
constexpr int kMidRegOps = 96;         // launch tiers between kSmallOps and kMaxRegOps (9 / 17 KiB)
constexpr int kLargeRegOps = 176;

template <int CAP>
struct RegParamsT {
  void* states;
  int64_t stride;
  uint64_t variant_base;
  int32_t tile_bits, low_bits, n_high, n_out, n_ops, init_basis, n_states;
  uint32_t zmask;           // tile-local bits whose amplitudes are known 0 (Sweep::zero_local_mask): not loaded
  int8_t hq[kMaxTileBits];
  int8_t oq[64];
  RegOp ops[CAP];
};
using RegParams = RegParamsT<kMaxRegOps>;
using RegParamsSmall = RegParamsT<kSmallOps>;
static_assert(sizeof(RegParams) <= 32760, "kernel parameter limit");

// merge_terms: out[s][h - row_begin][l] (+)= sum_t coef[s,t] hi[hidx[s,t]][h] lo[lidx[s,t]][l]
constexpr int kMaxMergeTerms = 1024;

struct MergeParams {
  const void* hi;           // [n_hi][hi_len]
  const void* lo;           // [n_lo][lo_len]
  void* out;                // slot s at out + s * out_slot_stride; row h at (h - row_begin) * W
  int64_t hi_len;           // amplitudes per hi state (= rows)
  int64_t lo_len;           // W = amplitudes per lo state (= columns)
  int64_t row_begin, row_end;
  int64_t out_slot_stride;
  int32_t log_w;
  int32_t S, K;             // slots, terms per slot
  int32_t accumulate;       // 0: overwrite, 1: add into out
  int32_t cols;             // min(W, C) columns covered by one row group
  int32_t log_cols;
  int32_t rows_per_iter;    // C / cols
  int32_t iters;            // row groups per CTA
  int32_t streaming;        // st.global.cs for the output
  int32_t hidx[kMaxMergeTerms];
  int32_t lidx[kMaxMergeTerms];
  double coef[2 * kMaxMergeTerms];
};
static_assert(sizeof(MergeParams) <= 32760, "kernel parameter limit");

}  // namespace cutsim
