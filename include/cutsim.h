/*
 * libcutsim — C-ABI of the B200 (sm_100a) circuit-cutting state-vector path.
 *
 * The reference (`cutbench`, /root/reference/pkg/src/cutbench) is a Python +
 * numba package with no FFI; its internal compute seam is two numba kernels
 * called from Python:
 *     engine._run_gates(amps, kinds, qa, qb, start, stop)   engine.py:122-139
 *     merging._axpy_outer(acc, hi, lo, alpha)               merging.py:86-94
 * driven by simulate() (engine.py:158-168) and merge() (merging.py:156-186).
 * Each entry point below states which of those it replaces. A ctypes binding
 * is the reference-side integration.
 *
 * Conventions (identical to the reference): amplitudes are complex128
 * interleaved (re, im) little-endian (or complex64 with dtype CS_C64), index
 * order with qubit j = bit j (qubit 0 = LSB); segment 0 on the low bits; gate
 * kind codes H=0 X=1 T=2 S=3 Sdg=4 CX=5 CZ=6 (+ U3=7 with params[g] = theta,
 * phi, lambda); CX/CZ first qubit = control.
 *
 * Memory: every state pointer is caller-owned device memory (e.g. a torch
 * tensor's data_ptr()); the library never allocates or frees caller memory.
 * All calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default stream) except the reductions, which synchronise the stream to
 * return a host value. Every function returns CS_OK (0) or an error code;
 * cs_last_error() gives the thread's last message.
 */
#ifndef CUTSIM_H
#define CUTSIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_OK 0
#define CS_ERR_INVALID 1
#define CS_ERR_CAPACITY 2
#define CS_ERR_CUDA 3
#define CS_ERR_NCCL 4
#define CS_ERR_INTERNAL 5
#define CS_ERR_NODEVICE 6
#define CS_ERR_TOPOLOGY 7
#define CS_ERR_TIMEOUT 8   /* BudgetExceededError (cs_sim_batch_until) */

#define CS_C128 0
#define CS_C64 1

int cs_version(void);
const char* cs_last_error(void);
int cs_device_count(int32_t* count);

/* Options: "tile_bits" (multi-sweep tile, default 12 for c128),
 * "low_bits" (contiguous low qubits per tile, default 5), "fuse" (1q gate
 * fusion, default 1; 2 = U3 split into phase . Ry . phase with phases
 * commuted through diagonal gates), "threads" (0 = auto), "merge_streaming" (evict-first
 * output stores, default 1), "merge_iters" (0 = auto), "merge_dmma" (FP64
 * tensor-core merge for K = 8..64: 0 off, 1 four real GEMMs per complex
 * product, 2 three (3M); default 2), "engine" (1 register-tile
 * sweep kernel, 0 shared-memory tile kernel), "jit" (0 never, 1 from a
 * program's second use, 2 always: NVRTC-specialised sweep kernels compiled
 * on first use, 3 tiered: interpreter until a background compile is done —
 * see cs_jit_wait), "jit_struct" (structure-keyed modules with the
 * coefficients passed as kernel parameters, so circuits differing only in
 * angles share compiled code: 0 never, 1 small programs such as variant
 * batches (default; their 2x2s are not normalised), 2 always),
 * "jit_units_compiled" / "jit_units_reused" (read-only counters),
 * "merge_ozaki" (int8 tcgen05 tensor-core merge with exact FP64 splitting
 * for one-slot products of K >= "merge_ozaki_min_k" terms, lo_len % 128 == 0,
 * row ranges % 16 == 0, outputs * K >= 2^"merge_ozaki_min_work" (default
 * 24: smaller products run faster on the FP64 kernels); 1 = default: short-
 * lived unit CTAs for K <= 16 and >= 2^27 outputs, the persistent kernel
 * otherwise, 2 = unit CTAs,
 * 3 = persistent, 0 = off; min K 16), "merge_ozaki_digits" (8: 7
 * balanced base-256 digits per operand, 7 int32 diagonals per output,
 * truncation ~1e-15 of max|out| — default, q=30 K=16 in 3.0 ms; 7: 8
 * base-128 digits, 8 diagonals, ~6e-16, 8 % slower at K = 16), "cluster" (cluster-resident
 * variant batches: one NVRTC kernel per program, the 2^12..2^16-amplitude
 * states in the distributed shared memory of a CTA cluster; default 1),
 * "cluster_max" (CTAs per cluster at most: 2..16, default 16), "cluster_loop"
 * (the ahead-of-time cluster kernel that reads the program as an op stream,
 * cluster.cu: 1 = default, while a new program's NVRTC cluster kernel
 * compiles (it replaces the per-launch interpreter there); 2 = always; 0 = off),
 * "zero_start_tiles" (simulations
 * from |0..0> zero the states once and launch only the tiles that can be
 * non-zero; default 1), "zero_skip" (with zero-start tiles and the register-tile
 * kernels: a sweep does not load the amplitudes its tile-local zero mask marks as
 * still 0, and the zeroing pass is dropped when the sweeps hold every qubit;
 * default 1),
 * "jit_max_cost", "vb", "sweep_minb", "merge_smem_kb", "merge_dmma3_warps", "jit_minb", "dense_norm" (normalised 2x2s:
 * 0 off, 1 on, 2 = with the NVRTC kernels), "reg_bits", "plan_json" (tuning /
 * testing). */
int cs_set_option(const char* key, int64_t value);
int64_t cs_get_option(const char* key);

/* Kernels launched by this library since load (bench `gpu_launches`). */
int64_t cs_launch_count(void);

/* jit = 3 (tiered): programs run on the interpreter kernel while their
 * NVRTC modules compile on a background thread. Block until that queue is
 * drained (timeout_s < 0: no limit); CS_ERR_TIMEOUT if it is still busy. */
int cs_jit_wait(double timeout_s);

/* Set every state of a batch to the basis state |index>.
 * Replaces StateVec.zero_state (engine.py:47-51). */
int cs_init_basis(void* states, int32_t nq, int64_t n_states, int64_t index, int32_t dtype,
                  void* stream);

/* Apply a gate table to a batch of n_states states of nq qubits (state v at
 * states + v * state_stride amplitudes). slots may be NULL; slots[g] >= 0
 * marks an S gate that is Sdg for states whose variant id
 * (variant_base + v) has bit slots[g] set — one template serves all cut
 * variants of a segment. init_zero != 0 starts from |0..0> without reading.
 * Replaces _run_gates (engine.py:122-139) over the per-variant simulate()
 * loop (harness.py:136-139) and the variant tables of cutting.py:237-247. */
int cs_sim_batch(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                 const double* params, const int32_t* slots, int64_t n_gates, void* states,
                 int64_t n_states, int64_t state_stride, uint64_t variant_base, int32_t init_zero,
                 int32_t dtype, void* stream);

/* Every segment family of one decomposition in ONE call: family f has
 * nq[f] qubits, gate_count[f] consecutive rows of the concatenated tables
 * (kinds/qa/qb/params/slots, the layout cs_cut_tables writes) and
 * n_states[f] variant states (variant ids 0..n_states[f]-1, contiguous at
 * states[f], stride 2^nq[f]), all started from |0..0>. Families run
 * concurrently on the library's side streams forked from / joined into
 * `stream`. Replaces the per-variant simulate() loop of the reference's
 * harness (harness.py:136-139) for a whole SubcircuitSet
 * (pipeline.simulate_families). */
int cs_sim_families(int32_t n_fam, const int32_t* nq, const int64_t* gate_count, const uint8_t* kinds,
                    const int64_t* qa, const int64_t* qb, const double* params, const int32_t* slots,
                    void* const* states, const int64_t* n_states, int32_t dtype, void* stream);

/* cs_sim_batch with a cooperative budget (the reference's `deadline`,
 * engine.py:142-155): deadline_s is CLOCK_MONOTONIC seconds (Python's
 * time.monotonic()); the stream is synchronised after every sweep launch and
 * CS_ERR_TIMEOUT returned once the deadline has passed. The fused program is
 * the same as cs_sim_batch's. */
int cs_sim_batch_until(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                       const double* params, const int32_t* slots, int64_t n_gates, void* states,
                       int64_t n_states, int64_t state_stride, uint64_t variant_base, int32_t init_zero,
                       int32_t dtype, void* stream, double deadline_s);
/* Host-only: the sweep schedule cs_sim_batch would run, as JSON. tile_bits
 * <= 0 uses the current option. Writes up to buflen bytes, *needed = full
 * length + 1. */
int cs_sweep_plan_json(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                       const double* params, const int32_t* slots, int64_t n_gates,
                       int32_t tile_bits, int32_t dtype, char* buf, int64_t buflen, int64_t* needed);

/* Host-only self-test of the NVRTC path: schedule the gate table as
 * cs_sim_batch would, emit the specialised sweep kernels and compile them to
 * an sm_100a CUBIN (no device needed). *cubin_bytes = CUBIN size. */
int cs_jit_selftest(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                    const double* params, const int32_t* slots, int64_t n_gates, int64_t n_states,
                    int32_t dtype, int64_t* cubin_bytes);

/* out[s][h - row_begin][l] (+)= sum_{t<K} coef[s,t] * hi[hidx[s,t]][h] * lo[lidx[s,t]][l]
 * for h in [row_begin, row_end), l in [0, lo_len); hi states have hi_len
 * amplitudes, lo states lo_len (a power of two); slot s of out starts at
 * out + s * out_slot_stride amplitudes. hidx/lidx/coef are HOST arrays of
 * S*K (coef: 2*S*K doubles, (re, im)). accumulate != 0 adds into out.
 * Replaces _axpy_outer/_outer_into/_iadd and the per-term loop
 * (merging.py:86-186) with one write-once pass per output. */
int cs_merge_terms(int32_t S, int32_t K, const int32_t* hidx, const int32_t* lidx,
                   const double* coef, const void* hi, int64_t hi_len, const void* lo,
                   int64_t lo_len, int64_t row_begin, int64_t row_end, void* out,
                   int64_t out_slot_stride, int32_t accumulate, int32_t dtype, void* stream);

/* Plan of the chain-contracted merge (host only). Segments 0..n-1 (segment 0
 * on the low bits) with seg_nq[j] qubits hold 2^{seg_ncuts[j]} states each;
 * seg_cut_ids lists, per segment and concatenated, the global cut ids
 * adjacent to it in circuit order (local variant bit k = k-th id); cut c sits
 * on boundary cut_boundary[c]; term_coef = {t0.re, t0.im, t1.re, t1.im}.
 * This is exactly the reference merge table r_i(m) (cutting.py:251-263) and
 * alpha_m (cutting.py:266-272). force_bond < 0 picks the bond by cost. */
int cs_merge_chain_plan(int32_t n, const int32_t* seg_nq, const int32_t* seg_ncuts,
                        const int32_t* seg_cut_ids, int32_t c_total, const int32_t* cut_boundary,
                        const double* term_coef, int32_t force_bond, int32_t dtype,
                        int64_t* workspace_bytes, int32_t* bond, int32_t* q_low);

/* Full-state reconstruction sum_m alpha_m psi_{n-1}^{r(m)} (x) ... (x) psi_0^{r(m)}
 * for output amplitudes [out_begin, out_end) (multiples of 2^{q_low}; out
 * points at amplitude out_begin) — the shard a GPU owns. seg_states[j] is a
 * device pointer to segment j's 2^{seg_ncuts[j]} x 2^{seg_nq[j]} states.
 * Replaces merge() (merging.py:156-186). */
int cs_merge_chain(int32_t n, const int32_t* seg_nq, const void* const* seg_states,
                   const int32_t* seg_ncuts, const int32_t* seg_cut_ids, int32_t c_total,
                   const int32_t* cut_boundary, const double* term_coef, int32_t force_bond,
                   int64_t out_begin, int64_t out_end, void* out, void* workspace,
                   int64_t workspace_bytes, int32_t dtype, void* stream);

/* ---- the cut pipeline as one call -------------------------------------------
 * Preprocess (reference plan_cut_sizes + decompose, cutting.py:82-136,
 * 190-283) on the host in C++, simulate every segment's variant family in
 * batched sweeps (segments on internal side streams joined back into
 * `stream`), and write amplitudes [out_begin, out_end) of the reconstructed
 * state (chain merge) into `out` — the reference's _cut_once
 * (harness.py:125-145) behind one entry point. seg_sizes has n_seg entries
 * summing to nq. The variant states and merge intermediates live in the
 * caller's `workspace` (size from cs_cut_workspace); out_begin/out_end must
 * be multiples of 2^q_low. stage_events (nullable: 3 cudaEvent_t) are
 * recorded on `stream` before the subcircuit stage, between it and the merge,
 * and after the merge (no synchronisation). stage_ms (nullable, 3 doubles)
 * receives the host preprocess time and the event-timed subcircuit and merge
 * stages (the call then synchronises `stream`). */
int cs_cut_workspace(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                     const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                     int32_t force_bond, int32_t dtype, int64_t* workspace_bytes, int32_t* q_low,
                     int32_t* c_total);
int cs_cut_run(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
               const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
               int32_t force_bond, int64_t out_begin, int64_t out_end, void* out, void* workspace,
               int64_t workspace_bytes, int32_t dtype, void* stream, void* const* stage_events,
               double* stage_ms);
/* Copy `bytes` of device memory to host memory and return when the host copy
 * is complete (after the work queued on `stream`). A pinned destination is
 * one cudaMemcpyAsync; a pageable one (e.g. a numpy array) goes through a
 * ring of pinned staging buffers drained by a pool of host threads, near the
 * PCIe rate instead of the driver's pageable path. Replaces the host copy
 * behind the reference's numpy results (StateVec.amps, engine.py:30-45). */
int cs_copy_to_host(void* host, const void* device, int64_t bytes, void* stream);

/* The same pipeline delivering the full 2^nq state into HOST memory
 * (host_out: 2^nq amplitudes, ideally pinned) — the reference API's contract
 * of a host-resident result. The merge runs in `chunks` row ranges into two
 * device staging buffers (part of `workspace`, size from
 * cs_cut_host_workspace) and each chunk's device-to-host copy overlaps the
 * next chunk's merge; returns when host_out is complete. stage_ms
 * (nullable): host preprocess, variant stage, merge + copies. */
int cs_cut_host_workspace(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                          const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                          int32_t chunks, int32_t dtype, int64_t* workspace_bytes);
int cs_cut_run_to_host(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                       const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                       int32_t chunks, void* host_out, void* workspace, int64_t workspace_bytes,
                       int32_t dtype, void* stream, double* stage_ms);
/* ---- the sharded (multi-GPU) cut pipeline, one call per rank -----------------
 * the output is sharded on its high amplitude bits and the
 * subcircuit variants are split across ranks. All segments must have equal
 * qubit counts: the segments' variant batches, concatenated segment-major,
 * form one array of `total` states split into `world` chunks of `per` states;
 * rank r simulates chunk r IN PLACE in its workspace and one in-place NCCL
 * all-gather (the pipeline's only exchange) completes the array on every rank
 * — it is exactly the segment batches the chain merge reads. Each rank then
 * writes output amplitudes [out_begin, out_end) (its rows of the reference
 * merge's result, merging.py:156-186) into `out`. comm = NULL: no exchange,
 * the rank simulates every variant itself (one GPU computing any rank's
 * share). The reference is single-process; this has no reference
 * counterpart beyond computing rows of merge().
 * cs_cut_shard_plan (host only) fills info[8] = {workspace bytes, q_low,
 * default out_begin, default out_end (rank's rows), first and end flat
 * variant index of the rank's chunk, per, total}.
 * stage_events (nullable): 4 cudaEvent_t recorded before the variant stage,
 * after it, after the all-gather and after the merge; stage_ms (nullable,
 * 4 doubles): host preprocess, variant stage, exchange, merge (synchronises). */
int cs_cut_shard_plan(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                      const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int32_t world,
                      int32_t rank, int32_t dtype, int64_t* info);
int cs_cut_run_sharded(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                       int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, void* comm, int32_t world,
                       int32_t rank, int64_t out_begin, int64_t out_end, void* out, void* workspace,
                       int64_t workspace_bytes, int32_t dtype, void* stream, void* const* stage_events,
                       double* stage_ms);
/* Host-only: the C++ preprocess as flat tables — replaces plan_cut_sizes +
 * decompose (cutting.py:70-136, 190-248). cuts[4j..4j+3] = position,
 * boundary, control segment, target segment of cut j; seg_counts[2s],
 * [2s+1] = template gates and adjacent cuts of segment s; the segments'
 * template tables (local qubits; slots[g] = cut bit patching gate g, or -1)
 * and adjacent-cut ids are concatenated in segment order. needed[0..1] =
 * total template gates, c_total; when they exceed gate_cap / cut_cap only
 * `needed` is written. */
int cs_cut_tables(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                  const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                  int64_t* cuts, int32_t* seg_counts, uint8_t* out_kinds, int64_t* out_qa,
                  int64_t* out_qb, double* out_params, int32_t* out_slots, int32_t* out_cut_ids,
                  int64_t gate_cap, int64_t cut_cap, int64_t* needed);
/* Host-only: the C++ preprocess result as JSON (cuts and per-segment
 * template tables with their cut slots) — checked against the Python
 * planner and the reference's golden tables in the CPU tests. */
int cs_cut_describe_json(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                         const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                         char* buf, int64_t buflen, int64_t* needed);

/* Device reductions (synchronise `stream`). */
int cs_maxabsdiff(const void* a, const void* b, int64_t n, int32_t dtype, double* result,
                  void* stream);
int cs_maxabs(const void* a, int64_t n, int32_t dtype, double* result, void* stream);
/* result[0..1] = sum conj(a) * b */
int cs_inner(const void* a, const void* b, int64_t n, int32_t dtype, double* result, void* stream);

/* out[i] = state[idx[i]] (idx, out: device pointers). */
int cs_gather(const void* state, const int64_t* idx, int64_t m, void* out, int32_t dtype,
              void* stream);

/* Multi-GPU plumbing over NCCL (NVLink / NVSwitch), one process per GPU
 * (SURVEY.md §8(b) item 6, §8(e)). The reference is single-process, so these
 * replace no reference symbol; they carry the sharded pipeline's single
 * exchange (parallel.gather_states) and the distributed simulator's
 * half-shard swaps (distributed.simulate_distributed). libnccl.so.2 is
 * dlopen'ed on first use (or from `path` via cs_nccl_load). */
int cs_nccl_load(const char* path);
/* rank 0 creates the 128-byte id; the caller distributes it to all ranks */
int cs_nccl_unique_id(uint8_t* id128);
int cs_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id128, int32_t device, void** comm);
int cs_nccl_comm_destroy(void* comm);
/* recv[r * bytes_per_rank ...] = rank r's send buffer, for every rank r */
int cs_allgather_states(void* comm, const void* send, int64_t bytes_per_rank, void* recv, void* stream);
/* exchange `bytes` with `peer` (grouped ncclSend + ncclRecv) */
int cs_sendrecv(void* comm, const void* send, void* recv, int64_t bytes, int32_t peer, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CUTSIM_H */
