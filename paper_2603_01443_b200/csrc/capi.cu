// extern "C" entry points of libcutsim (see include/cutsim.h for the contract
// and the reference interfaces each one replaces).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <thread>
#include <chrono>
#include <cstdlib>
#include <csignal>
#include <execinfo.h>
#include <unistd.h>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/cutsim.h"
#include "ops.hpp"
#include "plan.hpp"
#include "jit.hpp"
#include "cluster.hpp"

#include <nvtx3/nvToolsExt.h>

namespace cutsim {
extern int g_sweep_minb;
size_t sweep_smem_bytes(int tile_bits, int low_bits, int dtype, int n_ops, int vb);
cudaError_t launch_sweep(const SweepParams& p, uint32_t n_tiles, int vb, int threads, cudaStream_t stream,
                         int dtype);
cudaError_t launch_rsweep(const RegParams& p, int rb, uint32_t n_tiles, uint32_t n_states, cudaStream_t stream,
                          int dtype);
cudaError_t launch_merge(const MergeParams& p, int K, dim3 grid, int threads, size_t smem, bool wide,
                         cudaStream_t stream, int dtype);
int merge_cols_per_thread(int K);
cudaError_t launch_merge_dmma(const MergeParams& p, int K, dim3 grid, int threads, size_t smem,
                              cudaStream_t stream);
int merge_dmma_cols_per_warp(int K);
cudaError_t launch_merge_dmma3(const MergeParams& p, int K, int warps, dim3 grid, size_t smem,
                               cudaStream_t stream);
int merge_dmma3_cols_per_warp(int K);
int merge_dmma3_row_blocks(int K);
bool merge_ozaki_supported(int K, int64_t lo_len, int64_t nrows);
cudaError_t launch_merge_ozaki(const MergeParams& mp, int64_t nrows, void* out, int accumulate, int sms, bool unit,
                               cudaStream_t stream, int digit_bits);
cudaError_t launch_init_basis(void* states, int64_t len, int64_t n_states, int64_t index, int dtype,
                              cudaStream_t stream);
cudaError_t launch_reduce(const void* a, const void* b, int64_t n, int mode, int dtype, double2* scratch,
                          cudaStream_t stream);
int reduce_scratch_elems();
cudaError_t launch_gather(const void* state, const int64_t* idx, int64_t m, void* out, int dtype,
                          cudaStream_t stream);
}  // namespace cutsim

using namespace cutsim;

namespace {

// Debug aid (env CUTSIM_SEGV_TRACE=1 at load): a SIGSEGV prints the native
// backtrace of the faulting thread to stderr before the default action.
void segv_trace(int sig) {
  void* fr[64];
  const int n = backtrace(fr, 64);
  const char msg[] = "libcutsim: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(fr, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvTraceInstaller {
  SegvTraceInstaller() {
    const char* e = std::getenv("CUTSIM_SEGV_TRACE");
    if (e && *e == '1') signal(SIGSEGV, segv_trace);
  }
} g_segv_trace_installer;

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

struct Options {
  int64_t tile_bits_c128 = 12;
  int64_t tile_bits_c64 = 13;
  int64_t tile_bits = 0;  // 0 = per-dtype default
  int64_t low_bits = 5;
  int64_t fuse = 1;
  int64_t dense_norm = 2;  // normalised dense 2x2s: 0 off, 1 on, 2 when NVRTC kernels are enabled
  int64_t threads = 0;
  int64_t merge_streaming = 1;
  int64_t merge_iters = 0;
  int64_t vb = 0;  // states per CTA in a variant batch (0 = auto)
  int64_t merge_dmma3_warps = 8;  // warps per CTA of the 3M kernel (8: 2 CTAs/SM, 4: 4 CTAs/SM)
  int64_t merge_smem_kb = 96;  // staged-row budget per CTA of the tensor-core merge
  int64_t merge_dmma = 2;  // FP64 tensor-core merge: 1 = four real GEMMs, 2 = three (3M)
  int64_t zero_start_tiles = 1;   // from |0..0>: zero the states once, launch only the tiles that can be non-zero
  int64_t zero_skip = 1;  // with zero-start tiles: skip loads of still-zero amplitudes, and the zeroing when the sweeps hold every qubit
  int64_t merge_ozaki = 1;        // int8 tcgen05 merge (exact FP64 splitting) for K >= merge_ozaki_min_k: 1 auto (unit CTAs for K <= 16, else persistent), 2 unit CTAs, 3 persistent; 0 off
  int64_t merge_ozaki_min_k = 16;
  int64_t merge_ozaki_min_work = 24;  // log2 of outputs * K below which the FP64 kernels run
  int64_t merge_ozaki_digits = 8;  // digit bits of the int8 merge: 8 (7 base-256 slices, default: q=30 K=16 3.0 vs 3.27 ms) or 7 (8 base-128 slices, half the truncation)
  int64_t engine = 1;      // 1: register-tile kernel (rsweep), 0: shared-memory tile kernel (sweep)
  int64_t jit = 0;         // 0 never, 1 from a program's 2nd use, 2 always (compile on first use, blocking),
                           // 3 tiered: the interpreter runs while the module compiles on a background thread
  int64_t cluster = 1;      // cluster-resident variant batches (one kernel, states in DSMEM) with the NVRTC kernels
  int64_t cluster_max = 16; // CTAs per cluster at most (16 = the non-portable size)
  int64_t cluster_loop = 1; // cluster.cu's op-stream kernel: 1 = until the NVRTC cluster kernel is compiled, 2 = always
  int64_t jit_struct = 1;  // param-mode (structure-keyed) modules: 0 never, 1 for small programs (< 2^22
                           // amplitudes: variant batches), 2 always
  int64_t jit_max_cost = 40000;  // FP64 instructions per specialised launch (code-size guard)
  int64_t plan_json = 0;   // cs_sweep_plan_json: 0 sweeps, 1 register programs
} g_opt;
std::mutex g_opt_mu;

// NVTX ranges (header-only nvtx3: free without an attached tool): every
// entry point and the pipeline's stages show up by name in Nsight
// Systems / Compute (e.g. ncu --nvtx --nvtx-include "cs_cut_run/merge/")
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(CS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t elem_bytes(int dtype) { return dtype == CS_C128 ? 16 : 8; }

bool valid_dtype(int dtype) { return dtype == CS_C128 || dtype == CS_C64; }

int multi_tile_bits(int dtype) {
  if (g_opt.tile_bits > 0) return int(g_opt.tile_bits);
  return int(dtype == CS_C128 ? g_opt.tile_bits_c128 : g_opt.tile_bits_c64);
}

struct ScratchCache {
  std::mutex mu;
  std::vector<double2*> per_device;
} g_scratch;

double2* reduce_scratch(int* err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *err = cuda_fail(e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  if (int(g_scratch.per_device.size()) <= dev) g_scratch.per_device.resize(size_t(dev) + 1, nullptr);
  if (!g_scratch.per_device[size_t(dev)]) {
    double2* p = nullptr;
    e = cudaMalloc(&p, sizeof(double2) * size_t(reduce_scratch_elems()));
    if (e != cudaSuccess) {
      *err = cuda_fail(e, "cudaMalloc(reduce scratch)");
      return nullptr;
    }
    g_scratch.per_device[size_t(dev)] = p;
  }
  return g_scratch.per_device[size_t(dev)];
}

int choose_vb(int64_t n_states) {
  if (g_opt.engine == 1) return 1;
  if (g_opt.vb > 0) return int(std::min<int64_t>(g_opt.vb, 4));
  // measured (tools/tune_sub.py): 2 states per CTA beats 1 and 4 for cut variants
  return n_states >= 2 ? 2 : 1;
}

int group_budget(int vb, int dtype) {
  const int minb = vb == 1 ? g_sweep_minb : 2;
  const int values = (dtype == CS_C128 ? 8 : 16) * 2 / minb / vb;
  return values >= 16 ? 4 : values >= 8 ? 3 : values >= 4 ? 2 : 1;
}

int single_tile_max_vb(int dtype, int vb) {
  // the tile of vb states must fit shared memory next to the op list; the
  // register kernel runs at most 512 threads x 16 amplitudes
  if (g_opt.engine == 1) return 13;
  int t = dtype == CS_C128 ? 13 : 14;
  while (t > 6 && ((size_t(1) << t) * (dtype == CS_C128 ? 16 : 8) * size_t(vb)) > size_t(128 * 1024)) --t;
  return t;
}

int choose_tile_bits(int nq, int64_t n_states, int tile_bits, int dtype) {
  const int vb = choose_vb(n_states);
  if (tile_bits > 0) return std::min(tile_bits, nq);
  if (g_opt.tile_bits > 0) return std::min(int(g_opt.tile_bits), nq);
  // one CTA per state runs the whole circuit in shared memory; for 12-13
  // qubit states in small batches that leaves most SMs idle and runs long
  // straight-line code once per CTA, so they take the chip-filling
  // multi-tile path below (measured, NVRTC kernels, 4 variants per segment:
  // 12 qubits 63 -> 46 us, 13 qubits 104 -> 49 us; at <= 11 qubits the
  // single tile stays faster: 10 qubits 26 vs 37 us)
  const bool small_batch = n_states > 1 && n_states < 148 && nq >= 12;
  if (nq <= single_tile_max_vb(dtype, vb) && !small_batch) return nq;
  const int dflt = multi_tile_bits(dtype);
  if (n_states > 1) {
    // small batches of mid-size states (cut variants): shrink the tile until
    // the grid covers the chip (the states are L2-resident anyway)
    const int64_t groups = (n_states + vb - 1) / vb;
    const int64_t want = (148 + groups - 1) / groups;
    int lg = 0;
    while ((int64_t(1) << lg) < want) ++lg;
    return std::max(9, std::min(std::min(dflt, single_tile_max_vb(dtype, vb)), nq - lg));
  }
  return dflt;
}

// Cluster size (log2) of the cluster-resident form, 0 = not used: the NVRTC
// kernels must be on, the state 2^12..2^16 amplitudes, and a CTA's chunk
// plus its transpose scratch within 64 KiB (T <= 11 for complex128, 12 for
// complex64). Clusters as large as cluster_max allows while the batch's CTAs
// still fit the chip once (more CTAs per state = more SMs on the FP64 work).
int choose_cluster_bits(int nq, int64_t n_states, int dtype) {
  if (!g_opt.cluster || g_opt.jit == 0 || g_opt.engine != 1 || nq < 12 || nq > 16) return 0;
  // chunks of 2^11 amplitudes (32 KiB complex128: 8 amplitudes per thread,
  // 128 registers); 2^12-amplitude chunks (16 per thread, ~220 registers,
  // one 8-warp CTA per SM) measured 2-3x slower than the per-launch kernels
  const int tmax = dtype == CS_C128 ? 11 : 12;
  int cmax = 0;
  while ((int64_t(2) << cmax) <= g_opt.cluster_max) ++cmax;  // log2(cluster_max)
  int want = 0;
  while (want < cmax && (n_states << (want + 1)) <= 148) ++want;
  const int cb = std::max(nq - tmax, want);
  if (cb > cmax || nq - cb < 8) return 0;
  return cb;
}

struct Launch {
  int sweep = 0;
  std::vector<SweepOp> entries;  // engine 0
  std::vector<RegOp> reg;        // engine 1
};
struct Program {
  std::vector<Sweep> sweeps;
  std::vector<Launch> launches;
  int engine = 1;
  // NVRTC-specialised kernels, built once the program is hot (jit.cpp)
  mutable std::mutex jit_mu;
  mutable std::shared_ptr<JitModule> jit;
  mutable bool jit_tried = false;
  mutable std::atomic<int> uses{0};
  int64_t n_states = 1;  // states per launch the program was scheduled for
  bool param_mode = false;  // structure-keyed kernels with the coefficients as kernel parameters
  int cluster_bits = 0;     // > 0: every sweep tiles the state into 2^cluster_bits tiles (one per cluster CTA)
  // the sweeps' tiles together hold every qubit: a start from |0..0> with
  // zero-start tiles writes every amplitude and never reads one before it
  // was written (Sweep::zero_local_mask), so the states need no zeroing
  bool covers_all_qubits = false;
  // cluster_loop: the program as an op stream for cluster.cu's
  // ahead-of-time kernel (null: the NVRTC cluster kernel / per-launch form)
  std::unique_ptr<ClusterBlob> cloop;
};

// content-keyed program cache with least-recently-used eviction (a clear-all
// policy recompiled the NVRTC kernels of a program between a sweep point's
// warm-up and its timed repetitions once 256 programs had accumulated)
struct CacheEntry {
  std::shared_ptr<const Program> prog;
  uint64_t last_use = 0;
};
constexpr size_t kProgramCacheCap = 512;
std::mutex g_cache_mu;
std::unordered_map<std::string, CacheEntry> g_cache;
uint64_t g_cache_clock = 0;

// Split each sweep's entries into launches that fit the kernel parameter
// block (never splitting a slotted pair); the register kernel's chunks are
// smaller because its REMAPs add entries.
void build_launches(Program& prog) {
  const size_t cap = prog.engine == 1 ? size_t(kMaxRegOps / 2 - 4) : size_t(kMaxOpsPerLaunch);
  for (size_t s = 0; s < prog.sweeps.size(); ++s) {
    const Sweep& sw = prog.sweeps[s];
    size_t i0 = 0;
    do {
      size_t i1 = i0;
      while (i1 < sw.entries.size()) {
        const size_t w = sw.entries[i1].slot >= 0 ? 2 : 1;
        if (i1 + w - i0 > cap) break;
        i1 += w;
      }
      Launch l;
      l.sweep = int(s);
      l.entries.assign(sw.entries.begin() + long(i0), sw.entries.begin() + long(i1));
      if (prog.engine == 1) {
        if (i0 == 0 && i1 == sw.entries.size()) {
          l.reg = reg_program(sw, reg_bits_for(sw.tile_bits));
        } else {
          Sweep part;
          part.tile_bits = sw.tile_bits;
          part.low_bits = sw.low_bits;
          part.hq = sw.hq;
          part.oq = sw.oq;
          part.zero_tiles_log2 = sw.zero_tiles_log2;
          part.entries = l.entries;
          l.reg = reg_program(part, reg_bits_for(sw.tile_bits));
        }
      }
      prog.launches.push_back(std::move(l));
      i0 = i1;
    } while (i0 < sw.entries.size());
  }
}

// Zero-start tiles pay from a few MiB of states up (below, the extra zeroing
// launch costs more than the tiles it saves: the variant stage's small
// L2-resident batches)
bool zero_start_pays(int64_t n_states, int nq) { return (n_states << nq) >= (int64_t(1) << 22); }

// Lowered, fused and scheduled program for a gate table; cached by content.
std::shared_ptr<const Program> build_schedule(int nq, const uint8_t* kinds, const int64_t* qa,
                                                         const int64_t* qb, const double* params,
                                                         const int32_t* slots, int64_t n_gates, int64_t n_states,
                                                         int tile_bits, int dtype, bool zero_start) {
  // cluster-resident form (started from |0..0>, NVRTC kernels, 12..16
  // qubits): the state lives in the shared memory of a cluster of 2^cb CTAs,
  // each holding a 2^T chunk (T = nq - cb); sweeps become phases of ONE kernel
  const int cb = (zero_start && tile_bits <= 0) ? choose_cluster_bits(nq, n_states, dtype) : 0;
  const int T = cb ? nq - cb : choose_tile_bits(nq, n_states, tile_bits, dtype);
  const int L = (T == nq) ? nq : std::max(3, std::min(int(g_opt.low_bits), T - 6));
  const int vb = choose_vb(n_states);
  std::string key;
  key.reserve(size_t(n_gates) * 45 + 32);
  // fuse 2 (split U3 + commuted phases) measured slower than fused complex
  // 2x2s even with the specialised kernels (cfg4a uncut 286 vs 212 ms: a
  // phase on a thread bit diverges, and the longer op list grows the
  // straight-line code), so it stays opt-in
  const int fuse = int(g_opt.fuse);
  // normalised 2x2s only pay where the 1-coefficients become free (the
  // NVRTC-specialised kernels); the interpreter keeps the plain matrices
  // param mode: small (latency-bound) programs get structure-keyed kernels;
  // their 2x2s are normalised by the diagonal entries (a structural pivot,
  // plan.cpp normalize_dense) so the kernel source does not depend on angles
  const bool param_mode = g_opt.jit != 0 && g_opt.engine == 1 &&
                          (g_opt.jit_struct == 2 || (g_opt.jit_struct == 1 && !zero_start_pays(n_states, nq)));
  const int norm = g_opt.dense_norm == 2 ? (g_opt.jit != 0 && g_opt.engine == 1 ? 1 : 0) : int(g_opt.dense_norm);
  // the cost-aware tile-set policy (3) only pays for a start from |0..0>
  // (zero-start tiles); other starts keep the most-absorbed-ops policy
  const int windows = (g_sweep_windows == 3 && !(zero_start && g_opt.zero_start_tiles &&
                                                 zero_start_pays(n_states, nq)))
                          ? 1
                          : g_sweep_windows;
  const int32_t hdr[16] = {nq, T, L, int32_t(fuse), slots ? 1 : 0, dtype, vb, g_sweep_minb,
                           int32_t(g_opt.engine), norm, g_reg_bits * 8 + g_reg_reorder * 4 + windows, g_jit_minb,
                           g_jit_persistent, param_mode ? 1 : 0, cb, int32_t(g_opt.cluster_loop)};
  key.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
  key.append(reinterpret_cast<const char*>(kinds), size_t(n_gates));
  key.append(reinterpret_cast<const char*>(qa), size_t(n_gates) * 8);
  key.append(reinterpret_cast<const char*>(qb), size_t(n_gates) * 8);
  if (params) key.append(reinterpret_cast<const char*>(params), size_t(n_gates) * 24);
  if (slots) key.append(reinterpret_cast<const char*>(slots), size_t(n_gates) * 4);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      it->second.last_use = ++g_cache_clock;
      return it->second.prog;
    }
  }
  std::vector<LOp> ops = lower_gates(nq, kinds, qa, qb, params, slots, n_gates, fuse == 2);
  if (fuse == 2) ops = fuse_ops(commute_phases(ops), true);
  else if (fuse == 1) ops = fuse_ops(ops);
  // growth budget: amplitudes stay below 2^200 (c128) / 2^20 (c64)
  if (norm) ops = normalize_dense(ops, nq, dtype == CS_C128 ? 200.0 : 20.0, param_mode);
  // register groups hold 2^k x vb complex values: 8 (c128) / 16 (c64) per thread
  const int max_group = std::min(sweep_max_group(T), group_budget(vb, dtype));
  auto built = std::make_shared<Program>();
  built->engine = int(g_opt.engine);
  built->n_states = n_states;
  built->param_mode = param_mode;
  built->cluster_bits = cb;
  built->sweeps = schedule_sweeps(ops, nq, T, L, max_group, windows);
  {
    uint64_t held = 0;
    for (const Sweep& sw : built->sweeps) {
      for (int q = 0; q < sw.low_bits; ++q) held |= 1ull << q;
      for (int q : sw.hq) held |= 1ull << q;
    }
    built->covers_all_qubits = held == (nq >= 64 ? ~0ull : (1ull << nq) - 1ull);
  }
  build_launches(*built);
  if (cb > 0 && g_opt.cluster_loop && built->engine == 1) {
    std::vector<const Sweep*> sw;
    std::vector<const std::vector<RegOp>*> rp;
    for (const Launch& ln : built->launches) {
      sw.push_back(&built->sweeps[size_t(ln.sweep)]);
      rp.push_back(&ln.reg);
    }
    auto cl = std::make_unique<ClusterBlob>();
    std::string why;
    if (cluster_blob_build(sw, rp, T, dtype, cl.get(), &why)) built->cloop = std::move(cl);
  }
  std::shared_ptr<const Program> prog = built;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cache.size() >= kProgramCacheCap) {
    auto lru = g_cache.begin();
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
      if (it->second.last_use < lru->second.last_use) lru = it;
    g_cache.erase(lru);
  }
  g_cache[std::move(key)] = CacheEntry{prog, ++g_cache_clock};
  return prog;
}

bool dmma_eligible(int K, int dtype, int64_t lo_len) {
  return g_opt.merge_dmma && dtype == CS_C128 && (K == 8 || K == 16 || K == 32 || K == 64) &&
         lo_len >= merge_dmma_cols_per_warp(K);
}

// SMs of the current device (cached per device: a process may drive several)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev & 63];
  int n = slot.load();
  if (!n) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
    slot.store(n);
  }
  return n;
}

// merge_dmma = 2: the three-GEMM (3M) tensor-core kernel where it is
// instantiated (K = 8, 16, 32); K = 64 keeps the four-GEMM kernel
bool dmma3_eligible(int K, int dtype, int64_t lo_len) {
  return g_opt.merge_dmma == 2 && dtype == CS_C128 && (K == 8 || K == 16 || K == 32 || K == 64) &&
         lo_len >= merge_dmma3_cols_per_warp(K);
}

// merge_ozaki: the int8 tcgen05 kernel (ozaki.cu) for K >= merge_ozaki_min_k
// and the product is big enough to amortise its digit-prep launch:
// outputs * K >= 2^merge_ozaki_min_work (tools/merge_small_q.py, one
// combined 4-lane prep launch: q=20 K=16 16 vs 15 us FP64, K=64 23 vs 35;
// q=22 K=16 27 vs 34; q=24 K=16 61 vs 95; K = 8 stays on the FP64 kernels)
bool ozaki_eligible(int K, int dtype, int64_t lo_len, int64_t nrows) {
  return g_opt.merge_ozaki && dtype == CS_C128 && K >= g_opt.merge_ozaki_min_k &&
         double(nrows) * double(lo_len) * double(K) >= std::ldexp(1.0, int(g_opt.merge_ozaki_min_work)) &&
         merge_ozaki_supported(K, lo_len, nrows);
}

// Launch one merge_terms problem whose K is one instantiated width.
int merge_launch_one(int S, int Kc, const int32_t* hidx, const int32_t* lidx, const double* coef,
                     int64_t stride_terms, const void* hi, int64_t hi_len, const void* lo, int64_t lo_len,
                     int64_t row_begin, int64_t row_end, void* out, int64_t out_slot_stride, int accumulate,
                     int dtype, cudaStream_t stream) {
  // stride_terms: distance between consecutive slots' term lists in hidx/lidx
  const int threads = 256;
  const size_t eb0 = elem_bytes(dtype);
  if (ozaki_eligible(Kc, dtype, lo_len, row_end - row_begin)) {
    // int8 tensor-core merge (ozaki.cu): one problem per slot
    static MergeParams po;
    static std::mutex pom;
    std::lock_guard<std::mutex> lk(pom);
    for (int s = 0; s < S; ++s) {
      std::memset(&po, 0, offsetof(MergeParams, hidx));
      po.hi = hi;
      po.lo = lo;
      po.hi_len = hi_len;
      po.lo_len = lo_len;
      po.row_begin = row_begin;
      po.row_end = row_end;
      po.S = 1;
      po.K = Kc;
      for (int t = 0; t < Kc; ++t) {
        const int64_t src = int64_t(s) * stride_terms + t;
        po.hidx[t] = hidx[src];
        po.lidx[t] = lidx[src];
        po.coef[2 * t] = coef[2 * src];
        po.coef[2 * t + 1] = coef[2 * src + 1];
      }
      void* o = static_cast<char*>(out) + size_t(s) * size_t(out_slot_stride) * elem_bytes(dtype);
      // short-lived unit CTAs (two per SM) for K <= 16 and >= 2^27 outputs,
      // the persistent kernel otherwise (tools/ozaki_ab.py merge_ozaki=2,3:
      // K=16 at q=30 2.97 vs 3.23 ms, q=28 0.74 vs 0.76, q=26 0.215 vs
      // 0.204, q=24 71 vs 64 us; K=32 at q=30 4.40 vs 4.25 ms)
      const bool unit = g_opt.merge_ozaki == 2 ||
                        (g_opt.merge_ozaki == 1 && Kc <= 16 && double(row_end - row_begin) * double(lo_len) >= 0x1p27);
      cudaError_t e = launch_merge_ozaki(po, row_end - row_begin, o, accumulate, sm_count(), unit,
                                         stream, int(g_opt.merge_ozaki_digits));
      g_launches.fetch_add(3);
      if (e != cudaSuccess) return cuda_fail(e, "merge_ozaki launch");
    }
    return CS_OK;
  }
  const bool m3 = dmma3_eligible(Kc, dtype, lo_len);
  if (m3 || dmma_eligible(Kc, dtype, lo_len)) {
    // tensor-core path: 8 warps over ncg column groups of (16, 8 or 4)
    // complex columns; a CTA spans >= 128 columns so row staging is amortised
    const int64_t cw = m3 ? merge_dmma3_cols_per_warp(Kc) : merge_dmma_cols_per_warp(Kc);
    const int64_t ncg = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(8, 256 / cw), lo_len / cw));
    const int warps3 = Kc == 64 ? 8 : int(g_opt.merge_dmma3_warps);
    // K = 64 (3M) runs one CTA per SM: twice the staging budget
    const int64_t smem_budget = m3 ? g_opt.merge_smem_kb * 1024 * warps3 / 8 * (Kc == 64 ? 2 : 1)
                                   : g_opt.merge_smem_kb * 1024;
    const int64_t C = cw * ncg;
    const int64_t nrows = row_end - row_begin;
    const int RS = m3 ? 3 * Kc + 4 : 2 * Kc + 4;
    // row blocks processed together
    const int64_t rbg = m3 ? merge_dmma3_row_blocks(Kc) : 8 / (merge_dmma_cols_per_warp(Kc) / 4);
    int64_t iters = std::max<int64_t>(1, std::min<int64_t>(smem_budget / (8 * RS * 8), (nrows + 7) / 8));
    iters = std::min<int64_t>(iters, 64);
    // keep at least two CTAs per SM for small products
    const int64_t col_blocks = std::max<int64_t>(1, lo_len / C);
    iters = std::min<int64_t>(iters, std::max<int64_t>(1, ((nrows + 7) / 8) * col_blocks * S / (2 * 148)));
    iters = std::max<int64_t>(rbg, iters / rbg * rbg);
    const int64_t rows_cta = iters * 8;
    const size_t smem = size_t(rows_cta) * size_t(RS) * sizeof(double);
    const int slots_per_launch = std::max(1, kMaxMergeTerms / Kc);
    static MergeParams pd;
    static std::mutex pdm;
    std::lock_guard<std::mutex> lk(pdm);
    for (int s0 = 0; s0 < S; s0 += slots_per_launch) {
      const int sc = std::min(slots_per_launch, S - s0);
      std::memset(&pd, 0, offsetof(MergeParams, hidx));
      pd.hi = hi;
      pd.lo = lo;
      pd.hi_len = hi_len;
      pd.lo_len = lo_len;
      pd.out_slot_stride = out_slot_stride;
      pd.S = sc;
      pd.K = Kc;
      pd.accumulate = accumulate;
      pd.iters = int32_t(iters);
      pd.cols = int32_t(ncg);
      pd.streaming = int32_t(g_opt.merge_streaming);
      for (int s = 0; s < sc; ++s)
        for (int t = 0; t < Kc; ++t) {
          const int64_t src = int64_t(s0 + s) * stride_terms + t;
          pd.hidx[s * Kc + t] = hidx[src];
          pd.lidx[s * Kc + t] = lidx[src];
          pd.coef[2 * (s * Kc + t)] = coef[2 * src];
          pd.coef[2 * (s * Kc + t) + 1] = coef[2 * src + 1];
        }
      const int64_t max_rows_per_launch = rows_cta * 65535;
      for (int64_t r0 = row_begin; r0 < row_end; r0 += max_rows_per_launch) {
        const int64_t r1 = std::min(row_end, r0 + max_rows_per_launch);
        pd.row_begin = r0;
        pd.row_end = r1;
        char* base_out = static_cast<char*>(out) + size_t(s0) * size_t(out_slot_stride) * eb0;
        pd.out = base_out + size_t(r0 - row_begin) * size_t(lo_len) * eb0;
        dim3 grid(unsigned(lo_len / C), unsigned((r1 - r0 + rows_cta - 1) / rows_cta), unsigned(sc));
        cudaError_t e = m3 ? launch_merge_dmma3(pd, Kc, warps3, grid, smem, stream)
                           : launch_merge_dmma(pd, Kc, grid, threads, smem, stream);
        g_launches.fetch_add(1);
        if (e != cudaSuccess) return cuda_fail(e, "merge_dmma_kernel launch");
      }
    }
    return CS_OK;
  }
  const int CC = merge_cols_per_thread(Kc);
  const int64_t C = int64_t(threads) * CC;
  const int64_t W = lo_len;
  const bool wide = W >= C;
  const int64_t cols = wide ? C : W;
  const int64_t rows_per_iter = wide ? 1 : C / W;
  const size_t eb = elem_bytes(dtype);
  const int64_t nrows = row_end - row_begin;
  int64_t iters = g_opt.merge_iters > 0 ? g_opt.merge_iters
                                        : std::max<int64_t>(1, (256 * 1024) / int64_t(C * int64_t(eb)));
  const int64_t smem_cap = 32 * 1024;
  iters = std::min<int64_t>(iters, std::max<int64_t>(1, smem_cap / (rows_per_iter * Kc * int64_t(eb))));
  iters = std::min<int64_t>(iters, (nrows + rows_per_iter - 1) / rows_per_iter);
  iters = std::max<int64_t>(iters, 1);
  const int64_t rows_cta = iters * rows_per_iter;
  const size_t smem = size_t(rows_cta) * size_t(Kc) * eb;
  int log_w = 0;
  while ((int64_t(1) << log_w) < W) ++log_w;
  int log_cols = 0;
  while ((int64_t(1) << log_cols) < cols) ++log_cols;

  const int slots_per_launch = std::max(1, kMaxMergeTerms / Kc);
  static MergeParams p;  // large; filled per launch (launch copies it)
  static std::mutex pm;
  std::lock_guard<std::mutex> lk(pm);
  for (int s0 = 0; s0 < S; s0 += slots_per_launch) {
    const int sc = std::min(slots_per_launch, S - s0);
    std::memset(&p, 0, offsetof(MergeParams, hidx));
    p.hi = hi;
    p.lo = lo;
    p.out = static_cast<char*>(out) + size_t(s0) * size_t(out_slot_stride) * eb;
    p.hi_len = hi_len;
    p.lo_len = lo_len;
    p.out_slot_stride = out_slot_stride;
    p.log_w = log_w;
    p.S = sc;
    p.K = Kc;
    p.accumulate = accumulate;
    p.cols = int32_t(cols);
    p.log_cols = log_cols;
    p.rows_per_iter = int32_t(rows_per_iter);
    p.iters = int32_t(iters);
    p.streaming = int32_t(g_opt.merge_streaming);
    for (int s = 0; s < sc; ++s)
      for (int t = 0; t < Kc; ++t) {
        const int64_t src = int64_t(s0 + s) * stride_terms + t;
        p.hidx[s * Kc + t] = hidx[src];
        p.lidx[s * Kc + t] = lidx[src];
        p.coef[2 * (s * Kc + t)] = coef[2 * src];
        p.coef[2 * (s * Kc + t) + 1] = coef[2 * src + 1];
      }
    // row chunks so that grid.y stays within limits
    const int64_t max_rows_per_launch = rows_cta * 65535;
    for (int64_t r0 = row_begin; r0 < row_end; r0 += max_rows_per_launch) {
      const int64_t r1 = std::min(row_end, r0 + max_rows_per_launch);
      p.row_begin = r0;
      p.row_end = r1;
      char* base_out = static_cast<char*>(out) + size_t(s0) * size_t(out_slot_stride) * eb;
      p.out = base_out + size_t(r0 - row_begin) * size_t(W) * eb;
      dim3 grid(unsigned(wide ? W / C : 1), unsigned((r1 - r0 + rows_cta - 1) / rows_cta), unsigned(sc));
      cudaError_t e = launch_merge(p, Kc, grid, threads, smem, wide, stream, dtype);
      g_launches.fetch_add(1);
      if (e != cudaSuccess) return cuda_fail(e, "merge_kernel launch");
    }
  }
  return CS_OK;
}

int merge_terms_impl(int S, int K, const int32_t* hidx, const int32_t* lidx, const double* coef,
                     const void* hi, int64_t hi_len, const void* lo, int64_t lo_len, int64_t row_begin,
                     int64_t row_end, void* out, int64_t out_slot_stride, int accumulate, int dtype,
                     cudaStream_t stream) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (S < 1 || K < 0) return fail(CS_ERR_INVALID, "merge needs S >= 1 and K >= 0");
  if (lo_len < 1 || (lo_len & (lo_len - 1))) return fail(CS_ERR_INVALID, "lo_len must be a power of two");
  if (hi_len < 1 || row_begin < 0 || row_end > hi_len || row_begin > row_end)
    return fail(CS_ERR_INVALID, "row range outside [0, hi_len]");
  if (S > 1 && out_slot_stride < (row_end - row_begin) * lo_len)
    return fail(CS_ERR_INVALID, "out_slot_stride smaller than one slot");
  if (!out || (K > 0 && (!hi || !lo))) return fail(CS_ERR_INVALID, "null device pointer");
  if (row_end == row_begin) return CS_OK;
  const size_t eb = elem_bytes(dtype);
  if (K == 0) {
    if (accumulate) return CS_OK;
    for (int s = 0; s < S; ++s) {
      cudaError_t e = cudaMemsetAsync(static_cast<char*>(out) + size_t(s) * size_t(out_slot_stride) * eb, 0,
                                      size_t(row_end - row_begin) * size_t(lo_len) * eb, stream);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    }
    return CS_OK;
  }
  // split K into instantiated chunk widths: {64, 32} on the tensor-core path,
  // then {16, 8, 4, 2, 1}
  int t0 = 0;
  int acc = accumulate;
  while (t0 < K) {
    int rem = K - t0;
    int kc = rem >= 16 ? 16 : rem >= 8 ? 8 : rem >= 4 ? 4 : rem >= 2 ? 2 : 1;
    if (rem >= 64 && (dmma_eligible(64, dtype, lo_len) || ozaki_eligible(64, dtype, lo_len, row_end - row_begin)))
      kc = 64;
    else if (rem >= 32 && (dmma_eligible(32, dtype, lo_len) || ozaki_eligible(32, dtype, lo_len, row_end - row_begin)))
      kc = 32;
    int rc = merge_launch_one(S, kc, hidx + t0, lidx + t0, coef + 2 * t0, K, hi, hi_len, lo, lo_len, row_begin,
                              row_end, out, out_slot_stride, acc, dtype, stream);
    if (rc != CS_OK) return rc;
    t0 += kc;
    acc = 1;
  }
  return CS_OK;
}

// Compile a program's specialised kernels (sets prog.jit; caller holds jit_mu).
void compile_program_jit(const Program& prog, int dtype) {
  std::vector<const Sweep*> sw;
  std::vector<const std::vector<RegOp>*> rp;
  std::vector<int> minb;
  std::vector<char> pers;
  bool any = false;
  for (const Launch& ln : prog.launches) {
    const Sweep& s = prog.sweeps[size_t(ln.sweep)];
    sw.push_back(&s);
    // two CTAs per SM only pays when the launch has CTAs to fill them (and
    // whole-state tiles can spill under the 128-register cap)
    const int64_t ctas = (int64_t(1) << s.oq.size()) * prog.n_states;
    // many tiles of one state: the persistent prefetching form (one CTA per
    // SM); else one CTA per tile, two per SM when there are enough
    const bool p = g_jit_persistent && prog.n_states == 1 && (int64_t(1) << s.oq.size()) >= 4 * 148;
    pers.push_back(p ? 1 : 0);
    minb.push_back(p ? 1 : (ctas >= 2 * 148 ? g_jit_minb : 1));
    const bool ok = jit_cost(ln.reg, reg_bits_for(s.tile_bits)) <= g_opt.jit_max_cost;
    rp.push_back(ok ? &ln.reg : nullptr);
    any |= ok;
  }
  if (!any) return;
  std::string err;
  if (prog.cluster_bits > 0 && std::all_of(rp.begin(), rp.end(), [](const auto* r) { return r != nullptr; })) {
    // the whole program as one cluster-resident kernel; if that cannot be
    // built the same schedule runs as per-launch kernels
    auto cm = jit_compile_cluster(sw, rp, prog.sweeps[0].tile_bits, dtype, &err, prog.param_mode);
    if (cm) {
      prog.jit = cm;
      return;
    }
  }
  auto mod = jit_compile(sw, rp, dtype, &err, &minb, &pers, prog.param_mode);
  if (!mod) g_err = "JIT unavailable, using the interpreter kernel: " + err;
  prog.jit = mod;
}

// Tiered compilation (jit = 3): one background thread compiles queued
// programs while their calls run on the interpreter kernel.
struct JitQueue {
  std::mutex mu;
  std::condition_variable cv, idle_cv;
  std::deque<std::pair<std::shared_ptr<const Program>, int>> q;
  int busy = 0;
  bool started = false;
  bool stopping = false;  // process exit: no new jobs (drain_jit_queue)
};
// never destroyed: the detached worker waits on cv for the life of the
// process, and destroying a condition variable with a waiter blocks exit
JitQueue& g_jitq = *new JitQueue;

void jit_worker(int device) {
  cudaSetDevice(device);
  for (;;) {
    std::pair<std::shared_ptr<const Program>, int> job;
    {
      std::unique_lock<std::mutex> lk(g_jitq.mu);
      g_jitq.cv.wait(lk, [] { return !g_jitq.q.empty() || g_jitq.stopping; });
      if (g_jitq.stopping) return;
      job = std::move(g_jitq.q.front());
      g_jitq.q.pop_front();
      ++g_jitq.busy;
    }
    {
      std::lock_guard<std::mutex> lk(job.first->jit_mu);
      compile_program_jit(*job.first, job.second);
    }
    std::lock_guard<std::mutex> lk(g_jitq.mu);
    --g_jitq.busy;
    g_jitq.idle_cv.notify_all();
  }
}

// At process exit: drop the queued programs and wait for the one being
// compiled, so the worker never runs inside (or after) the destruction of
// the unit cache, NVRTC and the CUDA context it uses — a process that exited
// mid-compile crashed inside nvrtcCompileProgram (CUTSIM_SEGV_TRACE
// backtrace). Exit handlers and library destructors run in reverse order of
// registration, so this is registered after NVRTC (and the builtins library
// its first compile loads) is loaded: jit_warm_nvrtc() first.
void drain_jit_queue() {
  std::unique_lock<std::mutex> lk(g_jitq.mu);
  g_jitq.q.clear();
  g_jitq.stopping = true;
  g_jitq.cv.notify_all();
  g_jitq.idle_cv.wait_for(lk, std::chrono::seconds(60), [] { return g_jitq.busy == 0; });
}

void enqueue_jit(std::shared_ptr<const Program> prog, int dtype) {
  std::lock_guard<std::mutex> lk(g_jitq.mu);
  if (g_jitq.stopping) return;
  if (!g_jitq.started) {
    int dev = 0;
    cudaGetDevice(&dev);
    jit_warm_nvrtc();  // once per process, ~0.1 s: see drain_jit_queue
    std::atexit(drain_jit_queue);
    std::thread(jit_worker, dev).detach();
    g_jitq.started = true;
  }
  g_jitq.q.emplace_back(std::move(prog), dtype);
  g_jitq.cv.notify_one();
}

// The program's specialised kernels, compiling them on first demand (engine
// 1). jit = 3: never blocks — a program whose kernels are not compiled yet is
// queued for the background compiler and runs on the interpreter meanwhile.
std::shared_ptr<JitModule> program_jit(const std::shared_ptr<const Program>& pp, int dtype) {
  const Program& prog = *pp;
  if (prog.engine != 1 || g_opt.jit == 0) return nullptr;
  const int uses = ++prog.uses;
  if (g_opt.jit == 1 && uses < 2) return nullptr;
  if (g_opt.jit == 3) {
    std::unique_lock<std::mutex> lk(prog.jit_mu, std::try_to_lock);
    if (!lk.owns_lock()) return nullptr;  // the background compiler holds it
    if (prog.jit_tried) return prog.jit;
    prog.jit_tried = true;
    lk.unlock();
    enqueue_jit(pp, dtype);
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(prog.jit_mu);
  if (prog.jit_tried) return prog.jit;
  prog.jit_tried = true;
  compile_program_jit(prog, dtype);
  return prog.jit;
}

std::mutex g_cluster_launch_mu;  // launch_cluster_prog's static parameter blocks

// deadline_s > 0: CLOCK_MONOTONIC seconds (Python's time.monotonic()); the
// stream is synchronised after every launch and CS_ERR_TIMEOUT returned once
// it has passed (the reference's cooperative budget, engine.py:142-155)
int run_program(const std::shared_ptr<const Program>& prog_ptr, int nq, void* states, int64_t n_states,
                int64_t state_stride, uint64_t variant_base, int init_zero, int dtype, cudaStream_t st,
                double deadline_s = 0.0) {
  const Program* prog = prog_ptr.get();
  // cluster-resident op-stream kernel (cluster.cu): no NVRTC, one launch.
  // cluster_loop 1: the first tier while the NVRTC cluster kernel compiles
  // (it replaces the per-launch interpreter there); 2: always
  auto run_cloop = [&]() -> int {
    std::lock_guard<std::mutex> lk(g_cluster_launch_mu);
    for (int64_t v0 = 0; v0 < n_states; v0 += 65535) {
      const int64_t vc = std::min<int64_t>(65535, n_states - v0);
      void* sp = static_cast<char*>(states) + size_t(v0) * size_t(state_stride) * elem_bytes(dtype);
      const cudaError_t e =
          launch_cluster_prog(*prog->cloop, sp, state_stride, variant_base + uint64_t(v0), uint32_t(vc), st);
      g_launches.fetch_add(1);
      if (e != cudaSuccess) return cuda_fail(e, "cluster program launch");
    }
    return CS_OK;
  };
  const bool cloop_ok = prog->cloop && deadline_s <= 0.0;
  if (cloop_ok && g_opt.cluster_loop == 2) return run_cloop();
  std::shared_ptr<JitModule> jit = program_jit(prog_ptr, dtype);
  if (cloop_ok && !jit) return run_cloop();
  static SweepParams p;
  static RegParams rp;
  static std::mutex pm;
  std::lock_guard<std::mutex> lk(pm);
  bool first = true;
  size_t li = 0;
  // Started from |0..0>, a sweep's tiles beyond 2^zero_tiles_log2 are still
  // all zero (Sweep::zero_tiles_log2): zero the states once and launch only
  // the others (cfg4a uncut: the first sweep is one tile instead of 2^18)
  const bool sparse = init_zero && g_opt.zero_start_tiles && zero_start_pays(n_states, nq) &&
                      std::any_of(prog->launches.begin(), prog->launches.end(), [&](const Launch& l) {
                        const Sweep& s0 = prog->sweeps[size_t(l.sweep)];
                        return s0.zero_tiles_log2 < nq - s0.tile_bits;
                      });
  // with the register-tile kernels, a sweep skips the loads of amplitudes its
  // zero_local_mask marks as still 0; when the sweeps hold every qubit, every
  // amplitude is then written before it is read and the zeroing pass (16 B
  // per amplitude) goes (cfg4a uncut: 2.6 ms of HBM writes)
  const bool skip_zero_loads = sparse && prog->engine == 1 && g_opt.zero_skip;
  if (sparse && !(skip_zero_loads && prog->covers_all_qubits)) {
    // exactly the states (the caller may keep other data between strided states)
    const size_t eb = elem_bytes(dtype);
    cudaError_t e = state_stride == (int64_t(1) << nq)
                        ? cudaMemsetAsync(states, 0, size_t(n_states) * (size_t(1) << nq) * eb, st)
                        : cudaMemset2DAsync(states, size_t(state_stride) * eb, 0, (size_t(1) << nq) * eb,
                                            size_t(n_states), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  }
  if (jit && jit->cluster > 0 && jit->units[0] && deadline_s <= 0.0) {
    // the cluster-resident kernel: one launch, one cluster of jit->cluster
    // CTAs per state (blockIdx.y = variant), the whole program in DSMEM
    JitUnit* ju = jit->units[0].get();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaSuccess;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(ju->attrs_set.load(std::memory_order_relaxed) & bit)) {
      e = cudaKernelSetAttributeForDevice(ju->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ju->smem), dev);
      if (e == cudaSuccess && jit->cluster > 8)
        e = cudaKernelSetAttributeForDevice(ju->kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1, dev);
      if (e != cudaSuccess) return cuda_fail(e, "cluster kernel attributes");
      ju->attrs_set.fetch_or(bit);
    }
    const std::vector<unsigned char>& blob = jit->blobs[0];
    for (int64_t v0 = 0; v0 < n_states; v0 += 65535) {
      const int64_t vc = std::min<int64_t>(65535, n_states - v0);
      void* sp_arg = static_cast<char*>(states) + size_t(v0) * size_t(state_stride) * elem_bytes(dtype);
      long long stride_arg = state_stride;
      unsigned long long vbase_arg = variant_base + uint64_t(v0);
      int init_arg = 1;
      unsigned long long ntiles_arg = uint64_t(jit->cluster);
      void* args[] = {&sp_arg, &stride_arg, &vbase_arg, &init_arg, &ntiles_arg,
                      blob.empty() ? nullptr : const_cast<unsigned char*>(blob.data())};
      e = cudaLaunchKernel(reinterpret_cast<const void*>(ju->kernel), dim3(unsigned(jit->cluster), unsigned(vc), 1),
                           dim3(unsigned(ju->threads), 1, 1), args, ju->smem, st);
      g_launches.fetch_add(1);
      if (e != cudaSuccess) return cuda_fail(e, "cluster kernel launch");
    }
    return CS_OK;
  }
  int prev_sweep = -1;
  for (const Launch& ln : prog->launches) {
    JitUnit* jk = (jit && jit->cluster == 0 && li < jit->units.size() && jit->units[li])
                      ? jit->units[li].get() : nullptr;
    // only the first launch of a sweep sees the sweep's known-zero amplitudes
    const uint32_t zmask =
        (skip_zero_loads && !(first && init_zero) && ln.sweep != prev_sweep)
            ? prog->sweeps[size_t(ln.sweep)].zero_local_mask : 0u;
    prev_sweep = ln.sweep;
    const std::vector<unsigned char>* blob = jk ? &jit->blobs[li] : nullptr;
    ++li;
    const Sweep& sw = prog->sweeps[size_t(ln.sweep)];
    const int T = sw.tile_bits;
    if (sw.hq.size() > size_t(kMaxTileBits) || sw.oq.size() > 64)
      return fail(CS_ERR_INTERNAL, "sweep geometry exceeds the kernel limits");
    const uint32_t n_tiles = uint32_t(1) << (sparse ? std::min(sw.zero_tiles_log2, nq - T) : nq - T);
    for (int64_t v0 = 0; v0 < n_states; v0 += 65535) {
      const int64_t vc = std::min<int64_t>(65535, n_states - v0);
      void* sp = static_cast<char*>(states) + size_t(v0) * size_t(state_stride) * elem_bytes(dtype);
      cudaError_t e;
      if (jk) {
        void* sp_arg = sp;
        long long stride_arg = state_stride;
        unsigned long long vbase_arg = variant_base + uint64_t(v0);
        int init_arg = (first && init_zero) ? 1 : 0;
        unsigned long long ntiles_arg = n_tiles;
        unsigned zmask_arg = zmask;
        // param mode: the launch's coefficients travel as the 7th argument
        void* args[] = {&sp_arg, &stride_arg, &vbase_arg, &init_arg, &ntiles_arg, &zmask_arg,
                        blob && !blob->empty() ? const_cast<unsigned char*>(blob->data()) : nullptr};
        e = cudaSuccess;
        if (jk->smem > 48 * 1024) {
          int dev = 0;
          cudaGetDevice(&dev);
          const uint64_t bit = uint64_t(1) << (dev & 63);
          if (!(jk->attrs_set.load(std::memory_order_relaxed) & bit)) {
            e = cudaKernelSetAttributeForDevice(jk->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(jk->smem), dev);
            if (e == cudaSuccess) jk->attrs_set.fetch_or(bit);
          }
        }
        if (e == cudaSuccess)
          e = cudaLaunchKernel(reinterpret_cast<const void*>(jk->kernel),
                               dim3(jk->persistent ? std::min<uint32_t>(n_tiles, uint32_t(sm_count())) : n_tiles,
                                    unsigned(vc), 1),
                               dim3(unsigned(jk->threads), 1, 1), args, jk->smem, st);
      } else if (prog->engine == 1) {
        if (ln.reg.size() > size_t(kMaxRegOps)) return fail(CS_ERR_INTERNAL, "register program too long");
        std::memset(&rp, 0, offsetof(RegParams, ops));
        rp.states = sp;
        rp.stride = state_stride;
        rp.variant_base = variant_base + uint64_t(v0);
        rp.tile_bits = T;
        rp.low_bits = sw.low_bits;
        rp.n_high = int32_t(sw.hq.size());
        rp.n_out = int32_t(sw.oq.size());
        rp.n_ops = int32_t(ln.reg.size());
        rp.init_basis = (first && init_zero) ? 1 : 0;
        rp.n_states = int32_t(vc);
        rp.zmask = zmask;
        for (size_t j = 0; j < sw.hq.size() && j < size_t(kMaxTileBits); ++j) rp.hq[j] = int8_t(sw.hq[j]);
        for (size_t j = 0; j < sw.oq.size() && j < 64; ++j) rp.oq[j] = int8_t(sw.oq[j]);
        if (!ln.reg.empty()) std::memcpy(rp.ops, ln.reg.data(), sizeof(RegOp) * ln.reg.size());
        e = launch_rsweep(rp, reg_bits_for(T), n_tiles, uint32_t(vc), st, dtype);
      } else {
        std::memset(&p, 0, offsetof(SweepParams, ops));
        p.nq = nq;
        p.tile_bits = T;
        p.low_bits = sw.low_bits;
        p.n_high = int32_t(sw.hq.size());
        p.n_out = int32_t(sw.oq.size());
        for (size_t j = 0; j < sw.hq.size() && j < size_t(kMaxTileBits); ++j) p.hq[j] = int8_t(sw.hq[j]);
        for (size_t j = 0; j < sw.oq.size() && j < 64; ++j) p.oq[j] = int8_t(sw.oq[j]);
        p.n_ops = int32_t(ln.entries.size());
        if (!ln.entries.empty()) std::memcpy(p.ops, ln.entries.data(), sizeof(SweepOp) * ln.entries.size());
        p.init_basis = (first && init_zero) ? 1 : 0;
        p.stride = state_stride;
        int threads = int(g_opt.threads);
        if (threads == 0) threads = sweep_threads(T);
        threads = std::min(threads, 256);
        p.states = sp;
        p.variant_base = variant_base + uint64_t(v0);
        p.n_states = int32_t(vc);
        e = launch_sweep(p, n_tiles, choose_vb(n_states), threads, st, dtype);
      }
      g_launches.fetch_add(1);
      if (e != cudaSuccess) return cuda_fail(e, "sweep kernel launch");
    }
    first = false;
    if (deadline_s > 0.0 && li < prog->launches.size()) {
      cudaError_t se = cudaStreamSynchronize(st);
      if (se != cudaSuccess) return cuda_fail(se, "cudaStreamSynchronize");
      const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      if (now > deadline_s)
        return fail(CS_ERR_TIMEOUT, "simulation exceeded its deadline after " + std::to_string(li) + "/" +
                                        std::to_string(prog->launches.size()) + " sweep launches");
    }
  }
  return CS_OK;
}


int run_chain(const ChainPlan& plan, int n, const void* const* seg_states, int64_t out_begin, int64_t out_end,
              void* out, void* workspace, int64_t workspace_bytes, int dtype, cudaStream_t st) {
  const size_t eb = elem_bytes(dtype);
  std::vector<const void*> bufs(size_t(n) + plan.buf_amps.size(), nullptr);
  for (int j = 0; j < n; ++j) {
    if (!seg_states[j]) return fail(CS_ERR_INVALID, "null segment state pointer");
    bufs[size_t(j)] = seg_states[j];
  }
  int64_t off = 0;
  for (size_t b = 0; b < plan.buf_amps.size(); ++b) {
    const int64_t bytes = (plan.buf_amps[b] * int64_t(eb) + 255) / 256 * 256;
    if (off + bytes > workspace_bytes || !workspace)
      return fail(CS_ERR_INVALID, "merge workspace too small (query cs_merge_chain_plan)");
    bufs[size_t(n) + b] = static_cast<char*>(workspace) + off;
    off += bytes;
  }
  const int64_t unit = int64_t(1) << plan.q_low;
  if (out_begin < 0 || out_end < out_begin || (out_begin % unit) || (out_end % unit))
    return fail(CS_ERR_INVALID, "output range must be aligned to 2^q_low = " + std::to_string(unit) + " amplitudes");
  for (const MergeStep& s : plan.steps) {
    const void* hi = bufs[size_t(s.hi_buf)];
    const void* lo = bufs[size_t(s.lo_buf)];
    int rc;
    if (s.final_step) {
      const int64_t r0 = out_begin / unit, r1 = out_end / unit;
      if (r1 > s.hi_len) return fail(CS_ERR_INVALID, "output range beyond the state");
      rc = merge_terms_impl(1, s.K, s.hidx.data(), s.lidx.data(), s.coef.data(), hi, s.hi_len, lo, s.lo_len, r0,
                            r1, out, (r1 - r0) * s.lo_len, 0, dtype, st);
    } else {
      void* dst = const_cast<void*>(bufs[size_t(s.out_buf)]);
      rc = merge_terms_impl(s.S, s.K, s.hidx.data(), s.lidx.data(), s.coef.data(), hi, s.hi_len, lo, s.lo_len, 0,
                            s.hi_len, dst, s.hi_len * s.lo_len, 0, dtype, st);
    }
    if (rc != CS_OK) return rc;
  }
  return CS_OK;
}



// ---- the whole cut pipeline behind one call ---------------------------------
struct CutJob {
  CutPrep prep;
  ChainPlan plan;
  std::vector<int32_t> seg_nq, seg_ncuts, seg_cut_ids;
  std::vector<int64_t> seg_off;  // workspace byte offsets of the segment batches
  int64_t chain_off = 0, total_bytes = 0;
};

const double kTermCoef[4] = {0.5, -0.5, 0.5, 0.5};  // (1-i)/2, (1+i)/2 (reference cutting.py:34-35)

bool cut_job(int nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
             int64_t n_gates, int n_seg, const int32_t* sizes, int force_bond, int dtype, CutJob* job, int* rc) {
  try {
    job->prep = cut_prepare(nq, kinds, qa, qb, params, n_gates, n_seg, sizes);
  } catch (const PlanError& pe) {
    *rc = fail(pe.code, pe.msg);
    return false;
  }
  const CutPrep& pr = job->prep;
  for (const SegmentPlan& sp : pr.segs) {
    job->seg_nq.push_back(sp.nq);
    job->seg_ncuts.push_back(int32_t(sp.cut_ids.size()));
    for (int32_t c : sp.cut_ids) job->seg_cut_ids.push_back(c);
  }
  PlanError err{0, ""};
  const int32_t dummy = 0;
  if (!plan_chain(pr.n, job->seg_nq.data(), job->seg_ncuts.data(),
                  job->seg_cut_ids.empty() ? &dummy : job->seg_cut_ids.data(), pr.c_total(),
                  pr.cut_boundary.empty() ? &dummy : pr.cut_boundary.data(), kTermCoef, force_bond, &job->plan,
                  &err)) {
    *rc = fail(err.code, err.msg);
    return false;
  }
  const int64_t eb = int64_t(elem_bytes(dtype));
  int64_t off = 0;
  for (const SegmentPlan& sp : pr.segs) {
    if (sp.cut_ids.size() > 30 || sp.nq > 40) {
      *rc = fail(CS_ERR_CAPACITY, "segment too large for a variant batch");
      return false;
    }
    job->seg_off.push_back(off);
    off += ((int64_t(1) << (sp.cut_ids.size() + size_t(sp.nq))) * eb + 255) / 256 * 256;
  }
  job->chain_off = off;
  for (int64_t a : job->plan.buf_amps) off += (a * eb + 255) / 256 * 256;
  job->total_bytes = off;
  return true;
}

struct SideStreams {
  std::mutex mu;
  std::vector<std::vector<cudaStream_t>> per_device;
} g_side;

cudaStream_t side_stream(int i) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_side.mu);
  if (int(g_side.per_device.size()) <= dev) g_side.per_device.resize(size_t(dev) + 1);
  auto& v = g_side.per_device[size_t(dev)];
  while (int(v.size()) <= i) {
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    v.push_back(s);
  }
  return v[size_t(i)];
}

}  // namespace

// error hook for the library's other translation units (comm.cpp)
namespace cutsim {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace cutsim

extern "C" {

int cs_version(void) { return 10000; }

const char* cs_last_error(void) { return g_err.c_str(); }

int cs_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(CS_ERR_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  *count = c;
  return CS_OK;
}

int cs_set_option(const char* key, int64_t value) {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  const std::string k(key ? key : "");
  if (k == "tile_bits") {
    if (value != 0 && (value < 2 || value > 13)) return fail(CS_ERR_INVALID, "tile_bits must be 0 or in [2, 13]");
    g_opt.tile_bits = value;
  } else if (k == "low_bits") {
    if (value < 1 || value > 12) return fail(CS_ERR_INVALID, "low_bits must be in [1, 12]");
    g_opt.low_bits = value;
  } else if (k == "fuse") {
    if (value < 0 || value > 2) return fail(CS_ERR_INVALID, "fuse must be 0, 1 or 2");
    g_opt.fuse = value;
  } else if (k == "threads") {
    if (value != 0 && (value < 32 || value > 256 || (value & 31)))
      return fail(CS_ERR_INVALID, "threads must be 0 or a multiple of 32 in [32, 256]");
    g_opt.threads = value;
  } else if (k == "merge_streaming") {
    g_opt.merge_streaming = value ? 1 : 0;
  } else if (k == "merge_iters") {
    if (value < 0 || value > 4096) return fail(CS_ERR_INVALID, "merge_iters out of range");
    g_opt.merge_iters = value;
  } else if (k == "sweep_minb") {
    if (value < 2 || value > 4) return fail(CS_ERR_INVALID, "sweep_minb must be 2, 3 or 4");
    g_sweep_minb = int(value);
  } else if (k == "merge_smem_kb") {
    if (value < 8 || value > 112) return fail(CS_ERR_INVALID, "merge_smem_kb must be in [8, 112]");
    g_opt.merge_smem_kb = value;
  } else if (k == "sweep_windows") {
    if (value < 0 || value > 3) return fail(CS_ERR_INVALID, "sweep_windows must be 0, 1, 2 or 3");
    g_sweep_windows = int(value);
  } else if (k == "reg_reorder") {
    g_reg_reorder = value ? 1 : 0;
  } else if (k == "reg_bits") {
    if (value != 0 && (value < 2 || value > 4)) return fail(CS_ERR_INVALID, "reg_bits must be 0 or 2..4");
    g_reg_bits = int(value);
  } else if (k == "dense_norm") {
    if (value < 0 || value > 2) return fail(CS_ERR_INVALID, "dense_norm must be 0, 1 or 2");
    g_opt.dense_norm = value;
  } else if (k == "jit_persistent") {
    g_jit_persistent = value ? 1 : 0;
  } else if (k == "jit_minb") {
    if (value < 1 || value > 4) return fail(CS_ERR_INVALID, "jit_minb must be in [1, 4]");
    g_jit_minb = int(value);
  } else if (k == "merge_dmma3_warps") {
    if (value != 4 && value != 8) return fail(CS_ERR_INVALID, "merge_dmma3_warps must be 4 or 8");
    g_opt.merge_dmma3_warps = value;
  } else if (k == "zero_start_tiles") {
    g_opt.zero_start_tiles = value ? 1 : 0;
  } else if (k == "zero_skip") {
    g_opt.zero_skip = value ? 1 : 0;
  } else if (k == "merge_ozaki") {
    if (value < 0 || value > 3) return fail(CS_ERR_INVALID, "merge_ozaki must be 0, 1, 2 or 3");
    g_opt.merge_ozaki = value;
  } else if (k == "merge_ozaki_min_work") {
    if (value < 0 || value > 62) return fail(CS_ERR_INVALID, "merge_ozaki_min_work must be 0..62");
    g_opt.merge_ozaki_min_work = value;
  } else if (k == "merge_ozaki_min_k") {
    if (value != 8 && value != 16 && value != 32 && value != 64)
      return fail(CS_ERR_INVALID, "merge_ozaki_min_k must be 8, 16, 32 or 64");
    g_opt.merge_ozaki_min_k = value;
  } else if (k == "merge_dmma") {
    if (value < 0 || value > 2) return fail(CS_ERR_INVALID, "merge_dmma must be 0, 1 or 2");
    g_opt.merge_dmma = value;
  } else if (k == "jit") {
    if (value < 0 || value > 3) return fail(CS_ERR_INVALID, "jit must be 0, 1, 2 or 3");
    g_opt.jit = value;
  } else if (k == "merge_ozaki_digits") {
    if (value != 7 && value != 8) return fail(CS_ERR_INVALID, "merge_ozaki_digits must be 7 or 8");
    g_opt.merge_ozaki_digits = value;
  } else if (k == "cluster") {
    g_opt.cluster = value ? 1 : 0;
  } else if (k == "cluster_loop") {
    if (value < 0 || value > 2) return fail(CS_ERR_INVALID, "cluster_loop must be 0, 1 or 2");
    g_opt.cluster_loop = value;
  } else if (k == "cluster_max") {
    if (value != 2 && value != 4 && value != 8 && value != 16) return fail(CS_ERR_INVALID, "cluster_max must be 2, 4, 8 or 16");
    g_opt.cluster_max = value;
  } else if (k == "jit_struct") {
    if (value < 0 || value > 2) return fail(CS_ERR_INVALID, "jit_struct must be 0, 1 or 2");
    g_opt.jit_struct = value;
  } else if (k == "jit_max_cost") {
    if (value < 0) return fail(CS_ERR_INVALID, "jit_max_cost must be >= 0");
    g_opt.jit_max_cost = value;
  } else if (k == "engine") {
    if (value != 0 && value != 1) return fail(CS_ERR_INVALID, "engine must be 0 or 1");
    g_opt.engine = value;
  } else if (k == "plan_json") {
    g_opt.plan_json = value ? 1 : 0;
  } else if (k == "vb") {
    if (value < 0 || value > 4 || value == 3) return fail(CS_ERR_INVALID, "vb must be 0, 1, 2 or 4");
    g_opt.vb = value;
  } else {
    return fail(CS_ERR_INVALID, "unknown option '" + k + "'");
  }
  return CS_OK;
}

int64_t cs_get_option(const char* key) {
  const std::string k(key ? key : "");
  if (k == "tile_bits") return g_opt.tile_bits;
  if (k == "low_bits") return g_opt.low_bits;
  if (k == "fuse") return g_opt.fuse;
  if (k == "threads") return g_opt.threads;
  if (k == "merge_streaming") return g_opt.merge_streaming;
  if (k == "merge_iters") return g_opt.merge_iters;
  if (k == "vb") return g_opt.vb;
  if (k == "engine") return g_opt.engine;
  if (k == "jit") return g_opt.jit;
  if (k == "jit_struct") return g_opt.jit_struct;
  if (k == "cluster") return g_opt.cluster;
  if (k == "cluster_max") return g_opt.cluster_max;
  if (k == "cluster_loop") return g_opt.cluster_loop;
  if (k == "merge_ozaki_digits") return g_opt.merge_ozaki_digits;
  if (k == "jit_units_compiled") return jit_units_compiled();
  if (k == "jit_units_reused") return jit_units_reused();
  if (k == "jit_max_cost") return g_opt.jit_max_cost;
  if (k == "merge_dmma") return g_opt.merge_dmma;
  if (k == "merge_ozaki") return g_opt.merge_ozaki;
  if (k == "zero_start_tiles") return g_opt.zero_start_tiles;
  if (k == "zero_skip") return g_opt.zero_skip;
  if (k == "merge_ozaki_min_k") return g_opt.merge_ozaki_min_k;
  if (k == "merge_ozaki_min_work") return g_opt.merge_ozaki_min_work;
  if (k == "merge_smem_kb") return g_opt.merge_smem_kb;
  if (k == "merge_dmma3_warps") return g_opt.merge_dmma3_warps;
  if (k == "jit_minb") return g_jit_minb;
  if (k == "jit_persistent") return g_jit_persistent;
  if (k == "dense_norm") return g_opt.dense_norm;
  if (k == "reg_bits") return g_reg_bits;
  if (k == "reg_reorder") return g_reg_reorder;
  if (k == "sweep_windows") return g_sweep_windows;
  if (k == "plan_json") return g_opt.plan_json;
  if (k == "sweep_minb") return g_sweep_minb;
  return -1;
}

int64_t cs_launch_count(void) { return g_launches.load(); }

int cs_jit_wait(double timeout_s) {
  std::unique_lock<std::mutex> lk(g_jitq.mu);
  auto done = [] { return g_jitq.q.empty() && g_jitq.busy == 0; };
  if (timeout_s < 0) {
    g_jitq.idle_cv.wait(lk, done);
    return CS_OK;
  }
  if (!g_jitq.idle_cv.wait_for(lk, std::chrono::duration<double>(timeout_s), done))
    return fail(CS_ERR_TIMEOUT, "background kernel compilation still running");
  return CS_OK;
}

int cs_init_basis(void* states, int32_t nq, int64_t n_states, int64_t index, int32_t dtype, void* stream) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 0 || nq > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
  if (!states || n_states < 1) return fail(CS_ERR_INVALID, "empty state batch");
  if (index < 0 || index >= (int64_t(1) << nq)) return fail(CS_ERR_INVALID, "basis index out of range");
  cudaError_t e = launch_init_basis(states, int64_t(1) << nq, n_states, index, dtype, as_stream(stream));
  g_launches.fetch_add(1);
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "init_basis launch");
}

int cs_sim_batch(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                 const int32_t* slots, int64_t n_gates, void* states, int64_t n_states, int64_t state_stride,
                 uint64_t variant_base, int32_t init_zero, int32_t dtype, void* stream) {
  Nvtx nvtx_entry("cs_sim_batch");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 0 || nq > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
  if (!states || n_states < 1) return fail(CS_ERR_INVALID, "empty state batch");
  if (state_stride < (int64_t(1) << nq)) return fail(CS_ERR_INVALID, "state_stride smaller than 2^nq");
  if (n_gates < 0 || (n_gates > 0 && (!kinds || !qa || !qb))) return fail(CS_ERR_INVALID, "bad gate table");
  cudaStream_t st = as_stream(stream);
  if (nq == 0) {
    if (!init_zero) return CS_OK;
    return cs_init_basis(states, 0, n_states, 0, dtype, stream);
  }
  std::shared_ptr<const Program> prog;
  try {
    prog = build_schedule(nq, kinds, qa, qb, params, slots, n_gates, n_states, 0, dtype, init_zero != 0);
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  return run_program(prog, nq, states, n_states, state_stride, variant_base, init_zero, dtype, st);
}

// Run n independent launch sequences concurrently: items 1..n-1 on the
// library's side streams (forked from `st` by one event, joined back into
// it), item 0 on `st` itself, launched last so every item starts together.
// Keeping one item on `st` saves it the fork and join hops (cfg4a variant
// stage: family batches 28-30 us each, 43 us both through two side streams).
extern "C++" {
template <typename F>
int run_forked(int n, cudaStream_t st, F&& launch) {
  if (n <= 1) return n == 1 ? launch(0, st) : CS_OK;
  cudaEvent_t fork = nullptr;
  cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
  cudaEventRecord(fork, st);
  int rc = CS_OK;
  std::vector<cudaEvent_t> done;
  for (int i = 1; i < n && rc == CS_OK; ++i) {
    cudaStream_t ss = side_stream((i - 1) % 4);
    cudaStreamWaitEvent(ss, fork, 0);
    rc = launch(i, ss);
    cudaEvent_t d = nullptr;
    cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
    cudaEventRecord(d, ss);
    done.push_back(d);
  }
  if (rc == CS_OK) rc = launch(0, st);
  for (cudaEvent_t d : done) {
    cudaStreamWaitEvent(st, d, 0);
    cudaEventDestroy(d);
  }
  cudaEventDestroy(fork);
  return rc;
}
}  // extern "C++"

int cs_sim_families(int32_t n_fam, const int32_t* nq, const int64_t* gate_count, const uint8_t* kinds,
                    const int64_t* qa, const int64_t* qb, const double* params, const int32_t* slots,
                    void* const* states, const int64_t* n_states, int32_t dtype, void* stream) {
  Nvtx nvtx_entry("cs_sim_families");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (n_fam < 1 || !nq || !gate_count || !states || !n_states) return fail(CS_ERR_INVALID, "empty family list");
  std::vector<std::shared_ptr<const Program>> progs(static_cast<size_t>(n_fam));
  int64_t g0 = 0;
  for (int f = 0; f < n_fam; ++f) {
    const int64_t m = gate_count[f];
    if (nq[f] < 1 || nq[f] > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
    if (!states[f] || n_states[f] < 1) return fail(CS_ERR_INVALID, "empty state batch");
    if (m < 0 || (m > 0 && (!kinds || !qa || !qb))) return fail(CS_ERR_INVALID, "bad gate table");
    try {
      progs[size_t(f)] = build_schedule(nq[f], kinds + g0, qa + g0, qb + g0, params ? params + 3 * g0 : nullptr,
                                        slots ? slots + g0 : nullptr, m, n_states[f], 0, dtype, true);
    } catch (const PlanError& pe) {
      return fail(pe.code, pe.msg);
    }
    g0 += m;
  }
  return run_forked(n_fam, as_stream(stream), [&](int f, cudaStream_t ss) {
    return run_program(progs[size_t(f)], nq[f], states[f], n_states[f], int64_t(1) << nq[f], 0, 1, dtype, ss);
  });
}

int cs_sim_batch_until(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                       const double* params, const int32_t* slots, int64_t n_gates, void* states, int64_t n_states,
                       int64_t state_stride, uint64_t variant_base, int32_t init_zero, int32_t dtype, void* stream,
                       double deadline_s) {
  Nvtx nvtx_entry("cs_sim_batch_until");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 1 || nq > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
  if (!states || n_states < 1) return fail(CS_ERR_INVALID, "empty state batch");
  if (state_stride < (int64_t(1) << nq)) return fail(CS_ERR_INVALID, "state_stride smaller than 2^nq");
  if (n_gates < 0 || (n_gates > 0 && (!kinds || !qa || !qb))) return fail(CS_ERR_INVALID, "bad gate table");
  std::shared_ptr<const Program> prog;
  try {
    prog = build_schedule(nq, kinds, qa, qb, params, slots, n_gates, n_states, 0, dtype, init_zero != 0);
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  return run_program(prog, nq, states, n_states, state_stride, variant_base, init_zero, dtype, as_stream(stream),
                     deadline_s);
}

int cs_sweep_plan_json(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                       const double* params, const int32_t* slots, int64_t n_gates, int32_t tile_bits,
                       int32_t dtype, char* buf, int64_t buflen, int64_t* needed) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 1 || nq > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
  std::string js;
  try {
    auto prog = build_schedule(nq, kinds, qa, qb, params, slots, n_gates, 1, tile_bits, dtype, true);
    js = g_opt.plan_json ? reg_programs_to_json(prog->sweeps, nq) : sweeps_to_json(prog->sweeps, nq);
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  if (needed) *needed = int64_t(js.size()) + 1;
  if (buf && buflen > 0) {
    const size_t n = std::min(size_t(buflen - 1), js.size());
    std::memcpy(buf, js.data(), n);
    buf[n] = 0;
  }
  return CS_OK;
}

int cs_jit_selftest(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                    const int32_t* slots, int64_t n_gates, int64_t n_states, int32_t dtype, int64_t* cubin_bytes) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 1 || nq > 62) return fail(CS_ERR_INVALID, "qubit count out of range");
  std::shared_ptr<const Program> prog;
  try {
    prog = build_schedule(nq, kinds, qa, qb, params, slots, n_gates, n_states, 0, dtype, true);
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  if (prog->engine != 1) return fail(CS_ERR_INVALID, "JIT needs engine 1");
  std::vector<const Sweep*> sw;
  std::vector<const std::vector<RegOp>*> rp;
  for (const Launch& ln : prog->launches) {
    sw.push_back(&prog->sweeps[size_t(ln.sweep)]);
    rp.push_back(&ln.reg);
  }
  std::vector<char> cubin;
  std::vector<std::string> names;
  std::string err;
  if (prog->cluster_bits > 0) {  // the form cs_sim_batch would run: one cluster-resident kernel
    if (!jit_cluster_cubin(sw, rp, prog->sweeps[0].tile_bits, dtype, &cubin, &err, prog->param_mode))
      return fail(CS_ERR_INTERNAL, err);
  } else if (!jit_cubin(sw, rp, dtype, &cubin, &names, &err, prog->param_mode)) {
    return fail(CS_ERR_INTERNAL, err);
  }
  if (cubin_bytes) *cubin_bytes = int64_t(cubin.size());
  return CS_OK;
}

int cs_merge_terms(int32_t S, int32_t K, const int32_t* hidx, const int32_t* lidx, const double* coef,
                   const void* hi, int64_t hi_len, const void* lo, int64_t lo_len, int64_t row_begin,
                   int64_t row_end, void* out, int64_t out_slot_stride, int32_t accumulate, int32_t dtype,
                   void* stream) {
  Nvtx nvtx_entry("cs_merge_terms");
  return merge_terms_impl(S, K, hidx, lidx, coef, hi, hi_len, lo, lo_len, row_begin, row_end, out,
                          out_slot_stride, accumulate, dtype, as_stream(stream));
}

int cs_merge_chain_plan(int32_t n, const int32_t* seg_nq, const int32_t* seg_ncuts, const int32_t* seg_cut_ids,
                        int32_t c_total, const int32_t* cut_boundary, const double* term_coef, int32_t force_bond,
                        int32_t dtype, int64_t* workspace_bytes, int32_t* bond, int32_t* q_low) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  ChainPlan plan;
  PlanError err{0, ""};
  if (!plan_chain(n, seg_nq, seg_ncuts, seg_cut_ids, c_total, cut_boundary, term_coef, force_bond, &plan, &err))
    return fail(err.code, err.msg);
  int64_t bytes = 0;
  for (int64_t a : plan.buf_amps) bytes += (a * int64_t(elem_bytes(dtype)) + 255) / 256 * 256;
  if (workspace_bytes) *workspace_bytes = bytes;
  if (bond) *bond = plan.bond;
  if (q_low) *q_low = plan.q_low;
  return CS_OK;
}

int cs_merge_chain(int32_t n, const int32_t* seg_nq, const void* const* seg_states, const int32_t* seg_ncuts,
                   const int32_t* seg_cut_ids, int32_t c_total, const int32_t* cut_boundary, const double* term_coef,
                   int32_t force_bond, int64_t out_begin, int64_t out_end, void* out, void* workspace,
                   int64_t workspace_bytes, int32_t dtype, void* stream) {
  Nvtx nvtx_entry("cs_merge_chain");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  ChainPlan plan;
  PlanError err{0, ""};
  if (!plan_chain(n, seg_nq, seg_ncuts, seg_cut_ids, c_total, cut_boundary, term_coef, force_bond, &plan, &err))
    return fail(err.code, err.msg);
  return run_chain(plan, n, seg_states, out_begin, out_end, out, workspace, workspace_bytes, dtype,
                   as_stream(stream));
}


int cs_cut_workspace(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                     int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int32_t force_bond, int32_t dtype,
                     int64_t* workspace_bytes, int32_t* q_low, int32_t* c_total) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, force_bond, dtype, &job, &rc)) return rc;
  if (workspace_bytes) *workspace_bytes = job.total_bytes;
  if (q_low) *q_low = job.plan.q_low;
  if (c_total) *c_total = job.prep.c_total();
  return CS_OK;
}

int cs_cut_describe_json(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                         const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, char* buf,
                         int64_t buflen, int64_t* needed) {
  if (nq < 2 || nq > 62 || !seg_sizes) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  std::string js;
  try {
    js = cut_prep_to_json(cut_prepare(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes));
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  if (needed) *needed = int64_t(js.size()) + 1;
  if (buf && buflen > 0) {
    const size_t m = std::min(size_t(buflen - 1), js.size());
    std::memcpy(buf, js.data(), m);
    buf[m] = 0;
  }
  return CS_OK;
}

int cs_cut_tables(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                  int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int64_t* cuts, int32_t* seg_counts,
                  uint8_t* out_kinds, int64_t* out_qa, int64_t* out_qb, double* out_params, int32_t* out_slots,
                  int32_t* out_cut_ids, int64_t gate_cap, int64_t cut_cap, int64_t* needed) {
  if (nq < 2 || nq > 62 || !seg_sizes || !needed) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  CutPrep pr;
  try {
    pr = cut_prepare(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes);
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  int64_t total = 0, adj = 0;
  for (const SegmentPlan& sp : pr.segs) {
    total += int64_t(sp.kinds.size());
    adj += int64_t(sp.cut_ids.size());
  }
  needed[0] = total;
  needed[1] = pr.c_total();
  if (total > gate_cap || pr.c_total() > cut_cap || adj > 2 * cut_cap) return CS_OK;  // sizes only
  if (!cuts || !seg_counts || !out_kinds || !out_qa || !out_qb || !out_params || !out_slots || !out_cut_ids)
    return fail(CS_ERR_INVALID, "null output buffer");
  for (int j = 0; j < pr.c_total(); ++j) {
    cuts[4 * j] = pr.cut_pos[size_t(j)];
    cuts[4 * j + 1] = pr.cut_boundary[size_t(j)];
    cuts[4 * j + 2] = pr.cut_ctrl[size_t(j)];
    cuts[4 * j + 3] = pr.cut_tgt[size_t(j)];
  }
  int64_t g = 0, c = 0;
  for (size_t s = 0; s < pr.segs.size(); ++s) {
    const SegmentPlan& sp = pr.segs[s];
    const size_t m = sp.kinds.size();
    seg_counts[2 * s] = int32_t(m);
    seg_counts[2 * s + 1] = int32_t(sp.cut_ids.size());
    std::memcpy(out_kinds + g, sp.kinds.data(), m);
    std::memcpy(out_qa + g, sp.qa.data(), m * sizeof(int64_t));
    std::memcpy(out_qb + g, sp.qb.data(), m * sizeof(int64_t));
    std::memcpy(out_params + 3 * g, sp.params.data(), 3 * m * sizeof(double));
    std::memcpy(out_slots + g, sp.slots.data(), m * sizeof(int32_t));
    std::memcpy(out_cut_ids + c, sp.cut_ids.data(), sp.cut_ids.size() * sizeof(int32_t));
    g += int64_t(m);
    c += int64_t(sp.cut_ids.size());
  }
  return CS_OK;
}

namespace {

// One batch of consecutive variants [v0, v1) of segment `seg`, simulated
// into `dst` (state v0 first). The single-GPU pipeline runs one piece per
// segment (its whole family); a rank of the sharded pipeline runs the pieces
// of its slice of the flattened variant list.
struct Piece {
  int seg = 0;
  int64_t v0 = 0, v1 = 0;
  void* dst = nullptr;
};

// Programs of the pieces' variant batches, NVRTC-compiled if enabled (host
// side of the variant stage; compile before any timing).
int piece_programs(const CutJob& job, const std::vector<Piece>& pieces, int dtype,
                   std::vector<std::shared_ptr<const Program>>* progs) {
  try {
    for (const Piece& pc : pieces) {
      const SegmentPlan& sp = job.prep.segs[size_t(pc.seg)];
      progs->push_back(build_schedule(sp.nq, sp.kinds.data(), sp.qa.data(), sp.qb.data(), sp.params.data(),
                                      sp.slots.data(), int64_t(sp.kinds.size()), pc.v1 - pc.v0, 0, dtype, true));
    }
  } catch (const PlanError& pe) {
    return fail(pe.code, pe.msg);
  }
  for (const auto& pg : *progs) program_jit(pg, dtype);
  return CS_OK;
}

// Batched subcircuit simulation of every piece, pieces on side streams
// forked from / joined into `st` (segments are independent).
int run_pieces(const CutJob& job, const std::vector<Piece>& pieces,
               const std::vector<std::shared_ptr<const Program>>& progs, int dtype, cudaStream_t st) {
  return run_forked(int(pieces.size()), st, [&](int i, cudaStream_t ss) {
    const Piece& pc = pieces[size_t(i)];
    const SegmentPlan& sp = job.prep.segs[size_t(pc.seg)];
    return run_program(progs[size_t(i)], sp.nq, pc.dst, pc.v1 - pc.v0, int64_t(1) << sp.nq, uint64_t(pc.v0), 1, dtype,
                       ss);
  });
}

// The single-GPU pieces: every segment's whole family at its workspace slot.
std::vector<Piece> family_pieces(const CutJob& job, void* workspace, std::vector<const void*>* seg_states) {
  std::vector<Piece> pieces;
  for (size_t s = 0; s < job.prep.segs.size(); ++s) {
    Piece pc;
    pc.seg = int(s);
    pc.v1 = int64_t(1) << job.prep.segs[s].cut_ids.size();
    pc.dst = static_cast<char*>(workspace) + job.seg_off[s];
    seg_states->push_back(pc.dst);
    pieces.push_back(pc);
  }
  return pieces;
}

int cut_programs(const CutJob& job, int dtype, std::vector<std::shared_ptr<const Program>>* progs) {
  std::vector<const void*> dummy;
  return piece_programs(job, family_pieces(job, nullptr, &dummy), dtype, progs);
}

int cut_segments(const CutJob& job, const std::vector<std::shared_ptr<const Program>>& progs, void* workspace,
                 int dtype, cudaStream_t st, std::vector<const void*>* seg_states) {
  return run_pieces(job, family_pieces(job, workspace, seg_states), progs, dtype, st);
}

// ---- the sharded (multi-GPU) pipeline ----------------------------------------
// Every segment has the same qubit count, so the segments' variant batches,
// concatenated segment-major, are one array of `total` equal states. It is
// split into `world` chunks of `per` states (the last padded); rank r
// simulates chunk r in place and one in-place all-gather fills every chunk on
// every rank — the gathered array IS the segment batches the merge reads, no
// reassembly copies. Then each rank merges its own rows of the output.
struct ShardLayout {
  int64_t L = 0;                  // amplitudes per state
  int64_t total = 0, per = 0;     // states overall / per rank
  std::vector<int64_t> seg_first; // flat index of each segment's first variant
  int64_t gather_bytes = 0;       // world * per states (256-byte aligned)
  int64_t chain_off = 0, total_bytes = 0;
  int64_t row_amps = 0, rows = 0; // the final product's row length and count
};

bool shard_layout(const CutJob& job, int nq, int world, int dtype, ShardLayout* lay, int* rc) {
  const CutPrep& pr = job.prep;
  for (const SegmentPlan& sp : pr.segs)
    if (sp.nq != pr.segs[0].nq) {
      *rc = fail(CS_ERR_INVALID, "the sharded pipeline needs equal segment sizes");
      return false;
    }
  if (world < 1) {
    *rc = fail(CS_ERR_INVALID, "world must be >= 1");
    return false;
  }
  const int64_t eb = int64_t(elem_bytes(dtype));
  lay->L = int64_t(1) << pr.segs[0].nq;
  lay->total = 0;
  for (const SegmentPlan& sp : pr.segs) {
    lay->seg_first.push_back(lay->total);
    lay->total += int64_t(1) << sp.cut_ids.size();
  }
  lay->per = (lay->total + world - 1) / world;
  lay->gather_bytes = (int64_t(world) * lay->per * lay->L * eb + 255) / 256 * 256;
  lay->chain_off = lay->gather_bytes;
  int64_t off = lay->chain_off;
  for (int64_t a : job.plan.buf_amps) off += (a * eb + 255) / 256 * 256;
  lay->total_bytes = off;
  lay->row_amps = int64_t(1) << job.plan.q_low;
  lay->rows = (int64_t(1) << nq) >> job.plan.q_low;
  return true;
}

// rank's rows [r0, r1) of the final product (parallel.shard_range)
void shard_rows(const ShardLayout& lay, int world, int rank, int64_t* r0, int64_t* r1) {
  *r0 = lay.rows * rank / world;
  *r1 = lay.rows * (rank + 1) / world;
}

// rank's slice [g0, g1) of the flattened variant list, as per-segment pieces
std::vector<Piece> shard_pieces(const CutJob& job, const ShardLayout& lay, int64_t g0, int64_t g1, void* ws,
                                int dtype) {
  std::vector<Piece> pieces;
  const int64_t eb = int64_t(elem_bytes(dtype));
  for (size_t s = 0; s < job.prep.segs.size(); ++s) {
    const int64_t base = lay.seg_first[s];
    const int64_t cnt = int64_t(1) << job.prep.segs[s].cut_ids.size();
    const int64_t a = std::max(g0, base), b = std::min(g1, base + cnt);
    if (a >= b) continue;
    Piece pc;
    pc.seg = int(s);
    pc.v0 = a - base;
    pc.v1 = b - base;
    pc.dst = static_cast<char*>(ws) + a * lay.L * eb;
    pieces.push_back(pc);
  }
  return pieces;
}

int64_t host_chunk_amps(const CutJob& job, int nq, int chunks) {
  const int64_t unit = int64_t(1) << job.plan.q_low;
  const int64_t total = int64_t(1) << nq;
  const int64_t c = std::max<int64_t>(1, chunks);
  return std::max(unit, (total / c) / unit * unit);
}

cudaStream_t copy_stream() {
  static std::mutex mu;
  static std::vector<cudaStream_t> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (int(per_device.size()) <= dev) per_device.resize(size_t(dev) + 1, nullptr);
  if (!per_device[size_t(dev)]) cudaStreamCreateWithFlags(&per_device[size_t(dev)], cudaStreamNonBlocking);
  return per_device[size_t(dev)];
}

// ---- device -> pageable host memory through pinned staging ----------------
// cudaMemcpy into pageable memory runs at ~20 GB/s behind the driver's own
// staging (q=30: 0.8 s for the 16 GiB state into a fresh numpy array, first
// touch included). Here device data is copied in 64 MiB pieces into a ring
// of pinned buffers on the copy stream while a pool of host threads copies
// the previous piece out (first-touching the destination pages in parallel),
// so the transfer runs near the PCIe rate (the reference returns host numpy
// arrays: StateVec.amps, run_cut_to_host into numpy).
bool host_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// A fixed pool of host threads for one parallel memcpy at a time.
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool* pool = new HostCopyPool;  // never destroyed: detached workers
    return *pool;
  }
  void copy(void* dst, const void* src, size_t n) {
    if (n < (size_t(4) << 20) || nthreads_ <= 1) {
      std::memcpy(dst, src, n);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_ = n;
    left_ = nthreads_;
    ++gen_;
    cv_.notify_all();
    done_cv_.wait(lk, [this] { return left_ == 0; });
  }

 private:
  HostCopyPool() {
    const unsigned hc = std::thread::hardware_concurrency();
    nthreads_ = int(std::min(16u, std::max(1u, hc)));
    for (int t = 0; t < nthreads_; ++t) std::thread([this, t] { worker(t); }).detach();
  }
  void worker(int t) {
    uint64_t seen = 0;
    for (;;) {
      char* d;
      const char* sp;
      size_t n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        d = dst_;
        sp = src_;
        n = n_;
      }
      // slice t of n, 4 KiB aligned boundaries (one page per thread at a time)
      const size_t per = ((n / size_t(nthreads_)) + 4095) & ~size_t(4095);
      const size_t b = std::min(n, per * size_t(t)), e = std::min(n, b + per);
      if (e > b) std::memcpy(d + b, sp + b, e - b);
      std::lock_guard<std::mutex> lk(mu_);
      if (--left_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  int left_ = 0, nthreads_ = 1;
  uint64_t gen_ = 0;
};

// Ring of pinned staging buffers (per process, reused) feeding the pool.
class StagedHostWriter {
 public:
  static constexpr int kSlots = 3;
  static constexpr size_t kPiece = size_t(64) << 20;
  explicit StagedHostWriter(cudaStream_t cp) : cp_(cp) {}
  ~StagedHostWriter() {
    for (auto& e : done_)
      if (e) cudaEventDestroy(e);
  }
  // copy n bytes at device `src` to host `dst` once `ready` (may be null)
  // has fired on the device; returns a CUDA error of the enqueue
  cudaError_t write(char* dst, const char* src, size_t n, cudaEvent_t ready) {
    cudaError_t e = staging();
    if (e != cudaSuccess) return e;
    if (ready) cudaStreamWaitEvent(cp_, ready, 0);
    for (size_t off = 0; off < n; off += kPiece) {
      const size_t len = std::min(kPiece, n - off);
      const int s = next_;
      next_ = (next_ + 1) % kSlots;
      e = drain(s);  // the slot's previous piece is copied out first
      if (e != cudaSuccess) return e;
      if (!done_[s]) cudaEventCreateWithFlags(&done_[s], cudaEventDisableTiming);
      e = cudaMemcpyAsync(pin()[s], src + off, len, cudaMemcpyDeviceToHost, cp_);
      if (e != cudaSuccess) return e;
      cudaEventRecord(done_[s], cp_);
      dst_[s] = dst + off;
      len_[s] = len;
    }
    return cudaSuccess;
  }
  // every piece written to its destination
  cudaError_t finish() {
    for (int i = 0; i < kSlots; ++i) {
      cudaError_t e = drain((next_ + i) % kSlots);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

 private:
  static char** pin() {
    static char* bufs[kSlots] = {nullptr, nullptr, nullptr};
    return bufs;
  }
  static cudaError_t staging() {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (int s = 0; s < kSlots; ++s)
      if (!pin()[s]) {
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&pin()[s]), kPiece, cudaHostAllocPortable);
        if (e != cudaSuccess) {
          pin()[s] = nullptr;
          return e;
        }
      }
    return cudaSuccess;
  }
  cudaError_t drain(int s) {
    if (!dst_[s]) return cudaSuccess;
    cudaError_t e = cudaEventSynchronize(done_[s]);
    if (e != cudaSuccess) return e;
    HostCopyPool::get().copy(dst_[s], pin()[s], len_[s]);
    dst_[s] = nullptr;
    return cudaSuccess;
  }
  cudaStream_t cp_;
  cudaEvent_t done_[kSlots] = {nullptr, nullptr, nullptr};
  char* dst_[kSlots] = {nullptr, nullptr, nullptr};
  size_t len_[kSlots] = {0, 0, 0};
  int next_ = 0;
};

// one staged writer at a time (the pinned ring is shared by the process)
std::mutex g_staged_mu;

}  // namespace

int cs_cut_host_workspace(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                          const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes,
                          int32_t chunks, int32_t dtype, int64_t* workspace_bytes) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes || !workspace_bytes) return fail(CS_ERR_INVALID, "bad arguments");
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, -1, dtype, &job, &rc)) return rc;
  const int64_t chunk_bytes = host_chunk_amps(job, nq, chunks) * int64_t(elem_bytes(dtype));
  *workspace_bytes = job.total_bytes + 2 * ((chunk_bytes + 255) / 256 * 256);
  return CS_OK;
}

int cs_cut_run_to_host(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                       int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int32_t chunks, void* host_out,
                       void* workspace, int64_t workspace_bytes, int32_t dtype, void* stream, double* stage_ms) {
  Nvtx nvtx_entry("cs_cut_run_to_host");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  if (!host_out) return fail(CS_ERR_INVALID, "null host output pointer");
  const auto t0 = std::chrono::steady_clock::now();
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, -1, dtype, &job, &rc)) return rc;
  const size_t eb = elem_bytes(dtype);
  const int64_t step = host_chunk_amps(job, nq, chunks);
  const int64_t buf_bytes = (step * int64_t(eb) + 255) / 256 * 256;
  if (!workspace || workspace_bytes < job.total_bytes + 2 * buf_bytes)
    return fail(CS_ERR_INVALID, "workspace too small (query cs_cut_host_workspace)");
  std::vector<std::shared_ptr<const Program>> progs;
  rc = cut_programs(job, dtype, &progs);
  if (rc != CS_OK) return rc;
  const double t_pre = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  cudaStream_t st = as_stream(stream);
  cudaStream_t cp = copy_stream();
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  if (stage_ms) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventRecord(e0, st);
  }
  std::vector<const void*> seg_states;
  rc = cut_segments(job, progs, workspace, dtype, st, &seg_states);
  if (rc != CS_OK) return rc;
  if (e1) cudaEventRecord(e1, st);
  // chunked merge into two device buffers; each chunk's device-to-host copy
  // runs on the copy stream while the next chunk is merged (PCIe-bound)
  char* bufs[2] = {static_cast<char*>(workspace) + job.total_bytes,
                   static_cast<char*>(workspace) + job.total_bytes + buf_bytes};
  cudaEvent_t ready[2], copied[2] = {nullptr, nullptr};
  for (auto& e : ready) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  const int64_t total = int64_t(1) << nq;
  // pageable destination (e.g. a numpy array): pinned staging ring + host
  // copy threads instead of the driver's pageable path
  const bool staged = !host_is_pinned(host_out);
  std::unique_lock<std::mutex> staged_lk(g_staged_mu, std::defer_lock);
  if (staged) staged_lk.lock();
  StagedHostWriter writer(cp);
  int i = 0;
  for (int64_t b = 0; b < total && rc == CS_OK; b += step, ++i) {
    const int64_t e = std::min(total, b + step);
    const int k = i & 1;
    if (copied[k]) cudaStreamWaitEvent(st, copied[k], 0);  // buffer k free again
    rc = run_chain(job.plan, job.prep.n, seg_states.data(), b, e, bufs[k],
                   static_cast<char*>(workspace) + job.chain_off, job.total_bytes - job.chain_off, dtype, st);
    if (rc != CS_OK) break;
    cudaEventRecord(ready[k], st);
    char* dst = static_cast<char*>(host_out) + size_t(b) * eb;
    cudaError_t ce;
    if (staged) {
      ce = writer.write(dst, bufs[k], size_t(e - b) * eb, ready[k]);
    } else {
      cudaStreamWaitEvent(cp, ready[k], 0);
      ce = cudaMemcpyAsync(dst, bufs[k], size_t(e - b) * eb, cudaMemcpyDeviceToHost, cp);
    }
    if (ce != cudaSuccess) rc = cuda_fail(ce, "device to host copy");
    if (!copied[k]) cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming);
    cudaEventRecord(copied[k], cp);
  }
  if (staged && rc == CS_OK) {
    cudaError_t fe = writer.finish();
    if (fe != cudaSuccess) rc = cuda_fail(fe, "staged device to host copy");
  }
  // the host state is complete when this returns (the reference returns host memory)
  cudaError_t se = cudaStreamSynchronize(cp);
  if (e2) {
    cudaEventRecord(e2, st);
    cudaEventSynchronize(e2);
    float a = 0, m = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&m, e1, e2);
    stage_ms[0] = t_pre;
    stage_ms[1] = a;
    stage_ms[2] = m;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
  }
  for (auto& e : ready) cudaEventDestroy(e);
  for (auto& e : copied)
    if (e) cudaEventDestroy(e);
  if (rc != CS_OK) return rc;
  if (se != cudaSuccess) return cuda_fail(se, "device-to-host copy");
  cudaError_t le = cudaGetLastError();
  return le == cudaSuccess ? CS_OK : cuda_fail(le, "cut pipeline to host");
}

int cs_copy_to_host(void* host, const void* device, int64_t bytes, void* stream) {
  Nvtx nvtx_entry("cs_copy_to_host");
  if (bytes < 0 || (bytes > 0 && (!host || !device))) return fail(CS_ERR_INVALID, "bad copy arguments");
  if (bytes == 0) return CS_OK;
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  if (host_is_pinned(host)) {
    e = cudaMemcpyAsync(host, device, size_t(bytes), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? CS_OK : cuda_fail(e, "device to host copy");
  }
  // the copies run on the copy stream after everything queued on `stream`
  cudaEvent_t ready = nullptr;
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaEventRecord(ready, st);
  std::lock_guard<std::mutex> lk(g_staged_mu);
  {
    StagedHostWriter writer(copy_stream());
    e = writer.write(static_cast<char*>(host), static_cast<const char*>(device), size_t(bytes), ready);
    if (e == cudaSuccess) e = writer.finish();
  }
  // no staging copy may still be in flight when the ring is next used
  const cudaError_t se = cudaStreamSynchronize(copy_stream());
  if (e == cudaSuccess) e = se;
  cudaEventDestroy(ready);
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "staged device to host copy");
}

int cs_cut_run(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
               int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int32_t force_bond, int64_t out_begin,
               int64_t out_end, void* out, void* workspace, int64_t workspace_bytes, int32_t dtype, void* stream,
               void* const* stage_events, double* stage_ms) {
  Nvtx nvtx_entry("cs_cut_run");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  if (!out) return fail(CS_ERR_INVALID, "null output pointer");
  const auto t0 = std::chrono::steady_clock::now();
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, force_bond, dtype, &job, &rc)) return rc;
  if (!workspace || workspace_bytes < job.total_bytes)
    return fail(CS_ERR_INVALID, "cut workspace too small (query cs_cut_workspace)");
  const CutPrep& pr = job.prep;
  std::vector<std::shared_ptr<const Program>> progs;
  rc = cut_programs(job, dtype, &progs);  // compile before any timing
  if (rc != CS_OK) return rc;
  const double t_pre = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  cudaStream_t st = as_stream(stream);
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  if (stage_events) {
    for (int i = 0; i < 3; ++i) ev[i] = static_cast<cudaEvent_t>(stage_events[i]);
  } else if (stage_ms) {
    for (auto& e : ev) cudaEventCreate(&e);
  }
  if (ev[0]) cudaEventRecord(ev[0], st);
  std::vector<const void*> seg_states;
  {
    Nvtx r("variant_stage");
    rc = cut_segments(job, progs, workspace, dtype, st, &seg_states);
  }
  if (rc != CS_OK) return rc;
  if (ev[1]) cudaEventRecord(ev[1], st);
  Nvtx r_merge("merge");
  rc = run_chain(job.plan, pr.n, seg_states.data(), out_begin, out_end, out,
                 static_cast<char*>(workspace) + job.chain_off, job.total_bytes - job.chain_off, dtype, st);
  if (rc != CS_OK) return rc;
  if (ev[2]) cudaEventRecord(ev[2], st);
  if (stage_ms) {
    cudaError_t e = cudaEventSynchronize(ev[2]);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    if (!stage_events)
      for (auto& x : ev) cudaEventDestroy(x);
    if (e != cudaSuccess) return cuda_fail(e, "cut pipeline");
    stage_ms[0] = t_pre;
    stage_ms[1] = a;
    stage_ms[2] = b;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "cut pipeline");
}

int cs_cut_shard_plan(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb,
                      const double* params, int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, int32_t world,
                      int32_t rank, int32_t dtype, int64_t* info) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes || !info) return fail(CS_ERR_INVALID, "bad arguments");
  if (world < 1 || rank < 0 || rank >= world) return fail(CS_ERR_INVALID, "bad rank / world");
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, -1, dtype, &job, &rc)) return rc;
  ShardLayout lay;
  if (!shard_layout(job, nq, world, dtype, &lay, &rc)) return rc;
  if (world > lay.rows) return fail(CS_ERR_INVALID, "more ranks than output rows");
  int64_t r0, r1;
  shard_rows(lay, world, rank, &r0, &r1);
  info[0] = lay.total_bytes;
  info[1] = job.plan.q_low;
  info[2] = r0 * lay.row_amps;
  info[3] = r1 * lay.row_amps;
  info[4] = std::min(lay.total, int64_t(rank) * lay.per);
  info[5] = std::min(lay.total, int64_t(rank + 1) * lay.per);
  info[6] = lay.per;
  info[7] = lay.total;
  return CS_OK;
}

int cs_cut_run_sharded(int32_t nq, const uint8_t* kinds, const int64_t* qa, const int64_t* qb, const double* params,
                       int64_t n_gates, int32_t n_seg, const int32_t* seg_sizes, void* comm, int32_t world,
                       int32_t rank, int64_t out_begin, int64_t out_end, void* out, void* workspace,
                       int64_t workspace_bytes, int32_t dtype, void* stream, void* const* stage_events,
                       double* stage_ms) {
  Nvtx nvtx_entry("cs_cut_run_sharded");
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (nq < 2 || nq > 62 || !seg_sizes) return fail(CS_ERR_INVALID, "bad qubit count or segment sizes");
  if (world < 1 || rank < 0 || rank >= world) return fail(CS_ERR_INVALID, "bad rank / world");
  if (!out && out_end > out_begin) return fail(CS_ERR_INVALID, "null output pointer");
  const auto t0 = std::chrono::steady_clock::now();
  CutJob job;
  int rc = CS_OK;
  if (!cut_job(nq, kinds, qa, qb, params, n_gates, n_seg, seg_sizes, -1, dtype, &job, &rc)) return rc;
  ShardLayout lay;
  if (!shard_layout(job, nq, world, dtype, &lay, &rc)) return rc;
  if (!workspace || workspace_bytes < lay.total_bytes)
    return fail(CS_ERR_INVALID, "sharded cut workspace too small (query cs_cut_shard_plan)");
  // with a communicator: this rank's chunk, then the all-gather; without one
  // (comm == NULL): every variant here and no exchange (one GPU computing any
  // rank's rows, e.g. a share of the q=34 job)
  const bool exchange = comm != nullptr && world > 1;
  const int64_t g0 = exchange ? std::min(lay.total, int64_t(rank) * lay.per) : 0;
  const int64_t g1 = exchange ? std::min(lay.total, int64_t(rank + 1) * lay.per) : lay.total;
  std::vector<Piece> pieces = shard_pieces(job, lay, g0, g1, workspace, dtype);
  std::vector<std::shared_ptr<const Program>> progs;
  rc = piece_programs(job, pieces, dtype, &progs);
  if (rc != CS_OK) return rc;
  const double t_pre = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  cudaStream_t st = as_stream(stream);
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (stage_events) {
    for (int i = 0; i < 4; ++i) ev[i] = static_cast<cudaEvent_t>(stage_events[i]);
  } else if (stage_ms) {
    for (auto& e : ev) cudaEventCreate(&e);
  }
  if (ev[0]) cudaEventRecord(ev[0], st);
  {
    Nvtx r("variant_stage");
    rc = run_pieces(job, pieces, progs, dtype, st);
  }
  if (rc != CS_OK) return rc;
  if (ev[1]) cudaEventRecord(ev[1], st);
  if (exchange) {
    const int64_t chunk = lay.per * lay.L * int64_t(elem_bytes(dtype));
    rc = cs_allgather_states(comm, static_cast<char*>(workspace) + int64_t(rank) * chunk, chunk, workspace, st);
    if (rc != CS_OK) return rc;
  }
  if (ev[2]) cudaEventRecord(ev[2], st);
  std::vector<const void*> seg_states;
  for (size_t s = 0; s < job.prep.segs.size(); ++s)
    seg_states.push_back(static_cast<char*>(workspace) + lay.seg_first[s] * lay.L * int64_t(elem_bytes(dtype)));
  if (out_end > out_begin) {
    Nvtx r("merge");
    rc = run_chain(job.plan, job.prep.n, seg_states.data(), out_begin, out_end, out,
                   static_cast<char*>(workspace) + lay.chain_off, lay.total_bytes - lay.chain_off, dtype, st);
    if (rc != CS_OK) return rc;
  }
  if (ev[3]) cudaEventRecord(ev[3], st);
  if (stage_ms) {
    cudaError_t e = cudaEventSynchronize(ev[3]);
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    if (!stage_events)
      for (auto& x : ev) cudaEventDestroy(x);
    if (e != cudaSuccess) return cuda_fail(e, "sharded cut pipeline");
    stage_ms[0] = t_pre;
    stage_ms[1] = a;
    stage_ms[2] = b;
    stage_ms[3] = c;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "sharded cut pipeline");
}

static int reduce_common(const void* a, const void* b, int64_t n, int mode, int32_t dtype, double* result,
                         void* stream) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (!a || (mode != 2 && !b) || n < 0 || !result) return fail(CS_ERR_INVALID, "bad reduction arguments");
  int err = CS_OK;
  double2* scratch = reduce_scratch(&err);
  if (!scratch) return err;
  cudaStream_t st = as_stream(stream);
  cudaError_t e = launch_reduce(a, b ? b : a, n, mode, dtype, scratch, st);
  g_launches.fetch_add(2);
  if (e != cudaSuccess) return cuda_fail(e, "reduce launch");
  double2 host;
  e = cudaMemcpyAsync(&host, scratch + reduce_scratch_elems() - 1, sizeof(double2), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(reduce)");
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize(reduce)");
  result[0] = host.x;
  if (mode == 1) result[1] = host.y;
  return CS_OK;
}

int cs_maxabsdiff(const void* a, const void* b, int64_t n, int32_t dtype, double* result, void* stream) {
  return reduce_common(a, b, n, 0, dtype, result, stream);
}

int cs_maxabs(const void* a, int64_t n, int32_t dtype, double* result, void* stream) {
  return reduce_common(a, nullptr, n, 2, dtype, result, stream);
}

int cs_inner(const void* a, const void* b, int64_t n, int32_t dtype, double* result, void* stream) {
  return reduce_common(a, b, n, 1, dtype, result, stream);
}

int cs_gather(const void* state, const int64_t* idx, int64_t m, void* out, int32_t dtype, void* stream) {
  if (!valid_dtype(dtype)) return fail(CS_ERR_INVALID, "dtype must be CS_C128 or CS_C64");
  if (m == 0) return CS_OK;
  if (!state || !idx || !out || m < 0) return fail(CS_ERR_INVALID, "bad gather arguments");
  cudaError_t e = launch_gather(state, idx, m, out, dtype, as_stream(stream));
  g_launches.fetch_add(1);
  return e == cudaSuccess ? CS_OK : cuda_fail(e, "gather launch");
}

}  // extern "C"
