// NVRTC specialisation of register-tile sweep programs (see jit.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <memory>
#include <string>
#include <vector>

#include "ops.hpp"
#include "plan.hpp"

namespace cutsim {

// One compiled launch kernel (one NVRTC program): shared by every launch
// whose generated source is identical (jit.cpp's unit cache).
struct JitUnit {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  size_t smem = 0;
  int threads = 0;
  bool persistent = false;  // one CTA per SM walking the tiles, next tile prefetched
  // devices whose launch attributes (dynamic smem, cluster size) are set: one
  // bit per device, so the per-launch path makes no attribute calls
  std::atomic<uint64_t> attrs_set{0};
  ~JitUnit();
};

// A program's specialised launches: unit i (null = interpreter) and, in param
// mode, the kernel-parameter block of launch i (its matrices and phases).
struct JitModule {
  std::vector<std::shared_ptr<JitUnit>> units;
  std::vector<std::vector<unsigned char>> blobs;
  int cluster = 0;  // > 0: ONE cluster-resident kernel (units[0]) of this many CTAs per state
};

// CUDA C++ source of one launch: straight-line code for the register program
// (dense/phase/remap) with the tile geometry, masks, matrices (hex-float
// literals) and remap index maps baked in.
// pvals != null: param mode (coefficients other than 0 / +-1 go to the
// kernel-parameter block, appended to *pvals in order)
std::string jit_source(const Sweep& sw, const std::vector<RegOp>& prog, int reg_bits, int dtype,
                       const std::string& name, int minb = 1, bool persistent = false,
                       std::vector<double>* pvals = nullptr);

// Compile every launch of a program into one module (sm_100a CUBIN via
// NVRTC, loaded with cudaLibraryLoadData). Returns null and sets *err on
// failure (NVRTC missing, compile error).
// minb[i]: __launch_bounds__ min CTAs per SM of launch i (null: 1);
// persistent[i]: the prefetching tile-walking form (null: none)
std::shared_ptr<JitModule> jit_compile(const std::vector<const Sweep*>& sweeps,
                                       const std::vector<const std::vector<RegOp>*>& progs, int dtype,
                                       std::string* err, const std::vector<int>* minb = nullptr,
                                       const std::vector<char>* persistent = nullptr, bool param_mode = false);

// The whole program as one cluster-resident kernel (jit.cpp
// jit_cluster_source): every launch's sweep must use tile_bits T with
// 2^(nq - T) tiles = the cluster size.
std::string jit_cluster_source(const std::vector<const Sweep*>& sweeps,
                               const std::vector<const std::vector<RegOp>*>& progs, int T, int RB, int dtype,
                               const std::string& name, std::vector<double>* pvals);
std::shared_ptr<JitModule> jit_compile_cluster(const std::vector<const Sweep*>& sweeps,
                                               const std::vector<const std::vector<RegOp>*>& progs, int T,
                                               int dtype, std::string* err, bool param_mode);
bool jit_cluster_cubin(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
                       int T, int dtype, std::vector<char>* cubin, std::string* err, bool param_mode);

// NVRTC loaded and one trivial compile done on this thread (libraries a
// compile needs are loaded); false when NVRTC is unavailable
bool jit_warm_nvrtc();

// units compiled / served from the unit cache since load (cs_get_option
// "jit_units_compiled" / "jit_units_reused")
int64_t jit_units_compiled();
int64_t jit_units_reused();

// NVRTC step only (no device needed): the CUBIN and kernel names.
bool jit_cubin(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
               int dtype, std::vector<char>* cubin, std::vector<std::string>* names, std::string* err,
               bool param_mode = false);

// min CTAs per SM requested from the generated kernels that stream many
// tiles (option "jit_minb", default 2: <= 128 registers, two 256-thread CTAs
// per SM; measured uncut q=30 182 ms vs 261 ms at one CTA per SM)
extern int g_jit_minb;
// option "jit_persistent": streaming sweeps as persistent kernels that
// prefetch the next tile with cp.async (1) or one CTA per tile (0, default:
// the persistent form needs 128 KB of shared memory = one 8-warp CTA per SM
// and measured 171 vs 146 ms on the q=30 uncut circuit)
extern int g_jit_persistent;

// FP64 instructions the specialised code would contain (size guard).
int64_t jit_cost(const std::vector<RegOp>& prog, int reg_bits);

}  // namespace cutsim
