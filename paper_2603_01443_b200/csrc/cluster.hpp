// Cluster-resident variant batches as ONE ahead-of-time compiled kernel
// (cluster.cu): the register program is data, not code.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "ops.hpp"
#include "plan.hpp"

namespace cutsim {

// A program packed for cluster_prog_kernel: per phase (one launch of the
// schedule) a 32-byte geometry record, then the op stream (8 bytes per op),
// then the coefficient sets (1, 2 or 4 complex values by op kind; a slotted
// op's alternative set follows its own); at most 32000 bytes (the kernel
// parameter block).
struct ClusterBlob {
  std::vector<unsigned char> bytes;
  uint32_t ops_off = 0, coef_off = 0;
  int T = 0, RB = 0, cluster = 0, dtype = 0;
  int64_t n_ops = 0;
};

// false (and *err) when the program does not fit the encoding (the NVRTC
// cluster kernel then runs it)
bool cluster_blob_build(const std::vector<const Sweep*>& sweeps, const std::vector<const std::vector<RegOp>*>& progs,
                        int T, int dtype, ClusterBlob* out, std::string* err);

// one launch: a cluster of blob.cluster CTAs per state, n_states states
// (blockIdx.y = state, variant id vbase + y); the blob travels as the
// kernel-parameter block. Not thread-safe (callers hold capi's launch lock).
cudaError_t launch_cluster_prog(const ClusterBlob& blob, void* states, int64_t stride, uint64_t vbase,
                                uint32_t n_states, cudaStream_t st);

}  // namespace cutsim
