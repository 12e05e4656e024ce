// Return codes of the libcutsim C-ABI (mirrored in include/cutsim.h).
#pragma once

#define CS_OK 0
#define CS_ERR_INVALID 1   /* -> ValidationError */
#define CS_ERR_CAPACITY 2  /* -> CapacityError */
#define CS_ERR_CUDA 3      /* -> DeviceError */
#define CS_ERR_NCCL 4      /* -> DeviceError */
#define CS_ERR_INTERNAL 5  /* -> CutbenchError */
#define CS_ERR_NODEVICE 6  /* -> NativeUnavailableError */
#define CS_ERR_TOPOLOGY 7  /* -> UnsupportedTopologyError */
#define CS_ERR_TIMEOUT 8   /* -> BudgetExceededError */
