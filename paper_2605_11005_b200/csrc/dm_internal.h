// Host-side internals shared by the .cu translation units of libdm_moe.so.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dm_moe.h"

namespace dm {

// Records a message for dm_last_error_string() and returns `code`.
int set_error(int code, const char* fmt, ...);
// Records a CUDA runtime error; returns the (positive) cudaError_t value.
int set_cuda_error(cudaError_t err, const char* what);

// Cached per-device multiprocessor count of the current device.
int num_sms_current();

// cuTensorMapEncodeTiled resolved once through the runtime's driver entry point.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

// Raises `func`'s dynamic shared-memory limit to `bytes` on the current device, once per
// (kernel, device), thread-safe (cudaFuncSetAttribute is per device).
int ensure_smem_attr(const void* func, int bytes, const char* what);
// Cached cudaOccupancyMaxActiveBlocksPerMultiprocessor per (kernel, device); >= 1.
int max_active_blocks(const void* func, int threads, size_t smem);

// Counts kernel launches issued through the ABI (reported by dm_launch_count()).
void note_launch();

}  // namespace dm
