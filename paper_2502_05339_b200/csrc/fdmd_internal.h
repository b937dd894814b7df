// Private hooks shared by the CUDA unit (fdmd_abi.cu) and the host
// orchestration unit (fdmd_fit.cpp). Not part of the public C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif
/* stores msg in the thread-local slot read by fdmd_last_error(); returns code */
int fdmdi_set_error(int code, const char* msg);
/* stream-ordered scratch from the device's default pool (fdmd_abi.cu:scratch_alloc) */
cudaError_t fdmdi_scratch_alloc(void** p, size_t bytes, void* stream);
/* per-thread, per-device cuSOLVER handle bound to `stream` (cusolverDnHandle_t) */
void* fdmdi_solver_handle(void* stream);
#ifdef __cplusplus
}
#endif
