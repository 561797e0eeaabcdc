// Internal (not part of the C ABI): the one per-thread record of the cudaError_t
// behind a TDES_ERR_CUDA, shared by every translation unit of the library so
// that tdes_last_cuda_error() (include/tdes.h) is right after a failure in any
// entry point -- tdes.h, tdes_bench.h or tdes_paper.h.
#ifndef TDES_ERROR_H_
#define TDES_ERROR_H_

#include <cuda_runtime.h>

namespace tdes_internal {
// Records e for tdes_last_cuda_error() on this host thread; returns TDES_ERR_CUDA.
int cuda_fail(cudaError_t e);
// TDES_DEBUG builds: TDES_OK if p (nbytes > 0) is device-accessible memory of the
// current device (cudaPointerGetAttributes), else TDES_ERR_INVALID_ARG.  Release
// builds: always TDES_OK (no driver call on the launch path).
int check_device_pointer(const void* p);
}  // namespace tdes_internal

#endif  // TDES_ERROR_H_
