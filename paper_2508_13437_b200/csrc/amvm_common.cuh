// amvm_common.cuh — host helpers shared by the libamvm translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/amvm.h"

namespace amvm {
inline int cuda_rc(cudaError_t e) { return e == cudaSuccess ? AMVM_OK : AMVM_ERR_CUDA; }
}  // namespace amvm
