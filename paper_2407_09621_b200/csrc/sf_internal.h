// Internal (non-ABI) launchers shared between translation units.
#pragma once
#include <cuda_runtime.h>

#include "sf_common.cuh"

namespace sf {
// FP64 Q7 vmult on DMMA tensor cores (sf_dmma.cu); returns 0 or SF_ECUDA
int launch_vmult_dmma8(const Geom& g, const double* level_op, const void* u, void* v, int batch, cudaStream_t st);
}  // namespace sf
