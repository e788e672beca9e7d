// Internal (non-ABI) launchers shared between translation units.
#pragma once
#include <cuda_runtime.h>

#include "sf_common.cuh"

namespace sf {
// FP64 Q7 vmult on DMMA tensor cores (sf_dmma.cu); returns 0 or SF_ECUDA
int launch_vmult_dmma8(const Geom& g, const double* level_op, const void* u, void* v, int batch, cudaStream_t st);
// FP64 Q7 smoother colour pass on DMMA (sf_dmma.cu)
int launch_colour_dmma8(const Geom& g, const double* level_op, const double* patch_eig, const void* x_old,
                        const void* b, void* x_new, cudaStream_t st);
}  // namespace sf
