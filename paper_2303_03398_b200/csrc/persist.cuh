// persist.cuh -- the persistent PCG iteration kernel (persist.cu), MASPCG_OPT_PATH = 5.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace maspcg {

// co-resident grid of the persistent kernel on `device` (SMs x blocks per SM)
unsigned persist_grid(int device);
// `iters` PCG iterations (or until done) in one cooperative launch; single rank, nr even, x 16-byte aligned
cudaError_t launch_persist(const Dims &d, const DevArrays &a, double *x, int iters, int ring, unsigned grid, bool exact,
                           cudaStream_t st);

}  // namespace maspcg
