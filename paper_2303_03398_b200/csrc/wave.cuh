// wave.cuh -- p-update + stencil in one flag-ordered persistent kernel (wave.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace maspcg {

constexpr int kWaveTile = 4096;   // cells per tile (contiguous inside one phi-plane)

struct WaveArgs {
    unsigned *counter;        // work-item dispatch counter (reset by the last block)
    unsigned *flags;          // [nloc] A-tiles completed per plane (reset by the last block)
    double *tile_partials;    // [nloc * tpp][2] Dot2 pairs of p.q per B-tile
    int tpp;                  // tiles per plane
    int lag;                  // B trails A by lag planes (> the planes in progress across the grid)
};

inline int wave_tiles_per_plane(uint32_t plane) { return (int)((plane + kWaveTile - 1) / kWaveTile); }
int wave_grid(int device);
void launch_wave(const Dims &d, const DevArrays &a, const WaveArgs &w, double *x, int chunk, int grid, bool exact,
                 cudaStream_t st);

}  // namespace maspcg
