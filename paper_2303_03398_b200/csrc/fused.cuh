// fused.cuh -- two-pass PCG iteration (fused.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace maspcg {

struct FusedArgs {
    const double *p_old;               // p_{it-1}  [nloc][nt][nr]
    double *p_new;                     // p_it      [nloc][nt][nr]
    double *x;                         // caller's x
    const double *r;                   // r_{it-1}
    const double *r_lo, *r_hi;         // plane -1 / nloc of r   (wrap planes or received halos)
    const double *d_lo, *d_hi;         // plane -1 / nloc of D
    const double *p_lo, *p_hi;         // plane -1 / nloc of p_old
    int bj;                            // theta rows per tile (TMA variant: the tallest tile)
    int n_jt;                          // number of j-tiles
    int nch;                           // TMA variant: plane chunks (grid = n_jt * nch)
    int tma;                           // 1: k_pass_a_tma (bulk-copy staged), 0: k_pass_a
    FastDiv div_r;                     // / nr
};

int fused_bj(int nr, int nt);
size_t fused_smem_bytes(int nr, int bj);
int fused_blocks(int nr, int nt, int nloc, int bj, int device);
// Lockstep tiling of the TMA variant: n_jt x nch blocks (<= SMs), tallest tile hmax; false if
// unsupported (odd nr, or no tile height fits the shared memory).
bool fused_tma_geometry(int nr, int nt, int nloc, int device, int *njt, int *nch, int *hmax);
size_t tma_smem_bytes(int nr, int hmax);
void launch_pass_a(const Dims &d, const DevArrays &a, const FusedArgs &f, int blocks, bool exact, cudaStream_t st);
void launch_pass_b(const Dims &d, const DevArrays &a, bool exact, cudaStream_t st);

}  // namespace maspcg
