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
    int bj;                            // theta rows per tile
    int n_jt;                          // number of j-tiles
    FastDiv div_r;                     // / nr
};

int fused_bj(int nr, int nt);
size_t fused_smem_bytes(int nr, int bj);
int fused_blocks(int nr, int nt, int nloc, int bj, int device);
void launch_pass_a(const Dims &d, const DevArrays &a, const FusedArgs &f, int blocks, bool exact, cudaStream_t st);
void launch_pass_b(const Dims &d, const DevArrays &a, bool exact, cudaStream_t st);

}  // namespace maspcg
