// aniso.cuh -- field-aligned anisotropic conduction (reading R33 of DESIGN.md): the
// 19-point operator A = (7-point operator of K_aa = kappa_perp + kappa_par b_a^2) + cross terms
// kappa_par b_a b_b on the edges where an a-face meets a b-face.  The CPU oracle (oracle/) implements the
// same reading independently; this file shares nothing with it.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace maspcg {

// Library-owned arrays of the cross terms (a caller-owned workspace of its own), Xq = X / 4.
struct AnisoArrays {
    double *Xrt;   // [nloc][nt][nr]    edge (lower r-face i, lower theta-face j) of plane k; 0 at i = 0 or j = 0
    double *Xrp;   // [nloc+1][nt][nr]  plane kk: edge (lower r-face i, row j) on phi face (k0 + kk - 1) + 1/2; 0 at i = 0
    double *Xtp;   // [nloc+1][nt][nr]  plane kk: edge (lower theta-face j, column i) on that phi face; 0 at j = 0
    double *D7;    // [nloc][nt][nr]    diagonal of the 7-point part (the Jacobi diagonal a.D = D7 + cross diagonal)
    double *gr;    // [nr]  (rc_i^2 + rc_i rc_{i-1} + rc_{i-1}^2) / (3 r_f[i]), i >= 1
    double *qr;    // [nr]  R3_i / rc_i^2
    double *gt;    // [nt]  2 sin((tc_{j-1} + tc_j)/2) sin(h^t_j/2) / h^t_j, j >= 1
    double *cs;    // [nt]  2 sin(dtheta_j / 2)
    double *gts;   // [nt]  gt_j / sin t_f[j]
};

// Xrt, Xrp (planes 1..nloc), Xtp (planes 1..nloc) from the caller's edge coefficients krt [nloc][nt+1][nr+1],
// krp [nloc][nt][nr+1], ktp [nloc][nt+1][nr]; a non-finite entry sets sc->vinvalid.
void launch_aniso_edges(const Dims &d, const DevArrays &a, const AnisoArrays &x, const double *krt, const double *krp,
                        const double *ktp, cudaStream_t st);
// x.D7 := a.D (the 7-point diagonal of k_finalize_D), a.D := D7 + sum_e Xq_e (2 s_a s_b)
void launch_aniso_diag(const Dims &d, const DevArrays &a, const AnisoArrays &x, cudaStream_t st);
// y = A p over `part` of the slab (as launch_matvec), optional Dot2 partial of p.y
void launch_aniso_matvec(const Dims &d, const DevArrays &a, const AnisoArrays &x, double *y, StencilPart part,
                         bool with_dot, bool loop, unsigned red_slot0, unsigned red_total, bool exact, cudaStream_t st);
unsigned aniso_stencil_blocks(const Dims &d, StencilPart part, const double *y);

}  // namespace maspcg
