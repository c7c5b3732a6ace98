// kernels.cuh -- launchers of the sm_100a kernels (kernels.cu, stencil_tiled.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace maspcg {

enum class StencilPart { Full, Interior, Boundary };

void launch_assemble(const Dims &d, const DevArrays &a, const double *kr, const double *kt, const double *kp,
                     const double *s, cudaStream_t st);
// Face coefficients kr, kt, kp and shift s of the local slab from a cell field (NEXT-1, R25).
void launch_face_coeffs(const Dims &d, const double *f, const double *f_hi, const double *rho, double kappa0,
                        int half_power, int mean, double inv_dt, double *kr, double *kt, double *kp, double *s,
                        cudaStream_t st);
void launch_finalize_D(const Dims &d, const DevArrays &a, int bc_in, int bc_out, cudaStream_t st);
void launch_fill_p(const Dims &d, const DevArrays &a, const double *x, cudaStream_t st);

// The cells of `part` of the local slab as a launch range.
Range make_range(const Dims &d, StencilPart part);
// Number of blocks launch_matvec uses for `part` (0: nothing to do).
unsigned stencil_blocks(const Dims &d, StencilPart part, const double *y);
// y = A p over `part` of the slab.  with_dot: partial p.y into partial slots
// [red_slot0, red_slot0 + blocks); the last of red_total blocks writes
// sc->red1[0].  loop: early exit when sc->done.
// exact: the oracle-identical arithmetic of arith.cuh (no FMA contraction, Dot2 dot products).
void launch_matvec(const Dims &d, const DevArrays &a, double *y, StencilPart part, bool with_dot, bool loop,
                   unsigned red_slot0, unsigned red_total, bool exact, cudaStream_t st);

void launch_setup_residual(const Dims &d, const DevArrays &a, const double *f, int din, int dout, bool exact,
                           cudaStream_t st);
void launch_setup_scalars(const DevArrays &a, double tol, int maxit, cudaStream_t st);
void launch_update(const Dims &d, const DevArrays &a, bool exact, cudaStream_t st);
void launch_pupdate(const Dims &d, const DevArrays &a, double *x, int chunk, bool exact, cudaStream_t st);
// out[2t..2t+1] = rank-ordered Dot2 combination of gather[r][2t..2t+1], t < npairs.
void launch_dd_combine(const double *gather, int nranks, int npairs, double *out, bool exact, cudaStream_t st);
// RKL2 super-time-stepping stages (NEXT-4, R26); *p arguments are padded [nloc+2][nt][nr] arrays.
void launch_sts_first(const Dims &d, const DevArrays &a, const double *y0p, double *l0, double *y1p, double m1,
                      int din, int dout, bool exact, cudaStream_t st);
void launch_sts_stage(const Dims &d, const DevArrays &a, const double *yj1p, const double *yj2p, const double *y0p,
                      const double *l0, double *yjp, double mu, double nu, double w0, double mt, double gt, int din,
                      int dout, bool exact, cudaStream_t st);
// per-block maxima of the Gershgorin bound of lambda_max(V^-1 K) into out[0..blocks); returns blocks
unsigned launch_sts_gershgorin(const Dims &d, const DevArrays &a, double *out, cudaStream_t st);
void launch_zero_x_if(const Dims &d, const DevArrays &a, double *x, cudaStream_t st);
// inside the body of a conditional WHILE node: set the condition to "not done"
void launch_loop_cond(cudaGraphConditionalHandle h, const Scalars *sc, cudaStream_t st);
// applypriority L2::evict_normal over the 128-byte lines of [p, p + bytes) (undoes an L2_KEEP policy)
void launch_l2_demote(const void *p, size_t bytes, cudaStream_t st);

}  // namespace maspcg
