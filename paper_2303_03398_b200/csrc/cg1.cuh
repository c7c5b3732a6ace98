// cg1.cuh -- the single-reduction point-Jacobi PCG (Chronopoulos & Gear 1989; SURVEY.md 8(f) NEXT-3,
// reading R32 of DESIGN.md): one operator application and ONE fused reduction (gamma = r.u,
// delta = w.u, r.r) per iteration -- one all-reduce instead of two on P > 1 -- in two streaming kernels
// (128 B/cell, the same traffic as the three-kernel path).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace maspcg {

// The convergence test of the previous iterate (r.r in red2[2..3]), then beta (gamma = r.u in red2[0..1]),
// alpha (delta = w.u in red1), p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s, u = r / D
// (into the padded cgr, periodic copies on one rank) and the local Dot2 r.u, r.r of the new iterate.
// The matvec w = A u is launch_matvec of kernels.cuh on a DevArrays whose p is cgr.
void launch_cg1_update(const Dims &d, const DevArrays &a, double *x, bool exact, cudaStream_t st);

}  // namespace maspcg
