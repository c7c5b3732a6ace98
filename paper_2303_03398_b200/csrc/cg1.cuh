// cg1.cuh -- the single-reduction point-Jacobi PCG (Chronopoulos & Gear 1989; SURVEY.md 8(f) NEXT-3,
// reading R32 of DESIGN.md): one operator application and ONE fused reduction (gamma = r.u,
// delta = w.u, r.r) per iteration -- one all-reduce instead of two on P > 1 -- in two streaming kernels
// (128 B/cell, the same traffic as the three-kernel path).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace maspcg {

// w = A u with u = r / D formed on the fly (r from the padded cgr, D with its halo planes: periodic
// on one rank, a.dh otherwise) over `part` of the slab; Dot2 partials of r.u, w.u, r.r into partial
// slots [red_slot0, red_slot0 + blocks); the last of red_total blocks writes sc->red_cg.
// loop: early exit when sc->done.
void launch_cg1_matvec(const Dims &d, const DevArrays &a, StencilPart part, bool loop, unsigned red_slot0,
                       unsigned red_total, bool exact, cudaStream_t st);
unsigned cg1_matvec_blocks(const Dims &d, StencilPart part);
// The convergence test of the previous iterate (from red_cg), then beta, alpha and p = u + beta p,
// s = w + beta s, x += alpha p, r -= alpha s (r into cgr, periodic copies on one rank).
void launch_cg1_update(const Dims &d, const DevArrays &a, double *x, bool exact, cudaStream_t st);

}  // namespace maspcg
