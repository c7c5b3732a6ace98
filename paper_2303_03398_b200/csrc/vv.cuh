// vv.cuh -- the staggered vector viscosity operator (R27-R31):
// s v + curl(nu curl v) - grad(nu div v) on MAS's staggered spherical grid, v_r / v_theta / v_phi on
// the r- / theta- / phi-faces (Sec. III), the polar axis one r-edge per radius whose
// circulation is the per-radius sum over the pole ring -- the array reduction sum0(i) of
// PAPER.md:147-157 (Listing 3), here a Dot2 ring reduction plus, across phi-slabs, an all-gather.
//
// Vectors are [nloc][3][nt][nr]: inside each phi-plane the three components (0 r, 1 theta, 2 phi)
// of the LOWER faces of the plane's cells, so a plane of all three components is contiguous (halo
// exchange without packing) and the flat PCG kernels of kernels.cu run unchanged over
// n = nloc * 3 nt * nr values.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace maspcg {

struct VVDims {
    int nr, nt, nloc;
    uint32_t plane1;        // nt * nr
    uint32_t plane3;        // 3 * nt * nr
    uint32_t ncell;         // nloc * nt * nr
    FastDiv div_r, div_t;
    int wall_in, wall_out;  // 0 no-slip, 1 free-slip
    // chunked matvec (the pair kernels, homogeneous operator): the rows of planes [kb, ke) from the terms of
    // planes [kb - 1, ke], which live in rings of `ring` planes (slot (k + 1) % ring) kept in the L2
    // (evict_last inside a persisting set-aside); ring == 0: full-size term arrays, one chunk [0, nloc)
    int kb, ke;
    uint32_t ring;
    int chunk, nchunks;     // the rows' Dot2: per-chunk pairs, combined by the last chunk's last block
};

struct VVArrays {
    // 1-D metric (host-computed, same expressions as the oracle)
    double *rf, *rf2, *hr, *dr, *R3, *rce, *rhor, *dR2, *rc2;   // nr+1, nr+1, nr+1, nr, nr, nr+2, nr+1, nr, nr
    double *C, *dt, *ht, *Cs, *sinc, *sinf;                     // nt, nt, nt+1, nt+1, nt, nt+1
    double *dpp, *hmp;                                          // [nloc+2]: planes k0-1 .. k0+nloc (periodic)
    double *cap;                                                // [2]: capN, capS
    // coefficients
    double *wc;     // [nloc+2][nt][nr] nu / V (halo planes)
    double *Wr;     // [nloc+2][nt][nr] r-edge at theta-face j (j >= 1), phi-face k
    double *Wt;     // [nloc+2][nt][nr] theta-edge at r-face i (< nr), phi-face k
    double *WtO;    // [nloc+2][nt]     theta-edge on the outer wall (r-face nr)
    double *Wp;     // [nloc][nt][nr]   phi-edge at r-face i (< nr), theta-face j (j >= 1)
    double *WpO;    // [nloc][nt]       phi-edge on the outer wall
    double *WN, *WS;   // [nr] polar axes
    double *sM;     // [nloc][3][nt][nr] s_f M_f
    double *D;      // [nloc][3][nt][nr] Jacobi diagonal (1 on non-unknown slots)
    double *bw;     // [nloc][3][nt][nr] A(0; g): the wall-data part of the rhs
    // matvec phase-1 terms (planes -1 .. nloc; padded like wc)
    double *E;      // [nloc+2][nt][nr] wc * delta
    double *TR, *TT, *TP;   // [nloc+2][nt][nr] W Gamma of the lower r-, theta-, phi-edges of each cell
    double *TTO, *TPO;      // [nloc+2][nt]     the same on the outer wall (r-face nr)
    // inputs (consumed copies) and wall data
    double *nu, *s;          // [nloc][nt][nr]
    double *nulo, *slo;      // [nt][nr] plane k0-1 of nu, s (received, nranks > 1)
    double *gin, *gout;      // [nloc+2][3][nt] wall data (halo planes)
    // PCG vectors
    double *p;      // [nloc+2][3][nt][nr]
    double *q, *r;  // [nloc][3][nt][nr]
    // ring reductions
    double *ring;   // [2 poles][nr][2] Dot2 pairs (north, south); global after the all-gather
    double *nuring; // [2][nr][2]
    double *gather; // [kMaxRanks][4 nr]
};

// Validation of nu, s (>= 0, finite) into sc->vinvalid.
void launch_vv_validate(const VVDims &v, const double *nu, const double *s, int *flag, cudaStream_t st);
// Coefficients of the local planes (wc, Wr, Wt, WtO, Wp, WpO, sM) from the consumed nu, s and their
// plane k0-1 (nulo, slo).
void launch_vv_coef(const VVDims &v, const VVArrays &a, cudaStream_t st);
// Ring sums: mode 0 -- sum_k nu(i, pole row, k) into a.nuring; mode 1 -- sum_k l_p v_p(i, pole row, k)
// of p into a.ring.  Dot2 pairs per (pole, i), fixed-tree order.
void launch_vv_ring(const VVDims &v, const VVArrays &a, int mode, bool exact, cudaStream_t st);
// WN, WS from the global nu rings; np = global plane count.
void launch_vv_axis_weights(const VVDims &v, const VVArrays &a, int np, cudaStream_t st);
void launch_vv_diag(const VVDims &v, const VVArrays &a, cudaStream_t st);
// y = A p (homogeneous) or, wall = true, y = A(p; g) (used with p = 0 for bw).  with_dot: Dot2
// partial p.y -> sc->red1 via the last block; loop: early exit when sc->done.
void launch_vv_matvec(const VVDims &v, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                      bool wall, bool exact, cudaStream_t st);
// The same (homogeneous operator, nr even) as ONE plane-marching kernel with TMA-staged input planes
// (vv_march.cu); false when not applicable (odd nr, unaligned y, MASPCG_VV_MARCH=0) -- nothing launched.
bool launch_vv_march(const VVDims &v, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                     bool exact, cudaStream_t st);
// Planes per term ring of the chunked matvec for an L2 budget of `bytes` (0: the chunked form is off --
// MASPCG_VV_CHUNK=0, odd nr, or a slab of at most two chunks), and the ring's bytes (4 term arrays).
uint32_t vv_ring_planes(const VVDims &v, size_t bytes);
size_t vv_ring_bytes(const VVDims &v, uint32_t ring);
// b = M f - bw; r = b - q; z = r / D; p = z (padded, periodic copies when periodic_local);
// Dot2 partials r.z, r.r, b.b -> sc->red3.
void launch_vv_setup_residual(const VVDims &v, const VVArrays &a, const DevArrays &base, const Dims &dv,
                              const double *f, bool exact, cudaStream_t st);
// zero x on the non-unknown slots (v_r on r-face 0, v_theta on theta-face 0)
void launch_vv_mask(const VVDims &v, double *x, cudaStream_t st);

}  // namespace maspcg
