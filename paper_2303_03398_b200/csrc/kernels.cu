// kernels.cu -- sm_100a fp64 kernels of the MAS implicit parabolic PCG solve.
//
// Hot path per PCG iteration (BASELINE.json north_star):
//   stencil_matvec_dot  q = A p, partial p.q          48 B/cell algorithmic
//   update_jacobi_dots  x += a p, r -= a q, z = r/D,  56 B/cell
//                       partials r.z and r.r
//   p_update            p = r/D + b p                 32 B/cell
// All three are HBM-bandwidth bound (~0.2 flop/B, "highly
// memory-bound"): no tensor cores.  Reductions are warp shuffles + one
// partial per block + a last-block (atomic ticket) fixed-order final sum, so
// results are bitwise deterministic run to run and independent of block
// scheduling.  Scalars (alpha, beta, rho, convergence) live in device memory
// (Scalars) and are consumed at kernel entry: no host round trip per
// iteration (the "gaps between kernel launches" of PAPER.md:292).
//
// Setup kernels (assembly, D, rhs) use __dmul_rn/__dadd_rn/__ddiv_rn so the
// operator is computed with exactly one IEEE rounding per operation in the
// order of the formulas of SURVEY.md 8(c) items 3-5 (no FMA contraction).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "arith.cuh"
#include "p2p_ll.cuh"
#include "loopdev.cuh"

namespace maspcg {

namespace {

constexpr int kMinBlocks = kRedBlocks / 148;   // 8 resident blocks of 256 threads per SM (<= 32 registers)
constexpr int kVecBlocks = 4;                   // vector kernels: 4 blocks of 256 threads per SM (<= 64 registers)
constexpr int kMvBlocks = 5;                    // the vector stencil: 5 blocks per SM (<= 51 registers)
static_assert(kPartialSlots >= 2 * kRedBlocks && kPartialSlots >= 2 * 148 * kMvBlocks,
              "a split stencil (interior + boundary launches) must fit the Dot2 partial slots");

// Write a freshly computed p value of local cell c (plane k) into the padded
// p array and, on a single rank, into the periodic halo copies.
__device__ __forceinline__ void store_p(const Dims &d, double *p, uint32_t c, double v) {
    p[(size_t)c + d.plane] = v;
    if (d.periodic_local) {
        if (c < d.plane) p[(size_t)c + (size_t)(d.nloc + 1) * d.plane] = v;    // hi halo <- first plane
        if (c >= d.n - d.plane) p[(size_t)c - (size_t)(d.nloc - 1) * d.plane] = v; // lo halo <- last plane
    }
}

// ---------------------------------------------------------------- assembly
// SURVEY 8(c) item 3 (R3-R5, R8): face transmissibilities, s*V, validation.
__global__ void __launch_bounds__(kThreads) k_assemble(Dims d, DevArrays a, const double *__restrict__ kr,
                                                       const double *__restrict__ kt,
                                                       const double *__restrict__ kp,
                                                       const double *__restrict__ s) {
    int bad = 0, pos = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        const uint32_t row = (uint32_t)k * d.nt + j;
        const double dpk = a.dp[k];
        // r-face i (lower face of the cell; i = 0 is the inner boundary face)
        const double kri = kr[(size_t)row * (d.nr + 1) + i];
        bad |= !(kri >= 0.0) | !isfinite(kri);
        a.Tr[c] = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(kri, a.rf2[i]), a.C[j]), dpk), a.hr[i]);
        if (i == d.nr - 1) {
            const double kro = kr[(size_t)row * (d.nr + 1) + d.nr];
            bad |= !(kro >= 0.0) | !isfinite(kro);
            a.TrB[row] = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(kro, a.rf2[d.nr]), a.C[j]), dpk), a.hr[d.nr]);
        }
        // theta-face j (lower); boundary faces j = 0, nt carry no flux (R8)
        const size_t tbase = ((size_t)k * (d.nt + 1) + j) * d.nr + i;
        const double ktj = kt[tbase];
        bad |= !(ktj >= 0.0) | !isfinite(ktj);
        a.Tt[c] = (j == 0) ? 0.0
                           : __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(ktj, a.sinf[j]), a.dr[i]), dpk), a.ht[j]);
        if (j == d.nt - 1) {
            const double kte = kt[tbase + d.nr];
            bad |= !(kte >= 0.0) | !isfinite(kte);
        }
        // phi-face k+1/2 -> Tp plane k+1
        const double kpc = kp[c];
        bad |= !(kpc >= 0.0) | !isfinite(kpc);
        a.Tp[(size_t)c + d.plane] =
            __ddiv_rn(__dmul_rn(__dmul_rn(kpc, a.dr[i]), a.dt[j]), __dmul_rn(a.sinc[j], a.hp[k]));
        // s * V, V = R3_i C_j dphi_k
        const double sc = s[c];
        bad |= !(sc >= 0.0) | !isfinite(sc);
        pos |= (sc > 0.0);
        const double V = __dmul_rn(__dmul_rn(a.R3[i], a.C[j]), dpk);
        a.sV[c] = __dmul_rn(sc, V);
    }
    bad = __syncthreads_or(bad);
    pos = __syncthreads_or(pos);
    if (threadIdx.x == 0) {
        if (bad) atomicOr(&a.sc->vinvalid, 1);
        if (pos) atomicOr(&a.sc->vshift, 1);
    }
}

// D = sV + Tr_lo + Tr_hi + Tt_lo + Tt_hi + Tp_lo + Tp_hi  (R7, R10)
// ---------------------------------------------------------------- coefficients from fields (NEXT-1)
// kappa_c = kappa0 f_c^(m/2) as ((kappa0 f) f ...) sqrt(f) -- the same product as the oracle (R25).
// The same assembly, two r-neighbour cells per thread (nr even): 16-byte loads of kt, kp, s and 16-byte
// stores of T_r, T_theta, T_phi, sV; each cell's products and divisions in the order of k_assemble.
__global__ void __launch_bounds__(kThreads) k_assemble_vec2(Dims d, DevArrays a, const double *__restrict__ kr,
                                                            const double *__restrict__ kt,
                                                            const double *__restrict__ kp,
                                                            const double *__restrict__ s) {
    int bad = 0, pos = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = d.n >> 1;
    const int nr = d.nr, nt = d.nt;
    auto fin = [](double v) { return !(v >= 0.0) | !isfinite(v); };
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < npair; v += stride) {
        const uint32_t c = 2u * v;
        int i, j, k;
        decompose(d, c, i, j, k);
        const uint32_t row = (uint32_t)k * nt + j;
        const size_t rb = (size_t)row * (nr + 1) + i;
        const size_t tb = ((size_t)k * (nt + 1) + j) * nr + i;
        const double kr0 = __ldg(kr + rb), kr1 = __ldg(kr + rb + 1);
        const double2 ktv = __ldg(reinterpret_cast<const double2 *>(kt + tb));
        const double2 kpv = __ldg(reinterpret_cast<const double2 *>(kp + c));
        const double2 sv = __ldg(reinterpret_cast<const double2 *>(s + c));
        const double dpk = a.dp[k], Cj = a.C[j];
        bad |= fin(kr0) | fin(kr1) | fin(ktv.x) | fin(ktv.y) | fin(kpv.x) | fin(kpv.y) | fin(sv.x) | fin(sv.y);
        pos |= (sv.x > 0.0) | (sv.y > 0.0);
        const double tr0 = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(kr0, a.rf2[i]), Cj), dpk), a.hr[i]);
        const double tr1 = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(kr1, a.rf2[i + 1]), Cj), dpk), a.hr[i + 1]);
        *reinterpret_cast<double2 *>(a.Tr + c) = make_double2(tr0, tr1);
        if (i + 2 == nr) {
            const double kro = __ldg(kr + rb + 2);
            bad |= fin(kro);
            a.TrB[row] = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(kro, a.rf2[nr]), Cj), dpk), a.hr[nr]);
        }
        double tt0 = 0.0, tt1 = 0.0;
        if (j != 0) {
            const double sf = a.sinf[j], htj = a.ht[j];
            tt0 = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(ktv.x, sf), a.dr[i]), dpk), htj);
            tt1 = __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(ktv.y, sf), a.dr[i + 1]), dpk), htj);
        }
        *reinterpret_cast<double2 *>(a.Tt + c) = make_double2(tt0, tt1);
        if (j == nt - 1) {
            const double2 kte = __ldg(reinterpret_cast<const double2 *>(kt + tb + nr));
            bad |= fin(kte.x) | fin(kte.y);
        }
        const double dtj = a.dt[j], den = __dmul_rn(a.sinc[j], a.hp[k]);
        const double tp0 = __ddiv_rn(__dmul_rn(__dmul_rn(kpv.x, a.dr[i]), dtj), den);
        const double tp1 = __ddiv_rn(__dmul_rn(__dmul_rn(kpv.y, a.dr[i + 1]), dtj), den);
        *reinterpret_cast<double2 *>(a.Tp + (size_t)c + d.plane) = make_double2(tp0, tp1);
        const double V0 = __dmul_rn(__dmul_rn(a.R3[i], Cj), dpk), V1 = __dmul_rn(__dmul_rn(a.R3[i + 1], Cj), dpk);
        *reinterpret_cast<double2 *>(a.sV + c) = make_double2(__dmul_rn(sv.x, V0), __dmul_rn(sv.y, V1));
    }
    bad = __syncthreads_or(bad);
    pos = __syncthreads_or(pos);
    if (threadIdx.x == 0) {
        if (bad) atomicOr(&a.sc->vinvalid, 1);
        if (pos) atomicOr(&a.sc->vshift, 1);
    }
}

__device__ __forceinline__ double kappa_of(double kappa0, int half_power, double f) {
    double v = kappa0;
    for (int m = 0; m < half_power / 2; ++m) v = __dmul_rn(v, f);
    if (half_power & 1) v = __dmul_rn(v, __dsqrt_rn(f));
    return v;
}
__device__ __forceinline__ double face_mean(int mode, double a, double b) {
    if (mode == 0) return __dmul_rn(0.5, __dadd_rn(a, b));
    const double sum = __dadd_rn(a, b);
    return sum == 0.0 ? 0.0 : __ddiv_rn(__dmul_rn(__dmul_rn(2.0, a), b), sum);
}

// Face coefficients of the local slab into kr [nloc][nt][nr+1], kt [nloc][nt+1][nr], kp, s.
// f_hi: the plane after the slab (plane 0 on a single rank, the right neighbour's first plane otherwise).
__global__ void __launch_bounds__(kThreads) k_face_coeffs(Dims d, const double *__restrict__ f,
                                                          const double *__restrict__ f_hi,
                                                          const double *__restrict__ rho, double kappa0,
                                                          int half_power, int mean, double inv_dt,
                                                          double *__restrict__ kr, double *__restrict__ kt,
                                                          double *__restrict__ kp, double *__restrict__ s) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        const uint32_t row = (uint32_t)k * d.nt + j;
        const double kc = kappa_of(kappa0, half_power, f[c]);
        // r-faces: lower face i (one-sided at i = 0) and, on the last cell, the outer face nr
        kr[(size_t)row * (d.nr + 1) + i] = (i == 0) ? kc : face_mean(mean, kappa_of(kappa0, half_power, f[c - 1]), kc);
        if (i == d.nr - 1) kr[(size_t)row * (d.nr + 1) + d.nr] = kc;
        // theta-faces: lower face j (one-sided at j = 0) and, on the last row, face nt
        const size_t tb = ((size_t)k * (d.nt + 1) + j) * d.nr + i;
        kt[tb] = (j == 0) ? kc : face_mean(mean, kappa_of(kappa0, half_power, f[c - d.nr]), kc);
        if (j == d.nt - 1) kt[tb + d.nr] = kc;
        // phi-face k+1/2
        const double fn = (k == d.nloc - 1) ? f_hi[c - (size_t)k * d.plane] : f[c + d.plane];
        kp[c] = face_mean(mean, kc, kappa_of(kappa0, half_power, fn));
        s[c] = rho ? __dmul_rn(inv_dt, rho[c]) : inv_dt;
    }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_finalize_D(Dims d, DevArrays a, int bc_in, int bc_out) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        const uint32_t row = (uint32_t)k * d.nt + j;
        const double trlo = (i > 0 || bc_in == BC_DIRICHLET) ? a.Tr[c] : 0.0;
        const double trhi = (i < d.nr - 1) ? a.Tr[c + 1] : (bc_out == BC_DIRICHLET ? a.TrB[row] : 0.0);
        const double ttlo = a.Tt[c];
        const double tthi = (j < d.nt - 1) ? a.Tt[c + d.nr] : 0.0;
        const double tplo = a.Tp[c];
        const double tphi = a.Tp[(size_t)c + d.plane];
        double v = a.sV[c];
        v = __dadd_rn(v, trlo);
        v = __dadd_rn(v, trhi);
        v = __dadd_rn(v, ttlo);
        v = __dadd_rn(v, tthi);
        v = __dadd_rn(v, tplo);
        v = __dadd_rn(v, tphi);
        a.D[c] = v;
    }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_fill_p(Dims d, DevArrays a, const double *__restrict__ x) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        store_p(d, a.p, c, x[c]);
    }
}

// ---------------------------------------------------------------- stencil
// y = A p over a virtual range: c = v + off0 + (v >= split ? off1 : 0).
// WITH_DOT: block partials of p.y -> last block writes sc->red1 (Dot2 pair).
// LOOP: returns at entry once sc->done is set.
// Sum order = the oracle's: r_lo, r_hi, theta_lo, theta_hi, phi_lo, phi_hi, then D p - sum.
template <bool WITH_DOT, bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_matvec_flat(Dims d, DevArrays a, double *__restrict__ y,
                                                                      Range rg, unsigned red_slot0,
                                                                      unsigned red_total) {
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (LOOP && a.peer_wait) acquire_p_halo(a);
    using A = Ar<EXACT>;
    const double *__restrict__ p = a.p;
    const double *__restrict__ Tr = a.Tr;
    const double *__restrict__ Tt = a.Tt;
    const double *__restrict__ Tp = a.Tp;
    const double *__restrict__ D = a.D;
    const size_t plane = d.plane;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rg.vend; v += stride) {
        const uint32_t c = v + rg.off0 + (v >= rg.split ? rg.off1 : 0u);
        int i, j, k;
        decompose(d, c, i, j, k);
        const size_t cp = (size_t)c + plane;
        const double pc = __ldg(p + cp);
        double s = 0.0;
        if (i > 0) s = A::acc(s, __ldg(Tr + c), __ldg(p + cp - 1));
        if (i < d.nr - 1) s = A::acc(s, __ldg(Tr + c + 1), __ldg(p + cp + 1));
        if (j > 0) s = A::acc(s, __ldg(Tt + c), __ldg(p + cp - d.nr));
        if (j < d.nt - 1) s = A::acc(s, __ldg(Tt + c + d.nr), __ldg(p + cp + d.nr));
        s = A::acc(s, __ldg(Tp + c), __ldg(p + cp - plane));
        s = A::acc(s, __ldg(Tp + c + plane), __ldg(p + cp + plane));
        const double q = A::diag_minus(__ldg(D + c), pc, s);
        y[c] = q;
        if (WITH_DOT) dot[0].add(pc, q);
    }
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kThreads, 1>(dot, a.partials, &a.sc->ticket[0], red_slot0 + blockIdx.x, red_total,
                                            out)) {
            if (threadIdx.x == 0) {
                a.sc->red1[0] = out[0].p;
                a.sc->red1[1] = out[0].s;
                if (a.p2p_ll) ll_push_pairs(a, a.sc->red1, 1);   // to every rank (peer communicator)
            }
        }
    }
}

// ---------------------------------------------------------------- setup of a solve
// b = V f + Dirichlet face terms (R5); r0 = b - q (q = A x0); z0 = r0/D; p0 = z0;
// Dot2 partials r.z, r.r, b.b -> sc->red3.
template <bool EXACT>
__global__ void __launch_bounds__(kThreads) k_setup_residual(Dims d, DevArrays a, const double *__restrict__ f,
                                                             int din, int dout, unsigned total) {
    Acc<EXACT> acc[3];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        const uint32_t row = (uint32_t)k * d.nt + j;
        const double V = __dmul_rn(__dmul_rn(a.R3[i], a.C[j]), a.dp[k]);
        double b = __dmul_rn(V, f[c]);
        if (din && i == 0) b = __dadd_rn(b, __dmul_rn(a.Tr[c], a.gin[row]));
        if (dout && i == d.nr - 1) b = __dadd_rn(b, __dmul_rn(a.TrB[row], a.gout[row]));
        const double r = __dsub_rn(b, a.q[c]);
        const double z = __ddiv_rn(r, a.D[c]);
        a.r[c] = r;
        store_p(d, a.p, c, z);
        acc[0].add(r, z);
        acc[1].add(r, r);
        acc[2].add(b, b);
    }
    Acc<EXACT> out[3];
    if (reduce_last<EXACT, kThreads, 3>(acc, a.partials, &a.sc->ticket[3], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            for (int k = 0; k < 3; ++k) {
                a.sc->red3[2 * k] = out[k].p;
                a.sc->red3[2 * k + 1] = out[k].s;
            }
        }
    }
}

// PCG start, after red3 holds the global Dot2 pairs.
__global__ void k_setup_scalars(DevArrays a, double tol, int maxit) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Scalars *sc = a.sc;
    sc->tol = tol;
    sc->maxit = maxit;
    const double rz = __dadd_rn(sc->red3[0], sc->red3[1]);
    const double rr = __dadd_rn(sc->red3[2], sc->red3[3]);
    const double bb = __dadd_rn(sc->red3[4], sc->red3[5]);
    const double bn = sqrt(bb), h0 = sqrt(rr);
    sc->bn = bn;
    sc->tolbn = __dmul_rn(sc->tol, bn);
    sc->iter = 0;
    sc->hist_count = 0;
    sc->rho = rz;
    sc->zero_x = 0;
    sc->done = 1;
    if (!isfinite(bn)) {
        sc->hist0 = bn;
        sc->rn = bn;
        sc->status = ST_E_BREAKDOWN;
    } else if (bn == 0.0) {
        sc->hist0 = 0.0;
        sc->rn = 0.0;
        sc->zero_x = 1;
        sc->status = ST_OK;
    } else {
        sc->hist0 = h0;
        sc->rn = h0;
        if (!isfinite(h0) || !isfinite(rz)) sc->status = ST_E_BREAKDOWN;
        else if (h0 <= sc->tolbn) sc->status = ST_OK;
        else if (sc->maxit == 0) sc->status = ST_NOT_CONVERGED;
        else {
            sc->status = ST_NOT_CONVERGED;
            sc->done = 0;
        }
    }
}

// Value of Dot2 pair t of `npairs`: the local / already combined pair, or -- gather_ranks > 0 -- the
// rank-ordered combination of the all-gathered pairs, exactly as k_dd_combine forms it (so the consumer
// kernel replaces the combine kernel on the critical path of every reduction).
template <bool EXACT>
__device__ __forceinline__ double pair_value(const DevArrays &a, const double *local, int t, int npairs) {
    if (a.p2p_ll) {   // LL words of every rank, polled by the block at once; the first call fetches all pairs
        __shared__ double v_s[2];
        if (t == 0) {
            __syncthreads();
            ll_block_values<EXACT>(a, npairs, v_s);
        }
        return v_s[t];
    }
    if (a.gather_ranks == 0) return __dadd_rn(local[2 * t], local[2 * t + 1]);
    if (EXACT) {
        Acc<true> acc;
        for (int r = 0; r < a.gather_ranks; ++r) {
            Acc<true> o;
            o.p = a.gather[r * 2 * npairs + 2 * t];
            o.s = a.gather[r * 2 * npairs + 2 * t + 1];
            acc.add(o);
        }
        return __dadd_rn(acc.p, acc.s);
    }
    double v = 0.0;
    for (int r = 0; r < a.gather_ranks; ++r) v = __dadd_rn(v, a.gather[r * 2 * npairs + 2 * t]);
    return __dadd_rn(v, 0.0);
}

// ---------------------------------------------------------------- PCG loop (three-kernel path)
// alpha = rho / p.Ap; r -= alpha q; z = r / D; Dot2 partials r.z, r.r.  The x update of this
// iteration (x += alpha p) is deferred to k_pupdate, which reads p anyway (32 instead of 56 B/cell
// here, +16 there).
template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_update(Dims d, DevArrays a, unsigned total) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const double pi = pair_value<EXACT>(a, sc->red1, 0, 1);
    if (!(pi > 0.0) || !isfinite(pi)) {        // breakdown: uniform decision in every block; x = x_{k-1}
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sc->status = ST_E_BREAKDOWN;
            sc->done = 1;
        }
        return;
    }
    const double alpha = __ddiv_rn(sc->rho, pi);
    const double *__restrict__ q = a.q;
    const double *__restrict__ D = a.D;
    double *__restrict__ r = a.r;
    Acc<EXACT> acc[2];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        const double rc = A::ymax(r[c], alpha, __ldg(q + c));
        r[c] = rc;
        const double z = __ddiv_rn(rc, __ldg(D + c));
        acc[0].add(rc, z);
        acc[1].add(rc, rc);
    }
    Acc<EXACT> out[2];
    if (reduce_last<EXACT, kThreads, 2>(acc, a.partials, &sc->ticket[1], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            sc->red2[0] = out[0].p;
            sc->red2[1] = out[0].s;
            sc->red2[2] = out[1].p;
            sc->red2[3] = out[1].s;
            sc->alpha = alpha;
            if (a.p2p_ll) ll_push_pairs(a, sc->red2, 2);
        }
    }
}

// Convergence test on ||r|| (R12); beta = r.z / rho (R11); p = r/D + beta p.
// The last block advances the iteration counter and the scalars.
// x += alpha p (the deferred update of this iteration); then, unless this iteration ends the
// solve, p = r/D + beta p.  The last block advances the iteration counter and the scalars.
template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_pupdate(Dims d, DevArrays a, double *__restrict__ x,
                                                                  int chunk, unsigned total) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const double rz = pair_value<EXACT>(a, sc->red2, 0, 2);
    const double rr = pair_value<EXACT>(a, sc->red2, 1, 2);
    const double rn = sqrt(rr);
    const bool conv = rn <= sc->tolbn;
    const bool bad = !isfinite(rn) || !isfinite(rz);
    const bool last = conv || bad || sc->iter + 1 >= sc->maxit;
    const double alpha = sc->alpha;
    const double beta = last ? 0.0 : __ddiv_rn(rz, sc->rho);
    int peer_st = 0;
    const double *__restrict__ r = a.r;
    const double *__restrict__ D = a.D;
    const uint32_t stride = gridDim.x * blockDim.x;
    if (last) {
        for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride)
            x[c] = A::axpy(alpha, a.p[(size_t)c + d.plane], x[c]);
    } else {
        for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
            const double pold = a.p[(size_t)c + d.plane];
            x[c] = A::axpy(alpha, pold, x[c]);
            const double pn = A::axpy(beta, pold, __ddiv_rn(__ldg(r + c), __ldg(D + c)));
            store_p(d, a.p, c, pn);
            if (a.peer_p_lo) {   // peer mode: the boundary planes straight into the neighbours' halos
                if (c < d.plane) a.peer_p_hi[c] = pn, peer_st = 1;
                if (c >= d.n - d.plane) a.peer_p_lo[c - (d.n - d.plane)] = pn, peer_st = 1;
            }
        }
    }
    __shared__ bool am_last;
    peer_st = __syncthreads_or(peer_st);   // only blocks that stored into a peer pay the system-scope fence
    if (threadIdx.x == 0) {
        if (peer_st) fence_acq_rel_sys();
        am_last = atom_add_acq_rel_gpu(&sc->ticket[2], 1u) == total - 1;
    }
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
        if (a.peer_p_lo && !last) release_p_halo(a);
        const int it = sc->iter + 1;
        sc->iter = it;
        sc->rn = rn;
        sc->hist_ring[(it - 1) % chunk] = rn;
        if (a.hist_dev_on) a.hist_dev[it - 1] = rn;   // the device loop's full history
        if (conv) {
            sc->status = ST_OK;
            sc->done = 1;
        } else if (bad) {
            sc->status = ST_E_BREAKDOWN;
            sc->done = 1;
        } else if (it >= sc->maxit) {
            sc->status = ST_NOT_CONVERGED;
            sc->done = 1;
        }
        sc->rho = rz;
        sc->ticket[2] = 0u;
    }
}


// ---------------------------------------------------------------- 16-byte vector variants (nr even)
// Two r-neighbour cells (i, i+1), i even, per thread: every stream is one 16-byte load or store
// (LDG.E.128), halving the load/store instructions of the memory-bound kernels.  Same per-cell
// arithmetic in the same order as the scalar kernels; used when nr is even and x is 16-B aligned.
__device__ __forceinline__ void st2(double *p, double a, double b) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}

// HINT: the loads and stores carry the L2 residency policies of Dims::l2_mask and the peer-written halo
// planes are read coherently (loop stencil with an L2 plan or the peer communicator); without it the plain
// __ldg path (the policy registers and the per-load selection cost ~9 % on the P = 1 stencil).
template <bool WITH_DOT, bool LOOP, bool EXACT, bool MV2, bool HINT>
__global__ void __launch_bounds__(kThreads, kMvBlocks) k_matvec_vec2(Dims d, DevArrays a, double *__restrict__ y,
                                                                      Range rg, unsigned red_slot0,
                                                                      unsigned red_total) {
    pdl_wait();
    pdl_trigger();
    // peer mode: done is checked before the halo acquire (a finished solve releases no halo)
    const bool pw = LOOP && a.peer_wait;
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (pw) acquire_p_halo(a);
    using A = Ar<EXACT>;
    const double *__restrict__ p = a.p;
    const double *__restrict__ Tr = a.Tr;
    const double *__restrict__ Tt = a.Tt;
    const double *__restrict__ Tp = a.Tp;
    const double *__restrict__ D = a.D;
    const size_t plane = d.plane;
    const int nr = d.nr, nt = d.nt;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = rg.vend >> 1;
    // the loads of one pair (all issued before its first use), then its arithmetic
    struct PairIn {
        double2 pc, trv, ttl, tpl, tph, pkm, pkp, dv, ptm, ptp, tth;
        double pm, pp2, tr2;
        uint32_t c;
        bool jlo, jhi, ilo, ihi;
    };
    uint64_t pol_p = 0, pol_t = 0, pol_d = 0, pol_q = 0;
    if (HINT) {
        pol_p = l2_policy(d, L2A_P), pol_t = l2_policy(d, L2A_T), pol_d = l2_policy(d, L2A_D);
        pol_q = l2_policy(d, L2A_Q);
    }
    // peer mode: the halo planes k = -1 and k = nloc were stored by the neighbours during this kernel's
    // lifetime (acquired above), so they are read coherently
    const bool coh = HINT && LOOP && a.peer_wait;
    auto load = [&](uint32_t v) {
        PairIn q;
        const uint32_t v2 = 2u * v;
        q.c = v2 + rg.off0 + (v2 >= rg.split ? rg.off1 : 0u);
        int i, j, k;
        decompose(d, q.c, i, j, k);
        const size_t cp = (size_t)q.c + plane;
        if (!HINT) {   // plain read-only loads
            q.pc = __ldg(reinterpret_cast<const double2 *>(p + cp));
            q.trv = __ldg(reinterpret_cast<const double2 *>(Tr + q.c));
            q.ttl = __ldg(reinterpret_cast<const double2 *>(Tt + q.c));
            q.tpl = __ldg(reinterpret_cast<const double2 *>(Tp + q.c));
            q.tph = __ldg(reinterpret_cast<const double2 *>(Tp + q.c + plane));
            q.pkm = __ldg(reinterpret_cast<const double2 *>(p + cp - plane));
            q.pkp = __ldg(reinterpret_cast<const double2 *>(p + cp + plane));
            q.dv = __ldg(reinterpret_cast<const double2 *>(D + q.c));
            q.jlo = j > 0, q.jhi = j < nt - 1, q.ilo = i > 0, q.ihi = i + 2 < nr;
            q.ptm = make_double2(0.0, 0.0), q.ptp = q.ptm, q.tth = q.ptm;
            if (q.jlo) q.ptm = __ldg(reinterpret_cast<const double2 *>(p + cp - nr));
            if (q.jhi) {
                q.ptp = __ldg(reinterpret_cast<const double2 *>(p + cp + nr));
                q.tth = __ldg(reinterpret_cast<const double2 *>(Tt + q.c + nr));
            }
            q.pm = q.ilo ? __ldg(p + cp - 1) : 0.0;
            q.pp2 = q.ihi ? __ldg(p + cp + 2) : 0.0;
            q.tr2 = q.ihi ? __ldg(Tr + q.c + 2) : 0.0;
            return q;
        }
        q.pc = ld2h(p + cp, pol_p);
        q.trv = ld2h(Tr + q.c, pol_t);
        q.ttl = ld2h(Tt + q.c, pol_t);
        q.tpl = ld2h(Tp + q.c, pol_t);
        q.tph = ld2h(Tp + q.c + plane, pol_t);
        q.pkm = (coh && k == 0) ? ld2coh(p + cp - plane) : ld2h(p + cp - plane, pol_p);
        q.pkp = (coh && k == d.nloc - 1) ? ld2coh(p + cp + plane) : ld2h(p + cp + plane, pol_p);
        q.dv = ld2h(D + q.c, pol_d);
        q.jlo = j > 0, q.jhi = j < nt - 1, q.ilo = i > 0, q.ihi = i + 2 < nr;
        q.ptm = make_double2(0.0, 0.0), q.ptp = q.ptm, q.tth = q.ptm;
        if (q.jlo) q.ptm = ld2h(p + cp - nr, pol_p);
        if (q.jhi) {
            q.ptp = ld2h(p + cp + nr, pol_p);
            q.tth = ld2h(Tt + q.c + nr, pol_t);
        }
        q.pm = q.ilo ? ld1h(p + cp - 1, pol_p) : 0.0;
        q.pp2 = q.ihi ? ld1h(p + cp + 2, pol_p) : 0.0;
        q.tr2 = q.ihi ? ld1h(Tr + q.c + 2, pol_t) : 0.0;
        return q;
    };
    auto compute = [&](const PairIn &q) {
        // cell i
        double s = 0.0;
        if (q.ilo) s = A::acc(s, q.trv.x, q.pm);
        s = A::acc(s, q.trv.y, q.pc.y);
        if (q.jlo) s = A::acc(s, q.ttl.x, q.ptm.x);
        if (q.jhi) s = A::acc(s, q.tth.x, q.ptp.x);
        s = A::acc(s, q.tpl.x, q.pkm.x);
        s = A::acc(s, q.tph.x, q.pkp.x);
        const double q0 = A::diag_minus(q.dv.x, q.pc.x, s);
        // cell i+1
        s = 0.0;
        s = A::acc(s, q.trv.y, q.pc.x);
        if (q.ihi) s = A::acc(s, q.tr2, q.pp2);
        if (q.jlo) s = A::acc(s, q.ttl.y, q.ptm.y);
        if (q.jhi) s = A::acc(s, q.tth.y, q.ptp.y);
        s = A::acc(s, q.tpl.y, q.pkm.y);
        s = A::acc(s, q.tph.y, q.pkp.y);
        const double q1 = A::diag_minus(q.dv.y, q.pc.y, s);
        if (HINT) st2h(y + q.c, q0, q1, pol_q);
        else st2(y + q.c, q0, q1);
        if (WITH_DOT) {
            dot[0].add(q.pc.x, q0);
            dot[0].add(q.pc.y, q1);
        }
    };
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (MV2) {   // two pairs per trip: the second pair's loads are in flight during the first's arithmetic
        for (; v + stride < npair; v += 2 * stride) {
            const PairIn a0 = load(v), a1 = load(v + stride);
            compute(a0);
            compute(a1);
        }
    }
    for (; v < npair; v += stride) compute(load(v));
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kThreads, 1>(dot, a.partials, &a.sc->ticket[0], red_slot0 + blockIdx.x, red_total,
                                            out)) {
            if (threadIdx.x == 0) {
                a.sc->red1[0] = out[0].p;
                a.sc->red1[1] = out[0].s;
                if (a.p2p_ll) ll_push_pairs(a, a.sc->red1, 1);   // to every rank (peer communicator)
            }
        }
    }
}

template <bool EXACT, bool UP2>
__global__ void __launch_bounds__(kThreads, kVecBlocks) k_update_vec2(Dims d, DevArrays a, unsigned total, int rev) {
    pdl_wait();
    pdl_trigger();
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    double *__restrict__ r = a.r;
    const uint64_t pol_r = l2_policy(d, L2A_R), pol_q = l2_policy(d, L2A_Q), pol_d = l2_policy(d, L2A_D);
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = d.n >> 1;
    uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    auto cell = [&](uint32_t ww) { return 2u * (rev ? npair - 1 - ww : ww); };
    // The first trip's loads are issued BEFORE the scalars (done, p.q, rho): they do not depend on them,
    // so their latency overlaps the scalar reads at kernel entry instead of following them.
    const double2 z2 = make_double2(0.0, 0.0);
    const bool two = UP2 && w + stride < npair, one = w < npair;
    const uint32_t f0 = cell(one ? w : 0u), f1 = cell(two ? w + stride : 0u);
    double2 rv0 = z2, qv0 = z2, dv0 = z2, rv1 = z2, qv1 = z2, dv1 = z2;
    if (one) rv0 = ld2rwh(r + f0, pol_r), qv0 = ld2h(a.q + f0, pol_q), dv0 = ld2h(a.D + f0, pol_d);
    if (two) rv1 = ld2rwh(r + f1, pol_r), qv1 = ld2h(a.q + f1, pol_q), dv1 = ld2h(a.D + f1, pol_d);
    if (*(volatile int *)&sc->done) return;
    const double pi = pair_value<EXACT>(a, sc->red1, 0, 1);
    if (!(pi > 0.0) || !isfinite(pi)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            sc->status = ST_E_BREAKDOWN;
            sc->done = 1;
        }
        return;
    }
    const double alpha = __ddiv_rn(sc->rho, pi);
    Acc<EXACT> acc[2];
    auto body = [&](uint32_t c, double2 rv, double2 qv, double2 dv) {
        const double r0 = A::ymax(rv.x, alpha, qv.x), r1 = A::ymax(rv.y, alpha, qv.y);
        st2h(r + c, r0, r1, pol_r);
        const double z0 = __ddiv_rn(r0, dv.x), z1 = __ddiv_rn(r1, dv.y);
        acc[0].add(r0, z0);
        acc[0].add(r1, z1);
        acc[1].add(r0, r0);
        acc[1].add(r1, r1);
    };
    // the same per-thread order of the sums as a plain grid-stride loop (two pairs per trip, then one)
    if (two) {
        body(f0, rv0, qv0, dv0);
        body(f1, rv1, qv1, dv1);
        w += 2 * stride;
        if (UP2) {
            for (; w + stride < npair; w += 2 * stride) {
                const uint32_t c0 = cell(w), c1 = cell(w + stride);
                const double2 ra = ld2rwh(r + c0, pol_r), qa = ld2h(a.q + c0, pol_q), da = ld2h(a.D + c0, pol_d);
                const double2 rb = ld2rwh(r + c1, pol_r), qb = ld2h(a.q + c1, pol_q), db = ld2h(a.D + c1, pol_d);
                body(c0, ra, qa, da);
                body(c1, rb, qb, db);
            }
        }
    } else if (one) {
        body(f0, rv0, qv0, dv0);
        w += stride;
    }
    for (; w < npair; w += stride) {
        const uint32_t c = cell(w);
        body(c, ld2rwh(r + c, pol_r), ld2h(a.q + c, pol_q), ld2h(a.D + c, pol_d));
    }
    Acc<EXACT> out[2];
    if (reduce_last<EXACT, kThreads, 2>(acc, a.partials, &sc->ticket[1], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            sc->red2[0] = out[0].p;
            sc->red2[1] = out[0].s;
            sc->red2[2] = out[1].p;
            sc->red2[3] = out[1].s;
            sc->alpha = alpha;
            if (a.p2p_ll) ll_push_pairs(a, sc->red2, 2);
        }
    }
}

template <bool EXACT, bool PU2>
__global__ void __launch_bounds__(kThreads, kVecBlocks) k_pupdate_vec2(Dims d, DevArrays a, double *__restrict__ x, int chunk,
                                                           unsigned total) {
    pdl_wait();
    pdl_trigger();
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = d.n >> 1;
    double *__restrict__ p = a.p;
    const uint64_t pol_p = l2_policy(d, L2A_P), pol_x = l2_policy(d, L2A_X), pol_r = l2_policy(d, L2A_R);
    const uint64_t pol_d = l2_policy(d, L2A_D);
    // the first pair's four loads before the scalars (see k_update_vec2); r and D are read even in the
    // last iteration, where p is not updated (harmless)
    const double2 z2 = make_double2(0.0, 0.0);
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const bool pre = !PU2 && v < npair;
    double2 po_f = z2, xv_f = z2, rv_f = z2, dv_f = z2;
    if (pre) {
        const uint32_t c = 2u * v;
        po_f = ld2rwh(p + (size_t)c + d.plane, pol_p), xv_f = ld2rwh(x + c, pol_x);
        rv_f = ld2h(a.r + c, pol_r), dv_f = ld2h(a.D + c, pol_d);
    }
    if (*(volatile int *)&sc->done) return;
    const double rz = pair_value<EXACT>(a, sc->red2, 0, 2);
    const double rr = pair_value<EXACT>(a, sc->red2, 1, 2);
    const double rn = sqrt(rr);
    const bool conv = rn <= sc->tolbn;
    const bool bad = !isfinite(rn) || !isfinite(rz);
    const bool last = conv || bad || sc->iter + 1 >= sc->maxit;
    const double alpha = sc->alpha;
    const double beta = last ? 0.0 : __ddiv_rn(rz, sc->rho);
    int peer_st = 0;
    auto store = [&](uint32_t c, double2 po, double2 xv, double2 rv, double2 dv) {
        st2h(x + c, A::axpy(alpha, po.x, xv.x), A::axpy(alpha, po.y, xv.y), pol_x);
        if (!last) {
            const double p0 = A::axpy(beta, po.x, __ddiv_rn(rv.x, dv.x));
            const double p1 = A::axpy(beta, po.y, __ddiv_rn(rv.y, dv.y));
            st2h(p + (size_t)c + d.plane, p0, p1, pol_p);
            if (d.periodic_local) {
                if (c < d.plane) st2h(p + (size_t)c + (size_t)(d.nloc + 1) * d.plane, p0, p1, pol_p);
                if (c >= d.n - d.plane) st2h(p + (size_t)c - (size_t)(d.nloc - 1) * d.plane, p0, p1, pol_p);
            } else if (a.peer_p_lo) {   // peer mode: the boundary planes straight into the neighbours' halos
                if (c < d.plane) st2(a.peer_p_hi + c, p0, p1), peer_st = 1;
                if (c >= d.n - d.plane) st2(a.peer_p_lo + (c - (d.n - d.plane)), p0, p1), peer_st = 1;
            }
        }
    };
    if (pre) {
        store(2u * v, po_f, xv_f, rv_f, dv_f);
        v += stride;
    }
    if (PU2) {
        // two pairs per thread and trip: all eight 16-byte loads issued before the first store
        for (; v + stride < npair; v += 2 * stride) {
            const uint32_t c0 = 2u * v, c1 = 2u * (v + stride);
            const double2 po0 = ld2rwh(p + (size_t)c0 + d.plane, pol_p), xv0 = ld2rwh(x + c0, pol_x);
            const double2 po1 = ld2rwh(p + (size_t)c1 + d.plane, pol_p), xv1 = ld2rwh(x + c1, pol_x);
            const double2 rv0 = last ? z2 : ld2h(a.r + c0, pol_r), dv0 = last ? z2 : ld2h(a.D + c0, pol_d);
            const double2 rv1 = last ? z2 : ld2h(a.r + c1, pol_r), dv1 = last ? z2 : ld2h(a.D + c1, pol_d);
            store(c0, po0, xv0, rv0, dv0);
            store(c1, po1, xv1, rv1, dv1);
        }
    }
    for (; v < npair; v += stride) {
        const uint32_t c = 2u * v;
        const double2 po = ld2rwh(p + (size_t)c + d.plane, pol_p), xv = ld2rwh(x + c, pol_x);
        const double2 rv = last ? z2 : ld2h(a.r + c, pol_r), dv = last ? z2 : ld2h(a.D + c, pol_d);
        store(c, po, xv, rv, dv);
    }
    __shared__ bool am_last;
    peer_st = __syncthreads_or(peer_st);   // only blocks that stored into a peer pay the system-scope fence
    if (threadIdx.x == 0) {
        if (peer_st) fence_acq_rel_sys();
        am_last = atom_add_acq_rel_gpu(&sc->ticket[2], 1u) == total - 1;
    }
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
        if (a.peer_p_lo && !last) release_p_halo(a);
        const int it = sc->iter + 1;
        sc->iter = it;
        sc->rn = rn;
        sc->hist_ring[(it - 1) % chunk] = rn;
        if (a.hist_dev_on) a.hist_dev[it - 1] = rn;   // the device loop's full history
        if (conv) {
            sc->status = ST_OK;
            sc->done = 1;
        } else if (bad) {
            sc->status = ST_E_BREAKDOWN;
            sc->done = 1;
        } else if (it >= sc->maxit) {
            sc->status = ST_NOT_CONVERGED;
            sc->done = 1;
        }
        sc->rho = rz;
        sc->ticket[2] = 0u;
    }
}

// ---------------------------------------------------------------- super-time-stepping (NEXT-4, R26)
// L(u) = (b_D - K u) / V with K u = (A u) - (s V) u, A u summed exactly like the stencil kernels.
template <bool EXACT>
__device__ __forceinline__ double sts_L(const Dims &d, const DevArrays &a, const double *__restrict__ u, uint32_t c,
                                        int din, int dout) {
    using A = Ar<EXACT>;
    int i, j, k;
    decompose(d, c, i, j, k);
    const size_t plane = d.plane, cp = (size_t)c + plane;
    const double pc = u[cp];
    double s = 0.0;
    if (i > 0) s = A::acc(s, a.Tr[c], u[cp - 1]);
    if (i < d.nr - 1) s = A::acc(s, a.Tr[c + 1], u[cp + 1]);
    if (j > 0) s = A::acc(s, a.Tt[c], u[cp - d.nr]);
    if (j < d.nt - 1) s = A::acc(s, a.Tt[c + d.nr], u[cp + d.nr]);
    s = A::acc(s, a.Tp[c], u[cp - plane]);
    s = A::acc(s, a.Tp[c + plane], u[cp + plane]);
    const double y = A::diag_minus(a.D[c], pc, s);
    const double Ku = __dsub_rn(y, __dmul_rn(a.sV[c], pc));
    const uint32_t row = (uint32_t)k * d.nt + j;
    double b = 0.0;
    if (din && i == 0) b = __dadd_rn(b, __dmul_rn(a.Tr[c], a.gin[row]));
    if (dout && i == d.nr - 1) b = __dadd_rn(b, __dmul_rn(a.TrB[row], a.gout[row]));
    const double V = __dmul_rn(__dmul_rn(a.R3[i], a.C[j]), a.dp[k]);
    return __ddiv_rn(__dsub_rn(b, Ku), V);
}

// stage 1: L0 = L(Y0); Y1 = Y0 + (mu~_1 tau) L0 (into a padded buffer, periodic copies on one rank)
template <bool EXACT>
__global__ void __launch_bounds__(kThreads) k_sts_first(Dims d, DevArrays a, const double *__restrict__ y0p,
                                                        double *__restrict__ l0, double *__restrict__ y1p,
                                                        double m1, int din, int dout) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        const double L = sts_L<EXACT>(d, a, y0p, c, din, dout);
        l0[c] = L;
        store_p(d, y1p, c, __dadd_rn(y0p[(size_t)c + d.plane], __dmul_rn(m1, L)));
    }
}

// stage j >= 2: Yj = mu Y_{j-1} + nu Y_{j-2} + w0 Y0 + mt L(Y_{j-1}) + gt L0, added left to right
template <bool EXACT>
__global__ void __launch_bounds__(kThreads) k_sts_stage(Dims d, DevArrays a, const double *__restrict__ yj1p,
                                                        const double *__restrict__ yj2p,
                                                        const double *__restrict__ y0p,
                                                        const double *__restrict__ l0, double *__restrict__ yjp,
                                                        double mu, double nu, double w0, double mt, double gt,
                                                        int din, int dout) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const size_t plane = d.plane;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        const double L = sts_L<EXACT>(d, a, yj1p, c, din, dout);
        double t = __dmul_rn(mu, yj1p[(size_t)c + plane]);
        t = __dadd_rn(t, __dmul_rn(nu, yj2p[(size_t)c + plane]));
        t = __dadd_rn(t, __dmul_rn(w0, y0p[(size_t)c + plane]));
        t = __dadd_rn(t, __dmul_rn(mt, L));
        t = __dadd_rn(t, __dmul_rn(gt, l0[c]));
        store_p(d, yjp, c, t);
    }
}

// Gershgorin bound of lambda_max(V^-1 K): max_c (K_cc + sum_f T_f) / V_c, block maxima -> out[block]
__global__ void __launch_bounds__(kThreads) k_sts_gershgorin(Dims d, DevArrays a, double *out) {
    double m = 0.0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        double off = 0.0;
        if (i > 0) off += a.Tr[c];
        if (i < d.nr - 1) off += a.Tr[c + 1];
        if (j > 0) off += a.Tt[c];
        if (j < d.nt - 1) off += a.Tt[c + d.nr];
        off += a.Tp[c] + a.Tp[(size_t)c + d.plane];
        const double kdiag = a.D[c] - a.sV[c];
        const double V = __dmul_rn(__dmul_rn(a.R3[i], a.C[j]), a.dp[k]);
        m = fmax(m, (kdiag + off) / V);
    }
    __shared__ double sm[kThreads / 32];
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) v = fmax(v, sm[w]);
        out[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_zero_x_if(Dims d, DevArrays a, double *__restrict__ x) {
    if (!a.sc->zero_x) return;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) x[c] = 0.0;
}

// 16-byte vector kernels: nr even (pairs never straddle a row; every plane offset even) and the
// caller's array 16-byte aligned (workspace arrays are 256-byte aligned).
inline bool use_vec2(const Dims &d, const void *x) {
    return d.vec_ok && (d.nr % 2 == 0) && (((uintptr_t)x & 15) == 0);
}

template <typename... KArgs, typename... Args>
void launch_pdl(bool pdl, void (*kern)(KArgs...), unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline unsigned grid_mv2(uint32_t n) {    // the vector stencil: n cells, two per thread
    uint64_t g = (n / 2 + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * kMvBlocks)) g = 148 * kMvBlocks;
    return (unsigned)g;
}

inline unsigned grid_vec2(uint32_t n) {   // n cells, two per thread
    uint64_t g = (n / 2 + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * kVecBlocks)) g = 148 * kVecBlocks;
    return (unsigned)g;
}

inline unsigned grid_for(uint32_t n) {
    uint64_t g = (n + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)kRedBlocks) g = kRedBlocks;
    return (unsigned)g;
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_assemble(const Dims &d, const DevArrays &a, const double *kr, const double *kt, const double *kp,
                     const double *s, cudaStream_t st) {
    const bool al = ((((uintptr_t)kt | (uintptr_t)kp | (uintptr_t)s) & 15) == 0);
    if (d.vec_ok && (d.nr % 2 == 0) && al) k_assemble_vec2<<<grid_for(d.n / 2), kThreads, 0, st>>>(d, a, kr, kt, kp, s);
    else k_assemble<<<grid_for(d.n), kThreads, 0, st>>>(d, a, kr, kt, kp, s);
}

void launch_face_coeffs(const Dims &d, const double *f, const double *f_hi, const double *rho, double kappa0,
                        int half_power, int mean, double inv_dt, double *kr, double *kt, double *kp, double *s,
                        cudaStream_t st) {
    k_face_coeffs<<<grid_for(d.n), kThreads, 0, st>>>(d, f, f_hi, rho, kappa0, half_power, mean, inv_dt, kr, kt,
                                                      kp, s);
}

void launch_finalize_D(const Dims &d, const DevArrays &a, int bc_in, int bc_out, cudaStream_t st) {
    k_finalize_D<<<grid_for(d.n), kThreads, 0, st>>>(d, a, bc_in, bc_out);
}

void launch_fill_p(const Dims &d, const DevArrays &a, const double *x, cudaStream_t st) {
    k_fill_p<<<grid_for(d.n), kThreads, 0, st>>>(d, a, x);
}

Range make_range(const Dims &d, StencilPart part) {
    Range rg{};
    const uint32_t pl = d.plane;
    switch (part) {
        case StencilPart::Full: rg = {d.n, 0u, 0xffffffffu, 0u}; break;
        case StencilPart::Interior:
            rg = {d.nloc > 2 ? (uint32_t)(d.nloc - 2) * pl : 0u, pl, 0xffffffffu, 0u};
            break;
        case StencilPart::Boundary:
            if (d.nloc == 1) rg = {pl, 0u, 0xffffffffu, 0u};
            else rg = {2u * pl, 0u, pl, (uint32_t)(d.nloc - 2) * pl};
            break;
    }
    return rg;
}

unsigned stencil_blocks(const Dims &d, StencilPart part, const double *y) {
    Range rg = make_range(d, part);
    if (!rg.vend) return 0u;
    return use_vec2(d, y) ? grid_mv2(rg.vend) : grid_for(rg.vend);
}

void launch_matvec(const Dims &d, const DevArrays &a, double *y, StencilPart part, bool with_dot, bool loop,
                   unsigned red_slot0, unsigned red_total, bool exact, cudaStream_t st) {
    Range rg = make_range(d, part);
    if (rg.vend == 0) return;
    const bool vec = use_vec2(d, y);
    const unsigned g = vec ? grid_mv2(rg.vend) : grid_for(rg.vend);
    // MASPCG_MATVEC2=1: two pairs per trip -- measured slower (5.98 vs 6.07 TB/s live: 64 registers, spills)
    static const int mv2 = getenv("MASPCG_MATVEC2") ? atoi(getenv("MASPCG_MATVEC2")) : 0;
    // the policy / coherent-halo variant only where it is needed (an L2 plan or peer-written halos)
    const bool hint = loop && (d.l2_mask != 0u || a.peer_wait != 0);
#define MV(W, L, E)                                                                             \
    do {                                                                                        \
        if (vec && mv2) launch_pdl(d.pdl != 0, k_matvec_vec2<W, L, E, true, false>, g, st, d, a, y, rg, red_slot0, red_total); \
        else if (vec && L && hint) launch_pdl(d.pdl != 0, k_matvec_vec2<W, L, E, false, true>, g, st, d, a, y, rg, red_slot0, red_total); \
        else if (vec) launch_pdl(d.pdl != 0, k_matvec_vec2<W, L, E, false, false>, g, st, d, a, y, rg, red_slot0, red_total); \
        else k_matvec_flat<W, L, E><<<g, kThreads, 0, st>>>(d, a, y, rg, red_slot0, red_total);     \
    } while (0)
    if (exact) {
        if (with_dot) {
            if (loop) MV(true, true, true);
            else MV(true, false, true);
        } else MV(false, false, true);
    } else {
        if (with_dot) {
            if (loop) MV(true, true, false);
            else MV(true, false, false);
        } else MV(false, false, false);
    }
#undef MV
}

void launch_setup_residual(const Dims &d, const DevArrays &a, const double *f, int din, int dout, bool exact,
                           cudaStream_t st) {
    const unsigned g = grid_for(d.n);
    if (exact) k_setup_residual<true><<<g, kThreads, 0, st>>>(d, a, f, din, dout, g);
    else k_setup_residual<false><<<g, kThreads, 0, st>>>(d, a, f, din, dout, g);
}

void launch_setup_scalars(const DevArrays &a, double tol, int maxit, cudaStream_t st) {
    k_setup_scalars<<<1, 32, 0, st>>>(a, tol, maxit);
}

void launch_update(const Dims &d, const DevArrays &a, bool exact, cudaStream_t st) {
    if (use_vec2(d, nullptr)) {
        const unsigned gv = grid_vec2(d.n);
        // descending traversal: it starts on the cells whose q and D the stencil touched last (still in L2)
        // and ends on the cells the ascending p-update reads first; +0.4 % iterations/s on c3.
        // MASPCG_REV_UPDATE=0 restores the ascending order.
        static const int rev = getenv("MASPCG_REV_UPDATE") ? atoi(getenv("MASPCG_REV_UPDATE")) : 1;
        // two pairs per thread and trip (6 loads in flight before the first use): 6.38 vs 5.96 TB/s live
        static const int up2 = getenv("MASPCG_UPDATE2") ? atoi(getenv("MASPCG_UPDATE2")) : 1;
        if (up2) {
            if (exact) launch_pdl(d.pdl != 0, k_update_vec2<true, true>, gv, st, d, a, gv, rev);
            else launch_pdl(d.pdl != 0, k_update_vec2<false, true>, gv, st, d, a, gv, rev);
        } else {
            if (exact) launch_pdl(d.pdl != 0, k_update_vec2<true, false>, gv, st, d, a, gv, rev);
            else launch_pdl(d.pdl != 0, k_update_vec2<false, false>, gv, st, d, a, gv, rev);
        }
        return;
    }
    const unsigned g = grid_for(d.n);
    if (exact) k_update<true><<<g, kThreads, 0, st>>>(d, a, g);
    else k_update<false><<<g, kThreads, 0, st>>>(d, a, g);
}

void launch_pupdate(const Dims &d, const DevArrays &a, double *x, int chunk, bool exact, cudaStream_t st) {
    if (use_vec2(d, x)) {
        const unsigned gv = grid_vec2(d.n);
        // one pair per trip with its four loads ahead of the x store (6.46 TB/s live; two pairs: 6.32)
        static const int pu2 = getenv("MASPCG_PUPDATE2") ? atoi(getenv("MASPCG_PUPDATE2")) : 0;
        if (pu2) {
            if (exact) launch_pdl(d.pdl != 0, k_pupdate_vec2<true, true>, gv, st, d, a, x, chunk, gv);
            else launch_pdl(d.pdl != 0, k_pupdate_vec2<false, true>, gv, st, d, a, x, chunk, gv);
        } else {
            if (exact) launch_pdl(d.pdl != 0, k_pupdate_vec2<true, false>, gv, st, d, a, x, chunk, gv);
            else launch_pdl(d.pdl != 0, k_pupdate_vec2<false, false>, gv, st, d, a, x, chunk, gv);
        }
        return;
    }
    const unsigned g = grid_for(d.n);
    if (exact) k_pupdate<true><<<g, kThreads, 0, st>>>(d, a, x, chunk, g);
    else k_pupdate<false><<<g, kThreads, 0, st>>>(d, a, x, chunk, g);
}

__global__ void k_dd_combine(const double *gather, int nranks, int npairs, double *out, bool exact) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < npairs; t += gridDim.x * blockDim.x) {
    if (exact) {
        Acc<true> acc;
        for (int r = 0; r < nranks; ++r) {   // rank order: identical bits on every rank
            Acc<true> o;
            o.p = gather[r * 2 * npairs + 2 * t];
            o.s = gather[r * 2 * npairs + 2 * t + 1];
            acc.add(o);
        }
        out[2 * t] = acc.p;
        out[2 * t + 1] = acc.s;
    } else {
        double v = 0.0;
        for (int r = 0; r < nranks; ++r) v = __dadd_rn(v, gather[r * 2 * npairs + 2 * t]);
        out[2 * t] = v;
        out[2 * t + 1] = 0.0;
    }
    }
}

void launch_dd_combine(const double *gather, int nranks, int npairs, double *out, bool exact, cudaStream_t st) {
    k_dd_combine<<<(npairs + 127) / 128, 128, 0, st>>>(gather, nranks, npairs, out, exact);
}

void launch_sts_first(const Dims &d, const DevArrays &a, const double *y0p, double *l0, double *y1p, double m1,
                      int din, int dout, bool exact, cudaStream_t st) {
    const unsigned g = grid_for(d.n);
    if (exact) k_sts_first<true><<<g, kThreads, 0, st>>>(d, a, y0p, l0, y1p, m1, din, dout);
    else k_sts_first<false><<<g, kThreads, 0, st>>>(d, a, y0p, l0, y1p, m1, din, dout);
}

void launch_sts_stage(const Dims &d, const DevArrays &a, const double *yj1p, const double *yj2p, const double *y0p,
                      const double *l0, double *yjp, double mu, double nu, double w0, double mt, double gt, int din,
                      int dout, bool exact, cudaStream_t st) {
    const unsigned g = grid_for(d.n);
    if (exact) k_sts_stage<true><<<g, kThreads, 0, st>>>(d, a, yj1p, yj2p, y0p, l0, yjp, mu, nu, w0, mt, gt, din, dout);
    else k_sts_stage<false><<<g, kThreads, 0, st>>>(d, a, yj1p, yj2p, y0p, l0, yjp, mu, nu, w0, mt, gt, din, dout);
}

unsigned launch_sts_gershgorin(const Dims &d, const DevArrays &a, double *out, cudaStream_t st) {
    const unsigned g = grid_for(d.n);
    k_sts_gershgorin<<<g, kThreads, 0, st>>>(d, a, out);
    return g;
}

// The device loop (conditional WHILE node of a CUDA graph): run the body (a chunk of iterations) again
// while the solve is not done.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const Scalars *sc) {
    cudaGraphSetConditional(h, (*(volatile const int *)&sc->done) ? 0u : 1u);
}

void launch_loop_cond(cudaGraphConditionalHandle h, const Scalars *sc, cudaStream_t st) {
    k_loop_cond<<<1, 1, 0, st>>>(h, sc);
}

// Return the lines of [p, p + bytes) to the normal eviction priority (after a solve that kept them).
__global__ void __launch_bounds__(kThreads) k_l2_demote(uintptr_t base, size_t lines) {
    for (size_t l = blockIdx.x * (size_t)blockDim.x + threadIdx.x; l < lines; l += (size_t)gridDim.x * blockDim.x)
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(base + 128 * l) : "memory");
}

void launch_l2_demote(const void *p, size_t bytes, cudaStream_t st) {
    if (!p || !bytes) return;
    const uintptr_t b = (uintptr_t)p & ~(uintptr_t)127;
    const size_t lines = ((uintptr_t)p + bytes - b + 127) / 128;
    size_t g = (lines + kThreads - 1) / kThreads;
    if (g > 4 * 148) g = 4 * 148;
    k_l2_demote<<<(unsigned)g, kThreads, 0, st>>>(b, lines);
}

void launch_zero_x_if(const Dims &d, const DevArrays &a, double *x, cudaStream_t st) {
    k_zero_x_if<<<grid_for(d.n), kThreads, 0, st>>>(d, a, x);
}

}  // namespace maspcg
