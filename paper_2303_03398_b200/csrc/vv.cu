// vv.cu -- sm_100a fp64 kernels of the staggered vector viscosity operator (
// readings R27-R31 of DESIGN.md; see vv.cuh for the layout).
//
// Every operator quantity -- face areas and distances, outflows delta, circulations Gamma, the rows
// -- is evaluated with one IEEE rounding per operation (__dmul_rn / __dadd_rn / __dsub_rn /
// __ddiv_rn) in the order of the oracle's formulas (the vector-viscosity oracle), so the operator and its
// rows are bit-identical to the oracle's; the ring sums (the polar axes) and the PCG dot products
// are Dot2 (R24).  The matvec is HBM-bound like the scalar stencil: per cell it streams p (3 values,
// with +-1-plane neighbours through L1/L2), wc, Wr, Wt, Wp, sM (3) and writes q (3): 104 B/cell,
// i.e. ~35 B per unknown, and recomputes the outflows and circulations it needs from p in
// registers instead of storing them (which would cost 64 B/cell more).
#include <cuda_runtime.h>

#include <cstdlib>

#include "arith.cuh"
#include "common.cuh"
#include "vv.cuh"

namespace maspcg {

namespace {

constexpr int kVVThreads = 256;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void cell_of(const VVDims &v, uint32_t c, int &i, int &j, int &k) {
    const uint32_t row = v.div_r.div(c);
    i = (int)(c - row * (uint32_t)v.nr);
    const uint32_t kk = v.div_t.div(row);
    j = (int)(row - kk * (uint32_t)v.nt);
    k = (int)kk;
}

// padded vector slot (plane k in [-1, nloc]), padded cell slot, unpadded vector slot, padded wall slot
__device__ __forceinline__ size_t PV(const VVDims &v, int k, int c, int j, int i) {
    return ((size_t)(k + 1) * 3 + c) * v.plane1 + (size_t)j * v.nr + i;
}
__device__ __forceinline__ size_t PC(const VVDims &v, int k, int j, int i) {
    return (size_t)(k + 1) * v.plane1 + (size_t)j * v.nr + i;
}
__device__ __forceinline__ size_t UV(const VVDims &v, int k, int c, int j, int i) {
    return ((size_t)k * 3 + c) * v.plane1 + (size_t)j * v.nr + i;
}
__device__ __forceinline__ size_t UC(const VVDims &v, int k, int j, int i) {
    return (size_t)k * v.plane1 + (size_t)j * v.nr + i;
}
__device__ __forceinline__ size_t GW(const VVDims &v, int k, int c, int j) { return ((size_t)(k + 1) * 3 + c) * v.nt + j; }
// term plane slot of plane k (-1 .. nloc): the full padded array, or the ring of the chunked matvec
__device__ __forceinline__ uint32_t tslot(const VVDims &v, int k) {
    const uint32_t kk = (uint32_t)(k + 1);
    return v.ring ? kk % v.ring : kk;
}
// L2 policy of the term rings: evict_last (kept in the persisting set-aside) in ring mode, else normal
__device__ __forceinline__ uint64_t term_policy(const VVDims &v) {
    uint64_t pol;
    if (v.ring) asm("createpolicy.fractional.L2::evict_last.b64 %0, 0f3F800000;" : "=l"(pol));
    else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 0f3F800000;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void S2T(double *p, double x, double y, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(x), "d"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 L2T(const double *p, uint64_t pol) {
    double2 r;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double L1T(const double *p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}

// ------------------------------------------------------------ face geometry (R27; oracle A_r .. L_p)
struct Geo {
    const VVArrays &a;
    __device__ __forceinline__ double dp(int k) const { return a.dpp[k + 1]; }
    __device__ __forceinline__ double hm(int k) const { return a.hmp[k + 1]; }
    __device__ __forceinline__ double A_r(int i, int j, int k) const { return mul(mul(a.rf2[i], a.C[j]), dp(k)); }
    __device__ __forceinline__ double A_t(int i, int j, int k) const { return mul(mul(a.sinf[j], a.dR2[i]), dp(k)); }
    __device__ __forceinline__ double A_p(int i, int j) const { return mul(a.dR2[i], a.dt[j]); }
    __device__ __forceinline__ double L_t(int e, int j) const { return mul(a.rce[e], a.ht[j]); }
    __device__ __forceinline__ double L_p(int e, int j, int k) const { return mul(mul(a.rce[e], a.sinc[j]), hm(k)); }
};

// ------------------------------------------------------------ outflow and circulations of p (+ walls)
template <bool WALL>
struct Field {
    const VVDims &v;
    const VVArrays &a;
    const double *__restrict__ p;
    Geo g;
    __device__ __forceinline__ double P(int k, int c, int j, int i) const { return __ldg(p + PV(v, k, c, j, i)); }
    __device__ __forceinline__ double gi(int k, int c, int j) const { return WALL ? __ldg(a.gin + GW(v, k, c, j)) : 0.0; }
    __device__ __forceinline__ double go(int k, int c, int j) const { return WALL ? __ldg(a.gout + GW(v, k, c, j)) : 0.0; }
    // v_r on r-face e of row (j, k), the wall normal velocity on e = 0, nr
    __device__ __forceinline__ double vr(int k, int j, int e) const {
        if (e == 0) return gi(k, 0, j);
        if (e == v.nr) return go(k, 0, j);
        return P(k, 0, j, e);
    }
    // e = wc * delta of cell (i, j, k), k in [-1, nloc-1], from the face values of the cell
    __device__ __forceinline__ double ediv_v(int i, int j, int k, double vrl, double vrh, double vtl, double vth,
                                             double vpl, double vph) const {
        return ediv_w(i, j, k, vrl, vrh, vtl, vth, vpl, vph, __ldg(a.wc + PC(v, k, j, i)));
    }
    __device__ __forceinline__ double ediv_w(int i, int j, int k, double vrl, double vrh, double vtl, double vth,
                                             double vpl, double vph, double wcv) const {
        const double fr_lo = mul(g.A_r(i, j, k), vrl);
        const double fr_hi = mul(g.A_r(i + 1, j, k), vrh);
        const double ft_lo = (j == 0) ? 0.0 : mul(g.A_t(i, j, k), vtl);
        const double ft_hi = (j == v.nt - 1) ? 0.0 : mul(g.A_t(i, j + 1, k), vth);
        const double ap = g.A_p(i, j);
        const double fp_lo = mul(ap, vpl);
        const double fp_hi = mul(ap, vph);
        double d = add(sub(fr_hi, fr_lo), sub(ft_hi, ft_lo));
        d = add(d, sub(fp_hi, fp_lo));
        return mul(wcv, d);
    }
    // r-edge at theta-face j (1..nt-1), phi-face k: v_phi(j), v_phi(j-1), v_theta(k), v_theta(k-1)
    __device__ __forceinline__ double Gr_v(int i, int j, int k, double vpj, double vpjm, double vtk, double vtkm) const {
        const double gp_a = mul(g.L_p(i + 1, j, k), vpj);
        const double gp_b = mul(g.L_p(i + 1, j - 1, k), vpjm);
        const double lt = g.L_t(i + 1, j);
        const double gt_a = mul(lt, vtk);
        const double gt_b = mul(lt, vtkm);
        return sub(sub(gp_a, gp_b), sub(gt_a, gt_b));
    }
    // theta-edge at r-face e (0..nr), phi-face k: v_r(e, k), v_r(e, k-1), v_phi above / below the face
    __device__ __forceinline__ double Gt_v(int e, int j, int k, double vrk, double vrkm, double up, double dn) const {
        const double gr_a = mul(a.hr[e], vrk);
        const double gr_b = mul(a.hr[e], vrkm);
        const double gp_a = mul(g.L_p(e + 1, j, k), up);
        const double gp_b = mul(g.L_p(e, j, k), dn);
        return sub(sub(gr_a, gr_b), sub(gp_a, gp_b));
    }
    // phi-edge at r-face e (0..nr), theta-face j (1..nt-1): v_theta above / below, v_r(e, j), v_r(e, j-1)
    __device__ __forceinline__ double Gp_v(int e, int j, double up, double dn, double vrj, double vrjm) const {
        const double gt_a = mul(g.L_t(e + 1, j), up);
        const double gt_b = mul(g.L_t(e, j), dn);
        const double gr_a = mul(a.hr[e], vrj);
        const double gr_b = mul(a.hr[e], vrjm);
        return sub(sub(gt_a, gt_b), sub(gr_a, gr_b));
    }
    __device__ __forceinline__ double ediv(int i, int j, int k) const {
        return ediv_v(i, j, k, vr(k, j, i), vr(k, j, i + 1), (j == 0) ? 0.0 : P(k, 1, j, i),
                      (j == v.nt - 1) ? 0.0 : P(k, 1, j + 1, i), P(k, 2, j, i), P(k + 1, 2, j, i));
    }
    __device__ __forceinline__ double Gr(int i, int j, int k) const {
        return Gr_v(i, j, k, P(k, 2, j, i), P(k, 2, j - 1, i), P(k, 1, j, i), P(k - 1, 1, j, i));
    }
    __device__ __forceinline__ double Gt(int e, int j, int k) const {
        return Gt_v(e, j, k, vr(k, j, e), vr(k - 1, j, e), (e < v.nr) ? P(k, 2, j, e) : go(k, 2, j),
                    (e > 0) ? P(k, 2, j, e - 1) : gi(k, 2, j));
    }
    __device__ __forceinline__ double Gp(int e, int j, int k) const {
        return Gp_v(e, j, (e < v.nr) ? P(k, 1, j, e) : go(k, 1, j), (e > 0) ? P(k, 1, j, e - 1) : gi(k, 1, j),
                    vr(k, j, e), vr(k, j - 1, e));
    }
};

__device__ __forceinline__ double Wt_at(const VVDims &v, const VVArrays &a, int e, int j, int k) {
    return (e < v.nr) ? __ldg(a.Wt + PC(v, k, j, e)) : __ldg(a.WtO + (size_t)(k + 1) * v.nt + j);
}
__device__ __forceinline__ double Wp_at(const VVDims &v, const VVArrays &a, int e, int j, int k) {
    return (e < v.nr) ? __ldg(a.Wp + UC(v, k, j, e)) : __ldg(a.WpO + (size_t)k * v.nt + j);
}

// ------------------------------------------------------------ validation
__global__ void __launch_bounds__(kVVThreads) k_vv_validate(VVDims v, const double *__restrict__ nu,
                                                            const double *__restrict__ s, int *flag) {
    int bad = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        const double a = nu[c], b = s[c];
        bad |= !(a >= 0.0) | !isfinite(a) | !(b >= 0.0) | !isfinite(b);
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && bad) atomicOr(flag, 1);
}

// ------------------------------------------------------------ coefficients (R28, R30; the oracle's coefficients)
__device__ __forceinline__ double nu_at(const VVDims &v, const VVArrays &a, int k, int j, int i) {
    return (k < 0) ? a.nulo[(size_t)j * v.nr + i] : a.nu[UC(v, k, j, i)];
}
__device__ __forceinline__ double s_at(const VVDims &v, const VVArrays &a, int k, int j, int i) {
    return (k < 0) ? a.slo[(size_t)j * v.nr + i] : a.s[UC(v, k, j, i)];
}

__global__ void __launch_bounds__(kVVThreads) k_vv_coef(VVDims v, VVArrays a) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const Geo g{a};
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        const int km = k - 1;
        const double V = mul(mul(a.R3[i], a.C[j]), g.dp(k));
        a.wc[PC(v, k, j, i)] = __ddiv_rn(nu_at(v, a, k, j, i), V);
        // r-edge at theta-face j, phi-face k
        double wr = 0.0;
        if (j >= 1) {
            const double nue = mul(add(add(nu_at(v, a, km, j - 1, i), nu_at(v, a, km, j, i)),
                                       add(nu_at(v, a, k, j - 1, i), nu_at(v, a, k, j, i))),
                                   0.25);
            wr = __ddiv_rn(mul(nue, a.dr[i]), mul(mul(a.rc2[i], a.Cs[j]), g.hm(k)));
        }
        a.Wr[PC(v, k, j, i)] = wr;
        // theta-edges at r-face i (and the outer wall nr on the last cell), phi-face k
        for (int e = i; e <= ((i == v.nr - 1) ? v.nr : i); ++e) {
            const int wall = (e == 0) ? v.wall_in : (e == v.nr ? v.wall_out : -1);
            double w = 0.0;
            if (wall != 1) {
                double nue;
                if (e == 0) nue = mul(add(nu_at(v, a, km, j, 0), nu_at(v, a, k, j, 0)), 0.5);
                else if (e == v.nr) nue = mul(add(nu_at(v, a, km, j, v.nr - 1), nu_at(v, a, k, j, v.nr - 1)), 0.5);
                else
                    nue = mul(add(add(nu_at(v, a, km, j, e - 1), nu_at(v, a, km, j, e)),
                                  add(nu_at(v, a, k, j, e - 1), nu_at(v, a, k, j, e))),
                              0.25);
                w = __ddiv_rn(mul(nue, mul(a.rf[e], a.dt[j])), mul(mul(a.sinc[j], a.rhor[e]), g.hm(k)));
            }
            if (e < v.nr) a.Wt[PC(v, k, j, e)] = w;
            else a.WtO[(size_t)(k + 1) * v.nt + j] = w;
        }
        // phi-edges at r-face i (and nr), theta-face j >= 1
        for (int e = i; e <= ((i == v.nr - 1) ? v.nr : i); ++e) {
            const int wall = (e == 0) ? v.wall_in : (e == v.nr ? v.wall_out : -1);
            double w = 0.0;
            if (j >= 1 && wall != 1) {
                double nue;
                if (e == 0) nue = mul(add(nu_at(v, a, k, j - 1, 0), nu_at(v, a, k, j, 0)), 0.5);
                else if (e == v.nr) nue = mul(add(nu_at(v, a, k, j - 1, v.nr - 1), nu_at(v, a, k, j, v.nr - 1)), 0.5);
                else
                    nue = mul(add(add(nu_at(v, a, k, j - 1, e - 1), nu_at(v, a, k, j - 1, e)),
                                  add(nu_at(v, a, k, j, e - 1), nu_at(v, a, k, j, e))),
                              0.25);
                w = __ddiv_rn(mul(nue, mul(mul(a.rf[e], a.sinf[j]), g.dp(k))), mul(a.rhor[e], a.ht[j]));
            }
            if (e < v.nr) a.Wp[UC(v, k, j, e)] = w;
            else a.WpO[(size_t)k * v.nt + j] = w;
        }
        // s_f M_f of the three lower faces
        double m0 = 0.0, m1 = 0.0;
        if (i >= 1) {
            const double sf = mul(add(s_at(v, a, k, j, i - 1), s_at(v, a, k, j, i)), 0.5);
            m0 = mul(sf, mul(g.A_r(i, j, k), a.hr[i]));
        }
        if (j >= 1) {
            const double sf = mul(add(s_at(v, a, k, j - 1, i), s_at(v, a, k, j, i)), 0.5);
            m1 = mul(sf, mul(g.A_t(i, j, k), g.L_t(i + 1, j)));
        }
        const double sf = mul(add(s_at(v, a, km, j, i), s_at(v, a, k, j, i)), 0.5);
        const double m2 = mul(sf, mul(g.A_p(i, j), g.L_p(i + 1, j, k)));
        a.sM[UV(v, k, 0, j, i)] = m0;
        a.sM[UV(v, k, 1, j, i)] = m1;
        a.sM[UV(v, k, 2, j, i)] = m2;
    }
}

// ------------------------------------------------------------ ring sums (the polar axes, Listing 3)
// One block per radius i: Dot2 over the local planes of (north row, south row), fixed tree.
template <bool EXACT>
__global__ void __launch_bounds__(kVVThreads) k_vv_ring(VVDims v, VVArrays a, int mode, const double *__restrict__ p,
                                                        double *out) {
    const int i = blockIdx.x;
    const Geo g{a};
    Acc<EXACT> acc[2];
    for (int k = threadIdx.x; k < v.nloc; k += blockDim.x) {
        if (mode == 0) {
            acc[0].add(a.nu[UC(v, k, 0, i)], 1.0);
            acc[1].add(a.nu[UC(v, k, v.nt - 1, i)], 1.0);
        } else {
            acc[0].add(__ldg(p + PV(v, k, 2, 0, i)), g.L_p(i + 1, 0, k));
            acc[1].add(__ldg(p + PV(v, k, 2, v.nt - 1, i)), g.L_p(i + 1, v.nt - 1, k));
        }
    }
    block_combine<EXACT, kVVThreads, 2>(acc);
    if (threadIdx.x == 0) {
        out[2 * i] = acc[0].p;
        out[2 * i + 1] = acc[0].s;
        out[2 * (v.nr + i)] = acc[1].p;
        out[2 * (v.nr + i) + 1] = acc[1].s;
    }
}

__global__ void k_vv_axis_weights(VVDims v, VVArrays a, double np) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < v.nr; i += gridDim.x * blockDim.x) {
        const double nN = __ddiv_rn(add(a.nuring[2 * i], a.nuring[2 * i + 1]), np);
        const double nS = __ddiv_rn(add(a.nuring[2 * (v.nr + i)], a.nuring[2 * (v.nr + i) + 1]), np);
        a.WN[i] = __ddiv_rn(mul(nN, a.dr[i]), mul(a.rc2[i], a.cap[0]));
        a.WS[i] = __ddiv_rn(mul(nS, a.dr[i]), mul(a.rc2[i], a.cap[1]));
    }
}

// ------------------------------------------------------------ Jacobi diagonal (the oracle's diagonal)
__global__ void __launch_bounds__(kVVThreads) k_vv_diag(VVDims v, VVArrays a) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const Geo g{a};
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        double d = 1.0;
        if (i >= 1) {
            const double A = g.A_r(i, j, k), l = a.hr[i];
            double w = add(Wt_at(v, a, i, j, k), Wt_at(v, a, i, j, k + 1));
            if (j >= 1) w = add(w, Wp_at(v, a, i, j, k));
            if (j + 1 <= v.nt - 1) w = add(w, Wp_at(v, a, i, j + 1, k));
            d = add(a.sM[UV(v, k, 0, j, i)], mul(mul(A, A), add(a.wc[PC(v, k, j, i - 1)], a.wc[PC(v, k, j, i)])));
            d = add(d, mul(mul(l, l), w));
        }
        a.D[UV(v, k, 0, j, i)] = d;
        d = 1.0;
        if (j >= 1) {
            const double A = g.A_t(i, j, k), l = g.L_t(i + 1, j);
            double w = add(a.Wr[PC(v, k, j, i)], a.Wr[PC(v, k + 1, j, i)]);
            w = add(w, Wp_at(v, a, i, j, k));
            w = add(w, Wp_at(v, a, i + 1, j, k));
            d = add(a.sM[UV(v, k, 1, j, i)], mul(mul(A, A), add(a.wc[PC(v, k, j - 1, i)], a.wc[PC(v, k, j, i)])));
            d = add(d, mul(mul(l, l), w));
        }
        a.D[UV(v, k, 1, j, i)] = d;
        {
            const double A = g.A_p(i, j), l = g.L_p(i + 1, j, k);
            const double lo = (j == 0) ? a.WN[i] : a.Wr[PC(v, k, j, i)];
            const double hi = (j == v.nt - 1) ? a.WS[i] : a.Wr[PC(v, k, j + 1, i)];
            double w = add(lo, hi);
            w = add(w, Wt_at(v, a, i, j, k));
            w = add(w, Wt_at(v, a, i + 1, j, k));
            d = add(a.sM[UV(v, k, 2, j, i)], mul(mul(A, A), add(a.wc[PC(v, k - 1, j, i)], a.wc[PC(v, k, j, i)])));
            d = add(d, mul(mul(l, l), w));
        }
        a.D[UV(v, k, 2, j, i)] = d;
    }
}

// ------------------------------------------------------------ the operator (the oracle's apply), two phases
// Phase 1 (k_vv_terms): per cell of planes -1 .. nloc the products the rows combine -- the outflow term
// e = wc delta (planes -1 .. nloc-1) and the edge terms tau = W Gamma of the cell's lower r-, theta- and
// phi-edges (planes 0 .. nloc; the outer-wall edges of the last radial cell into side arrays).
// Phase 2 (k_vv_rows): the three rows of every local cell from those terms, sM p and the polar-axis
// terms WN GN, WS GS of the ring sums; Dot2 partial of p.q.  Each product is the one the oracle forms
// (e = wc * delta, W * Gamma), so the rows are bit-identical.  48 + 32 + 80 + 24 = 184 B/cell instead
// of the 104 of a fused kernel, but every load is a coalesced stream with no recomputation: the fused
// form was issue- and occupancy-bound (152 registers, ~1,300 instructions per cell).
template <bool WALL>
__global__ void __launch_bounds__(kVVThreads) k_vv_terms(VVDims v, VVArrays a, DevArrays base, int loop) {
    if (loop && *(volatile int *)&base.sc->done) return;
    const Field<WALL> F{v, a, a.p, Geo{a}};
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t n = v.ncell + 2 * v.plane1;   // planes -1 .. nloc
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        k -= 1;
        const size_t pc = PC(v, k, j, i);
        if (k <= v.nloc - 1) a.E[pc] = F.ediv(i, j, k);
        if (k >= 0) {
            a.TR[pc] = (j >= 1) ? mul(__ldg(a.Wr + pc), F.Gr(i, j, k)) : 0.0;
            a.TT[pc] = mul(__ldg(a.Wt + pc), F.Gt(i, j, k));
            a.TP[pc] = (j >= 1 && k <= v.nloc - 1) ? mul(Wp_at(v, a, i, j, k), F.Gp(i, j, k)) : 0.0;
            if (i == v.nr - 1) {
                const size_t w = (size_t)(k + 1) * v.nt + j;
                a.TTO[w] = mul(__ldg(a.WtO + w), F.Gt(v.nr, j, k));
                a.TPO[w] = (j >= 1 && k <= v.nloc - 1) ? mul(Wp_at(v, a, v.nr, j, k), F.Gp(v.nr, j, k)) : 0.0;
            }
        }
    }
}

__device__ __forceinline__ double TT_at(const VVDims &v, const VVArrays &a, int e, int j, int k) {
    return (e < v.nr) ? __ldg(a.TT + PC(v, k, j, e)) : __ldg(a.TTO + (size_t)(k + 1) * v.nt + j);
}
__device__ __forceinline__ double TP_at(const VVDims &v, const VVArrays &a, int e, int j, int k) {
    return (e < v.nr) ? __ldg(a.TP + PC(v, k, j, e)) : __ldg(a.TPO + (size_t)(k + 1) * v.nt + j);
}

template <bool WITH_DOT, bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kVVThreads) k_vv_rows(VVDims v, VVArrays a, DevArrays base, double *__restrict__ y,
                                                        unsigned total) {
    if (LOOP && *(volatile int *)&base.sc->done) return;
    const Geo g{a};
    const double *__restrict__ E = a.E;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        const size_t pc = PC(v, k, j, i);
        const double e0 = __ldg(E + pc);
        // r-face i
        double yr = 0.0;
        const double pr = __ldg(a.p + PV(v, k, 0, j, i));
        if (i >= 1) {
            yr = mul(__ldg(a.sM + UV(v, k, 0, j, i)), pr);
            yr = add(yr, mul(g.A_r(i, j, k), sub(__ldg(E + pc - 1), e0)));
            double cc = __ldg(a.TT + pc);
            cc = sub(cc, __ldg(a.TT + pc + v.plane1));
            if (j >= 1) cc = sub(cc, __ldg(a.TP + pc));
            if (j + 1 <= v.nt - 1) cc = add(cc, __ldg(a.TP + pc + v.nr));
            yr = add(yr, mul(a.hr[i], cc));
        }
        // theta-face j
        double yt = 0.0;
        const double pt = __ldg(a.p + PV(v, k, 1, j, i));
        if (j >= 1) {
            yt = mul(__ldg(a.sM + UV(v, k, 1, j, i)), pt);
            yt = add(yt, mul(g.A_t(i, j, k), sub(__ldg(E + pc - v.nr), e0)));
            double cc = sub(__ldg(a.TR + pc + v.plane1), __ldg(a.TR + pc));
            cc = add(cc, __ldg(a.TP + pc));
            cc = sub(cc, TP_at(v, a, i + 1, j, k));
            yt = add(yt, mul(g.L_t(i + 1, j), cc));
        }
        // phi-face k
        const double pp = __ldg(a.p + PV(v, k, 2, j, i));
        double yp = mul(__ldg(a.sM + UV(v, k, 2, j, i)), pp);
        yp = add(yp, mul(g.A_p(i, j), sub(__ldg(E + pc - v.plane1), e0)));
        const double lo = (j == 0) ? mul(__ldg(a.WN + i), add(__ldg(a.ring + 2 * i), __ldg(a.ring + 2 * i + 1)))
                                   : __ldg(a.TR + pc);
        const double hi = (j == v.nt - 1)
                              ? mul(__ldg(a.WS + i), -add(__ldg(a.ring + 2 * (v.nr + i)), __ldg(a.ring + 2 * (v.nr + i) + 1)))
                              : __ldg(a.TR + pc + v.nr);
        double cc = sub(lo, hi);
        cc = sub(cc, __ldg(a.TT + pc));
        cc = add(cc, TT_at(v, a, i + 1, j, k));
        yp = add(yp, mul(g.L_p(i + 1, j, k), cc));
        y[UV(v, k, 0, j, i)] = yr;
        y[UV(v, k, 1, j, i)] = yt;
        y[UV(v, k, 2, j, i)] = yp;
        if (WITH_DOT) {
            dot[0].add(pr, yr);
            dot[0].add(pt, yt);
            dot[0].add(pp, yp);
        }
    }
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kVVThreads, 1>(dot, base.partials, &base.sc->ticket[0], blockIdx.x, total, out)) {
            if (threadIdx.x == 0) {
                base.sc->red1[0] = out[0].p;
                base.sc->red1[1] = out[0].s;
            }
        }
    }
}

// ------------------------------------------------------------ 16-byte pair variants (nr even)
// Two r-neighbour cells (i0, i0 + 1), i0 even, per thread: every stream is one 16-byte load / store and
// the shared neighbours are loaded once.  The per-cell arithmetic is the value-based helpers above, so
// the results are the scalar kernels' bit for bit.  The scalar kernels were latency-bound (about 40 %
// issue utilisation and 35-48 % of DRAM bandwidth at 50 % occupancy).
__device__ __forceinline__ double2 L2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ void S2(double *p, double x, double y) {
    *reinterpret_cast<double2 *>(p) = make_double2(x, y);
}

template <bool WALL>
__global__ void __launch_bounds__(kVVThreads, 3) k_vv_terms2(VVDims v, VVArrays a, DevArrays base, int loop) {
    if (loop && *(volatile int *)&base.sc->done) return;
    const Field<WALL> F{v, a, a.p, Geo{a}};
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = (v.ncell + 2 * v.plane1) >> 1;   // planes -1 .. nloc
    const int nr = v.nr, nt = v.nt;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += stride) {
        int i0, j, k;
        cell_of(v, 2 * t, i0, j, k);
        k -= 1;
        // every load up front (addresses clamped into the arrays; unused values are discarded), so the
        // memory system sees all of the thread's requests before the first use
        const int km = k > -1 ? k - 1 : -1, kp = k < v.nloc ? k + 1 : v.nloc, jm = j > 0 ? j - 1 : 0;
        const int jp = j < nt - 1 ? j + 1 : j, kw = k < 0 ? 0 : (k > v.nloc - 1 ? v.nloc - 1 : k);
        const size_t pc = PC(v, k, j, i0);
        const bool last = (i0 + 2 == nr);
        const double2 R = L2(a.p + PV(v, k, 0, j, i0));
        const double2 T = L2(a.p + PV(v, k, 1, j, i0));
        const double2 Pp = L2(a.p + PV(v, k, 2, j, i0));
        const double2 Tj1 = L2(a.p + PV(v, k, 1, jp, i0));
        const double2 Pk1 = L2(a.p + PV(v, kp, 2, j, i0));
        const double2 Rm = L2(a.p + PV(v, km, 0, j, i0));
        const double2 Pjm = L2(a.p + PV(v, k, 2, jm, i0));
        const double2 Tkm = L2(a.p + PV(v, km, 1, j, i0));
        const double2 Rjm = L2(a.p + PV(v, k, 0, jm, i0));
        const double r2 = __ldg(a.p + PV(v, k, 0, j, last ? i0 : i0 + 2));
        const double pm1 = __ldg(a.p + PV(v, k, 2, j, i0 > 0 ? i0 - 1 : 0));
        const double tm1 = __ldg(a.p + PV(v, k, 1, j, i0 > 0 ? i0 - 1 : 0));
        const double2 wt = L2(a.Wt + pc), wr = L2(a.Wr + pc), wp = L2(a.Wp + UC(v, kw, j, i0));
        const double vr0 = (i0 == 0) ? F.gi(k, 0, j) : R.x;          // v_r on r-face i0 (wall at 0)
        const double vr2 = last ? F.go(k, 0, j) : r2;
        if (k <= v.nloc - 1) {
            const double e0 = F.ediv_v(i0, j, k, vr0, R.y, T.x, Tj1.x, Pp.x, Pk1.x);
            const double e1 = F.ediv_v(i0 + 1, j, k, R.y, vr2, T.y, Tj1.y, Pp.y, Pk1.y);
            S2(a.E + pc, e0, e1);
        }
        if (k >= 0) {
            const double vrm0 = (i0 == 0) ? F.gi(k - 1, 0, j) : Rm.x;
            const double dn0 = (i0 == 0) ? F.gi(k, 2, j) : pm1;
            S2(a.TT + pc, mul(wt.x, F.Gt_v(i0, j, k, vr0, vrm0, Pp.x, dn0)),
               mul(wt.y, F.Gt_v(i0 + 1, j, k, R.y, Rm.y, Pp.y, Pp.x)));
            double tr0 = 0.0, tr1 = 0.0, tp0 = 0.0, tp1 = 0.0;
            if (j >= 1) {
                tr0 = mul(wr.x, F.Gr_v(i0, j, k, Pp.x, Pjm.x, T.x, Tkm.x));
                tr1 = mul(wr.y, F.Gr_v(i0 + 1, j, k, Pp.y, Pjm.y, T.y, Tkm.y));
                if (k <= v.nloc - 1) {
                    const double vrjm0 = (i0 == 0) ? F.gi(k, 0, j - 1) : Rjm.x;
                    const double tdn0 = (i0 == 0) ? F.gi(k, 1, j) : tm1;
                    tp0 = mul(wp.x, F.Gp_v(i0, j, T.x, tdn0, vr0, vrjm0));
                    tp1 = mul(wp.y, F.Gp_v(i0 + 1, j, T.y, T.x, R.y, Rjm.y));
                }
            }
            S2(a.TR + pc, tr0, tr1);
            S2(a.TP + pc, tp0, tp1);
            if (last) {
                const size_t w = (size_t)(k + 1) * nt + j;
                a.TTO[w] = mul(__ldg(a.WtO + w), F.Gt_v(nr, j, k, F.go(k, 0, j), F.go(k - 1, 0, j), F.go(k, 2, j), Pp.y));
                a.TPO[w] = (j >= 1 && k <= v.nloc - 1)
                               ? mul(__ldg(a.WpO + (size_t)k * nt + j),
                                     F.Gp_v(nr, j, F.go(k, 1, j), T.y, F.go(k, 0, j), F.go(k, 0, j - 1)))
                               : 0.0;
            }
        }
    }
}

// The same phase with its 16-byte streams staged by cp.async into shared memory one grid-stride
// iteration ahead (double-buffered, each thread copying and reading only its own slots, so no block
// barrier): the HBM latency of an iteration's loads overlaps the previous iteration's arithmetic.
constexpr int kStg = 13;   // staged streams per pair
__device__ __forceinline__ void cp16(double2 *dst, const double *src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <bool WALL>
__global__ void __launch_bounds__(kVVThreads, 2) k_vv_terms3(VVDims v, VVArrays a, DevArrays base, int loop) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // programmatic dependent launch (chunked matvec)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (loop && *(volatile int *)&base.sc->done) return;
    extern __shared__ double2 stg[];   // [2][kStg][kVVThreads]
    const Field<WALL> F{v, a, a.p, Geo{a}};
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = ((uint32_t)(v.ke - v.kb + 2) * v.plane1) >> 1;   // planes kb-1 .. ke
    const uint32_t c0 = (uint32_t)v.kb * v.plane1;
    const uint64_t polT = term_policy(v);
    const int nr = v.nr, nt = v.nt;
    auto slot = [&](int stage, int s) -> double2 * { return stg + ((size_t)stage * kStg + s) * kVVThreads + threadIdx.x; };
    auto issue = [&](uint32_t t, int stage) {
        if (t < npair) {
            int i0, j, k;
            cell_of(v, 2 * t + c0, i0, j, k);
            k -= 1;
            const int km = k > -1 ? k - 1 : -1, kp = k < v.nloc ? k + 1 : v.nloc;
            const int jp = j < nt - 1 ? j + 1 : j, kw = k < 0 ? 0 : (k > v.nloc - 1 ? v.nloc - 1 : k);
            const size_t pc = PC(v, k, j, i0);
            cp16(slot(stage, 0), a.p + PV(v, k, 0, j, i0));
            cp16(slot(stage, 1), a.p + PV(v, k, 1, j, i0));
            cp16(slot(stage, 2), a.p + PV(v, k, 2, j, i0));
            cp16(slot(stage, 3), a.p + PV(v, k, 1, jp, i0));
            cp16(slot(stage, 4), a.p + PV(v, kp, 2, j, i0));
            cp16(slot(stage, 5), a.p + PV(v, km, 0, j, i0));
            cp16(slot(stage, 6), a.p + PV(v, km, 1, j, i0));
            cp16(slot(stage, 7), a.Wt + pc);
            cp16(slot(stage, 8), a.Wr + pc);
            cp16(slot(stage, 9), a.Wp + UC(v, kw, j, i0));
            cp16(slot(stage, 10), a.wc + pc);
            const int jm = j > 0 ? j - 1 : 0;
            cp16(slot(stage, 11), a.p + PV(v, k, 2, jm, i0));
            cp16(slot(stage, 12), a.p + PV(v, k, 0, jm, i0));
        }
        cp_commit();
    };
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    issue(t, 0);
    for (int it = 0; t < npair; t += stride, ++it) {
        const int st = it & 1;
        const unsigned act = __activemask();
        __syncwarp(act);   // the neighbouring lanes have finished reading this lane's slots of stage st ^ 1
        issue(t + stride, st ^ 1);
        cp_wait1();        // this thread's copies of stage st have landed
        __syncwarp(act);   // ... and the other lanes' (r2, pm1, tm1 come from the neighbouring lanes' slots)
        int i0, j, k;
        cell_of(v, 2 * t + c0, i0, j, k);
        k -= 1;
        const size_t pc = PC(v, k, j, i0);
        const size_t pt = (size_t)tslot(v, k) * v.plane1 + (size_t)j * nr + i0;   // term slot
        const bool last = (i0 + 2 == nr);
        const double2 R = *slot(st, 0), T = *slot(st, 1), Pp = *slot(st, 2), Tj1 = *slot(st, 3), Pk1 = *slot(st, 4);
        const double2 Rm = *slot(st, 5), Tkm = *slot(st, 6), wt = *slot(st, 7), wr = *slot(st, 8), wp = *slot(st, 9);
        const double2 wcv = *slot(st, 10), Pjm = *slot(st, 11), Rjm = *slot(st, 12);
        // the r-neighbours of the pair: pair t + 1 (i0 + 2) and pair t - 1 (i0 - 1) of the same row are the
        // neighbouring lanes' staged pairs (grid-stride trips keep consecutive pairs in consecutive lanes)
        const int lane = threadIdx.x & 31;
        const bool up_in = lane < 31 && t + 1 < npair, dn_in = lane > 0;
        const double r2 = last ? 0.0 : (up_in ? slot(st, 0)[1].x : __ldg(a.p + PV(v, k, 0, j, i0 + 2)));
        const double pm1 = i0 == 0 ? 0.0 : (dn_in ? slot(st, 2)[-1].y : __ldg(a.p + PV(v, k, 2, j, i0 - 1)));
        const double tm1 = i0 == 0 ? 0.0 : (dn_in ? slot(st, 1)[-1].y : __ldg(a.p + PV(v, k, 1, j, i0 - 1)));
        const double vr0 = (i0 == 0) ? F.gi(k, 0, j) : R.x;          // v_r on r-face i0 (wall at 0)
        const double vr2 = last ? F.go(k, 0, j) : r2;
        if (k <= v.ke - 1) {   // (ke <= nloc)
            const double e0 = F.ediv_w(i0, j, k, vr0, R.y, T.x, Tj1.x, Pp.x, Pk1.x, wcv.x);
            const double e1 = F.ediv_w(i0 + 1, j, k, R.y, vr2, T.y, Tj1.y, Pp.y, Pk1.y, wcv.y);
            S2T(a.E + pt, e0, e1, polT);
        }
        if (k >= v.kb) {       // (kb >= 0)
            const double vrm0 = (i0 == 0) ? F.gi(k - 1, 0, j) : Rm.x;
            const double dn0 = (i0 == 0) ? F.gi(k, 2, j) : pm1;
            S2T(a.TT + pt, mul(wt.x, F.Gt_v(i0, j, k, vr0, vrm0, Pp.x, dn0)),
                mul(wt.y, F.Gt_v(i0 + 1, j, k, R.y, Rm.y, Pp.y, Pp.x)), polT);
            double tr0 = 0.0, tr1 = 0.0, tp0 = 0.0, tp1 = 0.0;
            if (j >= 1) {
                tr0 = mul(wr.x, F.Gr_v(i0, j, k, Pp.x, Pjm.x, T.x, Tkm.x));
                tr1 = mul(wr.y, F.Gr_v(i0 + 1, j, k, Pp.y, Pjm.y, T.y, Tkm.y));
                if (k <= v.nloc - 1) {
                    const double vrjm0 = (i0 == 0) ? F.gi(k, 0, j - 1) : Rjm.x;
                    const double tdn0 = (i0 == 0) ? F.gi(k, 1, j) : tm1;
                    tp0 = mul(wp.x, F.Gp_v(i0, j, T.x, tdn0, vr0, vrjm0));
                    tp1 = mul(wp.y, F.Gp_v(i0 + 1, j, T.y, T.x, R.y, Rjm.y));
                }
            }
            S2T(a.TR + pt, tr0, tr1, polT);
            S2T(a.TP + pt, tp0, tp1, polT);
            if (last) {
                const size_t w = (size_t)(k + 1) * nt + j;
                a.TTO[w] = mul(__ldg(a.WtO + w), F.Gt_v(nr, j, k, F.go(k, 0, j), F.go(k - 1, 0, j), F.go(k, 2, j), Pp.y));
                a.TPO[w] = (j >= 1 && k <= v.nloc - 1)
                               ? mul(__ldg(a.WpO + (size_t)k * nt + j),
                                     F.Gp_v(nr, j, F.go(k, 1, j), T.y, F.go(k, 0, j), F.go(k, 0, j - 1)))
                               : 0.0;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <bool WITH_DOT, bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kVVThreads, 2) k_vv_rows2(VVDims v, VVArrays a, DevArrays base, double *__restrict__ y,
                                                         unsigned total) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (LOOP && *(volatile int *)&base.sc->done) return;
    const Geo g{a};
    const double *__restrict__ E = a.E;
    const int nr = v.nr, nt = v.nt;
    const uint32_t pl = v.plane1;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = ((uint32_t)(v.ke - v.kb) * v.plane1) >> 1;   // planes kb .. ke-1
    const uint32_t c0 = (uint32_t)v.kb * v.plane1;
    const uint64_t polT = term_policy(v);
    // (staging these streams with cp.async as in k_vv_terms3 measured slower here: 643 vs 513 us)
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += stride) {
        int i0, j, k;
        cell_of(v, 2 * t + c0, i0, j, k);
        // term slots of planes k, k - 1, k + 1 (rings wrap)
        const uint32_t s0 = tslot(v, k);
        const uint32_t sm_ = v.ring ? (s0 == 0 ? v.ring - 1 : s0 - 1) : s0 - 1;
        const uint32_t sp_ = v.ring ? (s0 + 1 == v.ring ? 0 : s0 + 1) : s0 + 1;
        const size_t in = (size_t)j * nr + i0;
        const size_t pc = (size_t)s0 * pl + in, pcm = (size_t)sm_ * pl + in, pcp = (size_t)sp_ * pl + in;
        const bool last = (i0 + 2 == nr);
        const double2 e = L2T(E + pc, polT);
        const double2 pr = L2(a.p + PV(v, k, 0, j, i0));
        const double2 pt = L2(a.p + PV(v, k, 1, j, i0));
        const double2 pp = L2(a.p + PV(v, k, 2, j, i0));
        const double2 tt = L2T(a.TT + pc, polT);
        const double2 tr = L2T(a.TR + pc, polT);
        const double2 tp = L2T(a.TP + pc, polT);
        const double2 sm0 = L2(a.sM + UV(v, k, 0, j, i0));
        const double2 sm1 = L2(a.sM + UV(v, k, 1, j, i0));
        const double2 sm2 = L2(a.sM + UV(v, k, 2, j, i0));
        const double2 tt1 = L2T(a.TT + pcp, polT);
        const double tt2 = last ? __ldg(a.TTO + (size_t)(k + 1) * nt + j) : L1T(a.TT + pc + 2, polT);
        const double tp2 = last ? __ldg(a.TPO + (size_t)(k + 1) * nt + j) : L1T(a.TP + pc + 2, polT);
        // the remaining streams up front (addresses clamped inside the arrays; unused values discarded)
        const double em1 = L1T(E + pc - (i0 > 0 ? 1 : 0), polT);
        const double2 tpj = L2T(a.TP + pc + (j + 1 < nt ? nr : 0), polT);
        const double2 ej = L2T(E + pc - (j > 0 ? nr : 0), polT);
        const double2 ek = L2T(E + pcm, polT);
        const double2 tr1 = L2T(a.TR + pcp, polT);
        const double2 trj = L2T(a.TR + pc + (j + 1 < nt ? nr : 0), polT);
        // r-faces i0 (i0 >= 1) and i0 + 1
        double yr0 = 0.0, yr1;
        {
            const double2 sm = sm0;
            if (i0 >= 1) {
                yr0 = mul(sm.x, pr.x);
                yr0 = add(yr0, mul(g.A_r(i0, j, k), sub(em1, e.x)));
                double cc = sub(tt.x, tt1.x);
                if (j >= 1) cc = sub(cc, tp.x);
                if (j + 1 <= nt - 1) cc = add(cc, tpj.x);
                yr0 = add(yr0, mul(a.hr[i0], cc));
            }
            yr1 = mul(sm.y, pr.y);
            yr1 = add(yr1, mul(g.A_r(i0 + 1, j, k), sub(e.x, e.y)));
            double cc = sub(tt.y, tt1.y);
            if (j >= 1) cc = sub(cc, tp.y);
            if (j + 1 <= nt - 1) cc = add(cc, tpj.y);
            yr1 = add(yr1, mul(a.hr[i0 + 1], cc));
        }
        // theta-faces j (j >= 1)
        double yt0 = 0.0, yt1 = 0.0;
        if (j >= 1) {
            const double2 sm = sm1;
            yt0 = mul(sm.x, pt.x);
            yt0 = add(yt0, mul(g.A_t(i0, j, k), sub(ej.x, e.x)));
            double cc = sub(tr1.x, tr.x);
            cc = add(cc, tp.x);
            cc = sub(cc, tp.y);
            yt0 = add(yt0, mul(g.L_t(i0 + 1, j), cc));
            yt1 = mul(sm.y, pt.y);
            yt1 = add(yt1, mul(g.A_t(i0 + 1, j, k), sub(ej.y, e.y)));
            cc = sub(tr1.y, tr.y);
            cc = add(cc, tp.y);
            cc = sub(cc, tp2);
            yt1 = add(yt1, mul(g.L_t(i0 + 2, j), cc));
        }
        // phi-faces k
        double yp0, yp1;
        {
            const double2 sm = sm2;
            double2 lo, hi;
            if (j == 0) {
                lo.x = mul(__ldg(a.WN + i0), add(__ldg(a.ring + 2 * i0), __ldg(a.ring + 2 * i0 + 1)));
                lo.y = mul(__ldg(a.WN + i0 + 1), add(__ldg(a.ring + 2 * i0 + 2), __ldg(a.ring + 2 * i0 + 3)));
            } else {
                lo = tr;
            }
            if (j == nt - 1) {
                const double *rs = a.ring + 2 * (nr + i0);
                hi.x = mul(__ldg(a.WS + i0), -add(__ldg(rs), __ldg(rs + 1)));
                hi.y = mul(__ldg(a.WS + i0 + 1), -add(__ldg(rs + 2), __ldg(rs + 3)));
            } else {
                hi = trj;
            }
            yp0 = mul(sm.x, pp.x);
            yp0 = add(yp0, mul(g.A_p(i0, j), sub(ek.x, e.x)));
            double cc = sub(lo.x, hi.x);
            cc = sub(cc, tt.x);
            cc = add(cc, tt.y);
            yp0 = add(yp0, mul(g.L_p(i0 + 1, j, k), cc));
            yp1 = mul(sm.y, pp.y);
            yp1 = add(yp1, mul(g.A_p(i0 + 1, j), sub(ek.y, e.y)));
            cc = sub(lo.y, hi.y);
            cc = sub(cc, tt.y);
            cc = add(cc, tt2);
            yp1 = add(yp1, mul(g.L_p(i0 + 2, j, k), cc));
        }
        S2(y + UV(v, k, 0, j, i0), yr0, yr1);
        S2(y + UV(v, k, 1, j, i0), yt0, yt1);
        S2(y + UV(v, k, 2, j, i0), yp0, yp1);
        if (WITH_DOT) {
            dot[0].add(pr.x, yr0);
            dot[0].add(pt.x, yt0);
            dot[0].add(pp.x, yp0);
            dot[0].add(pr.y, yr1);
            dot[0].add(pt.y, yt1);
            dot[0].add(pp.y, yp1);
        }
    }
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kVVThreads, 1>(dot, base.partials, &base.sc->ticket[0], blockIdx.x, total, out)) {
            if (threadIdx.x == 0) {
                if (v.nchunks <= 1) {
                    base.sc->red1[0] = out[0].p;
                    base.sc->red1[1] = out[0].s;
                } else {
                    // chunked matvec: this chunk's pair into slot `chunk` of the fourth partial row; the last
                    // chunk combines all chunk pairs in chunk order (the earlier launches have completed)
                    double *cp = base.partials + 6 * kPartialSlots;
                    cp[v.chunk] = out[0].p;
                    cp[kPartialSlots + v.chunk] = out[0].s;
                    if (v.chunk == v.nchunks - 1) {
                        Acc<EXACT> acc;
                        for (int q = 0; q < v.nchunks; ++q) {
                            Acc<EXACT> o;
                            o.p = cp[q];
                            o.s = cp[kPartialSlots + q];
                            acc.add(o);
                        }
                        base.sc->red1[0] = acc.p;
                        base.sc->red1[1] = acc.s;
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------ setup of a solve (the oracle's rhs + PCG start)
template <bool EXACT>
__global__ void __launch_bounds__(kVVThreads) k_vv_setup_residual(VVDims v, VVArrays a, DevArrays base, Dims dv,
                                                                  const double *__restrict__ f, unsigned total) {
    const Geo g{a};
    Acc<EXACT> acc[3];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        for (int comp = 0; comp < 3; ++comp) {
            const size_t u = UV(v, k, comp, j, i);
            bool unknown = true;
            double M = 0.0;
            if (comp == 0) {
                unknown = i >= 1;
                if (unknown) M = mul(g.A_r(i, j, k), a.hr[i]);
            } else if (comp == 1) {
                unknown = j >= 1;
                if (unknown) M = mul(g.A_t(i, j, k), g.L_t(i + 1, j));
            } else {
                M = mul(g.A_p(i, j), g.L_p(i + 1, j, k));
            }
            const double b = unknown ? sub(mul(M, f[u]), a.bw[u]) : 0.0;
            const double r = sub(b, a.q[u]);
            const double z = __ddiv_rn(r, a.D[u]);
            a.r[u] = r;
            // p0 = z (padded; periodic copies on a single rank, as store_p of kernels.cu)
            a.p[u + dv.plane] = z;
            if (dv.periodic_local) {
                if (u < dv.plane) a.p[u + (size_t)(dv.nloc + 1) * dv.plane] = z;
                if (u >= (size_t)dv.n - dv.plane) a.p[u - (size_t)(dv.nloc - 1) * dv.plane] = z;
            }
            acc[0].add(r, z);
            acc[1].add(r, r);
            acc[2].add(b, b);
        }
    }
    Acc<EXACT> out[3];
    if (reduce_last<EXACT, kVVThreads, 3>(acc, base.partials, &base.sc->ticket[3], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            for (int t = 0; t < 3; ++t) {
                base.sc->red3[2 * t] = out[t].p;
                base.sc->red3[2 * t + 1] = out[t].s;
            }
        }
    }
}

__global__ void __launch_bounds__(kVVThreads) k_vv_mask(VVDims v, double *__restrict__ x) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        if (i == 0) x[UV(v, k, 0, j, i)] = 0.0;
        if (j == 0) x[UV(v, k, 1, j, i)] = 0.0;
    }
}

// all blocks resident at once (no partial last wave): SMs x the kernel's occupancy, at most one block per
// 256 work items
template <typename K>
unsigned resident_grid(K kern, uint32_t n, size_t smem = 0) {
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kVVThreads, smem);
        if (per_sm < 1) per_sm = 1;
    }
    uint64_t g = (n + kVVThreads - 1) / kVVThreads;
    const uint64_t cap = (uint64_t)sms * per_sm < (uint64_t)kRedBlocks ? (uint64_t)sms * per_sm : kRedBlocks;
    if (g > cap) g = cap;
    return g < 1 ? 1u : (unsigned)g;
}

// MASPCG_VV_STAGED=0 selects the register-only first phase (for comparisons)
inline bool vv_staged() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MASPCG_VV_STAGED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

inline unsigned vv_grid(uint32_t n) {
    uint64_t g = (n + kVVThreads - 1) / kVVThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)kRedBlocks) g = kRedBlocks;
    return (unsigned)g;
}

}  // namespace

void launch_vv_validate(const VVDims &v, const double *nu, const double *s, int *flag, cudaStream_t st) {
    k_vv_validate<<<vv_grid(v.ncell), kVVThreads, 0, st>>>(v, nu, s, flag);
}

void launch_vv_coef(const VVDims &v, const VVArrays &a, cudaStream_t st) {
    k_vv_coef<<<vv_grid(v.ncell), kVVThreads, 0, st>>>(v, a);
}

void launch_vv_ring(const VVDims &v, const VVArrays &a, int mode, bool exact, cudaStream_t st) {
    double *out = mode == 0 ? a.nuring : a.ring;
    if (exact) k_vv_ring<true><<<v.nr, kVVThreads, 0, st>>>(v, a, mode, a.p, out);
    else k_vv_ring<false><<<v.nr, kVVThreads, 0, st>>>(v, a, mode, a.p, out);
}

void launch_vv_axis_weights(const VVDims &v, const VVArrays &a, int np, cudaStream_t st) {
    k_vv_axis_weights<<<(v.nr + 127) / 128, 128, 0, st>>>(v, a, (double)np);
}

void launch_vv_diag(const VVDims &v, const VVArrays &a, cudaStream_t st) {
    k_vv_diag<<<vv_grid(v.ncell), kVVThreads, 0, st>>>(v, a);
}

// Opt-in (MASPCG_VV_CHUNK = ring planes, > 2): measured SLOWER than the one-pass two phases on c3v (1,491 vs
// 1,128 us per ring + matvec with the ring sized from 0.45 of the L2; 1,472-1,568 us for rings of 30-80
// planes): the terms did not stay in the L2 (ncu without cache control: the rows still read ~77 B/cell from
// DRAM, L2 hit rate 21 %) and the 32 launches per matvec lose ~20 % per chunk to ramp-up and tail
// (profiles/r02/vv_chunked_matvec.txt).  `bytes` is unused while the default is off.
uint32_t vv_ring_planes(const VVDims &v, size_t bytes) {
    (void)bytes;
    const char *e = getenv("MASPCG_VV_CHUNK");
    if (!e || atoi(e) <= 2 || (v.nr % 2)) return 0;
    const uint32_t r = (uint32_t)atoi(e);   // chunks of ring - 2 planes
    return (int)r - 2 < v.nloc ? r : 0;
}

size_t vv_ring_bytes(const VVDims &v, uint32_t ring) { return 4 * (size_t)v.plane1 * ring * sizeof(double); }

template <typename... KArgs, typename... Args>
void launch_pdl_vv(void (*kern)(KArgs...), unsigned grid, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kVVThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The chunked matvec: for chunks of K = ring - 2 planes, the terms of planes [kb - 1, ke] then the rows of
// [kb, ke); the two recomputed boundary planes per chunk cost 2/K of phase 1.
void launch_vv_chunked(const VVDims &v0, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                       bool exact, cudaStream_t st) {
    const int K = (int)v0.ring - 2;
    const int nch = (v0.nloc + K - 1) / K;
    const size_t sm = sizeof(double2) * 2 * kStg * kVVThreads;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_vv_terms3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = true;
    }
    for (int ch = 0; ch < nch; ++ch) {
        VVDims v = v0;
        v.kb = ch * K;
        v.ke = v.kb + K < v0.nloc ? v.kb + K : v0.nloc;
        v.chunk = ch;
        v.nchunks = nch;
        const uint32_t n1 = (uint32_t)(v.ke - v.kb + 2) * v.plane1;
        // every launch with programmatic dependent launch: the next chunk's blocks are resident while the
        // previous kernel drains (each kernel waits on griddepcontrol.wait before touching memory)
        launch_pdl_vv(k_vv_terms3<false>, resident_grid(k_vv_terms3<false>, n1 / 2, sm), sm, st, v, a, base,
                      loop ? 1 : 0);
        const uint32_t n2 = (uint32_t)(v.ke - v.kb) * v.plane1;
#define VRC(W, L, E)                                                                      \
    do {                                                                                  \
        const unsigned g = resident_grid(k_vv_rows2<W, L, E>, n2 / 2);                     \
        launch_pdl_vv(k_vv_rows2<W, L, E>, g, 0, st, v, a, base, y, g);                    \
    } while (0)
        if (!with_dot) VRC(false, false, true);
        else if (exact) {
            if (loop) VRC(true, true, true);
            else VRC(true, false, true);
        } else {
            if (loop) VRC(true, true, false);
            else VRC(true, false, false);
        }
#undef VRC
    }
}

void launch_vv_matvec(const VVDims &vin, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                      bool wall, bool exact, cudaStream_t st) {
    const bool pair0 = (vin.nr % 2 == 0) && (((uintptr_t)y & 15) == 0);
    if (pair0 && !wall && vin.ring && vv_staged()) {   // chunked: the terms of a chunk stay in the L2 rings
        launch_vv_chunked(vin, a, base, y, with_dot, loop, exact, st);
        return;
    }
    // one pass over the whole slab with full-size term arrays (also the wall-data operator of the setup)
    VVDims v = vin;
    v.kb = 0;
    v.ke = vin.nloc;
    v.ring = 0;
    v.chunk = 0;
    v.nchunks = 1;
    // default for the homogeneous operator: the plane-marching kernel with TMA-staged planes (vv_march.cu)
    if (!wall && launch_vv_march(v, a, base, y, with_dot, loop, exact, st)) return;
    const bool pair = pair0;
    const uint32_t nt1 = v.ncell + 2 * v.plane1;
    if (pair && vv_staged()) {
        const size_t sm = sizeof(double2) * 2 * kStg * kVVThreads;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_vv_terms3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaFuncSetAttribute(k_vv_terms3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            attr = true;
        }
        if (wall) k_vv_terms3<true><<<resident_grid(k_vv_terms3<true>, nt1 / 2, sm), kVVThreads, sm, st>>>(v, a, base, 0);
        else k_vv_terms3<false><<<resident_grid(k_vv_terms3<false>, nt1 / 2, sm), kVVThreads, sm, st>>>(v, a, base, loop ? 1 : 0);
    } else if (pair) {
        if (wall) k_vv_terms2<true><<<resident_grid(k_vv_terms2<true>, nt1 / 2), kVVThreads, 0, st>>>(v, a, base, 0);
        else k_vv_terms2<false><<<resident_grid(k_vv_terms2<false>, nt1 / 2), kVVThreads, 0, st>>>(v, a, base, loop ? 1 : 0);
    } else {
        const unsigned gt = vv_grid(nt1);
        if (wall) k_vv_terms<true><<<gt, kVVThreads, 0, st>>>(v, a, base, 0);
        else k_vv_terms<false><<<gt, kVVThreads, 0, st>>>(v, a, base, loop ? 1 : 0);
    }
#define VR(W, L, E)                                                                                   \
    do {                                                                                              \
        if (pair) {                                                                                   \
            const unsigned g = resident_grid(k_vv_rows2<W, L, E>, v.ncell / 2);                        \
            k_vv_rows2<W, L, E><<<g, kVVThreads, 0, st>>>(v, a, base, y, g);                          \
        } else {                                                                                      \
            const unsigned g = vv_grid(v.ncell);                                                      \
            k_vv_rows<W, L, E><<<g, kVVThreads, 0, st>>>(v, a, base, y, g);                           \
        }                                                                                             \
    } while (0)
    if (!with_dot) {
        VR(false, false, true);
    } else if (exact) {
        if (loop) VR(true, true, true);
        else VR(true, false, true);
    } else {
        if (loop) VR(true, true, false);
        else VR(true, false, false);
    }
#undef VR
}

void launch_vv_setup_residual(const VVDims &v, const VVArrays &a, const DevArrays &base, const Dims &dv,
                              const double *f, bool exact, cudaStream_t st) {
    const unsigned g = vv_grid(v.ncell);
    if (exact) k_vv_setup_residual<true><<<g, kVVThreads, 0, st>>>(v, a, base, dv, f, g);
    else k_vv_setup_residual<false><<<g, kVVThreads, 0, st>>>(v, a, base, dv, f, g);
}

void launch_vv_mask(const VVDims &v, double *x, cudaStream_t st) {
    k_vv_mask<<<vv_grid(v.ncell), kVVThreads, 0, st>>>(v, x);
}

}  // namespace maspcg
