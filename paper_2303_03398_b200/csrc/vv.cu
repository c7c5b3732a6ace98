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
    // e = wc * delta of cell (i, j, k), k in [-1, nloc-1]
    __device__ __forceinline__ double ediv(int i, int j, int k) const {
        const double fr_lo = mul(g.A_r(i, j, k), vr(k, j, i));
        const double fr_hi = mul(g.A_r(i + 1, j, k), vr(k, j, i + 1));
        const double ft_lo = (j == 0) ? 0.0 : mul(g.A_t(i, j, k), P(k, 1, j, i));
        const double ft_hi = (j == v.nt - 1) ? 0.0 : mul(g.A_t(i, j + 1, k), P(k, 1, j + 1, i));
        const double ap = g.A_p(i, j);
        const double fp_lo = mul(ap, P(k, 2, j, i));
        const double fp_hi = mul(ap, P(k + 1, 2, j, i));
        double d = add(sub(fr_hi, fr_lo), sub(ft_hi, ft_lo));
        d = add(d, sub(fp_hi, fp_lo));
        return mul(__ldg(a.wc + PC(v, k, j, i)), d);
    }
    // r-edge at theta-face j (1..nt-1), phi-face k (k in [0, nloc])
    __device__ __forceinline__ double Gr(int i, int j, int k) const {
        const double gp_a = mul(g.L_p(i + 1, j, k), P(k, 2, j, i));
        const double gp_b = mul(g.L_p(i + 1, j - 1, k), P(k, 2, j - 1, i));
        const double lt = g.L_t(i + 1, j);
        const double gt_a = mul(lt, P(k, 1, j, i));
        const double gt_b = mul(lt, P(k - 1, 1, j, i));
        return sub(sub(gp_a, gp_b), sub(gt_a, gt_b));
    }
    // theta-edge at r-face e (0..nr), phi-face k (k in [0, nloc])
    __device__ __forceinline__ double Gt(int e, int j, int k) const {
        const double gr_a = mul(a.hr[e], vr(k, j, e));
        const double gr_b = mul(a.hr[e], vr(k - 1, j, e));
        const double up = (e < v.nr) ? P(k, 2, j, e) : go(k, 2, j);
        const double dn = (e > 0) ? P(k, 2, j, e - 1) : gi(k, 2, j);
        const double gp_a = mul(g.L_p(e + 1, j, k), up);
        const double gp_b = mul(g.L_p(e, j, k), dn);
        return sub(sub(gr_a, gr_b), sub(gp_a, gp_b));
    }
    // phi-edge at r-face e (0..nr), theta-face j (1..nt-1)
    __device__ __forceinline__ double Gp(int e, int j, int k) const {
        const double up = (e < v.nr) ? P(k, 1, j, e) : go(k, 1, j);
        const double dn = (e > 0) ? P(k, 1, j, e - 1) : gi(k, 1, j);
        const double gt_a = mul(g.L_t(e + 1, j), up);
        const double gt_b = mul(g.L_t(e, j), dn);
        const double gr_a = mul(a.hr[e], vr(k, j, e));
        const double gr_b = mul(a.hr[e], vr(k, j - 1, e));
        return sub(sub(gt_a, gt_b), sub(gr_a, gr_b));
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

// ------------------------------------------------------------ the operator (the oracle's apply)
template <bool WITH_DOT, bool LOOP, bool WALL, bool EXACT>
__global__ void __launch_bounds__(kVVThreads) k_vv_matvec(VVDims v, VVArrays a, DevArrays base, double *__restrict__ y,
                                                          unsigned total) {
    if (LOOP && *(volatile int *)&base.sc->done) return;
    const Field<WALL> F{v, a, a.p, Geo{a}};
    const Geo &g = F.g;
    // the polar-axis circulations of this radius are read per cell from the ring pairs
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < v.ncell; c += stride) {
        int i, j, k;
        cell_of(v, c, i, j, k);
        const double e0 = F.ediv(i, j, k);
        // r-face i
        double yr = 0.0;
        const double pr = F.P(k, 0, j, i);
        if (i >= 1) {
            yr = mul(__ldg(a.sM + UV(v, k, 0, j, i)), pr);
            yr = add(yr, mul(g.A_r(i, j, k), sub(F.ediv(i - 1, j, k), e0)));
            double cc = mul(Wt_at(v, a, i, j, k), F.Gt(i, j, k));
            cc = sub(cc, mul(Wt_at(v, a, i, j, k + 1), F.Gt(i, j, k + 1)));
            if (j >= 1) cc = sub(cc, mul(Wp_at(v, a, i, j, k), F.Gp(i, j, k)));
            if (j + 1 <= v.nt - 1) cc = add(cc, mul(Wp_at(v, a, i, j + 1, k), F.Gp(i, j + 1, k)));
            yr = add(yr, mul(a.hr[i], cc));
        }
        // theta-face j
        double yt = 0.0;
        const double pt = F.P(k, 1, j, i);
        if (j >= 1) {
            yt = mul(__ldg(a.sM + UV(v, k, 1, j, i)), pt);
            yt = add(yt, mul(g.A_t(i, j, k), sub(F.ediv(i, j - 1, k), e0)));
            double cc = sub(mul(__ldg(a.Wr + PC(v, k + 1, j, i)), F.Gr(i, j, k + 1)),
                            mul(__ldg(a.Wr + PC(v, k, j, i)), F.Gr(i, j, k)));
            cc = add(cc, mul(Wp_at(v, a, i, j, k), F.Gp(i, j, k)));
            cc = sub(cc, mul(Wp_at(v, a, i + 1, j, k), F.Gp(i + 1, j, k)));
            yt = add(yt, mul(g.L_t(i + 1, j), cc));
        }
        // phi-face k
        const double pp = F.P(k, 2, j, i);
        double yp = mul(__ldg(a.sM + UV(v, k, 2, j, i)), pp);
        yp = add(yp, mul(g.A_p(i, j), sub(F.ediv(i, j, k - 1), e0)));
        double lo, hi;
        if (j == 0) lo = mul(__ldg(a.WN + i), add(__ldg(a.ring + 2 * i), __ldg(a.ring + 2 * i + 1)));
        else lo = mul(__ldg(a.Wr + PC(v, k, j, i)), F.Gr(i, j, k));
        if (j == v.nt - 1)
            hi = mul(__ldg(a.WS + i), -add(__ldg(a.ring + 2 * (v.nr + i)), __ldg(a.ring + 2 * (v.nr + i) + 1)));
        else hi = mul(__ldg(a.Wr + PC(v, k, j + 1, i)), F.Gr(i, j + 1, k));
        double cc = sub(lo, hi);
        cc = sub(cc, mul(Wt_at(v, a, i, j, k), F.Gt(i, j, k)));
        cc = add(cc, mul(Wt_at(v, a, i + 1, j, k), F.Gt(i + 1, j, k)));
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

void launch_vv_matvec(const VVDims &v, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                      bool wall, bool exact, cudaStream_t st) {
    const unsigned g = vv_grid(v.ncell);
#define VM(W, L, WL, E) k_vv_matvec<W, L, WL, E><<<g, kVVThreads, 0, st>>>(v, a, base, y, g)
    if (wall) {
        VM(false, false, true, true);
    } else if (!with_dot) {
        VM(false, false, false, true);
    } else if (exact) {
        if (loop) VM(true, true, false, true);
        else VM(true, false, false, true);
    } else {
        if (loop) VM(true, true, false, false);
        else VM(true, false, false, false);
    }
#undef VM
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
