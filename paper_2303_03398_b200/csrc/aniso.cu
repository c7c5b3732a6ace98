// aniso.cu -- sm_100a kernels of the field-aligned anisotropic conduction operator (
// reading R33 of DESIGN.md).  The operator: flux -K grad T, K = kappa_perp I + kappa_par b b^T, in the
// volume-weighted energy form -- the 7-point operator of the diagonal face coefficients K_aa (the
// caller's kr, kt, kp through the ordinary assembly) plus, on every edge between two interior faces of
// directions a and b, the cross term X_e (a_e.T)(b_e.T) of kappa_par b_a b_b (19-point stencil).  The
// thermal-conduction term of MAS's "full thermodynamic MHD model" (Sec. V-A) on its
// "non-uniform staggered spherical grid" (Sec. III); the paper gives no formula.
//
// Arithmetic (bitwise equal to the CPU oracle of R33): the edge weights with one IEEE rounding
// per operation in the order of the R33 formulas; per cell y = (D7 p - 7-point sum) + sum over the
// cell's 12 edges, in the fixed R33 order, of Xq (s_a db + s_b da), da and db the sums of the edge's
// two a- and b-differences.  Bandwidth: p (8, neighbours from L1/L2), T_r, T_theta, T_phi, D7 (32),
// Xrt, Xrp, Xtp (24), y (8) = 72 B/cell of algorithmic traffic per apply.
//
// Kernels: k_aniso_tma (default: p rows staged by 1-D bulk copies into double-buffered shared-memory tiles),
// k_aniso_vec2 (two cells per thread from global memory; the split boundary launch of a multi-rank stencil),
// k_aniso_flat (one cell per thread, odd nr), k_aniso_edges / k_aniso_diag (setup).
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "aniso.cuh"
#include "arith.cuh"
#include "common.cuh"
#include "loopdev.cuh"
#include "p2p_ll.cuh"

namespace maspcg {

namespace {

constexpr int kAnisoBlocks = 4;   // resident blocks of 256 threads per SM (<= 64 registers)


// ---------------------------------------------------------------- edge weights (setup)
__global__ void __launch_bounds__(kThreads) k_aniso_edges(Dims d, DevArrays a, AnisoArrays x,
                                                           const double *__restrict__ krt,
                                                           const double *__restrict__ krp,
                                                           const double *__restrict__ ktp) {
    int bad = 0;
    const int nr = d.nr, nt = d.nt;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        // r-theta edge (i, j) of plane k; the caller's krt row also holds the boundary edges i = nr, j = nt
        const size_t ert = ((size_t)k * (nt + 1) + j) * (nr + 1) + i;
        const double kq = krt[ert];
        bad |= !isfinite(kq);
        if (i == nr - 1) bad |= !isfinite(krt[ert + 1]);
        if (j == nt - 1) {
            bad |= !isfinite(krt[ert + nr + 1]);
            if (i == nr - 1) bad |= !isfinite(krt[ert + nr + 2]);
        }
        x.Xrt[c] = (i >= 1 && j >= 1)
                       ? __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(kq, x.gr[i]), x.gt[j]), a.dp[k]), 0.25)
                       : 0.0;
        // r-phi edge (i, row j) on face k+1/2 -> plane k+1
        const size_t erp = ((size_t)k * nt + j) * (nr + 1) + i;
        const double kp = krp[erp];
        bad |= !isfinite(kp);
        if (i == nr - 1) bad |= !isfinite(krp[erp + 1]);
        x.Xrp[(size_t)c + d.plane] = (i >= 1) ? __dmul_rn(__dmul_rn(__dmul_rn(kp, x.gr[i]), x.cs[j]), 0.25) : 0.0;
        // theta-phi edge (j, column i) on face k+1/2 -> plane k+1
        const size_t etp = ((size_t)k * (nt + 1) + j) * nr + i;
        const double kt = ktp[etp];
        bad |= !isfinite(kt);
        if (j == nt - 1) bad |= !isfinite(ktp[etp + nr]);
        x.Xtp[(size_t)c + d.plane] = (j >= 1) ? __dmul_rn(__dmul_rn(__dmul_rn(kt, x.qr[i]), x.gts[j]), 0.25) : 0.0;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && bad) atomicOr(&a.sc->vinvalid, 1);
}

// ---------------------------------------------------------------- Jacobi diagonal
// diag(A) = D7 + sum over the 12 edges (R33 order) of Xq (2 s_a s_b); 2 s_a s_b Xq is exact (+-2 Xq).
__global__ void __launch_bounds__(kThreads) k_aniso_diag(Dims d, DevArrays a, AnisoArrays x) {
    const int nr = d.nr, nt = d.nt;
    const size_t plane = d.plane;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        int i, j, k;
        decompose(d, c, i, j, k);
        double s = 0.0;
        auto add = [&](double X, bool plus) { s = __dadd_rn(s, plus ? __dmul_rn(X, 2.0) : __dmul_rn(X, -2.0)); };
        const size_t row = (size_t)j * nr;
        const size_t pk = (size_t)k * plane;
        // r-theta: (i, j) ++, (i+1, j) -+, (i, j+1) +-, (i+1, j+1) --
        if (i >= 1 && j >= 1) add(x.Xrt[pk + row + i], true);
        if (i + 1 <= nr - 1 && j >= 1) add(x.Xrt[pk + row + i + 1], false);
        if (i >= 1 && j + 1 <= nt - 1) add(x.Xrt[pk + row + nr + i], false);
        if (i + 1 <= nr - 1 && j + 1 <= nt - 1) add(x.Xrt[pk + row + nr + i + 1], true);
        // r-phi: (i, lo) ++, (i+1, lo) -+, (i, hi) +-, (i+1, hi) --
        const size_t lo = pk, hi = pk + plane;
        if (i >= 1) add(x.Xrp[lo + row + i], true);
        if (i + 1 <= nr - 1) add(x.Xrp[lo + row + i + 1], false);
        if (i >= 1) add(x.Xrp[hi + row + i], false);
        if (i + 1 <= nr - 1) add(x.Xrp[hi + row + i + 1], true);
        // theta-phi: (j, lo) ++, (j+1, lo) -+, (j, hi) +-, (j+1, hi) --
        if (j >= 1) add(x.Xtp[lo + row + i], true);
        if (j + 1 <= nt - 1) add(x.Xtp[lo + row + nr + i], false);
        if (j >= 1) add(x.Xtp[hi + row + i], false);
        if (j + 1 <= nt - 1) add(x.Xtp[hi + row + nr + i], true);
        const double d7 = a.D[c];
        x.D7[c] = d7;
        a.D[c] = __dadd_rn(d7, s);
    }
}

// ---------------------------------------------------------------- operator apply (one cell per thread)
template <bool EXACT>
struct Cross {
    double s = 0.0;
    // one edge: Xq (s_a db + s_b da), da = (a1 - a0) + (b1 - b0), db = (b0' ...) given as the four values of the
    // 2x2 block (u00 = lo a, lo b; u10 = hi a, lo b; u01 = lo a, hi b; u11 = hi a, hi b)
    __device__ __forceinline__ void edge(double X, double u00, double u10, double u01, double u11, bool sa_plus,
                                         bool sb_plus) {
        const double da = __dadd_rn(__dsub_rn(u10, u00), __dsub_rn(u11, u01));   // the two a-differences
        const double db = __dadd_rn(__dsub_rn(u01, u00), __dsub_rn(u11, u10));   // the two b-differences
        const double v = __dadd_rn(sa_plus ? db : -db, sb_plus ? da : -da);
        s = EXACT ? __dadd_rn(s, __dmul_rn(X, v)) : fma(X, v, s);
    }
};

template <bool WITH_DOT, bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kThreads, kAnisoBlocks) k_aniso_flat(Dims d, DevArrays a, AnisoArrays x,
                                                                       double *__restrict__ y, Range rg,
                                                                       unsigned red_slot0, unsigned red_total) {
    pdl_wait();
    pdl_trigger();
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (LOOP && a.peer_wait) acquire_p_halo(a);
    const bool coh = LOOP && a.peer_wait;   // peer-written halo planes: coherent loads (loopdev.cuh)
    using A = Ar<EXACT>;
    const double *__restrict__ p = a.p;
    const int nr = d.nr, nt = d.nt, nloc = d.nloc;
    const size_t plane = d.plane;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rg.vend; v += stride) {
        const uint32_t c = v + rg.off0 + (v >= rg.split ? rg.off1 : 0u);
        int i, j, k;
        decompose(d, c, i, j, k);
        // p of local plane kk (-1 .. nloc, halo planes included), row jj, column ii
        auto P = [&](int kk, int jj, int ii) -> double {
            const double *q = p + (size_t)(kk + 1) * plane + (size_t)jj * nr + ii;
            return (coh && (kk < 0 || kk >= nloc)) ? __ldcg(q) : __ldg(q);
        };
        const bool il = i > 0, ih = i < nr - 1, jl = j > 0, jh = j < nt - 1;
        const double pc = P(k, j, i);
        const double pim = il ? P(k, j, i - 1) : 0.0, pip = ih ? P(k, j, i + 1) : 0.0;
        const double pjm = jl ? P(k, j - 1, i) : 0.0, pjp = jh ? P(k, j + 1, i) : 0.0;
        const double pkm = P(k - 1, j, i), pkp = P(k + 1, j, i);
        // the 7-point part, the oracle's order (r_lo, r_hi, t_lo, t_hi, p_lo, p_hi; D7 p - sum)
        double s = 0.0;
        if (il) s = A::acc(s, __ldg(a.Tr + c), pim);
        if (ih) s = A::acc(s, __ldg(a.Tr + c + 1), pip);
        if (jl) s = A::acc(s, __ldg(a.Tt + c), pjm);
        if (jh) s = A::acc(s, __ldg(a.Tt + c + nr), pjp);
        s = A::acc(s, __ldg(a.Tp + c), pkm);
        s = A::acc(s, __ldg(a.Tp + c + plane), pkp);
        const double y7 = A::diag_minus(__ldg(x.D7 + c), pc, s);
        // the cross terms, R33 edge order
        Cross<EXACT> cr;
        const size_t pk = (size_t)k * plane, row = (size_t)j * nr;
        // r-theta edges of plane k: a = r, b = theta
        const double pjm_im = (jl && il) ? P(k, j - 1, i - 1) : 0.0, pjm_ip = (jl && ih) ? P(k, j - 1, i + 1) : 0.0;
        const double pjp_im = (jh && il) ? P(k, j + 1, i - 1) : 0.0, pjp_ip = (jh && ih) ? P(k, j + 1, i + 1) : 0.0;
        if (il && jl) cr.edge(__ldg(x.Xrt + pk + row + i), pjm_im, pjm, pim, pc, true, true);
        if (ih && jl) cr.edge(__ldg(x.Xrt + pk + row + i + 1), pjm, pjm_ip, pc, pip, false, true);
        if (il && jh) cr.edge(__ldg(x.Xrt + pk + row + nr + i), pim, pc, pjp_im, pjp, true, false);
        if (ih && jh) cr.edge(__ldg(x.Xrt + pk + row + nr + i + 1), pc, pip, pjp, pjp_ip, false, false);
        // r-phi edges of row j: a = r, b = phi; face k-1/2 (planes k-1, k: Xrp plane k), k+1/2 (k, k+1: plane k+1)
        const double pkm_im = il ? P(k - 1, j, i - 1) : 0.0, pkm_ip = ih ? P(k - 1, j, i + 1) : 0.0;
        const double pkp_im = il ? P(k + 1, j, i - 1) : 0.0, pkp_ip = ih ? P(k + 1, j, i + 1) : 0.0;
        if (il) cr.edge(__ldg(x.Xrp + pk + row + i), pkm_im, pkm, pim, pc, true, true);
        if (ih) cr.edge(__ldg(x.Xrp + pk + row + i + 1), pkm, pkm_ip, pc, pip, false, true);
        if (il) cr.edge(__ldg(x.Xrp + pk + plane + row + i), pim, pc, pkp_im, pkp, true, false);
        if (ih) cr.edge(__ldg(x.Xrp + pk + plane + row + i + 1), pc, pip, pkp, pkp_ip, false, false);
        // theta-phi edges of column i: a = theta, b = phi
        const double pkm_jm = jl ? P(k - 1, j - 1, i) : 0.0, pkm_jp = jh ? P(k - 1, j + 1, i) : 0.0;
        const double pkp_jm = jl ? P(k + 1, j - 1, i) : 0.0, pkp_jp = jh ? P(k + 1, j + 1, i) : 0.0;
        if (jl) cr.edge(__ldg(x.Xtp + pk + row + i), pkm_jm, pkm, pjm, pc, true, true);
        if (jh) cr.edge(__ldg(x.Xtp + pk + row + nr + i), pkm, pkm_jp, pc, pjp, false, true);
        if (jl) cr.edge(__ldg(x.Xtp + pk + plane + row + i), pjm, pc, pkp_jm, pkp, true, false);
        if (jh) cr.edge(__ldg(x.Xtp + pk + plane + row + nr + i), pc, pjp, pkp, pkp_jp, false, false);
        const double q = __dadd_rn(y7, cr.s);
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

// ---------------------------------------------------------------- operator apply, two cells per thread (nr even)
// The pair (i0, i0 + 1), i0 even: every stream is a 16-byte load, the pair's shared neighbours and the
// r-theta / r-phi edge between its two cells (face i0 + 1) are loaded and differenced once.  Each cell's
// cross terms are accumulated in the R33 edge order, with the same operations as the one-cell kernel, so
// the results are that kernel's (and the oracle's) bit for bit.
struct Row4 {   // p of one row at the pair's columns i0 - 1 (m, if i0 > 0), i0, i0 + 1, i0 + 2 (q, if i0 + 2 < nr)
    double m, c0, c1, q;
};

__device__ __forceinline__ double2 ldv2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ double2 ldv2c(const double *p, bool coherent) {
    return coherent ? __ldcg(reinterpret_cast<const double2 *>(p)) : __ldg(reinterpret_cast<const double2 *>(p));
}

template <bool EXACT>
__device__ __forceinline__ void xterm(double &s, double X, double da, double db, bool sa_plus, bool sb_plus) {
    const double v = __dadd_rn(sa_plus ? db : -db, sb_plus ? da : -da);
    s = EXACT ? __dadd_rn(s, __dmul_rn(X, v)) : fma(X, v, s);
}
// da (the two a-differences) and db (the two b-differences) of the 2x2 block u00 (lo a, lo b), u10 (hi a,
// lo b), u01 (lo a, hi b), u11 (hi a, hi b)
__device__ __forceinline__ void diffs(double u00, double u10, double u01, double u11, double &da, double &db) {
    da = __dadd_rn(__dsub_rn(u10, u00), __dsub_rn(u11, u01));
    db = __dadd_rn(__dsub_rn(u01, u00), __dsub_rn(u11, u10));
}

// The arithmetic of one pair (i0, i0 + 1) of plane k, row j, from its p values and coefficient streams: the
// 7-point part in the oracle's order, the cross terms in the R33 edge order, the store of y and the Dot2
// update.
// The pair's coefficient streams (T_r, T_theta, T_phi, D7, the three edge arrays): loaded unconditionally
// (clamped addresses), so the caller can issue them ahead of the p values.
struct PairCoef {
    double2 tr, ttl, tth, tpl, tph, d7, Xt0, Xt1, Xp0, Xp1, Xjl, Xjpl, Xjh, Xjph;
    double tr2, Xt0q, Xt1q, Xp0q, Xp1q;
};
__device__ __forceinline__ PairCoef load_coef(const Dims &d, const DevArrays &a, const AnisoArrays &x, uint32_t c,
                                              int i0, int j) {
    const int nr = d.nr, nt = d.nt;
    const size_t plane = d.plane;
    const size_t oq = (i0 + 2 < nr) ? 2 : 1, ojp = (j < nt - 1) ? nr : 0;
    const size_t e = c;   // (k, j, i0) in the [nloc][nt][nr] edge arrays
    PairCoef q;
    q.tr = ldv2(a.Tr + c);
    q.tr2 = __ldg(a.Tr + c + oq);
    q.ttl = ldv2(a.Tt + c), q.tth = ldv2(a.Tt + c + ojp);
    q.tpl = ldv2(a.Tp + c), q.tph = ldv2(a.Tp + c + plane);
    q.d7 = ldv2(x.D7 + c);
    q.Xt0 = ldv2(x.Xrt + e), q.Xt1 = ldv2(x.Xrt + e + ojp);
    q.Xt0q = __ldg(x.Xrt + e + oq), q.Xt1q = __ldg(x.Xrt + e + ojp + oq);
    q.Xp0 = ldv2(x.Xrp + e), q.Xp1 = ldv2(x.Xrp + e + plane);
    q.Xp0q = __ldg(x.Xrp + e + oq), q.Xp1q = __ldg(x.Xrp + e + plane + oq);
    q.Xjl = ldv2(x.Xtp + e), q.Xjpl = ldv2(x.Xtp + e + ojp);
    q.Xjh = ldv2(x.Xtp + e + plane), q.Xjph = ldv2(x.Xtp + e + plane + ojp);
    return q;
}

// Access to a pair's p values (the arithmetic below is written against these accessors).
__device__ __forceinline__ double g_m(const Row4 &r) { return r.m; }
__device__ __forceinline__ double g_c0(const Row4 &r) { return r.c0; }
__device__ __forceinline__ double g_c1(const Row4 &r) { return r.c1; }
__device__ __forceinline__ double g_q(const Row4 &r) { return r.q; }
__device__ __forceinline__ double g_x(const double2 &v) { return v.x; }
__device__ __forceinline__ double g_y(const double2 &v) { return v.y; }

template <bool WITH_DOT, bool EXACT, bool JIN = false, typename R4, typename R2>
__device__ __forceinline__ void aniso_pair(const Dims &d, const PairCoef &K, double *__restrict__ y, uint32_t c,
                                           int i0, int j, const R4 &Rj, const R4 &Rjm, const R4 &Rjp,
                                           const R4 &Mj, const R4 &Pj, const R2 &Mjm, const R2 &Mjp,
                                           const R2 &Pjm, const R2 &Pjp, Acc<EXACT> &dotacc) {
    using A = Ar<EXACT>;
    const int nr = d.nr, nt = d.nt;
    // JIN: the caller guarantees 0 < j < nt - 1 (a tile strictly between the poles)
    const bool il = i0 > 0, ih = i0 + 2 < nr, jl = JIN || j > 0, jh = JIN || j < nt - 1;
    // ---- the 7-point part, the oracle's order per cell
    const double2 tr = K.tr;
    const double tr2 = K.tr2;
    const double2 ttl = K.ttl, tth = K.tth;
    const double2 tpl = K.tpl, tph = K.tph;
    const double2 d7 = K.d7;
    double s0 = 0.0, s1 = 0.0;
    if (il) s0 = A::acc(s0, tr.x, g_m(Rj));
    s0 = A::acc(s0, tr.y, g_c1(Rj));
    if (jl) s0 = A::acc(s0, ttl.x, g_c0(Rjm));
    if (jh) s0 = A::acc(s0, tth.x, g_c0(Rjp));
    s0 = A::acc(s0, tpl.x, g_c0(Mj));
    s0 = A::acc(s0, tph.x, g_c0(Pj));
    const double y70 = A::diag_minus(d7.x, g_c0(Rj), s0);
    s1 = A::acc(s1, tr.y, g_c0(Rj));
    if (ih) s1 = A::acc(s1, tr2, g_q(Rj));
    if (jl) s1 = A::acc(s1, ttl.y, g_c1(Rjm));
    if (jh) s1 = A::acc(s1, tth.y, g_c1(Rjp));
    s1 = A::acc(s1, tpl.y, g_c1(Mj));
    s1 = A::acc(s1, tph.y, g_c1(Pj));
    const double y71 = A::diag_minus(d7.y, g_c1(Rj), s1);
    // ---- cross terms: x0 for cell i0, x1 for cell i0 + 1, each in the R33 edge order
    double x0 = 0.0, x1 = 0.0, da, db;
    // r-theta edges of plane k: je = j (rows j-1, j) and je = j + 1 (rows j, j+1); ie = i0, i0+1, i0+2
    const double2 Xt0 = K.Xt0, Xt1 = K.Xt1;
    const double Xt0q = K.Xt0q, Xt1q = K.Xt1q;
    const double2 Xp0 = K.Xp0, Xp1 = K.Xp1;
    const double Xp0q = K.Xp0q, Xp1q = K.Xp1q;
    const double2 Xjl = K.Xjl, Xjpl = K.Xjpl;
    const double2 Xjh = K.Xjh, Xjph = K.Xjph;
    if (jl) {
        const double2 X = Xt0;
        const double X2 = Xt0q;
        if (il) { diffs(g_m(Rjm), g_c0(Rjm), g_m(Rj), g_c0(Rj), da, db); xterm<EXACT>(x0, X.x, da, db, true, true); }
        diffs(g_c0(Rjm), g_c1(Rjm), g_c0(Rj), g_c1(Rj), da, db);
        xterm<EXACT>(x0, X.y, da, db, false, true);
        xterm<EXACT>(x1, X.y, da, db, true, true);
        if (ih) { diffs(g_c1(Rjm), g_q(Rjm), g_c1(Rj), g_q(Rj), da, db); xterm<EXACT>(x1, X2, da, db, false, true); }
    }
    if (jh) {
        const double2 X = Xt1;
        const double X2 = Xt1q;
        if (il) { diffs(g_m(Rj), g_c0(Rj), g_m(Rjp), g_c0(Rjp), da, db); xterm<EXACT>(x0, X.x, da, db, true, false); }
        diffs(g_c0(Rj), g_c1(Rj), g_c0(Rjp), g_c1(Rjp), da, db);
        xterm<EXACT>(x0, X.y, da, db, false, false);
        xterm<EXACT>(x1, X.y, da, db, true, false);
        if (ih) { diffs(g_c1(Rj), g_q(Rj), g_c1(Rjp), g_q(Rjp), da, db); xterm<EXACT>(x1, X2, da, db, false, false); }
    }
    // r-phi edges of row j: face k-1/2 (planes k-1, k; Xrp plane k) then k+1/2 (planes k, k+1; plane k+1)
    {
        const double2 X = Xp0;
        const double X2 = Xp0q;
        if (il) { diffs(g_m(Mj), g_c0(Mj), g_m(Rj), g_c0(Rj), da, db); xterm<EXACT>(x0, X.x, da, db, true, true); }
        diffs(g_c0(Mj), g_c1(Mj), g_c0(Rj), g_c1(Rj), da, db);
        xterm<EXACT>(x0, X.y, da, db, false, true);
        xterm<EXACT>(x1, X.y, da, db, true, true);
        if (ih) { diffs(g_c1(Mj), g_q(Mj), g_c1(Rj), g_q(Rj), da, db); xterm<EXACT>(x1, X2, da, db, false, true); }
    }
    {
        const double2 X = Xp1;
        const double X2 = Xp1q;
        if (il) { diffs(g_m(Rj), g_c0(Rj), g_m(Pj), g_c0(Pj), da, db); xterm<EXACT>(x0, X.x, da, db, true, false); }
        diffs(g_c0(Rj), g_c1(Rj), g_c0(Pj), g_c1(Pj), da, db);
        xterm<EXACT>(x0, X.y, da, db, false, false);
        xterm<EXACT>(x1, X.y, da, db, true, false);
        if (ih) { diffs(g_c1(Rj), g_q(Rj), g_c1(Pj), g_q(Pj), da, db); xterm<EXACT>(x1, X2, da, db, false, false); }
    }
    // theta-phi edges of each cell's column: (j, lo), (j+1, lo), (j, hi), (j+1, hi)
    {
        if (jl) {
            diffs(g_x(Mjm), g_c0(Mj), g_c0(Rjm), g_c0(Rj), da, db); xterm<EXACT>(x0, Xjl.x, da, db, true, true);
            diffs(g_y(Mjm), g_c1(Mj), g_c1(Rjm), g_c1(Rj), da, db); xterm<EXACT>(x1, Xjl.y, da, db, true, true);
        }
        if (jh) {
            diffs(g_c0(Mj), g_x(Mjp), g_c0(Rj), g_c0(Rjp), da, db); xterm<EXACT>(x0, Xjpl.x, da, db, false, true);
            diffs(g_c1(Mj), g_y(Mjp), g_c1(Rj), g_c1(Rjp), da, db); xterm<EXACT>(x1, Xjpl.y, da, db, false, true);
        }
        if (jl) {
            diffs(g_c0(Rjm), g_c0(Rj), g_x(Pjm), g_c0(Pj), da, db); xterm<EXACT>(x0, Xjh.x, da, db, true, false);
            diffs(g_c1(Rjm), g_c1(Rj), g_y(Pjm), g_c1(Pj), da, db); xterm<EXACT>(x1, Xjh.y, da, db, true, false);
        }
        if (jh) {
            diffs(g_c0(Rj), g_c0(Rjp), g_c0(Pj), g_x(Pjp), da, db); xterm<EXACT>(x0, Xjph.x, da, db, false, false);
            diffs(g_c1(Rj), g_c1(Rjp), g_c1(Pj), g_y(Pjp), da, db); xterm<EXACT>(x1, Xjph.y, da, db, false, false);
        }
    }
    const double q0 = __dadd_rn(y70, x0), q1 = __dadd_rn(y71, x1);
    *reinterpret_cast<double2 *>(y + c) = make_double2(q0, q1);
    if (WITH_DOT) {
        dotacc.add(g_c0(Rj), q0);
        dotacc.add(g_c1(Rj), q1);
    }
}

template <bool WITH_DOT, bool LOOP, bool EXACT, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_aniso_vec2(Dims d, DevArrays a, AnisoArrays x,
                                                            double *__restrict__ y, Range rg, unsigned red_slot0,
                                                            unsigned red_total) {
    pdl_wait();
    pdl_trigger();
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (LOOP && a.peer_wait) acquire_p_halo(a);
    const bool coh = LOOP && a.peer_wait;
    using A = Ar<EXACT>;
    const int nr = d.nr, nt = d.nt, nloc = d.nloc;
    const size_t plane = d.plane;
    Acc<EXACT> dot[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t npair = rg.vend >> 1;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < npair; v += stride) {
        const uint32_t v2 = 2u * v;
        const uint32_t c = v2 + rg.off0 + (v2 >= rg.split ? rg.off1 : 0u);
        int i0, j, k;
        decompose(d, c, i0, j, k);
        const bool il = i0 > 0, ih = i0 + 2 < nr, jl = j > 0, jh = j < nt - 1;
        const double *pk = a.p + plane + c;   // padded p at (plane k, row j, column i0)
        const bool cm = coh && k == 0, cp = coh && k == nloc - 1;   // halo planes written by the neighbours
        // Every load is unconditional (branch-free, so the compiler can issue them all ahead of their uses):
        // a neighbour that does not exist is replaced by an in-range address whose value is never used.
        const size_t om = il ? 1 : 0, oq = ih ? 2 : 1, ojm = jl ? nr : 0, ojp = jh ? nr : 0;
        auto row4 = [&](const double *q, bool coherent) {
            Row4 r;
            const double2 v = ldv2c(q, coherent);
            r.c0 = v.x, r.c1 = v.y;
            r.m = coherent ? __ldcg(q - om) : __ldg(q - om);
            r.q = coherent ? __ldcg(q + oq) : __ldg(q + oq);
            return r;
        };
        const Row4 Rj = row4(pk, false);
        const Row4 Rjm = row4(pk - ojm, false);
        const Row4 Rjp = row4(pk + ojp, false);
        const Row4 Mj = row4(pk - plane, cm);
        const Row4 Pj = row4(pk + plane, cp);
        const double2 Mjm = ldv2c(pk - plane - ojm, cm), Mjp = ldv2c(pk - plane + ojp, cm);
        const double2 Pjm = ldv2c(pk + plane - ojm, cp), Pjp = ldv2c(pk + plane + ojp, cp);
        const PairCoef K = load_coef(d, a, x, c, i0, j);
        aniso_pair<WITH_DOT, EXACT>(d, K, y, c, i0, j, Rj, Rjm, Rjp, Mj, Pj, Mjm, Mjp, Pjm, Pjp, dot[0]);
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

// ---------------------------------------------------------------- operator apply, TMA-staged tiles
// A block walks 256-pair chunks (512 consecutive cells: a few rows of one or two planes).  The p rows a chunk
// needs -- rows R0 - 1 .. R1 + 1 of planes k - 1, k, k + 1, three contiguous ranges of the padded p -- are
// brought into shared memory by three 1-D bulk copies (cp.async.bulk, the Tensor Memory Accelerator) issued
// by one thread and counted on an mbarrier, double-buffered: the copies of chunk n + 1 are in flight while
// chunk n is computed.  No per-element staging arithmetic, no global p loads in the compute; the coefficient
// streams are loaded per thread as in the pair kernel.
constexpr int kTilePairs = kThreads;

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init1(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
// p + off as one explicit 64-bit add (a bulk-copy source address; see fused.cu for the ptxas 12.9 issue)
__device__ __forceinline__ const double *gaddr64(const double *p, size_t off) {
    const double *r;
    asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(off * sizeof(double)));
    return r;
}

template <bool WITH_DOT, bool LOOP, bool EXACT, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_aniso_tma(Dims d, DevArrays a, AnisoArrays x, double *__restrict__ y,
                                                           Range rg, unsigned red_slot0, unsigned red_total,
                                                           int maxrows) {
    extern __shared__ __align__(128) double tiles[];   // [2 stages][3 planes][maxrows][nr]
    __shared__ __align__(8) uint64_t bars[2];
    pdl_wait();
    pdl_trigger();
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (LOOP && a.peer_wait) acquire_p_halo(a);   // before any copy of a (peer-written) halo plane
    const int nr = d.nr, nt = d.nt;
    const int rows_pad = (d.nloc + 2) * nt;         // rows of the padded p
    const uint32_t npair = rg.vend >> 1;            // a range without a split (full slab or interior planes)
    const uint32_t nch = (npair + kTilePairs - 1) / kTilePairs;
    const size_t stage = (size_t)3 * maxrows * nr;
    const double *const gp = a.p;
    if (threadIdx.x == 0) {
        mbar_init1(&bars[0]);
        mbar_init1(&bars[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the staged rows of chunk ch: Ra = R0 - 1 .. R1 + 1 (slab rows k nt + j)
    auto rows_of = [&](uint32_t ch, int &Ra, int &nrows) {
        const uint32_t v0 = ch * kTilePairs;
        const uint32_t v1 = v0 + kTilePairs < npair ? v0 + kTilePairs : npair;
        const int R0 = (int)d.div_r.div(2u * v0 + rg.off0);
        const int R1 = (int)d.div_r.div(2u * (v1 - 1) + 1u + rg.off0);
        Ra = R0 - 1;
        nrows = R1 - R0 + 3;
    };
    auto issue = [&](uint32_t ch, int st) {   // thread 0: three bulk copies into stage st
        int Ra, nrows;
        rows_of(ch, Ra, nrows);
        uint32_t bytes = 0;
        int lo[3], n[3];
        for (int pl = 0; pl < 3; ++pl) {
            int r0 = Ra + nt + (pl - 1) * nt, r1 = r0 + nrows;   // padded rows [r0, r1)
            lo[pl] = r0 < 0 ? -r0 : 0;                           // rows outside the padded array are never read
            r0 = r0 < 0 ? 0 : r0;
            r1 = r1 > rows_pad ? rows_pad : r1;
            n[pl] = r1 - r0;
            bytes += (uint32_t)(n[pl] * nr * sizeof(double));
        }
        mbar_expect(&bars[st], bytes);
        for (int pl = 0; pl < 3; ++pl) {
            const int r0 = Ra + nt + (pl - 1) * nt + lo[pl];
            double *dst = tiles + (size_t)st * stage + ((size_t)pl * maxrows + lo[pl]) * nr;
            bulk_copy(dst, gaddr64(gp, (size_t)r0 * nr), (uint32_t)(n[pl] * nr * sizeof(double)), &bars[st]);
        }
    };
    Acc<EXACT> dot[1];
    uint32_t use[2] = {0u, 0u};
    const uint32_t first = blockIdx.x;
    if (threadIdx.x == 0) {
        if (first < nch) issue(first, 0);
        if (first + gridDim.x < nch) issue(first + gridDim.x, 1);
    }
    int it = 0;
    for (uint32_t ch = first; ch < nch; ch += gridDim.x, ++it) {
        const int st = it & 1;
        const uint32_t v0 = ch * kTilePairs;
        const uint32_t v1 = v0 + kTilePairs < npair ? v0 + kTilePairs : npair;
        const uint32_t v = v0 + threadIdx.x;
        const bool mine = v < v1;
        const uint32_t c = 2u * (mine ? v : v0) + rg.off0;
        int i0, j, k;
        decompose(d, c, i0, j, k);
        int Ra, nrows;
        rows_of(ch, Ra, nrows);
        mbar_wait_parity(&bars[st], use[st] & 1u);
        ++use[st];
        if (mine) {
            // (loading the coefficients before the wait, or reading the tile lazily at each use, measured
            // slower: 625 vs 580-588 us per launch on c3a -- more registers live across the wait)
            const PairCoef K = load_coef(d, a, x, c, i0, j);
            const double *tb = tiles + (size_t)st * stage;
            const int lr = k * nt + j - Ra;   // 1 .. nrows - 2
            const int im = i0 > 0 ? i0 - 1 : i0, iq = i0 + 2 < nr ? i0 + 2 : i0 + 1;
            auto T = [&](int pl, int dr) -> const double * { return tb + ((size_t)pl * maxrows + lr + dr) * nr; };
            {
                auto row4 = [&](const double *r) {
                    const double2 v2 = *reinterpret_cast<const double2 *>(r + i0);
                    return Row4{r[im], v2.x, v2.y, r[iq]};
                };
                auto pr2 = [&](const double *r) { return *reinterpret_cast<const double2 *>(r + i0); };
                aniso_pair<WITH_DOT, EXACT>(d, K, y, c, i0, j, row4(T(1, 0)), row4(T(1, -1)), row4(T(1, 1)),
                                            row4(T(0, 0)), row4(T(2, 0)), pr2(T(0, -1)), pr2(T(0, 1)),
                                            pr2(T(2, -1)), pr2(T(2, 1)), dot[0]);
            }
        }
        __syncthreads();   // every thread is done with stage st
        if (threadIdx.x == 0 && ch + 2 * gridDim.x < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(ch + 2 * gridDim.x, st);
        }
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

// ---------------------------------------------------------------- operator apply, plane-marching (default)
// The same arithmetic (aniso_pair) with every operand staged by the Tensor Memory Accelerator: a block owns a
// theta-tile of tj rows x all nr radii and marches through a run of phi-planes.  Per plane it receives, by 1-D bulk
// copies counted on mbarriers, the p tile of plane s + 2 (rows j0 - 1 .. j0 + tj) into a 4-slot ring (planes
// s - 1, s, s + 1 read, s + 2 in flight) and the coefficient rows of step s + 1 into a 3-slot ring: T_r, T_theta,
// D7, X_rt of plane s + 1 and T_phi, X_rphi, X_thetaphi of the face above it (the face below is the previous
// step's); the threads read their pair's operands from shared memory (no global loads, no per-element index
// arithmetic), one block barrier per plane.  The pair kernels hold ~40 coefficient values in registers across a
// global-memory latency (latency-bound at 2 blocks per SM); here the bulk copies carry the memory parallelism.
constexpr int kAM = 512;   // threads per block (one block per SM)

struct AnisoMarch {
    int tj, njt;
    int k0, nk;           // planes [k0, k0 + nk) of the slab (Full: 0, nloc; Interior: 1, nloc - 2)
    uint32_t pslot;       // (tj + 2) rows of nr
    uint32_t cslot;       // (7 tj + 3) rows of nr: Tr [tj], Tt [tj+1], D7 [tj], Xrt [tj+1], Tp+ [tj], Xrp+ [tj], Xtp+ [tj+1]
    uint32_t units;       // njt * nk
};
inline size_t am_smem(const AnisoMarch &M) { return sizeof(double) * (4 * (size_t)M.pslot + 3 * (size_t)M.cslot); }

template <bool WITH_DOT, bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kAM, 1) k_aniso_march(Dims d, DevArrays a, AnisoArrays x, double *__restrict__ y,
                                                       AnisoMarch M, unsigned red_slot0, unsigned red_total) {
    extern __shared__ __align__(128) double amsm[];
    __shared__ __align__(8) uint64_t pbar[4], cbar[3];
    pdl_wait();
    pdl_trigger();
    if (LOOP && *(volatile int *)&a.sc->done) return;
    if (LOOP && a.peer_wait) acquire_p_halo(a);   // before any copy of a (peer-written) halo plane
    const int nr = d.nr, nt = d.nt, nh = nr >> 1, tj = M.tj;
    const size_t plane = d.plane;
    double *const pring = amsm;
    double *const cring = pring + 4 * (size_t)M.pslot;
    const uint32_t oTt = (uint32_t)tj * nr, oD7 = (uint32_t)(2 * tj + 1) * nr, oXrt = (uint32_t)(3 * tj + 1) * nr;
    const uint32_t oTp = (uint32_t)(4 * tj + 2) * nr, oXrp = (uint32_t)(5 * tj + 2) * nr, oXtp = (uint32_t)(6 * tj + 2) * nr;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) mbar_init1(&pbar[q]);
        for (int q = 0; q < 3; ++q) mbar_init1(&cbar[q]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int t = threadIdx.x;
    const bool member = t < tj * nh;
    const int lr = member ? t / nh : 0;
    const int i0 = member ? 2 * (t - lr * nh) : 0;
    const bool il = i0 > 0, ih = i0 + 2 < nr;
    const int om = il ? 1 : 0, oq = ih ? 2 : 1;
    Acc<EXACT> dot[1];
    const uint64_t u0 = (uint64_t)blockIdx.x * M.units / gridDim.x, u1 = (uint64_t)(blockIdx.x + 1) * M.units / gridDim.x;
    uint32_t pidx = 0, cidx = 0;   // running issue counts of the rings
    for (uint64_t u = u0; u < u1;) {
        const int jt = (int)(u / (uint32_t)M.nk);
        const int kb = M.k0 + (int)(u - (uint64_t)jt * M.nk);
        const int kend = M.k0 + M.nk;
        const int ke = (int)((uint64_t)kb + (u1 - u) < (uint64_t)kend ? kb + (u1 - u) : kend);
        u += (uint64_t)(ke - kb);
        const int j0 = jt * tj, j = j0 + lr;
        const bool act = member && j < nt;
        const bool jl = j > 0, jh = j < nt - 1;
        const int jlo = j0 - 1 > 0 ? j0 - 1 : 0;
        const int jhi1 = j0 + tj < nt - 1 ? j0 + tj : nt - 1;          // rows .. j0 + tj
        const int jhi0 = j0 + tj - 1 < nt - 1 ? j0 + tj - 1 : nt - 1;  // rows .. j0 + tj - 1
        // p plane k (-1 .. nloc) into ring slot idx % 4: rows jlo .. jhi1 to tile rows from j0 - 1
        auto issue_p = [&](int k, uint32_t idx) {
            const uint32_t q = idx & 3u, bytes = (uint32_t)(jhi1 - jlo + 1) * nr * 8u;
            mbar_expect(&pbar[q], bytes);
            bulk_copy(pring + (size_t)q * M.pslot + (size_t)(jlo - (j0 - 1)) * nr,
                      gaddr64(a.p, (size_t)(k + 1) * plane + (size_t)jlo * nr), bytes, &pbar[q]);
        };
        // coefficient stage of plane s (s = kb - 1: only the face above it, i.e. the faces of plane kb)
        auto issue_c = [&](int s, uint32_t idx) {
            const uint32_t q = idx % 3u;
            double *cs = cring + (size_t)q * M.cslot;
            const uint32_t b0 = (uint32_t)(jhi0 - j0 + 1) * nr * 8u, b1 = (uint32_t)(jhi1 - j0 + 1) * nr * 8u;
            const bool full = s >= kb;
            mbar_expect(&cbar[q], (full ? 2 * b0 + 2 * b1 : 0u) + 2 * b0 + b1);
            const size_t pu = (size_t)(s + 1) * plane + (size_t)j0 * nr;         // the face above plane s
            const size_t ps = full ? pu - plane : 0;                              // plane s (s >= kb >= 0)
            if (full) {
                bulk_copy(cs, gaddr64(a.Tr, ps), b0, &cbar[q]);
                bulk_copy(cs + oTt, gaddr64(a.Tt, ps), b1, &cbar[q]);
                bulk_copy(cs + oD7, gaddr64(x.D7, ps), b0, &cbar[q]);
                bulk_copy(cs + oXrt, gaddr64(x.Xrt, ps), b1, &cbar[q]);
            }
            bulk_copy(cs + oTp, gaddr64(a.Tp, pu), b0, &cbar[q]);
            bulk_copy(cs + oXrp, gaddr64(x.Xrp, pu), b0, &cbar[q]);
            bulk_copy(cs + oXtp, gaddr64(x.Xtp, pu), b1, &cbar[q]);
        };
        // ring index of p plane k: pb + k - (kb - 1) (planes kb - 1 .. ke); of stage s: cb + s - (kb - 1) (kb - 1 .. ke - 1)
        const uint32_t pb = pidx, cb = cidx;
        pidx += (uint32_t)(ke - kb + 2);
        cidx += (uint32_t)(ke - kb + 1);
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_p(kb - 1, pb);
            issue_p(kb, pb + 1);
            issue_p(kb + 1, pb + 2);
            issue_c(kb - 1, cb);
            issue_c(kb, cb + 1);
        }
        {   // the first step's older operands: planes kb - 1, kb and the faces of plane kb
            const uint32_t i1 = pb, i2 = pb + 1;
            mbar_wait_parity(&pbar[i1 & 3u], (i1 >> 2) & 1u);
            mbar_wait_parity(&pbar[i2 & 3u], (i2 >> 2) & 1u);
            mbar_wait_parity(&cbar[cb % 3u], (cb / 3u) & 1u);
        }
        // the own row's p of planes s - 1 and s, carried from step to step (plane s + 1 is the only new row4)
        Row4 Mj{0.0, 0.0, 0.0, 0.0}, Rj{0.0, 0.0, 0.0, 0.0};
        // and the coefficients of the face below plane s (the previous step's face above): T_phi, X_rphi, X_thetaphi
        double2 cTp = make_double2(0.0, 0.0), cXp = cTp, cXj = cTp, cXjp = cTp;
        double cXpq = 0.0;
        double2 Mjm2 = make_double2(0.0, 0.0), Mjp2 = Mjm2;   // plane s - 1, rows j -+ 1 (the previous step's)
        // the step loop, compiled for interior tiles (every row strictly between the poles: no j-boundary
        // predicates in aniso_pair) and generic for the first and last tiles
        auto march = [&](auto interior) {
            constexpr bool JIN = decltype(interior)::value;
            for (int s = kb; s < ke; ++s) {
                const uint32_t q = (uint32_t)(s - (kb - 1));
                if (threadIdx.x == 0) {   // into the slots of plane s - 2 and stage s - 2 (free: barrier of step s - 1)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (s + 2 <= ke) issue_p(s + 2, pb + q + 2);
                    if (s + 1 <= ke - 1) issue_c(s + 1, cb + q + 1);
                }
                const uint32_t ip = pb + q + 1, ic = cb + q;   // plane s + 1, stage s
                mbar_wait_parity(&pbar[ip & 3u], (ip >> 2) & 1u);
                mbar_wait_parity(&cbar[ic % 3u], (ic / 3u) & 1u);
                if (act) {
                    const double *Pm = pring + (size_t)((ip - 2) & 3u) * M.pslot;   // plane s - 1
                    const double *P0 = pring + (size_t)((ip - 1) & 3u) * M.pslot;   // plane s
                    const double *P1 = pring + (size_t)(ip & 3u) * M.pslot;         // plane s + 1
                    const double *C = cring + (size_t)(ic % 3u) * M.cslot;           // stage s
                    const double *Cb = cring + (size_t)((ic + 2) % 3u) * M.cslot;    // stage s - 1: the faces of plane s
                    const int r = lr + 1;                                            // tile row of j
                    const int rm = (JIN || jl) ? r - 1 : r, rp = (JIN || jh) ? r + 1 : r;
                    auto row4 = [&](const double *P, int rr) {
                        const double *w = P + (size_t)rr * nr + i0;
                        const double2 v2 = *reinterpret_cast<const double2 *>(w);
                        return Row4{w[-om], v2.x, v2.y, w[oq]};
                    };
                    auto pr2 = [&](const double *P, int rr) { return *reinterpret_cast<const double2 *>(P + (size_t)rr * nr + i0); };
                    const uint32_t o0 = (uint32_t)lr * nr + i0, o1 = (uint32_t)((JIN || jh) ? lr + 1 : lr) * nr + i0;
                    auto c2 = [&](const double *base, uint32_t off) { return *reinterpret_cast<const double2 *>(base + off); };
                    PairCoef K;
                    K.tr = c2(C, o0);
                    K.tr2 = C[o0 + oq];
                    K.ttl = c2(C + oTt, o0);
                    K.tth = c2(C + oTt, o1);
                    if (s == kb) {
                        cTp = c2(Cb + oTp, o0);
                        cXp = c2(Cb + oXrp, o0);
                        cXpq = Cb[oXrp + o0 + oq];
                        cXj = c2(Cb + oXtp, o0);
                        cXjp = c2(Cb + oXtp, o1);
                    }
                    K.tpl = cTp;
                    K.tph = c2(C + oTp, o0);
                    K.d7 = c2(C + oD7, o0);
                    K.Xt0 = c2(C + oXrt, o0);
                    K.Xt1 = c2(C + oXrt, o1);
                    K.Xt0q = C[oXrt + o0 + oq];
                    K.Xt1q = C[oXrt + o1 + oq];
                    K.Xp0 = cXp;
                    K.Xp1 = c2(C + oXrp, o0);
                    K.Xp0q = cXpq;
                    K.Xp1q = C[oXrp + o0 + oq];
                    K.Xjl = cXj;
                    K.Xjpl = cXjp;
                    K.Xjh = c2(C + oXtp, o0);
                    K.Xjph = c2(C + oXtp, o1);
                    const uint32_t c = (uint32_t)((size_t)s * plane + (size_t)j * nr + i0);
                    if (s == kb) {
                        Mj = row4(Pm, r);
                        Rj = row4(P0, r);
                        Mjm2 = pr2(Pm, rm);
                        Mjp2 = pr2(Pm, rp);
                    }
                    const Row4 Pj = row4(P1, r), Rjm = row4(P0, rm), Rjp = row4(P0, rp);
                    aniso_pair<WITH_DOT, EXACT, JIN>(d, K, y, c, i0, j, Rj, Rjm, Rjp, Mj, Pj, Mjm2, Mjp2, pr2(P1, rm),
                                                pr2(P1, rp), dot[0]);
                    Mjm2 = make_double2(Rjm.c0, Rjm.c1);
                    Mjp2 = make_double2(Rjp.c0, Rjp.c1);
                    Mj = Rj;
                    Rj = Pj;
                    cTp = K.tph;
                    cXp = K.Xp1;
                    cXpq = K.Xp1q;
                    cXj = K.Xjh;
                    cXjp = K.Xjph;
                }
                __syncthreads();
            }
        };
        if (j0 >= 1 && j0 + tj <= nt - 1) march(std::true_type{});
        else march(std::false_type{});
    }
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kAM, 1>(dot, a.partials, &a.sc->ticket[0], red_slot0 + blockIdx.x, red_total, out)) {
            if (threadIdx.x == 0) {
                a.sc->red1[0] = out[0].p;
                a.sc->red1[1] = out[0].s;
                if (a.p2p_ll) ll_push_pairs(a, a.sc->red1, 1);   // to every rank (peer communicator)
            }
        }
    }
}

inline int tile_rows(int nr) { return (2 * kTilePairs + nr - 1) / nr + 3; }
inline size_t tile_smem(int nr) { return sizeof(double) * 2 * 3 * (size_t)tile_rows(nr) * nr; }

inline unsigned grid_aniso(uint32_t n) {
    uint64_t g = (n + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * kAnisoBlocks)) g = 148 * kAnisoBlocks;
    return (unsigned)g;
}

// blocks per SM of the pair kernel: 2 (default, 128 registers, no spills) or 3 (MASPCG_ANISO_BLOCKS=3:
// 85 registers with spills)
inline int aniso2_blocks() {
    static const int b = getenv("MASPCG_ANISO_BLOCKS") ? atoi(getenv("MASPCG_ANISO_BLOCKS")) : 2;
    return b == 3 ? 3 : 2;
}

inline unsigned grid_aniso2(uint32_t n) {   // two cells per thread, a resident grid
    uint64_t g = (n / 2 + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * aniso2_blocks())) g = 148 * aniso2_blocks();
    return (unsigned)g;
}

// the pair kernel: nr even (pairs never straddle a row) and y 16-byte aligned (MASPCG_OPT_VEC)
inline bool aniso_vec2(const Dims &d, const double *y) {
    return d.vec_ok && (d.nr % 2 == 0) && (((uintptr_t)y & 15) == 0);
}

inline unsigned grid_setup(uint32_t n) {
    uint64_t g = (n + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)kRedBlocks) g = kRedBlocks;
    return (unsigned)g;
}

template <typename... KArgs, typename... Args>
void launch_pdl_aniso_smem(bool pdl, void (*kern)(KArgs...), unsigned grid, size_t smem, cudaStream_t st,
                           Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
void launch_pdl_aniso(bool pdl, void (*kern)(KArgs...), unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace

void launch_aniso_edges(const Dims &d, const DevArrays &a, const AnisoArrays &x, const double *krt, const double *krp,
                        const double *ktp, cudaStream_t st) {
    k_aniso_edges<<<grid_setup(d.n), kThreads, 0, st>>>(d, a, x, krt, krp, ktp);
}

void launch_aniso_diag(const Dims &d, const DevArrays &a, const AnisoArrays &x, cudaStream_t st) {
    k_aniso_diag<<<grid_setup(d.n), kThreads, 0, st>>>(d, a, x);
}

// the TMA tile kernel: pair layout and a range without a split (MASPCG_ANISO_TMA=0 selects the all-global
// pair kernel for comparisons)
inline bool aniso_tma(const Dims &d, const double *y, const Range &rg) {
    static const int on = getenv("MASPCG_ANISO_TMA") ? atoi(getenv("MASPCG_ANISO_TMA")) : 1;
    return on && aniso_vec2(d, y) && rg.split == 0xffffffffu;
}

// resident blocks per SM of the TMA kernel: 2 (default, 128 registers) or MASPCG_ANISO_TMA_BLOCKS = 3 (80
// registers with spills; measured slower, 882-897 vs 575-584 us; reading the tile lazily at each use instead
// of copying a pair's p values to registers measured 615 us at 2 blocks, 734 at 3 -- removed)
inline int tma_blocks() {
    static const int b = getenv("MASPCG_ANISO_TMA_BLOCKS") ? atoi(getenv("MASPCG_ANISO_TMA_BLOCKS")) : 2;
    return b == 3 ? 3 : 2;
}

inline unsigned grid_tma(uint32_t n) {   // n cells: 256-pair chunks, a resident grid
    uint64_t g = ((uint64_t)n / 2 + kTilePairs - 1) / kTilePairs;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * tma_blocks())) g = 148 * tma_blocks();
    return (unsigned)g;
}

// the plane-marching kernel (default; MASPCG_ANISO_MARCH=0 disables it, MASPCG_ANISO_MARCH_TJ / _GRID force
// smaller tiles / grids for the tests): the pair layout, the full slab or its interior planes
inline bool aniso_march(const Dims &d, const double *y, StencilPart part, AnisoMarch &M) {
    const char *e = getenv("MASPCG_ANISO_MARCH");
    if ((e && e[0] == '0') || !aniso_vec2(d, y) || part == StencilPart::Boundary) return false;
    M.k0 = part == StencilPart::Full ? 0 : 1;
    M.nk = part == StencilPart::Full ? d.nloc : d.nloc - 2;
    if (M.nk < 1 || d.nr < 2) return false;
    int tj = kAM / (d.nr / 2);
    if (tj > d.nt) tj = d.nt;
    const char *f = getenv("MASPCG_ANISO_MARCH_TJ");
    if (f && atoi(f) > 0 && atoi(f) < tj) tj = atoi(f);
    for (; tj >= 1; --tj) {
        M.tj = tj;
        M.pslot = (uint32_t)(tj + 2) * d.nr;
        M.cslot = (uint32_t)(7 * tj + 3) * d.nr;
        if (am_smem(M) <= 220u * 1024u) break;
    }
    if (tj < 1) return false;
    M.njt = (d.nt + tj - 1) / tj;
    M.units = (uint32_t)M.njt * (uint32_t)M.nk;
    return true;
}

inline unsigned grid_march(const AnisoMarch &M) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t g = (uint32_t)sms;
    const char *f = getenv("MASPCG_ANISO_MARCH_GRID");
    if (f && atoi(f) > 0) g = (uint32_t)atoi(f);
    if (g > M.units) g = M.units;
    if (g > (uint32_t)kRedBlocks) g = kRedBlocks;
    return g < 1 ? 1u : g;
}

unsigned aniso_stencil_blocks(const Dims &d, StencilPart part, const double *y) {
    const Range rg = make_range(d, part);
    if (!rg.vend) return 0u;
    AnisoMarch M;
    if (aniso_march(d, y, part, M)) return grid_march(M);
    if (aniso_tma(d, y, rg)) return grid_tma(rg.vend);
    return aniso_vec2(d, y) ? grid_aniso2(rg.vend) : grid_aniso(rg.vend);
}

void launch_aniso_matvec(const Dims &d, const DevArrays &a, const AnisoArrays &x, double *y, StencilPart part,
                         bool with_dot, bool loop, unsigned red_slot0, unsigned red_total, bool exact, cudaStream_t st) {
    const Range rg = make_range(d, part);
    if (rg.vend == 0) return;
    const bool pdl = d.pdl != 0;
    AnisoMarch M;
    if (aniso_march(d, y, part, M)) {
        const unsigned g = grid_march(M);
        const size_t sm = am_smem(M);
#define AM(W, L, E)                                                                                           \
    do {                                                                                                      \
        cudaFuncSetAttribute(k_aniso_march<W, L, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        cudaLaunchConfig_t cfg{};                                                                             \
        cfg.gridDim = dim3(g);                                                                                \
        cfg.blockDim = dim3(kAM);                                                                             \
        cfg.dynamicSmemBytes = sm;                                                                            \
        cfg.stream = st;                                                                                      \
        cudaLaunchAttribute attr[1];                                                                          \
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                      \
        attr[0].val.programmaticStreamSerializationAllowed = 1;                                               \
        cfg.attrs = attr;                                                                                     \
        cfg.numAttrs = pdl ? 1 : 0;                                                                           \
        cudaLaunchKernelEx(&cfg, k_aniso_march<W, L, E>, d, a, x, y, M, red_slot0, red_total);                \
    } while (0)
        if (exact) {
            if (with_dot) {
                if (loop) AM(true, true, true);
                else AM(true, false, true);
            } else AM(false, false, true);
        } else {
            if (with_dot) {
                if (loop) AM(true, true, false);
                else AM(true, false, false);
            } else AM(false, false, false);
        }
#undef AM
        return;
    }
    if (aniso_tma(d, y, rg)) {
        const unsigned g = grid_tma(rg.vend);
        const size_t sm = tile_smem(d.nr);
        const int mr = tile_rows(d.nr);
#define TM(W, L, E)                                                                                           \
    do {                                                                                                      \
        if (tma_blocks() == 2) {                                                                      \
            cudaFuncSetAttribute(k_aniso_tma<W, L, E, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
            launch_pdl_aniso_smem(pdl, k_aniso_tma<W, L, E, 2>, g, sm, st, d, a, x, y, rg, red_slot0, red_total, mr); \
        } else {                                                                                             \
            cudaFuncSetAttribute(k_aniso_tma<W, L, E, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
            launch_pdl_aniso_smem(pdl, k_aniso_tma<W, L, E, 3>, g, sm, st, d, a, x, y, rg, red_slot0, red_total, mr); \
        }                                                                                                    \
    } while (0)
        if (exact) {
            if (with_dot) {
                if (loop) TM(true, true, true);
                else TM(true, false, true);
            } else TM(false, false, true);
        } else {
            if (with_dot) {
                if (loop) TM(true, true, false);
                else TM(true, false, false);
            } else TM(false, false, false);
        }
#undef TM
        return;
    }
    const bool vec = aniso_vec2(d, y);
    const unsigned g = vec ? grid_aniso2(rg.vend) : grid_aniso(rg.vend);
#define AN(W, L, E)                                                                                      \
    do {                                                                                                 \
        if (vec && aniso2_blocks() == 3)                                                                 \
            launch_pdl_aniso(pdl, k_aniso_vec2<W, L, E, 3>, g, st, d, a, x, y, rg, red_slot0, red_total);   \
        else if (vec) launch_pdl_aniso(pdl, k_aniso_vec2<W, L, E, 2>, g, st, d, a, x, y, rg, red_slot0, red_total); \
        else launch_pdl_aniso(pdl, k_aniso_flat<W, L, E>, g, st, d, a, x, y, rg, red_slot0, red_total);     \
    } while (0)
    if (exact) {
        if (with_dot) {
            if (loop) AN(true, true, true);
            else AN(true, false, true);
        } else AN(false, false, true);
    } else {
        if (with_dot) {
            if (loop) AN(true, true, false);
            else AN(true, false, false);
        } else AN(false, false, false);
    }
#undef AN
}

}  // namespace maspcg
