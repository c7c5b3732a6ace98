// vv_march.cu -- the staggered vector viscosity operator (R27-R31, 10b) as
// ONE plane-marching kernel per matvec, its input planes staged by the Tensor Memory Accelerator.
//
// Why: the two-phase form (vv.cu: k_vv_terms3 + k_vv_rows2) writes the outflow and edge terms of every cell
// to HBM and reads them back -- 184 B/cell against the 104 B/cell of the operator's own streams (p 24, wc,
// W_r, W_theta, W_phi 32, sM 24 in; q 24 out), so it cannot pass 104/184 = 0.57 of its bound.  Here the
// terms never leave the SM.
//
// Shape of the kernel (one block of kMT threads per SM, persistent):
//  * work unit = (theta-tile of tj rows x all nr radii, one phi-plane); a block owns a contiguous run of
//    units (ordered tile-major), i.e. one or two "segments" = (tile, planes [kb, ke)), and marches through
//    each segment plane by plane: step s forms the terms of plane s (e = wc delta, tau_theta, tau_r,
//    tau_phi = W Gamma of the cell's lower edges) and the three rows of plane s - 1.
//  * thread = one r-pair (i0, i0 + 1) of one tile row, FIXED for the whole segment, so the products of the
//    1-D metric factors that do not depend on phi (rf2[i] C[j], sinf[j] dR2[i], dR2[i] dt[j], rce[e] ht[j],
//    rce[e] sinc[j]) are formed once (13 in registers, the six used once per step in a per-thread shared
//    table: the kernel then fits 128 registers without spills); per plane only the phi factors dp(k), hm(k)
//    (a shared table of the slab's planes) multiply in -- each product associated exactly as vv.cu's Geo forms
//    it, so every term and row is bit-identical to the oracle's.  Rows j0 - 1 (lower halo: e only) and j0 + tj
//    (upper halo: tau_r, tau_phi only) are computed by extra threads of the block.
//  * inputs: the p tile of a plane (3 components x rows j0-1 .. j0+tj, one contiguous range per component)
//    in a 3-slot ring (plane s + 2 in flight while planes s, s + 1 are read) and the coefficient rows of a
//    step (wc, W_r, W_theta, W_phi of plane s, sM of plane s - 1) in a 2-slot ring -- every one a 1-D bulk
//    copy (cp.async.bulk, UBLKCP) issued by one thread right after the step's barrier and counted on the
//    slot's mbarrier.  No per-element staging arithmetic; the memory-level parallelism comes from the bulk
//    copies, not from resident warps.
//  * terms: the neighbours' e, tau (i - 1, i + 1, j - 1, j + 1 of the same plane) through a double-buffered
//    shared tile [tj + 2][nr + 2] per term (slot nr: the outer-wall edge of the last radial cell); the own p of
//    plane s - 1 and tau_theta(s), tau_r(s) in registers, e(s - 2) read before e(s) overwrites it.  One block
//    barrier per plane (a hardware barrier: waiting warps issue nothing -- mbarrier-based split barriers with
//    spinning or sleeping waiters measured slower).
//  * Dot2 partial of p.q per thread, combined by the last block (reduce_last) as every matvec kernel.
// Homogeneous operator only (the loop's; the wall-data operator of the setup uses the two phases), nr even.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "arith.cuh"
#include "common.cuh"
#include "vv.cuh"

namespace maspcg {

namespace {

constexpr int kMT = 512;   // threads per block
constexpr int kMaxTR2 = 64;   // tile rows incl. the two halo rows

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk(double *dst, const double *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}
// base + off as one explicit 64-bit add (a bulk-copy source; see fused.cu for the ptxas 12.9 issue)
__device__ __forceinline__ const double *g64(const double *p, size_t off) {
    const double *r;
    asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(off * sizeof(double)));
    return r;
}
__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void st2(double *p, double x, double y) { *reinterpret_cast<double2 *>(p) = make_double2(x, y); }

}  // namespace

// Shared-memory layout (in doubles), computed on the host
struct MarchLayout {
    int tj, njt;            // theta rows per tile, tiles
    uint32_t pslot;         // one p slot: [3 comps][tj + 2 rows][nr]
    uint32_t cslot;         // one coefficient slot: wc [tj+1], Wr [tj+1], Wp [tj+1], Wt [tj], sM [3][tj] rows of nr
    uint32_t nphi;          // dp, hm of the slab's planes -1 .. nloc: 2 (nloc + 2)
    uint32_t tbuf;          // one term buffer: E, TT, TR, TP, each [tj + 2][nr + 2] (two buffers)
    uint32_t units;         // njt * nloc
};

inline size_t march_smem_bytes(const MarchLayout &L) {
    return sizeof(double) * (3 * (size_t)L.pslot + 2 * (size_t)L.cslot + 2 * (size_t)L.tbuf + L.nphi);
}

namespace {

// PROBE: the timing-probe build (tools/vv_march_probe.py), whose `dbg` bits switch parts off -- 1 arithmetic,
// 2 bulk copies, 4 block barrier, 8 rows, 16 terms, 32 everything; its results are wrong.  The product build
// (PROBE = false) compiles the switches out.
template <bool WITH_DOT, bool LOOP, bool EXACT, bool PROBE>
__global__ void __launch_bounds__(kMT, 1) k_vv_march(VVDims v, VVArrays a, DevArrays base, double *__restrict__ y,
                                                    MarchLayout L, unsigned total, int dbg_) {
    const int dbg = PROBE ? dbg_ : 0;
    if (LOOP && *(volatile int *)&base.sc->done) return;
    if (dbg & 32) return;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t pbar[3], cbar[2];   // p ring, coefficient ring
    __shared__ double2 cst[3][kMT];                       // per-thread metric products (see below)
    const int nr = v.nr, nt = v.nt, nh = nr >> 1, tj = L.tj, RL = nr + 2, TR2 = tj + 2;
    double *const pring = sm;
    double *const cring = pring + 3 * (size_t)L.pslot;
    double *const tb0 = cring + 2 * (size_t)L.cslot;
    double *const phi = tb0 + 2 * (size_t)L.tbuf;   // dp(k), hm(k) of planes -1 .. nloc (2 (nloc + 2))
    for (int q = threadIdx.x; q < v.nloc + 2; q += blockDim.x) {
        phi[2 * q] = a.dpp[q];
        phi[2 * q + 1] = a.hmp[q];
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < 3; ++q) mbar_init(&pbar[q], 1);
        for (int q = 0; q < 2; ++q) mbar_init(&cbar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // this thread's place in a tile: row lr (0 = lower halo j0 - 1, 1 .. tj own rows, tj + 1 upper halo), pair
    const int t = threadIdx.x;
    const bool member = t < TR2 * nh;
    const int lr = member ? t / nh : 0;
    const int i0 = member ? 2 * (t - lr * nh) : 0;
    const bool last = (i0 + 2 == nr);
    const int role = !member ? 0 : (lr == 0 ? 1 : (lr == tj + 1 ? 3 : 2));   // 1 low halo, 2 own, 3 up halo

    Acc<EXACT> dot[1];
    const uint64_t u0 = (uint64_t)blockIdx.x * L.units / gridDim.x, u1 = (uint64_t)(blockIdx.x + 1) * L.units / gridDim.x;
    uint32_t pidx = 0, cidx = 0;   // running issue counts of the two rings (slot = idx % n, parity = (idx / n) & 1)
    for (uint64_t u = u0; u < u1;) {
        const int jt = (int)(u / (uint32_t)v.nloc), kb = (int)(u - (uint64_t)jt * v.nloc);
        const int ke = (int)((uint64_t)kb + (u1 - u) < (uint64_t)v.nloc ? kb + (u1 - u) : v.nloc);
        u += (uint64_t)(ke - kb);
        const int j0 = jt * tj;
        const int j = j0 - 1 + lr;
        const bool act = role != 0 && j >= 0 && j < nt;
        // ---- the r-pair's metric products for row j (phi-independent; Geo's association)
        // ((atU0, atU1), (lpm0, lpm1), (arC2, lt0), one use each per step, live in shared memory: registers bind)
        double arC0 = 0, arC1 = 0, atS0 = 0, atS1 = 0, ap0 = 0, ap1 = 0;
        double lt1 = 0, lt2 = 0, lpc0 = 0, lpc1 = 0, lpc2 = 0, hr0 = 0, hr1 = 0;
        if (act) {
            const double Cj = a.C[j], sfj = a.sinf[j], sfu = a.sinf[j + 1], dtj = a.dt[j], htj = a.ht[j], scj = a.sinc[j];
            const double scm = j >= 1 ? a.sinc[j - 1] : 0.0;
            const double d0 = a.dR2[i0], d1 = a.dR2[i0 + 1];
            arC0 = mul(a.rf2[i0], Cj);
            arC1 = mul(a.rf2[i0 + 1], Cj);
            const double arC2 = mul(a.rf2[i0 + 2], Cj);
            atS0 = mul(sfj, d0);
            atS1 = mul(sfj, d1);
            cst[0][t] = make_double2(mul(sfu, d0), mul(sfu, d1));   // atU0, atU1
            ap0 = mul(d0, dtj);
            ap1 = mul(d1, dtj);
            const double c0 = a.rce[i0], c1 = a.rce[i0 + 1], c2 = a.rce[i0 + 2];
            cst[2][t] = make_double2(arC2, mul(c0, htj));            // arC2, lt0
            lt1 = mul(c1, htj);
            lt2 = mul(c2, htj);
            lpc0 = mul(c0, scj);
            lpc1 = mul(c1, scj);
            lpc2 = mul(c2, scj);
            cst[1][t] = make_double2(mul(c1, scm), mul(c2, scm));   // lpm0, lpm1
            hr0 = a.hr[i0];
            hr1 = a.hr[i0 + 1];
        }
        // ---- the bulk copies of a p plane and of a step's coefficient rows (thread 0)
        const int jlo = j0 - 1 > 0 ? j0 - 1 : 0;
        const int jhi_p = j0 + tj < nt - 1 ? j0 + tj : nt - 1;       // p, Wr, Wp rows .. j0 + tj
        const int jhi_o = j0 + tj - 1 < nt - 1 ? j0 + tj - 1 : nt - 1;   // wc, Wt, sM rows .. j0 + tj - 1
        auto issue_p = [&](int k, uint32_t idx) {
            const uint32_t q = idx % 3;
            double *dst = pring + (size_t)q * L.pslot;
            const uint32_t rows = (uint32_t)(jhi_p - jlo + 1), bytes = rows * nr * 8u;
            mbar_expect(&pbar[q], 3 * bytes);
            for (int c = 0; c < 3; ++c)
                bulk(dst + ((size_t)c * TR2 + (jlo - (j0 - 1))) * nr,
                     g64(a.p, ((size_t)(k + 1) * 3 + c) * v.plane1 + (size_t)jlo * nr), bytes, &pbar[q]);
        };
        auto issue_c = [&](int s, uint32_t idx) {
            const uint32_t q = idx & 1;
            double *cw = cring + (size_t)q * L.cslot;
            double *cr = cw + (size_t)(tj + 1) * nr, *cp = cr + (size_t)(tj + 1) * nr, *ct = cp + (size_t)(tj + 1) * nr;
            double *cs = ct + (size_t)tj * nr;
            const uint32_t bo = (uint32_t)(jhi_o - jlo + 1) * nr * 8u;         // wc rows jlo .. jhi_o
            const uint32_t bu = (uint32_t)(jhi_p - j0 + 1) * nr * 8u;          // Wr, Wp rows j0 .. jhi_p
            const uint32_t bt = (uint32_t)(jhi_o - j0 + 1) * nr * 8u;          // Wt, sM rows j0 .. jhi_o
            const bool e = s <= ke - 1, tt = s >= kb, tp = s >= kb && s <= ke - 1, rw = s - 1 >= kb;
            mbar_expect(&cbar[q], (e ? bo : 0u) + (tt ? bu + bt : 0u) + (tp ? bu : 0u) + (rw ? 3 * bt : 0u));
            const size_t pc = (size_t)(s + 1) * v.plane1;   // padded plane s
            if (e) bulk(cw + (size_t)(jlo - (j0 - 1)) * nr, g64(a.wc, pc + (size_t)jlo * nr), bo, &cbar[q]);
            if (tt) {
                bulk(cr, g64(a.Wr, pc + (size_t)j0 * nr), bu, &cbar[q]);
                bulk(ct, g64(a.Wt, pc + (size_t)j0 * nr), bt, &cbar[q]);
            }
            if (tp) bulk(cp, g64(a.Wp, (size_t)s * v.plane1 + (size_t)j0 * nr), bu, &cbar[q]);
            if (rw)
                for (int c = 0; c < 3; ++c)
                    bulk(cs + (size_t)c * tj * nr, g64(a.sM, ((size_t)(s - 1) * 3 + c) * v.plane1 + (size_t)j0 * nr), bt,
                         &cbar[q]);
        };
        // ring index of plane k: pb + k - (kb - 1); of step s: cb + s - (kb - 1)
        const uint32_t pb = pidx, cb = cidx;
        pidx += (uint32_t)(ke - kb + 2);   // planes kb - 1 .. ke, steps kb - 1 .. ke
        cidx += (uint32_t)(ke - kb + 2);
        if (t == 0 && !(dbg & 2)) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_p(kb - 1, pb);
            issue_p(kb, pb + 1);
            issue_c(kb - 1, cb);
        }
        double2 Rm = make_double2(0.0, 0.0), Tm = Rm, Pm = Rm;   // own p of plane s - 1
        // The step loop, specialised for interior tiles (every row of the tile and its halo rows strictly between
        // the poles: no pole / boundary-row predicates) and generic for the first and last tiles
        auto march = [&](auto interior) {
            constexpr bool IN = decltype(interior)::value;
            const bool ACT = IN ? member : act;
            for (int s = kb - 1; s <= ke; ++s) {
                const int q = s - (kb - 1);
                if (t == 0 && !(dbg & 2)) {   // into the slots of plane s - 1 and step s - 1 (free: the barrier of step s - 1)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (s + 2 <= ke) issue_p(s + 2, pb + (uint32_t)q + 2);
                    if (s + 1 <= ke) issue_c(s + 1, cb + (uint32_t)q + 1);
                }
                const bool e_on = s <= ke - 1;
                // the outer-wall edge weights of this step (last pair only), loaded ahead of the waits
                double wto = 0.0, wpo = 0.0;
                if (ACT && last && s >= kb) {
                    if (role == 2) wto = __ldg(a.WtO + (size_t)(s + 1) * nt + j);
                    if (e_on && (IN || j >= 1)) wpo = __ldg(a.WpO + (size_t)s * nt + j);
                }
                const uint32_t ps = pb + (uint32_t)q, ps1 = ps + 1, cs_ = cb + (uint32_t)q;
                const double *P0 = pring + (size_t)(ps % 3) * L.pslot;    // plane s
                const double *P1 = pring + (size_t)(ps1 % 3) * L.pslot;   // plane s + 1
                const double *Cw = cring + (size_t)(cs_ & 1) * L.cslot;
                const double *Cr = Cw + (size_t)(tj + 1) * nr, *Cp = Cr + (size_t)(tj + 1) * nr, *Ct = Cp + (size_t)(tj + 1) * nr;
                const double *Cs = Ct + (size_t)tj * nr;
                double *TBn = tb0 + (size_t)(s & 1) * L.tbuf;         // terms of plane s (still e of plane s - 2)
                const double *TBo = tb0 + (size_t)((s - 1) & 1) * L.tbuf;   // terms of plane s - 1
                const size_t TA = (size_t)TR2 * RL;                    // one term array
                if (!(dbg & 2)) {
                    mbar_wait(&pbar[ps % 3], (ps / 3) & 1u);
                    if (e_on) mbar_wait(&pbar[ps1 % 3], (ps1 / 3) & 1u);
                    mbar_wait(&cbar[cs_ & 1], (cs_ >> 1) & 1u);
                }
                if (ACT && !(dbg & 1)) {
                    const double dps = phi[2 * (s + 1)], hms = phi[2 * (s + 1) + 1];
                    auto PT = [&](const double *P, int c, int r) { return P + ((size_t)c * TR2 + r) * nr; };
                    const double2 R = ld2(PT(P0, 0, lr) + i0), T = ld2(PT(P0, 1, lr) + i0), Pp = ld2(PT(P0, 2, lr) + i0);
                    const double vr0 = i0 == 0 ? 0.0 : R.x;
                    const size_t o = (size_t)lr * RL + i0;
                    // -- e(s): rows j0 - 1 .. j0 + tj - 1 (stored after the rows have read e(s - 2) from the same slot)
                    double e0 = 0.0, e1 = 0.0;
                    if (role <= 2 && e_on && !(dbg & 16)) {
                        const double2 Tj1 = ld2(PT(P0, 1, lr + 1) + i0), Pk1 = ld2(PT(P1, 2, lr) + i0);
                        const double vr2 = last ? 0.0 : PT(P0, 0, lr)[i0 + 2];
                        const double2 wc = ld2(Cw + (size_t)lr * nr + i0);
                        const double2 aU = cst[0][t];
                        const double A0 = mul(arC0, dps), A1 = mul(arC1, dps), A2 = mul(cst[2][t].x, dps);
                        {
                            const double fr_lo = mul(A0, vr0), fr_hi = mul(A1, R.y);
                            const double ft_lo = (!IN && j == 0) ? 0.0 : mul(mul(atS0, dps), T.x);
                            const double ft_hi = (!IN && j == nt - 1) ? 0.0 : mul(mul(aU.x, dps), Tj1.x);
                            const double fp_lo = mul(ap0, Pp.x), fp_hi = mul(ap0, Pk1.x);
                            double d = add(sub(fr_hi, fr_lo), sub(ft_hi, ft_lo));
                            d = add(d, sub(fp_hi, fp_lo));
                            e0 = mul(wc.x, d);
                        }
                        {
                            const double fr_lo = mul(A1, R.y), fr_hi = mul(A2, vr2);
                            const double ft_lo = (!IN && j == 0) ? 0.0 : mul(mul(atS1, dps), T.y);
                            const double ft_hi = (!IN && j == nt - 1) ? 0.0 : mul(mul(aU.y, dps), Tj1.y);
                            const double fp_lo = mul(ap1, Pp.y), fp_hi = mul(ap1, Pk1.y);
                            double d = add(sub(fr_hi, fr_lo), sub(ft_hi, ft_lo));
                            d = add(d, sub(fp_hi, fp_lo));
                            e1 = mul(wc.y, d);
                        }
                    }
                    // -- tau_theta(s) (own rows), tau_r(s) (own + upper halo), tau_phi(s) (own + upper halo)
                    double tt0 = 0.0, tt1 = 0.0, tr0 = 0.0, tr1 = 0.0;
                    if (role >= 2 && s >= kb && !(dbg & 16)) {
                        const double hm = hms;
                        const double Lp0 = mul(lpc0, hm), Lp1 = mul(lpc1, hm), Lp2 = mul(lpc2, hm);
                        const size_t co = (size_t)(lr - 1) * nr + i0;
                        if (role == 2) {
                            const double pm1 = i0 == 0 ? 0.0 : PT(P0, 2, lr)[i0 - 1];
                            const double2 wt = ld2(Ct + co);
                            {
                                const double vrkm = i0 == 0 ? 0.0 : Rm.x;
                                const double gr_a = mul(hr0, vr0), gr_b = mul(hr0, vrkm);
                                const double gp_a = mul(Lp1, Pp.x), gp_b = mul(Lp0, pm1);
                                tt0 = mul(wt.x, sub(sub(gr_a, gr_b), sub(gp_a, gp_b)));
                            }
                            {
                                const double gr_a = mul(hr1, R.y), gr_b = mul(hr1, Rm.y);
                                const double gp_a = mul(Lp2, Pp.y), gp_b = mul(Lp1, Pp.x);
                                tt1 = mul(wt.y, sub(sub(gr_a, gr_b), sub(gp_a, gp_b)));
                            }
                            double *TT = TBn + TA + o;
                            st2(TT, tt0, tt1);
                            if (last) {   // the outer-wall theta-edge (r-face nr): Gt(nr) with zero wall data
                                const double hrn = a.hr[nr];
                                const double Lpn1 = mul(mul(a.rce[nr + 1], a.sinc[j]), hm);
                                const double gt = sub(sub(mul(hrn, 0.0), mul(hrn, 0.0)), sub(mul(Lpn1, 0.0), mul(Lp2, Pp.y)));
                                TT[2] = mul(wto, gt);
                            }
                        }
                        if (IN || j >= 1) {
                            const double2 Pjm = ld2(PT(P0, 2, lr - 1) + i0), lpm = cst[1][t];
                            const double2 wr = ld2(Cr + co);
                            {
                                const double gp_a = mul(Lp1, Pp.x), gp_b = mul(mul(lpm.x, hm), Pjm.x);
                                tr0 = mul(wr.x, sub(sub(gp_a, gp_b), sub(mul(lt1, T.x), mul(lt1, Tm.x))));
                            }
                            {
                                const double gp_a = mul(Lp2, Pp.y), gp_b = mul(mul(lpm.y, hm), Pjm.y);
                                tr1 = mul(wr.y, sub(sub(gp_a, gp_b), sub(mul(lt2, T.y), mul(lt2, Tm.y))));
                            }
                        }
                        st2(TBn + 2 * TA + o, tr0, tr1);
                        if (e_on) {   // tau_phi(s), planes kb .. ke - 1
                            double tp0 = 0.0, tp1 = 0.0, tpw = 0.0;
                            if (IN || j >= 1) {
                                const double2 Rjm = ld2(PT(P0, 0, lr - 1) + i0);
                                const double tm1 = i0 == 0 ? 0.0 : PT(P0, 1, lr)[i0 - 1];
                                const double2 wp = ld2(Cp + co);
                                {
                                    const double vrjm = i0 == 0 ? 0.0 : Rjm.x;
                                    const double gt_a = mul(lt1, T.x), gt_b = mul(cst[2][t].y, tm1);
                                    const double gr_a = mul(hr0, vr0), gr_b = mul(hr0, vrjm);
                                    tp0 = mul(wp.x, sub(sub(gt_a, gt_b), sub(gr_a, gr_b)));
                                }
                                {
                                    const double gt_a = mul(lt2, T.y), gt_b = mul(lt1, T.x);
                                    const double gr_a = mul(hr1, R.y), gr_b = mul(hr1, Rjm.y);
                                    tp1 = mul(wp.y, sub(sub(gt_a, gt_b), sub(gr_a, gr_b)));
                                }
                                if (last) {   // the outer-wall phi-edge: Gp(nr) with zero wall data
                                    const double hrn = a.hr[nr];
                                    const double Ltn1 = mul(a.rce[nr + 1], a.ht[j]);
                                    const double gt = sub(sub(mul(Ltn1, 0.0), mul(lt2, T.y)), sub(mul(hrn, 0.0), mul(hrn, 0.0)));
                                    tpw = mul(wpo, gt);
                                }
                            }
                            double *TP = TBn + 3 * TA + o;
                            st2(TP, tp0, tp1);
                            if (last) TP[2] = tpw;
                        }
                    }
                    // -- the rows of plane k = s - 1 (own rows)
                    if (role == 2 && s - 1 >= kb && !(dbg & 8)) {
                        const int k = s - 1;
                        const double dpk = phi[2 * (k + 1)], hmk = phi[2 * (k + 1) + 1];
                        const double *Eo = TBo + o, *TTo = TBo + TA + o, *TRo = TBo + 2 * TA + o, *TPo = TBo + 3 * TA + o;
                        const double2 e = ld2(Eo), tt = ld2(TTo), tr = ld2(TRo), tp = ld2(TPo);
                        const double2 ek = ld2(TBn + o);   // own e(k - 1): written at step s - 2, not yet overwritten
                        const double tt2 = TTo[2], tp2 = TPo[2];
                        const size_t so = (size_t)(lr - 1) * nr + i0;
                        const double2 sm0 = ld2(Cs + so), sm1 = ld2(Cs + (size_t)tj * nr + so), sm2 = ld2(Cs + 2 * (size_t)tj * nr + so);
                        double yr0 = 0.0, yr1;
                        {
                            const double2 tpj = (IN || j + 1 <= nt - 1) ? ld2(TPo + RL) : make_double2(0.0, 0.0);
                            if (i0 >= 1) {
                                yr0 = mul(sm0.x, Rm.x);
                                yr0 = add(yr0, mul(mul(arC0, dpk), sub(Eo[-1], e.x)));
                                double cc = sub(tt.x, tt0);
                                if (IN || j >= 1) cc = sub(cc, tp.x);
                                if (IN || j + 1 <= nt - 1) cc = add(cc, tpj.x);
                                yr0 = add(yr0, mul(hr0, cc));
                            }
                            yr1 = mul(sm0.y, Rm.y);
                            yr1 = add(yr1, mul(mul(arC1, dpk), sub(e.x, e.y)));
                            double cc = sub(tt.y, tt1);
                            if (IN || j >= 1) cc = sub(cc, tp.y);
                            if (IN || j + 1 <= nt - 1) cc = add(cc, tpj.y);
                            yr1 = add(yr1, mul(hr1, cc));
                        }
                        double yt0 = 0.0, yt1 = 0.0;
                        if (IN || j >= 1) {
                            const double2 ej = ld2(Eo - RL);
                            yt0 = mul(sm1.x, Tm.x);
                            yt0 = add(yt0, mul(mul(atS0, dpk), sub(ej.x, e.x)));
                            double cc = sub(tr0, tr.x);
                            cc = add(cc, tp.x);
                            cc = sub(cc, tp.y);
                            yt0 = add(yt0, mul(lt1, cc));
                            yt1 = mul(sm1.y, Tm.y);
                            yt1 = add(yt1, mul(mul(atS1, dpk), sub(ej.y, e.y)));
                            cc = sub(tr1, tr.y);
                            cc = add(cc, tp.y);
                            cc = sub(cc, tp2);
                            yt1 = add(yt1, mul(lt2, cc));
                        }
                        double yp0, yp1;
                        {
                            double2 lo, hi;
                            if (!IN && j == 0) {
                                lo.x = mul(__ldg(a.WN + i0), add(__ldg(a.ring + 2 * i0), __ldg(a.ring + 2 * i0 + 1)));
                                lo.y = mul(__ldg(a.WN + i0 + 1), add(__ldg(a.ring + 2 * i0 + 2), __ldg(a.ring + 2 * i0 + 3)));
                            } else {
                                lo = tr;
                            }
                            if (!IN && j == nt - 1) {
                                const double *rs = a.ring + 2 * (nr + i0);
                                hi.x = mul(__ldg(a.WS + i0), -add(__ldg(rs), __ldg(rs + 1)));
                                hi.y = mul(__ldg(a.WS + i0 + 1), -add(__ldg(rs + 2), __ldg(rs + 3)));
                            } else {
                                hi = ld2(TRo + RL);
                            }
                            yp0 = mul(sm2.x, Pm.x);
                            yp0 = add(yp0, mul(ap0, sub(ek.x, e.x)));
                            double cc = sub(lo.x, hi.x);
                            cc = sub(cc, tt.x);
                            cc = add(cc, tt.y);
                            yp0 = add(yp0, mul(mul(lpc1, hmk), cc));
                            yp1 = mul(sm2.y, Pm.y);
                            yp1 = add(yp1, mul(ap1, sub(ek.y, e.y)));
                            cc = sub(lo.y, hi.y);
                            cc = sub(cc, tt.y);
                            cc = add(cc, tt2);
                            yp1 = add(yp1, mul(mul(lpc2, hmk), cc));
                        }
                        const size_t yo = ((size_t)k * 3) * v.plane1 + (size_t)j * nr + i0;
                        st2(y + yo, yr0, yr1);
                        st2(y + yo + v.plane1, yt0, yt1);
                        st2(y + yo + 2 * (size_t)v.plane1, yp0, yp1);
                        if (WITH_DOT) {
                            dot[0].add(Rm.x, yr0);
                            dot[0].add(Tm.x, yt0);
                            dot[0].add(Pm.x, yp0);
                            dot[0].add(Rm.y, yr1);
                            dot[0].add(Tm.y, yt1);
                            dot[0].add(Pm.y, yp1);
                        }
                    }
                    if (role <= 2 && e_on) st2(TBn + o, e0, e1);
                    Rm = R;
                    Tm = T;
                    Pm = Pp;
                }
                if (!(dbg & 4)) __syncthreads();
            }
        };
        if (j0 - 1 >= 1 && j0 + tj <= nt - 2) march(std::true_type{});
        else march(std::false_type{});
        __syncthreads();   // segment end: every slot and term buffer free
    }
    if (WITH_DOT) {
        Acc<EXACT> out[1];
        if (reduce_last<EXACT, kMT, 1>(dot, base.partials, &base.sc->ticket[0], blockIdx.x, total, out)) {
            if (threadIdx.x == 0) {
                base.sc->red1[0] = out[0].p;
                base.sc->red1[1] = out[0].s;
            }
        }
    }
}

}  // namespace

// MASPCG_VV_MARCH=0 disables the marching operator (the two-phase kernels then run)
static bool vv_march_enabled() {
    const char *e = getenv("MASPCG_VV_MARCH");
    return !(e && e[0] == '0');
}

bool vv_march_layout(const VVDims &v, MarchLayout &L) {
    if (v.nr % 2 || v.nr < 2 || v.nt < 1 || v.nloc < 1) return false;
    const int nh = v.nr / 2;
    int tj = kMT / nh - 2;
    if (tj > v.nt) tj = v.nt;
    if (tj > kMaxTR2 - 2) tj = kMaxTR2 - 2;
    const char *f = getenv("MASPCG_VV_MARCH_TJ");   // (tests: force smaller tiles -- ragged tiles, many segments)
    if (f && atoi(f) > 0 && atoi(f) < tj) tj = atoi(f);
    for (; tj >= 1; --tj) {
        L.tj = tj;
        L.pslot = 3u * (tj + 2) * v.nr;
        L.cslot = (3u * (tj + 1) + 4u * tj) * v.nr;
        L.nphi = 2u * (v.nloc + 2);
        L.tbuf = 4u * (tj + 2) * (v.nr + 2);
        if (march_smem_bytes(L) <= 202u * 1024u + 512u) break;   // (+ 24.4 KB static: 227 KB per block)
    }
    if (tj < 1) return false;
    L.njt = (v.nt + tj - 1) / tj;
    L.units = (uint32_t)L.njt * (uint32_t)v.nloc;
    return true;
}

template <bool W, bool LP, bool E, bool PR>
static void launch_march(const VVDims &v, const VVArrays &a, const DevArrays &base, double *y, const MarchLayout &L,
                         cudaStream_t st) {
    const size_t sm = march_smem_bytes(L);
    cudaFuncSetAttribute(k_vv_march<W, LP, E, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t g = (uint32_t)sms;
    const char *f = getenv("MASPCG_VV_MARCH_GRID");   // (tests: fewer blocks -- several segments per block)
    if (f && atoi(f) > 0) g = (uint32_t)atoi(f);
    if (g > L.units) g = L.units;
    if (g > (uint32_t)kRedBlocks) g = kRedBlocks;
    if (g < 1) g = 1;
    const char *d = getenv("MASPCG_VV_MARCH_DEBUG");   // (timing probes only, see k_vv_march)
    k_vv_march<W, LP, E, PR><<<g, kMT, sm, st>>>(v, a, base, y, L, g, PR && d ? (atoi(d) & 0xff) : 0);
}

bool launch_vv_march(const VVDims &v, const VVArrays &a, const DevArrays &base, double *y, bool with_dot, bool loop,
                     bool exact, cudaStream_t st) {
    if (!vv_march_enabled() || ((uintptr_t)y & 15) != 0) return false;
    MarchLayout L;
    if (!vv_march_layout(v, L)) return false;
    const char *d = getenv("MASPCG_VV_MARCH_DEBUG");
    // the timing probe (tools/vv_march_probe.py sets the switch bits plus 0x100): never a loop matvec, and only with
    // the 0x100 marker, so a stray value cannot change a solve
    if (d && (atoi(d) & 0x100) && !with_dot && !loop) {
        launch_march<false, false, true, true>(v, a, base, y, L, st);
        return true;
    }
    if (!with_dot) launch_march<false, false, true, false>(v, a, base, y, L, st);
    else if (exact) {
        if (loop) launch_march<true, true, true, false>(v, a, base, y, L, st);
        else launch_march<true, false, true, false>(v, a, base, y, L, st);
    } else {
        if (loop) launch_march<true, true, false, false>(v, a, base, y, L, st);
        else launch_march<true, false, false, false>(v, a, base, y, L, st);
    }
    return true;
}

}  // namespace maspcg
