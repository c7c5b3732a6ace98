// cg1.cu -- the single-reduction (Chronopoulos-Gear) point-Jacobi PCG, MASPCG_OPT_PATH = 4 (SURVEY.md
// 8(f) NEXT-3; reading R32; the oracle's single-reduction variant step by step):
//
//   update  convergence of the previous iterate; beta = gamma / gamma_old,
//           alpha = gamma / (delta - beta gamma / alpha_old); u = r / D; p = u + beta p, s = w + beta s,
//           x += alpha p, r -= alpha s; u' = r / D (stored, with halo planes); Dot2 partials r.u', r.r
//                                                                   88 B/cell: r, D, w, p, s, x / p, s, x, r, u
//   matvec  w = A u (u with halo planes), Dot2 partial w.u          48 B/cell: u, D, T_r, T_t, T_p / w
//
// All three dot products of an iteration (r.u and r.r from the update, w.u from the matvec) are
// all-reduced TOGETHER after the matvec, so on P > 1 ranks they travel in ONE all-gather instead of
// two -- the latency floor of strong scaling.  136 B/cell per iteration (the three-kernel
// path: 128).  In exact arithmetic s = A p and the iterates are those of the Hestenes-Stiefel path; in
// floating point they differ at rounding level, hence the oracle's own variant.  Same rounding policy
// as kernels.cu: one IEEE operation per operation of the formulas, Dot2 dot products (R24), so the GPU
// reproduces the oracle's cg1 iterates bit for bit.  (A first version formed u = r / D on the fly in
// the matvec -- 128 B/cell but seven divisions per cell: 471 us per launch on c3, compute-bound.)
#include <cuda_runtime.h>

#include "arith.cuh"
#include "cg1.cuh"
#include "common.cuh"

namespace maspcg {

namespace {

constexpr int kCgBlocks = 4;   // resident 256-thread blocks per SM (<= 64 registers)

__device__ __forceinline__ void pdl_wait_cg() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_cg() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void decompose_cg(const Dims &d, uint32_t c, int &i, int &j, int &k) {
    const uint32_t row = d.div_r.div(c);
    i = (int)(c - row * (uint32_t)d.nr);
    const uint32_t kk = d.div_t.div(row);
    j = (int)(row - kk * (uint32_t)d.nt);
    k = (int)kk;
}

struct Range1 {
    uint32_t vend, off0, split, off1;
};

Range1 make_range1(const Dims &d, StencilPart part) {
    const uint32_t pl = d.plane;
    switch (part) {
        case StencilPart::Interior: return {d.nloc > 2 ? (uint32_t)(d.nloc - 2) * pl : 0u, pl, 0xffffffffu, 0u};
        case StencilPart::Boundary:
            if (d.nloc == 1) return {pl, 0u, 0xffffffffu, 0u};
            return {2u * pl, 0u, pl, (uint32_t)(d.nloc - 2) * pl};
        default: return {d.n, 0u, 0xffffffffu, 0u};
    }
}

// w of one cell: D u - sum T u_nb in the oracle's order (r_lo, r_hi, theta_lo, theta_hi, phi_lo, phi_hi)
template <bool EXACT>
__device__ __forceinline__ double cell_w(const Dims &d, const DevArrays &a, uint32_t c, int i, int j, double uc,
                                         double dc) {
    using A = Ar<EXACT>;
    const double *__restrict__ u = a.cgr + d.plane;   // u[c] of local cell c, halo planes at -plane / +n
    double s = 0.0;
    if (i > 0) s = A::acc(s, __ldg(a.Tr + c), __ldg(u + c - 1));
    if (i < d.nr - 1) s = A::acc(s, __ldg(a.Tr + c + 1), __ldg(u + c + 1));
    if (j > 0) s = A::acc(s, __ldg(a.Tt + c), __ldg(u + c - d.nr));
    if (j < d.nt - 1) s = A::acc(s, __ldg(a.Tt + c + d.nr), __ldg(u + c + d.nr));
    s = A::acc(s, __ldg(a.Tp + c), __ldg(u + (size_t)c - d.plane));
    s = A::acc(s, __ldg(a.Tp + c + d.plane), __ldg(u + (size_t)c + d.plane));
    return A::diag_minus(dc, uc, s);
}

template <bool LOOP, bool EXACT>
__global__ void __launch_bounds__(kThreads, kCgBlocks) k_cg1_matvec(Dims d, DevArrays a, Range1 rg, unsigned red_slot0,
                                                                    unsigned red_total, int pair) {
    pdl_wait_cg();
    pdl_trigger_cg();
    if (LOOP && *(volatile int *)&a.sc->done) return;
    const double *__restrict__ u = a.cgr + d.plane;
    Acc<EXACT> acc[1];
    const uint32_t stride = gridDim.x * blockDim.x;
    if (pair) {
        // two r-neighbour cells per thread (nr even): 16-byte loads of the pair's own streams
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; 2 * v < rg.vend; v += stride) {
            const uint32_t c0 = 2 * v + rg.off0 + (2 * v >= rg.split ? rg.off1 : 0u);
            int i, j, k;
            decompose_cg(d, c0, i, j, k);
            const double2 uu = __ldg(reinterpret_cast<const double2 *>(u + c0));
            const double2 dd = __ldg(reinterpret_cast<const double2 *>(a.D + c0));
            const double w0 = cell_w<EXACT>(d, a, c0, i, j, uu.x, dd.x);
            const double w1 = cell_w<EXACT>(d, a, c0 + 1, i + 1, j, uu.y, dd.y);
            *reinterpret_cast<double2 *>(a.cgw + c0) = make_double2(w0, w1);
            acc[0].add(w0, uu.x);
            acc[0].add(w1, uu.y);
        }
    } else {
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < rg.vend; v += stride) {
            const uint32_t c = v + rg.off0 + (v >= rg.split ? rg.off1 : 0u);
            int i, j, k;
            decompose_cg(d, c, i, j, k);
            const double uc = __ldg(u + c);
            const double w = cell_w<EXACT>(d, a, c, i, j, uc, __ldg(a.D + c));
            a.cgw[c] = w;
            acc[0].add(w, uc);
        }
    }
    Acc<EXACT> out[1];
    if (reduce_last<EXACT, kThreads, 1>(acc, a.partials, &a.sc->ticket[0], red_slot0 + blockIdx.x, red_total, out)) {
        if (threadIdx.x == 0) {
            a.sc->red_cg[2] = out[0].p;
            a.sc->red_cg[3] = out[0].s;
        }
    }
}

__device__ __forceinline__ void store_r(const Dims &d, double *rp, uint32_t c, double v) {
    rp[(size_t)c + d.plane] = v;
    if (d.periodic_local) {
        if (c < d.plane) rp[(size_t)c + (size_t)(d.nloc + 1) * d.plane] = v;
        if (c >= d.n - d.plane) rp[(size_t)c - (size_t)(d.nloc - 1) * d.plane] = v;
    }
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kCgBlocks) k_cg1_update(Dims d, DevArrays a, double *__restrict__ x,
                                                                    unsigned total) {
    pdl_wait_cg();
    pdl_trigger_cg();
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const int it = sc->iter;
    // the previous iterate r_it (its r.r came with this iteration's reduction): history, stopping test
    if (it > 0) {
        const double rn = sqrt(__dadd_rn(sc->red_cg[4], sc->red_cg[5]));
        const bool conv = rn <= sc->tolbn, bad = !isfinite(rn);
        if (conv || bad || it >= sc->maxit) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                sc->rn = rn;
                sc->hist_ring[(it - 1) % (2 * kMaxChunk)] = rn;
                sc->hist_count = it;
                sc->status = conv ? ST_OK : (bad ? ST_E_BREAKDOWN : ST_NOT_CONVERGED);
                sc->done = 1;
            }
            return;
        }
    }
    const double gamma = __dadd_rn(sc->red_cg[0], sc->red_cg[1]);
    const double delta = __dadd_rn(sc->red_cg[2], sc->red_cg[3]);
    double beta = 0.0, den = delta;
    if (it > 0) {
        beta = __ddiv_rn(gamma, sc->cg_gamma_old);
        den = __dsub_rn(delta, __ddiv_rn(__dmul_rn(beta, gamma), sc->cg_alpha_old));
    }
    if (!(den > 0.0) || !isfinite(den) || !isfinite(gamma)) {   // uniform decision in every block
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (it > 0) {
                const double rn = sqrt(__dadd_rn(sc->red_cg[4], sc->red_cg[5]));
                sc->rn = rn;
                sc->hist_ring[(it - 1) % (2 * kMaxChunk)] = rn;
                sc->hist_count = it;
            }
            sc->status = ST_E_BREAKDOWN;
            sc->done = 1;
        }
        return;
    }
    const double alpha = __ddiv_rn(gamma, den);
    double *__restrict__ up = a.cgr;
    double *__restrict__ r = a.r;
    double *__restrict__ p = a.q;
    double *__restrict__ s = a.cgs;
    Acc<EXACT> acc[2];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride) {
        const double rc = r[c], dc = __ldg(a.D + c);
        const double u = __ddiv_rn(rc, dc);
        const double pn = A::axpy(beta, p[c], u);
        const double sn = A::axpy(beta, s[c], __ldg(a.cgw + c));
        p[c] = pn;
        s[c] = sn;
        x[c] = A::axpy(alpha, pn, x[c]);
        const double rn = A::ymax(rc, alpha, sn);
        r[c] = rn;
        const double un = __ddiv_rn(rn, dc);
        store_r(d, up, c, un);
        acc[0].add(rn, un);
        acc[1].add(rn, rn);
    }
    Acc<EXACT> out[2];
    if (reduce_last<EXACT, kThreads, 2>(acc, a.partials, &sc->ticket[1], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            if (it > 0) {   // the history entry of r_it (checked above)
                const double rn = sqrt(__dadd_rn(sc->red_cg[4], sc->red_cg[5]));
                sc->rn = rn;
                sc->hist_ring[(it - 1) % (2 * kMaxChunk)] = rn;
                sc->hist_count = it;
            }
            sc->red_cg[0] = out[0].p;   // local r.u and r.r of the new iterate: all-reduced with w.u
            sc->red_cg[1] = out[0].s;
            sc->red_cg[4] = out[1].p;
            sc->red_cg[5] = out[1].s;
            sc->iter = it + 1;
            sc->cg_gamma_old = gamma;
            sc->cg_alpha_old = alpha;
        }
    }
}

template <typename... KArgs, typename... Args>
void launch_cg_pdl(bool pdl, void (*kern)(KArgs...), unsigned grid, cudaStream_t st, Args... args) {
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

inline bool cg_pair(const Dims &d) { return d.vec_ok && (d.nr % 2 == 0); }

inline unsigned cg_grid(uint32_t work) {
    uint64_t g = (work + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * kCgBlocks)) g = 148 * kCgBlocks;
    return (unsigned)g;
}

}  // namespace

unsigned cg1_matvec_blocks(const Dims &d, StencilPart part) {
    const Range1 rg = make_range1(d, part);
    if (!rg.vend) return 0u;
    return cg_grid(cg_pair(d) ? rg.vend / 2 : rg.vend);
}

void launch_cg1_matvec(const Dims &d, const DevArrays &a, StencilPart part, bool loop, unsigned red_slot0,
                       unsigned red_total, bool exact, cudaStream_t st) {
    const Range1 rg = make_range1(d, part);
    if (!rg.vend) return;
    const int pair = cg_pair(d) ? 1 : 0;
    const unsigned g = cg_grid(pair ? rg.vend / 2 : rg.vend);
    if (exact) {
        if (loop) launch_cg_pdl(d.pdl != 0, k_cg1_matvec<true, true>, g, st, d, a, rg, red_slot0, red_total, pair);
        else launch_cg_pdl(d.pdl != 0, k_cg1_matvec<false, true>, g, st, d, a, rg, red_slot0, red_total, pair);
    } else {
        if (loop) launch_cg_pdl(d.pdl != 0, k_cg1_matvec<true, false>, g, st, d, a, rg, red_slot0, red_total, pair);
        else launch_cg_pdl(d.pdl != 0, k_cg1_matvec<false, false>, g, st, d, a, rg, red_slot0, red_total, pair);
    }
}

void launch_cg1_update(const Dims &d, const DevArrays &a, double *x, bool exact, cudaStream_t st) {
    const unsigned g = cg_grid(d.n);
    if (exact) launch_cg_pdl(d.pdl != 0, k_cg1_update<true>, g, st, d, a, x, g);
    else launch_cg_pdl(d.pdl != 0, k_cg1_update<false>, g, st, d, a, x, g);
}

}  // namespace maspcg
