// cg1.cu -- the single-reduction (Chronopoulos-Gear) point-Jacobi PCG, MASPCG_OPT_PATH = 4 (SURVEY.md
// 8(f) NEXT-3; reading R32; the oracle's single-reduction variant step by step):
//
//   update  convergence of the previous iterate; beta = gamma / gamma_old,
//           alpha = gamma / (delta - beta gamma / alpha_old); u = r / D; p = u + beta p, s = w + beta s,
//           x += alpha p, r -= alpha s; u' = r / D (stored, with halo planes); Dot2 partials r.u', r.r
//                                                                   88 B/cell: r, D, w, p, s, x / p, s, x, r, u
//   matvec  w = A u (u with halo planes), Dot2 partial w.u          48 B/cell: u, D, T_r, T_t, T_p / w
//           -- the stencil kernel of the three-kernel path (kernels.cu) applied to u, writing w
//
// All three dot products of an iteration (r.u and r.r from the update into red2, w.u from the matvec
// into red1, adjacent in Scalars) are all-reduced TOGETHER after the matvec, so on P > 1 ranks they travel in ONE all-gather instead of
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

constexpr int kCgBlocks = 4;      // matvec: resident 256-thread blocks per SM (<= 64 registers)
constexpr int kCgUpdBlocks = 2;   // update: 2 per SM (1,694-1,698 vs 1,646-1,667 it/s at 3 and 1,557-1,561 at 4)

__device__ __forceinline__ void pdl_wait_cg() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_cg() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


__device__ __forceinline__ void store_r(const Dims &d, double *rp, uint32_t c, double v) {
    rp[(size_t)c + d.plane] = v;
    if (d.periodic_local) {
        if (c < d.plane) rp[(size_t)c + (size_t)(d.nloc + 1) * d.plane] = v;
        if (c >= d.n - d.plane) rp[(size_t)c - (size_t)(d.nloc - 1) * d.plane] = v;
    }
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kCgUpdBlocks) k_cg1_update(Dims d, DevArrays a, double *__restrict__ x,
                                                                    unsigned total, int pair) {
    pdl_wait_cg();
    pdl_trigger_cg();
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const int it = sc->iter;
    // the previous iterate r_it (its r.r came with this iteration's reduction): history, stopping test
    if (it > 0) {
        const double rn = sqrt(__dadd_rn(sc->red2[2], sc->red2[3]));
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
    const double gamma = __dadd_rn(sc->red2[0], sc->red2[1]);
    const double delta = __dadd_rn(sc->red1[0], sc->red1[1]);
    double beta = 0.0, den = delta;
    if (it > 0) {
        beta = __ddiv_rn(gamma, sc->cg_gamma_old);
        den = __dsub_rn(delta, __ddiv_rn(__dmul_rn(beta, gamma), sc->cg_alpha_old));
    }
    if (!(den > 0.0) || !isfinite(den) || !isfinite(gamma)) {   // uniform decision in every block
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (it > 0) {
                const double rn = sqrt(__dadd_rn(sc->red2[2], sc->red2[3]));
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
    if (pair) {   // two values per thread, 16-byte loads and stores (n and the plane are even)
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; 2 * v < d.n; v += stride) {
            const uint32_t c = 2 * v;
            const double2 rc = *reinterpret_cast<const double2 *>(r + c);
            const double2 dc = __ldg(reinterpret_cast<const double2 *>(a.D + c));
            const double2 po = *reinterpret_cast<const double2 *>(p + c);
            const double2 so = *reinterpret_cast<const double2 *>(s + c);
            const double2 wc = __ldg(reinterpret_cast<const double2 *>(a.cgw + c));
            const double2 xo = *reinterpret_cast<const double2 *>(x + c);
            const double p0 = A::axpy(beta, po.x, __ddiv_rn(rc.x, dc.x));
            const double p1 = A::axpy(beta, po.y, __ddiv_rn(rc.y, dc.y));
            const double s0 = A::axpy(beta, so.x, wc.x), s1 = A::axpy(beta, so.y, wc.y);
            *reinterpret_cast<double2 *>(p + c) = make_double2(p0, p1);
            *reinterpret_cast<double2 *>(s + c) = make_double2(s0, s1);
            *reinterpret_cast<double2 *>(x + c) = make_double2(A::axpy(alpha, p0, xo.x), A::axpy(alpha, p1, xo.y));
            const double r0 = A::ymax(rc.x, alpha, s0), r1 = A::ymax(rc.y, alpha, s1);
            *reinterpret_cast<double2 *>(r + c) = make_double2(r0, r1);
            const double u0 = __ddiv_rn(r0, dc.x), u1 = __ddiv_rn(r1, dc.y);
            *reinterpret_cast<double2 *>(up + (size_t)c + d.plane) = make_double2(u0, u1);
            if (d.periodic_local) {
                if (c < d.plane) *reinterpret_cast<double2 *>(up + (size_t)c + (size_t)(d.nloc + 1) * d.plane) = make_double2(u0, u1);
                if (c >= d.n - d.plane) *reinterpret_cast<double2 *>(up + (size_t)c - (size_t)(d.nloc - 1) * d.plane) = make_double2(u0, u1);
            }
            acc[0].add(r0, u0);
            acc[0].add(r1, u1);
            acc[1].add(r0, r0);
            acc[1].add(r1, r1);
        }
    } else
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
                const double rn = sqrt(__dadd_rn(sc->red2[2], sc->red2[3]));
                sc->rn = rn;
                sc->hist_ring[(it - 1) % (2 * kMaxChunk)] = rn;
                sc->hist_count = it;
            }
            sc->red2[0] = out[0].p;   // local r.u and r.r of the new iterate: all-reduced with w.u (red1)
            sc->red2[1] = out[0].s;
            sc->red2[2] = out[1].p;
            sc->red2[3] = out[1].s;
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

inline unsigned cg_grid(uint32_t work, int per_sm = kCgBlocks) {
    uint64_t g = (work + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)(148 * per_sm)) g = 148 * per_sm;
    return (unsigned)g;
}

}  // namespace

void launch_cg1_update(const Dims &d, const DevArrays &a, double *x, bool exact, cudaStream_t st) {
    const int pair = (cg_pair(d) && ((uintptr_t)x & 15) == 0) ? 1 : 0;
    const unsigned g = cg_grid(pair ? d.n / 2 : d.n, kCgUpdBlocks);
    if (exact) launch_cg_pdl(d.pdl != 0, k_cg1_update<true>, g, st, d, a, x, g, pair);
    else launch_cg_pdl(d.pdl != 0, k_cg1_update<false>, g, st, d, a, x, g, pair);
}

}  // namespace maspcg
