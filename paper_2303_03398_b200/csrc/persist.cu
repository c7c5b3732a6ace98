// persist.cu -- the persistent PCG iteration kernel, MASPCG_OPT_PATH = 5 (single rank; SURVEY.md 8(f)
// NEXT-3 "conditional ... device loop", 8(e) lever 1).
//
// One cooperative launch runs a whole chunk of iterations: every block owns the same grid-stride share
// of the slab in every phase, and the three phases of an iteration -- stencil + p.q, r-update + Jacobi
// + r.z, r.r, deferred x-update + p-update -- are separated by grid-wide barriers instead of kernel
// boundaries.  A reduction barrier is the last-block Dot2 combination of the three-kernel path
// (reduce_last: the same partials, the same fixed order, so the same bits) whose last block releases
// the barrier.  The arithmetic per cell is the 16-byte pair code of kernels.cu; the traffic is the
// three-kernel path's 128 B/cell.  What it removes is the launch and drain of three kernels per
// iteration -- the fixed cost that dominates small per-GPU slabs in strong scaling.
#include <cuda_runtime.h>

#include "arith.cuh"
#include "common.cuh"
#include "persist.cuh"

namespace maspcg {

namespace {

constexpr int kPersistBlocks = 3;   // resident 256-thread blocks per SM (<= 85 registers)

__device__ __forceinline__ void decompose_p(const Dims &d, uint32_t c, int &i, int &j, int &k) {
    const uint32_t row = d.div_r.div(c);
    i = (int)(c - row * (uint32_t)d.nr);
    const uint32_t kk = d.div_t.div(row);
    j = (int)(row - kk * (uint32_t)d.nt);
    k = (int)kk;
}
__device__ __forceinline__ double2 ld2p(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ double2 ld2v(const double *p) { return __ldcg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ void st2p(double *p, double a, double b) {
    *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}

// plain grid barrier (generation counter): every block's writes before it are visible after it
__device__ __forceinline__ void grid_sync(unsigned *count, unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *(volatile unsigned *)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned *)gen == g) __nanosleep(16);
        }
        __threadfence();
    }
    __syncthreads();
}

// reduction barrier: block partials -> the last-arriving block combines them (reduce_last, fixed order),
// writes out[N] to `dst` (Dot2 pairs) and releases the others; every block returns the global values
template <bool EXACT, int N>
__device__ __forceinline__ void grid_reduce(Acc<EXACT> (&acc)[N], double *partials, unsigned *ticket, unsigned *gen,
                                            unsigned nblocks, double *dst) {
    __shared__ unsigned g0;
    if (threadIdx.x == 0) g0 = *(volatile unsigned *)gen;   // before arriving: gen moves only after all arrive
    __syncthreads();
    Acc<EXACT> out[N];
    if (reduce_last<EXACT, kThreads, N>(acc, partials, ticket, blockIdx.x, nblocks, out)) {
        if (threadIdx.x == 0) {
            for (int t = 0; t < N; ++t) {
                dst[2 * t] = out[t].p;
                dst[2 * t + 1] = out[t].s;
            }
            __threadfence();
            atomicAdd(gen, 1u);
        }
    } else if (threadIdx.x == 0) {
        while (*(volatile unsigned *)gen == g0) __nanosleep(16);
        __threadfence();
    }
    __syncthreads();
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kPersistBlocks) k_persist(Dims d, DevArrays a, double *__restrict__ x,
                                                                      int iters, int ring) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    unsigned *bar_count = &sc->ticket[5], *bar_gen = &sc->ticket[6];
    const unsigned nb = gridDim.x;
    double *__restrict__ p = a.p;
    double *__restrict__ q = a.q;
    double *__restrict__ r = a.r;
    const double *__restrict__ Tr = a.Tr;
    const double *__restrict__ Tt = a.Tt;
    const double *__restrict__ Tp = a.Tp;
    const double *__restrict__ D = a.D;
    const size_t plane = d.plane;
    const int nr = d.nr, nt = d.nt;
    const uint32_t stride = gridDim.x * blockDim.x, npair = d.n >> 1;
    double rho = *(volatile double *)&sc->rho;
    for (int step = 0; step < iters; ++step) {
        if (*(volatile int *)&sc->done) break;   // uniform: written before the last barrier
        // read before the first barrier of the iteration: block 0 advances it in phase C, which no block
        // reaches before every block has passed the two reduction barriers
        const int it_done = *(volatile int *)&sc->iter;
        // ---- phase A: q = A p, p.q (the stencil of k_matvec_vec2)
        Acc<EXACT> dot[1];
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < npair; v += stride) {
            const uint32_t c = 2u * v;
            int i, j, k;
            decompose_p(d, c, i, j, k);
            const size_t cp = (size_t)c + plane;
            const double2 pc = ld2v(p + cp);
            const double2 trv = ld2p(Tr + c);
            const double2 ttl = ld2p(Tt + c);
            const double2 tpl = ld2p(Tp + c);
            const double2 tph = ld2p(Tp + c + plane);
            const double2 pkm = ld2v(p + cp - plane);
            const double2 pkp = ld2v(p + cp + plane);
            const double2 dv = ld2p(D + c);
            const bool jlo = j > 0, jhi = j < nt - 1, ilo = i > 0, ihi = i + 2 < nr;
            double2 ptm = make_double2(0.0, 0.0), ptp = ptm, tth = ptm;
            if (jlo) ptm = ld2v(p + cp - nr);
            if (jhi) {
                ptp = ld2v(p + cp + nr);
                tth = ld2p(Tt + c + nr);
            }
            const double pm = ilo ? __ldcg(p + cp - 1) : 0.0;
            const double pp2 = ihi ? __ldcg(p + cp + 2) : 0.0;
            const double tr2 = ihi ? __ldg(Tr + c + 2) : 0.0;
            double s = 0.0;
            if (ilo) s = A::acc(s, trv.x, pm);
            s = A::acc(s, trv.y, pc.y);
            if (jlo) s = A::acc(s, ttl.x, ptm.x);
            if (jhi) s = A::acc(s, tth.x, ptp.x);
            s = A::acc(s, tpl.x, pkm.x);
            s = A::acc(s, tph.x, pkp.x);
            const double q0 = A::diag_minus(dv.x, pc.x, s);
            s = 0.0;
            s = A::acc(s, trv.y, pc.x);
            if (ihi) s = A::acc(s, tr2, pp2);
            if (jlo) s = A::acc(s, ttl.y, ptm.y);
            if (jhi) s = A::acc(s, tth.y, ptp.y);
            s = A::acc(s, tpl.y, pkm.y);
            s = A::acc(s, tph.y, pkp.y);
            const double q1 = A::diag_minus(dv.y, pc.y, s);
            st2p(q + c, q0, q1);
            dot[0].add(pc.x, q0);
            dot[0].add(pc.y, q1);
        }
        grid_reduce<EXACT, 1>(dot, a.partials, &sc->ticket[0], bar_gen, nb, sc->red1);
        const double pi = __dadd_rn(__ldcg(&sc->red1[0]), __ldcg(&sc->red1[1]));
        if (!(pi > 0.0) || !isfinite(pi)) {   // breakdown: the same decision in every block; x = x_{k-1}
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                sc->status = ST_E_BREAKDOWN;
                sc->done = 1;
            }
            break;
        }
        const double alpha = __ddiv_rn(rho, pi);
        // ---- phase B: r -= alpha q; z = r / D; r.z, r.r (k_update_vec2)
        Acc<EXACT> acc[2];
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < npair; v += stride) {
            const uint32_t c = 2u * v;
            const double2 rv = ld2v(r + c), qv = ld2v(q + c), dv = ld2p(D + c);
            const double r0 = A::ymax(rv.x, alpha, qv.x), r1 = A::ymax(rv.y, alpha, qv.y);
            st2p(r + c, r0, r1);
            const double z0 = __ddiv_rn(r0, dv.x), z1 = __ddiv_rn(r1, dv.y);
            acc[0].add(r0, z0);
            acc[0].add(r1, z1);
            acc[1].add(r0, r0);
            acc[1].add(r1, r1);
        }
        grid_reduce<EXACT, 2>(acc, a.partials, &sc->ticket[1], bar_gen, nb, sc->red2);
        const double rz = __dadd_rn(__ldcg(&sc->red2[0]), __ldcg(&sc->red2[1]));
        const double rr = __dadd_rn(__ldcg(&sc->red2[2]), __ldcg(&sc->red2[3]));
        const double rn = sqrt(rr);
        const bool conv = rn <= sc->tolbn;
        const bool bad = !isfinite(rn) || !isfinite(rz);
        const bool last = conv || bad || it_done + 1 >= sc->maxit;
        const double beta = last ? 0.0 : __ddiv_rn(rz, rho);
        // ---- phase C: x += alpha p (deferred); p = r/D + beta p (k_pupdate_vec2)
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < npair; v += stride) {
            const uint32_t c = 2u * v;
            const double2 po = ld2v(p + (size_t)c + plane), xv = ld2v(x + c);
            st2p(x + c, A::axpy(alpha, po.x, xv.x), A::axpy(alpha, po.y, xv.y));
            if (!last) {
                const double2 rv = ld2v(r + c), dv = ld2p(D + c);
                const double p0 = A::axpy(beta, po.x, __ddiv_rn(rv.x, dv.x));
                const double p1 = A::axpy(beta, po.y, __ddiv_rn(rv.y, dv.y));
                st2p(p + (size_t)c + plane, p0, p1);
                if (c < d.plane) st2p(p + (size_t)c + (size_t)(d.nloc + 1) * plane, p0, p1);   // periodic halos
                if (c >= d.n - d.plane) st2p(p + (size_t)c - (size_t)(d.nloc - 1) * plane, p0, p1);
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const int it = it_done + 1;
            sc->iter = it;
            sc->rn = rn;
            sc->alpha = alpha;
            sc->hist_ring[(it - 1) % ring] = rn;
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
        }
        rho = rz;
        grid_sync(bar_count, bar_gen, nb);   // p complete, the scalars visible, before the next stencil
        if (last) break;
    }
}

}  // namespace

unsigned persist_grid(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_persist<true>, kThreads, 0);
    int per_sm2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_persist<false>, kThreads, 0);
    if (per_sm2 < per_sm) per_sm = per_sm2;
    if (per_sm < 1) per_sm = 1;
    unsigned g = (unsigned)(sms * per_sm);
    return g > (unsigned)kRedBlocks ? (unsigned)kRedBlocks : g;
}

cudaError_t launch_persist(const Dims &d, const DevArrays &a, double *x, int iters, int ring, unsigned grid, bool exact,
                           cudaStream_t st) {
    Dims dd = d;
    DevArrays aa = a;
    void *args[] = {&dd, &aa, &x, &iters, &ring};
    return exact ? cudaLaunchCooperativeKernel((const void *)k_persist<true>, dim3(grid), dim3(kThreads), args, 0, st)
                 : cudaLaunchCooperativeKernel((const void *)k_persist<false>, dim3(grid), dim3(kThreads), args, 0, st);
}

}  // namespace maspcg
