// wave.cu -- the p-update of iteration k and the stencil of iteration k+1 in ONE persistent kernel,
// ordered by plane-completion flags so that p_new and D are read back from L2 instead of HBM.
//
// Iteration (MASPCG_OPT_PATH = 3, single rank):
//   k_update_vec2   alpha, r -= alpha q, z = r/D, Dot2 r.z, r.r                32 B/cell
//   k_wave          A: x += alpha p, p = r/D + beta p  (in place)               48 B/cell
//                   B: q = A p_new, Dot2 p.q                                    32 B/cell from HBM
//                      (p_new and D of the B tile were written / read by A-tiles a few planes
//                       earlier: L2 hits, reuse distance ~10 MB << 126 MB)
// = 112 B/cell of HBM traffic per iteration with plain streaming access patterns -- the same
// saving as the tiled fused path (fused.cu) without recomputing p on halo rows.
//
// Scheduling: the slab is cut into tiles of kWaveTile consecutive cells inside a plane (TPP tiles
// per plane).  Work item u (dispatched in order through an atomic counter) = A on tile u and B on
// tile u - lag*TPP, where B visits the planes in the order 1, 2, ..., nloc-1, 0 (plane 0 needs
// plane nloc-1 through the periodic halo).  A B-tile on plane k waits (spin, nanosleep back-off)
// until all A-tiles of planes k-1, k, k+1 (mod nloc) have been published (store, __threadfence,
// atomicAdd on the plane's flag).  lag = planes in progress across the grid + 2, so waits are rare
// while the A->B reuse distance (lag planes of traffic, ~30 MB on c3) stays well inside the L2:
// small tiles (1024 cells) and 2 blocks per SM keep the in-progress window short.  A-tiles never
// wait, and the grid is exactly the co-resident capacity, so the scheme cannot deadlock.  B reads
// p through L2 (ld.global.cg) because another SM wrote it.  The p.q partial of every B-tile goes
// to its own slot and the last block combines the slots in tile order: deterministic.
#include <cuda_runtime.h>

#include "arith.cuh"
#include "common.cuh"
#include "wave.cuh"

namespace maspcg {

namespace {

constexpr int kWaveThreads = 256;
constexpr int kWaveBlocksPerSM = 4;

__device__ __forceinline__ void wdecompose(const Dims &d, uint32_t c, int &i, int &j, int &k) {
    const uint32_t row = d.div_r.div(c);
    i = (int)(c - row * (uint32_t)d.nr);
    const uint32_t kk = d.div_t.div(row);
    j = (int)(row - kk * (uint32_t)d.nt);
    k = (int)kk;
}


__device__ __forceinline__ double2 ldcg2(const double *p) { return __ldcg(reinterpret_cast<const double2 *>(p)); }

}  // namespace

template <bool EXACT>
__global__ void __launch_bounds__(kWaveThreads, kWaveBlocksPerSM) k_wave(Dims d, DevArrays a, WaveArgs w,
                                                                         double *__restrict__ x, int chunk) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const int tid = threadIdx.x;
    const double rz = __dadd_rn(sc->red2[0], sc->red2[1]);
    const double rr = __dadd_rn(sc->red2[2], sc->red2[3]);
    const double rn = sqrt(rr);
    const bool conv = rn <= sc->tolbn;
    const bool bad = !isfinite(rn) || !isfinite(rz);
    const bool last = conv || bad || sc->iter + 1 >= sc->maxit;
    const double alpha = sc->alpha;
    const double beta = last ? 0.0 : __ddiv_rn(rz, sc->rho);
    double *__restrict__ p = a.p;
    const size_t plane = d.plane;
    __shared__ bool am_last;

    if (last) {   // this iteration ends the solve: only its deferred x update
        const uint32_t stride = gridDim.x * blockDim.x;
        for (uint32_t c = blockIdx.x * blockDim.x + tid; c < d.n; c += stride)
            x[c] = A::axpy(alpha, p[(size_t)c + plane], x[c]);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            am_last = atomicAdd(&sc->ticket[7], 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (am_last && tid == 0) {
            __threadfence();
            const int it = sc->iter + 1;
            sc->iter = it;
            sc->rn = rn;
            sc->hist_ring[(it - 1) % chunk] = rn;
            sc->status = conv ? ST_OK : (bad ? ST_E_BREAKDOWN : ST_NOT_CONVERGED);
            sc->done = 1;
            sc->rho = rz;
            sc->ticket[7] = 0u;
        }
        return;
    }

    const int nloc = d.nloc, nr = d.nr, nt = d.nt;
    const int tpp = w.tpp;
    const uint32_t ntile = (uint32_t)nloc * tpp;
    const int lag = min(w.lag, nloc);
    const uint32_t nitems = ntile + (uint32_t)lag * tpp;
    const double *__restrict__ r = a.r;
    const double *__restrict__ D = a.D;
    const double *__restrict__ Tr = a.Tr;
    const double *__restrict__ Tt = a.Tt;
    const double *__restrict__ Tp = a.Tp;
    __shared__ uint32_t item_s;

    for (;;) {
        if (tid == 0) item_s = atomicAdd(w.counter, 1u);
        __syncthreads();
        const uint32_t u = item_s;
        __syncthreads();
        if (u >= nitems) break;
        // ---------------- A: x += alpha p, p = r/D + beta p on tile u
        if (u < ntile) {
            const int kA = (int)(u / tpp);
            const uint32_t c0 = (uint32_t)kA * plane + (u - (uint32_t)kA * tpp) * (uint32_t)kWaveTile;
            const uint32_t c1 = min(c0 + (uint32_t)kWaveTile, (uint32_t)(kA + 1) * (uint32_t)plane);
            // 16-byte accesses when every pair start is 16-byte aligned (even plane, aligned x)
            const bool vec = ((plane & 1u) == 0) && (((uintptr_t)x & 15) == 0);
            for (uint32_t c = c0 + 2u * tid; c < c1; c += 2u * kWaveThreads) {
                if (vec && c + 1 < c1) {
                    const double2 po = *reinterpret_cast<const double2 *>(p + (size_t)c + plane);
                    const double2 xv = *reinterpret_cast<const double2 *>(x + c);
                    const double2 rv = __ldg(reinterpret_cast<const double2 *>(r + c));
                    const double2 dv = __ldg(reinterpret_cast<const double2 *>(D + c));
                    *reinterpret_cast<double2 *>(x + c) =
                        make_double2(A::axpy(alpha, po.x, xv.x), A::axpy(alpha, po.y, xv.y));
                    const double p0 = A::axpy(beta, po.x, __ddiv_rn(rv.x, dv.x));
                    const double p1 = A::axpy(beta, po.y, __ddiv_rn(rv.y, dv.y));
                    *reinterpret_cast<double2 *>(p + (size_t)c + plane) = make_double2(p0, p1);
                    if (kA == 0)
                        *reinterpret_cast<double2 *>(p + (size_t)c + (size_t)(nloc + 1) * plane) = make_double2(p0, p1);
                    if (kA == nloc - 1)
                        *reinterpret_cast<double2 *>(p + (size_t)c - (size_t)(nloc - 1) * plane) = make_double2(p0, p1);
                } else {
                    for (uint32_t cc = c; cc < c + 2u && cc < c1; ++cc) {
                        const double po = p[(size_t)cc + plane];
                        x[cc] = A::axpy(alpha, po, x[cc]);
                        const double pn = A::axpy(beta, po, __ddiv_rn(r[cc], D[cc]));
                        p[(size_t)cc + plane] = pn;
                        if (kA == 0) p[(size_t)cc + (size_t)(nloc + 1) * plane] = pn;
                        if (kA == nloc - 1) p[(size_t)cc - (size_t)(nloc - 1) * plane] = pn;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(w.flags + kA, 1u);
            }
        }
        // ---------------- B: q = A p_new on tile b = u - kLag*TPP (planes in the order 1..nloc-1, 0)
        if (u >= (uint32_t)lag * tpp) {
            const uint32_t b = u - (uint32_t)lag * tpp;
            const int ord = (int)(b / tpp);
            const int kB = (ord + 1) % nloc;
            const uint32_t c0 = (uint32_t)kB * plane + (b - (uint32_t)ord * tpp) * (uint32_t)kWaveTile;
            const uint32_t c1 = min(c0 + (uint32_t)kWaveTile, (uint32_t)(kB + 1) * (uint32_t)plane);
            if (tid == 0) {
                const int km = (kB + nloc - 1) % nloc, kp = (kB + 1) % nloc;
                const unsigned target = (unsigned)tpp;
                unsigned ns = 32;
                while (*(volatile unsigned *)(w.flags + km) < target || *(volatile unsigned *)(w.flags + kB) < target ||
                       *(volatile unsigned *)(w.flags + kp) < target) {
                    __nanosleep(ns);
                    if (ns < 1024) ns *= 2;
                }
                __threadfence();
            }
            __syncthreads();
            Acc<EXACT> dot[1];
            const bool vecB = (nr % 2 == 0);   // pairs (i, i+1), i even, never straddle a row
            for (uint32_t c = c0 + 2u * tid; c < c1; c += 2u * kWaveThreads) {
                if (vecB) {
                    int i, j, k;
                    wdecompose(d, c, i, j, k);
                    const size_t cp = (size_t)c + plane;
                    const double2 pc = ldcg2(p + cp);
                    const double2 trv = __ldg(reinterpret_cast<const double2 *>(Tr + c));
                    const double2 ttl = __ldg(reinterpret_cast<const double2 *>(Tt + c));
                    const double2 tpl = __ldg(reinterpret_cast<const double2 *>(Tp + c));
                    const double2 tph = __ldg(reinterpret_cast<const double2 *>(Tp + c + plane));
                    const double2 pkm = ldcg2(p + cp - plane);
                    const double2 pkp = ldcg2(p + cp + plane);
                    const double2 dv = __ldg(reinterpret_cast<const double2 *>(D + c));
                    const bool jlo = j > 0, jhi = j < nt - 1, ilo = i > 0, ihi = i + 2 < nr;
                    double2 ptm = make_double2(0.0, 0.0), ptp = ptm, tth = ptm;
                    if (jlo) ptm = ldcg2(p + cp - nr);
                    if (jhi) {
                        ptp = ldcg2(p + cp + nr);
                        tth = __ldg(reinterpret_cast<const double2 *>(Tt + c + nr));
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
                    *reinterpret_cast<double2 *>(a.q + c) = make_double2(q0, q1);
                    dot[0].add(pc.x, q0);
                    dot[0].add(pc.y, q1);
                    continue;
                }
                const int nc = (c + 1 < c1) ? 2 : 1;
                for (int e = 0; e < nc; ++e) {
                    const uint32_t cc = c + e;
                    int i, j, k;
                    wdecompose(d, cc, i, j, k);
                    const size_t cp = (size_t)cc + plane;
                    const double pc = __ldcg(p + cp);
                    double s = 0.0;
                    if (i > 0) s = A::acc(s, __ldg(Tr + cc), __ldcg(p + cp - 1));
                    if (i < nr - 1) s = A::acc(s, __ldg(Tr + cc + 1), __ldcg(p + cp + 1));
                    if (j > 0) s = A::acc(s, __ldg(Tt + cc), __ldcg(p + cp - nr));
                    if (j < nt - 1) s = A::acc(s, __ldg(Tt + cc + nr), __ldcg(p + cp + nr));
                    s = A::acc(s, __ldg(Tp + cc), __ldcg(p + cp - plane));
                    s = A::acc(s, __ldg(Tp + cc + plane), __ldcg(p + cp + plane));
                    const double q = A::diag_minus(__ldg(D + cc), pc, s);
                    a.q[cc] = q;
                    dot[0].add(pc, q);
                }
            }
            block_combine<EXACT, kWaveThreads, 1>(dot);
            if (tid == 0) {
                w.tile_partials[2 * b] = dot[0].p;
                w.tile_partials[2 * b + 1] = dot[0].s;
            }
        }
    }

    // ---------------- last block: p.q over the tiles in order, iteration bookkeeping, reset
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        am_last = atomicAdd(&sc->ticket[7], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    Acc<EXACT> acc[1];
    for (uint32_t b = tid; b < ntile; b += kWaveThreads) {
        Acc<EXACT> o;
        o.p = __ldcg(w.tile_partials + 2 * b);
        o.s = __ldcg(w.tile_partials + 2 * b + 1);
        acc[0].add(o);
    }
    block_combine<EXACT, kWaveThreads, 1>(acc);
    for (int k = tid; k < nloc; k += kWaveThreads) w.flags[k] = 0u;
    if (tid == 0) {
        sc->red1[0] = acc[0].p;
        sc->red1[1] = acc[0].s;
        const int it = sc->iter + 1;
        sc->iter = it;
        sc->rn = rn;
        sc->hist_ring[(it - 1) % chunk] = rn;
        sc->rho = rz;
        *w.counter = 0u;
        sc->ticket[7] = 0u;
    }
}

int wave_grid(int device) {
    int sms = 148, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_wave<true>, kWaveThreads, 0);
    int occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_wave<false>, kWaveThreads, 0);
    if (occ2 < occ) occ = occ2;
    if (occ > kWaveBlocksPerSM) occ = kWaveBlocksPerSM;
    if (occ < 1) occ = 1;
    return sms * occ;   // all blocks co-resident: required by the flag waits
}

void launch_wave(const Dims &d, const DevArrays &a, const WaveArgs &w, double *x, int chunk, int grid, bool exact,
                 cudaStream_t st) {
    if (exact) k_wave<true><<<grid, kWaveThreads, 0, st>>>(d, a, w, x, chunk);
    else k_wave<false><<<grid, kWaveThreads, 0, st>>>(d, a, w, x, chunk);
}

}  // namespace maspcg
