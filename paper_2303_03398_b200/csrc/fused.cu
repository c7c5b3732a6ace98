// fused.cu -- the two-pass PCG iteration (SURVEY.md 8(f) NEXT-3 "fold p-update into the
// stencil", plus the deferred x update): 112 instead of 136 algorithmic bytes per cell.
//
//   pass A  k_pass_a  (it = iter + 1, reads the scalars of iteration `iter`)
//       finalise iteration `iter`: ||r||, convergence / breakdown / maxit  (R12, R13)
//       beta = rz / rho                                                      (R11)
//       p_it = r/D + beta p_{it-1}   computed ONCE per cell into a 3-plane shared-memory ring
//       x   += alpha_{iter} p_{it-1} (the x update of iteration `iter`, deferred one pass)
//       q    = A p_it,  partial p_it . q
//       reads r, D, p_old, x, T_r, T_theta, T_phi; writes p_new, q, x      80 B/cell
//   pass B  k_pass_b
//       alpha = rho / (p.q); r -= alpha q; z = r/D; partials r.z, r.r        32 B/cell
//
// Same arithmetic as the three-kernel path (kernels.cu) and, with the default exact policy of
// arith.cuh, as the oracle: identical iterates.  PAPER.md credits
// kernel fusion and asynchronous launches for the best GPU version; this is that
// fusion done by hand for sm_100a.
//
// Tiling (2.5-D phi march): the slab is cut into j-tiles of BJ theta rows; the (j-tile, plane)
// pairs are split into equal contiguous segments, one per persistent block (1 block of 512 threads
// per SM, ~160 KB of shared memory).  A block marches its segment plane by plane: phase 1 loads r,
// D, p_old, x of up to kAM tile cells per thread in one batch, computes p_new into ring slot k%3
// (plus the two halo rows), keeps D in a 2-plane shared ring and stores p_new and x; phase 2
// applies the 7-point stencil to plane k-1 from the rings, carrying the upper T_phi face of each
// cell in a register as the next plane's lower face -- so D and T_phi are read from HBM once
// (re-reads across plane steps would miss in L2: ~150 blocks x ~250 KB per step).  The halo rows / the two halo planes of a segment are
// recomputed from r, D, p_old (a few % extra reads, mostly L2 hits) instead of being exchanged.
// Planes -1 and nloc come from halo pointers: the wrap planes on a single rank, received halo
// buffers on several ranks.
#include <cuda_runtime.h>

#include "arith.cuh"
#include "common.cuh"
#include "fused.cuh"

namespace maspcg {

namespace {

constexpr int kAThreads = 512;   // one persistent block per SM (smem-bound)
constexpr int kAM = 8;           // tile cells per thread per plane (register batches)

// plane pointer of array `base` for local plane k in [-1, nloc] (halo pointers at the ends)
__device__ __forceinline__ const double *plane_ptr(const double *base, const double *lo, const double *hi, int k,
                                                   int nloc, size_t plane) {
    return k < 0 ? lo : (k >= nloc ? hi : base + (size_t)k * plane);
}

}  // namespace

// ------------------------------------------------------------------------ pass A
template <bool EXACT>
__global__ void __launch_bounds__(kAThreads, 1) k_pass_a(Dims d, DevArrays a, FusedArgs f) {
    using A = Ar<EXACT>;
    extern __shared__ double smem[];   // p ring [3][(bj+2) nr] | D ring [2][bj nr]
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const int it_done = sc->iter;
    const bool first = it_done == 0;
    double rz = 0.0, rn = 0.0;
    bool stop = false, conv = false, bad = false;
    if (!first) {
        rz = __dadd_rn(sc->red2[0], sc->red2[1]);
        rn = sqrt(__dadd_rn(sc->red2[2], sc->red2[3]));
        conv = rn <= sc->tolbn;
        bad = !isfinite(rn) || !isfinite(rz);
        stop = conv || bad || it_done >= sc->maxit;
    }
    const double alpha = first ? 0.0 : sc->alpha;
    const double beta = first ? 0.0 : __ddiv_rn(rz, sc->rho);
    const double *__restrict__ pold = f.p_old;
    double *__restrict__ x = f.x;
    const unsigned total = gridDim.x;

    if (stop) {
        // iteration `it_done` is the last: complete its deferred x update and finish
        const uint32_t stride = gridDim.x * blockDim.x;
        for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride)
            x[c] = A::axpy(alpha, __ldg(pold + c), x[c]);
        __shared__ bool am_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            am_last = atomicAdd(&sc->ticket[4], 1u) == total - 1;
        }
        __syncthreads();
        if (am_last && threadIdx.x == 0) {
            __threadfence();
            sc->hist_ring[(it_done - 1) % (2 * kMaxChunk)] = rn;
            sc->hist_count = it_done;
            sc->rn = rn;
            sc->status = conv ? ST_OK : (bad ? ST_E_BREAKDOWN : ST_NOT_CONVERGED);
            sc->done = 1;
            sc->ticket[4] = 0u;
        }
        return;
    }

    const int nr = d.nr, nt = d.nt, nloc = d.nloc;
    const size_t plane = d.plane;
    const int bj = f.bj;
    const int ext = (bj + 2) * nr;             // p ring slot: tile rows + one halo row on each side
    const int own = bj * nr;                   // D ring slot: tile rows
    double *ring = smem;                       // [3][ext]
    double *dring = smem + 3 * ext;            // [2][own]
    const uint32_t T = (uint32_t)f.n_jt * (uint32_t)nloc;
    const uint32_t t_beg = (uint32_t)(((uint64_t)T * blockIdx.x) / total);
    const uint32_t t_end = (uint32_t)(((uint64_t)T * (blockIdx.x + 1)) / total);
    const int tid = threadIdx.x;
    Acc<EXACT> dot[1];
    double tp_carry[kAM];                      // T_phi upper face of the previous plane = lower face of this one

    uint32_t t = t_beg;
    while (t < t_end) {
        const int jt = (int)(t / (uint32_t)nloc);
        const int ka = (int)(t - (uint32_t)jt * nloc);
        const int kb = min(nloc - 1, ka + (int)(t_end - t) - 1);
        t += (uint32_t)(kb - ka + 1);
        const int j0 = jt * bj;
        const int rows = min(bj, nt - j0);
        const int own_n = rows * nr;
        for (int k = ka - 1; k <= kb + 1; ++k) {
            // ---- phase 1: p_new on plane k for the tile rows (batched loads, kAM cells per thread)
            double *slot = ring + (size_t)((k + 3) % 3) * ext;
            double *dslot = dring + (size_t)(k & 1) * own;
            const double *rp = plane_ptr(f.r, f.r_lo, f.r_hi, k, nloc, plane);
            const double *dp = plane_ptr(a.D, f.d_lo, f.d_hi, k, nloc, plane);
            const double *pp = plane_ptr(pold, f.p_lo, f.p_hi, k, nloc, plane);
            const bool own_plane = k >= ka && k <= kb;
            const size_t tile0 = (size_t)j0 * nr;      // tile start within the plane
            {
                double rv[kAM], dv[kAM], pv[kAM], xv[kAM];
#pragma unroll
                for (int m = 0; m < kAM; ++m) {
                    const int o = tid + m * kAThreads;
                    rv[m] = dv[m] = 1.0;
                    pv[m] = xv[m] = 0.0;
                    if (o < own_n) {
                        rv[m] = __ldg(rp + tile0 + o);
                        dv[m] = __ldg(dp + tile0 + o);
                        if (!first) {
                            pv[m] = __ldg(pp + tile0 + o);
                            if (own_plane) xv[m] = x[(size_t)k * plane + tile0 + o];
                        }
                    }
                }
#pragma unroll
                for (int m = 0; m < kAM; ++m) {
                    const int o = tid + m * kAThreads;
                    if (o < own_n) {
                        const double z = __ddiv_rn(rv[m], dv[m]);
                        const double pn = first ? z : A::axpy(beta, pv[m], z);
                        slot[nr + o] = pn;
                        dslot[o] = dv[m];
                        if (own_plane) {
                            const size_t gc = (size_t)k * plane + tile0 + o;
                            f.p_new[gc] = pn;
                            if (!first) x[gc] = A::axpy(alpha, pv[m], xv[m]);
                        }
                    }
                }
            }
            // the two halo rows of the tile (recomputed from r, D, p_old; not stored)
            for (int h = tid; h < 2 * nr; h += kAThreads) {
                const int top = h >= nr;
                const int i = h - top * nr;
                const int j = top ? j0 + rows : j0 - 1;
                if (j < 0 || j >= nt) continue;
                const size_t g = (size_t)j * nr + i;
                const double z = __ddiv_rn(__ldg(rp + g), __ldg(dp + g));
                slot[(top ? (rows + 1) * nr : 0) + i] = first ? z : A::axpy(beta, __ldg(pp + g), z);
            }
            __syncthreads();
            // ---- phase 2: stencil on plane ks = k-1 from ring slots ks-1, ks, ks+1
            const int ks = k - 1;
            if (ks >= ka) {
                const double *sm_ = ring + (size_t)((ks + 2) % 3) * ext;   // plane ks-1
                const double *s0 = ring + (size_t)((ks + 3) % 3) * ext;    // plane ks
                const double *sp = slot;                                    // plane ks+1
                const double *dk = dring + (size_t)(ks & 1) * own;
                const size_t pbase = (size_t)ks * plane + tile0;
                double tr0[kAM], tr1[kAM], tt0[kAM], tt1[kAM], tph[kAM];
#pragma unroll
                for (int m = 0; m < kAM; ++m) {
                    const int o = tid + m * kAThreads;
                    tr0[m] = tr1[m] = tt0[m] = tt1[m] = tph[m] = 0.0;
                    if (o < own_n) {
                        const int jj = (int)f.div_r.div((uint32_t)o);
                        const int i = o - jj * nr;
                        const int j = j0 + jj;
                        const size_t c = pbase + o;
                        tr0[m] = __ldg(a.Tr + c);
                        if (i < nr - 1) tr1[m] = __ldg(a.Tr + c + 1);
                        tt0[m] = __ldg(a.Tt + c);
                        if (j < nt - 1) tt1[m] = __ldg(a.Tt + c + nr);
                        tph[m] = __ldg(a.Tp + c + plane);
                        if (ks == ka) tp_carry[m] = __ldg(a.Tp + c);
                    }
                }
#pragma unroll
                for (int m = 0; m < kAM; ++m) {
                    const int o = tid + m * kAThreads;
                    if (o < own_n) {
                        const int jj = (int)f.div_r.div((uint32_t)o);
                        const int i = o - jj * nr;
                        const int j = j0 + jj;
                        const int l = nr + o;
                        const double pc = s0[l];
                        double s = 0.0;
                        if (i > 0) s = A::acc(s, tr0[m], s0[l - 1]);
                        if (i < nr - 1) s = A::acc(s, tr1[m], s0[l + 1]);
                        if (j > 0) s = A::acc(s, tt0[m], s0[l - nr]);
                        if (j < nt - 1) s = A::acc(s, tt1[m], s0[l + nr]);
                        s = A::acc(s, tp_carry[m], sm_[l]);
                        s = A::acc(s, tph[m], sp[l]);
                        const double q = A::diag_minus(dk[o], pc, s);
                        a.q[pbase + o] = q;
                        dot[0].add(pc, q);
                        tp_carry[m] = tph[m];
                    }
                }
            }
            __syncthreads();
        }
    }

    Acc<EXACT> out[1];
    if (reduce_last<EXACT, kAThreads, 1>(dot, a.partials, &sc->ticket[5], blockIdx.x, total, out)) {
        if (threadIdx.x == 0) {
            sc->red1[0] = out[0].p;
            sc->red1[1] = out[0].s;
            if (!first) {
                sc->hist_ring[(it_done - 1) % (2 * kMaxChunk)] = rn;
                sc->hist_count = it_done;
                sc->rn = rn;
                sc->rho = rz;
            }
        }
    }
}

// ------------------------------------------------------------------------ pass B
template <bool EXACT>
__global__ void __launch_bounds__(kThreads, kRedBlocks / 148) k_pass_b(Dims d, DevArrays a) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    const double pi = __dadd_rn(sc->red1[0], sc->red1[1]);
    if (!(pi > 0.0) || !isfinite(pi)) {     // breakdown: x already holds x_{iter} (deferred update done)
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
    if (reduce_last<EXACT, kThreads, 2>(acc, a.partials, &sc->ticket[6], blockIdx.x, gridDim.x, out)) {
        if (threadIdx.x == 0) {
            sc->red2[0] = out[0].p;
            sc->red2[1] = out[0].s;
            sc->red2[2] = out[1].p;
            sc->red2[3] = out[1].s;
            sc->alpha = alpha;
            sc->iter = sc->iter + 1;
        }
    }
}

// ------------------------------------------------------------------------ launchers
int fused_bj(int nr, int nt) {
    // tile rows: bj * nr <= kAM * kAThreads cells (one register batch per thread) and the shared
    // memory (3 p planes of bj+2 rows + 2 D planes of bj rows) within ~200 KB.  0: not supported.
    int bj = (kAM * kAThreads) / nr;
    while (bj > 0 && fused_smem_bytes(nr, bj) > 200 * 1024) --bj;
    if (bj > nt) bj = nt;
    return bj;
}

size_t fused_smem_bytes(int nr, int bj) { return (size_t)(3 * (bj + 2) + 2 * bj) * nr * sizeof(double); }

int fused_blocks(int nr, int nt, int nloc, int bj, int device) {
    static int cached_dev = -1, sms = 148;
    if (cached_dev != device) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        cached_dev = device;
    }
    const size_t smem = fused_smem_bytes(nr, bj);
    cudaFuncSetAttribute(k_pass_a<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_pass_a<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0, occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pass_a<true>, kAThreads, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_pass_a<false>, kAThreads, smem);
    if (occ2 < occ) occ = occ2;
    if (occ < 1) occ = 1;
    if (occ > 1) occ = 1;
    const long long tiles = (long long)((nt + bj - 1) / bj) * nloc;
    long long b = (long long)sms * occ;
    if (b > tiles) b = tiles;
    if (b > kRedBlocks) b = kRedBlocks;
    return (int)b;
}

void launch_pass_a(const Dims &d, const DevArrays &a, const FusedArgs &f, int blocks, bool exact, cudaStream_t st) {
    const size_t smem = fused_smem_bytes(d.nr, f.bj);
    if (exact) k_pass_a<true><<<blocks, kAThreads, smem, st>>>(d, a, f);
    else k_pass_a<false><<<blocks, kAThreads, smem, st>>>(d, a, f);
}

void launch_pass_b(const Dims &d, const DevArrays &a, bool exact, cudaStream_t st) {
    uint64_t g = (d.n + kThreads - 1) / kThreads;
    if (g < 1) g = 1;
    if (g > (uint64_t)kRedBlocks) g = kRedBlocks;
    if (exact) k_pass_b<true><<<(unsigned)g, kThreads, 0, st>>>(d, a);
    else k_pass_b<false><<<(unsigned)g, kThreads, 0, st>>>(d, a);
}

}  // namespace maspcg
