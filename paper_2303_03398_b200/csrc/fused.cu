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
constexpr int kTThreads = 1024;  // TMA variant: all inputs staged in shared memory, 32 warps per SM

// plane pointer of array `base` for local plane k in [-1, nloc] (halo pointers at the ends)
__device__ __forceinline__ const double *plane_ptr(const double *base, const double *lo, const double *hi, int k,
                                                   int nloc, size_t plane) {
    return k < 0 ? lo : (k >= nloc ? hi : base + (size_t)k * plane);
}

// Scalars of pass A: finalise iteration `iter` (R12, R13) and form beta (R11).
struct PassAScalars {
    bool first;
    double alpha, beta, rz, rn;
    int it_done;
};

// Reads the scalars; when iteration `iter` was the last, completes its deferred x update, lets the
// last block publish status / history and returns true (the caller returns).
template <bool EXACT>
__device__ __forceinline__ bool pass_a_prologue(const Dims &d, const DevArrays &a, const FusedArgs &f,
                                                PassAScalars &S) {
    using A = Ar<EXACT>;
    Scalars *sc = a.sc;
    S.it_done = sc->iter;
    S.first = S.it_done == 0;
    S.rz = 0.0;
    S.rn = 0.0;
    bool stop = false, conv = false, bad = false;
    if (!S.first) {
        S.rz = __dadd_rn(sc->red2[0], sc->red2[1]);
        S.rn = sqrt(__dadd_rn(sc->red2[2], sc->red2[3]));
        conv = S.rn <= sc->tolbn;
        bad = !isfinite(S.rn) || !isfinite(S.rz);
        stop = conv || bad || S.it_done >= sc->maxit;
    }
    S.alpha = S.first ? 0.0 : sc->alpha;
    S.beta = S.first ? 0.0 : __ddiv_rn(S.rz, sc->rho);
    if (!stop) return false;
    // iteration `it_done` is the last: complete its deferred x update and finish
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < d.n; c += stride)
        f.x[c] = A::axpy(S.alpha, __ldg(f.p_old + c), f.x[c]);
    __shared__ bool am_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        am_last = atomicAdd(&sc->ticket[4], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
        __threadfence();
        sc->hist_ring[(S.it_done - 1) % (2 * kMaxChunk)] = S.rn;
        sc->hist_count = S.it_done;
        sc->rn = S.rn;
        sc->status = conv ? ST_OK : (bad ? ST_E_BREAKDOWN : ST_NOT_CONVERGED);
        sc->done = 1;
        sc->ticket[4] = 0u;
    }
    return true;
}

// p.q -> red1 (Dot2 pair); the last block also publishes the history entry and rho of iteration `iter`.
template <bool EXACT, int NT>
__device__ __forceinline__ void pass_a_epilogue(const DevArrays &a, const PassAScalars &S, Acc<EXACT> (&dot)[1]) {
    Scalars *sc = a.sc;
    Acc<EXACT> out[1];
    if (reduce_last<EXACT, NT, 1>(dot, a.partials, &sc->ticket[5], blockIdx.x, gridDim.x, out)) {
        if (threadIdx.x == 0) {
            sc->red1[0] = out[0].p;
            sc->red1[1] = out[0].s;
            if (!S.first) {
                sc->hist_ring[(S.it_done - 1) % (2 * kMaxChunk)] = S.rn;
                sc->hist_count = S.it_done;
                sc->rn = S.rn;
                sc->rho = S.rz;
            }
        }
    }
}

}  // namespace

// ------------------------------------------------------------------------ pass A
template <bool EXACT>
__global__ void __launch_bounds__(kAThreads, 1) k_pass_a(Dims d, DevArrays a, FusedArgs f) {
    using A = Ar<EXACT>;
    extern __shared__ double smem[];   // p ring [3][(bj+2) nr] | D ring [2][bj nr]
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    PassAScalars S;
    if (pass_a_prologue<EXACT>(d, a, f, S)) return;
    const bool first = S.first;
    const double alpha = S.alpha, beta = S.beta;
    const double *__restrict__ pold = f.p_old;
    double *__restrict__ x = f.x;
    const unsigned total = gridDim.x;

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

    pass_a_epilogue<EXACT, kAThreads>(a, S, dot);
}

// ------------------------------------------------------------------------ pass A, TMA variant
// Same arithmetic as k_pass_a.  The grid is a lockstep tiling: block b owns j-tile b % njt (rows
// [jt*nt/njt, (jt+1)*nt/njt)) over the plane chunk b / njt, so blocks on neighbouring tiles march
// through the same planes at the same time and the halo rows both read are L2 hits.  EVERY input
// of a plane is staged by the Tensor Memory Accelerator -- one 1-D bulk copy (cp.async.bulk, i.e.
// UBLKCP) per array and plane, completion counted on an mbarrier -- into a 3-stage shared ring
// two planes ahead of the compute: r, D, p_old on the tile rows plus one halo row each side, x,
// T_r, both T_phi faces on the tile rows, T_theta on the tile rows plus the row above.  No warp
// ever waits on a global load; global memory sees only the bulk copies and the streaming stores
// of p_new, x and q.  Requires nr even (16-byte aligned rows).
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// p + off (elements) as one explicit 64-bit add.  ptxas 12.9 lowered `(base + c0) + plane` feeding a
// bulk-copy source operand to a 32-bit uniform LEA (dropping the high word of the address); forming
// every bulk-copy source address here keeps it 64-bit.
__device__ __forceinline__ const double *gaddr(const double *p, size_t off) {
    const double *r;
    asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(off * sizeof(double)));
    return r;
}

// one stage = all inputs of one plane of the tile (doubles; sext = (H+2) nr, sown = H nr, H = tallest tile)
struct TmaStage {
    double *r, *D, *P;           // ext rows: row 0 = tile row j0 - 1
    double *X, *Tr, *Tplo, *Tphi; // tile rows
    double *Tt;                   // tile rows + the row above
};
__device__ __forceinline__ TmaStage tma_stage(double *base, int sext, int sown) {
    TmaStage t;
    t.r = base;
    t.D = base + sext;
    t.P = base + 2 * sext;
    t.X = base + 3 * sext;
    t.Tr = t.X + sown;
    t.Tplo = t.Tr + sown;
    t.Tphi = t.Tplo + sown;
    t.Tt = t.Tphi + sown;
    return t;
}

}  // namespace

__host__ __device__ size_t tma_stage_doubles(int nr, int hmax) { return (size_t)nr * (3 * (hmax + 2) + 4 * hmax + hmax + 1); }
size_t tma_smem_bytes(int nr, int hmax) {
    return 8 * (3 * tma_stage_doubles(nr, hmax) + (size_t)3 * (hmax + 2) * nr);
}

template <bool EXACT>
__global__ void __launch_bounds__(kTThreads, 1) k_pass_a_tma(Dims d, DevArrays a, FusedArgs f) {
    using A = Ar<EXACT>;
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t bars[3];
    Scalars *sc = a.sc;
    if (*(volatile int *)&sc->done) return;
    PassAScalars S;
    if (pass_a_prologue<EXACT>(d, a, f, S)) return;
    const bool first = S.first;
    const double alpha = S.alpha, beta = S.beta;
    double *__restrict__ x = f.x;

    const int nr = d.nr, nt = d.nt, nloc = d.nloc;
    const size_t plane = d.plane;
    const int njt = f.n_jt;
    const int jt = blockIdx.x % njt, ch = blockIdx.x / njt;
    const int j0 = (int)(((long long)jt * nt) / njt), j1 = (int)(((long long)(jt + 1) * nt) / njt);
    const int ka = (int)(((long long)ch * nloc) / f.nch), kb = (int)(((long long)(ch + 1) * nloc) / f.nch) - 1;
    const int h = j1 - j0;
    const int sext = (f.bj + 2) * nr, sown = f.bj * nr;   // f.bj = tallest tile
    const size_t stage_sz = tma_stage_doubles(nr, f.bj);
    double *ring = smem + 3 * stage_sz;                     // [3][sext] p_new
    const int tid = threadIdx.x;
    uint32_t parity[3] = {0u, 0u, 0u};
    if (tid == 0) {
        for (int q = 0; q < 3; ++q) mbar_init(&bars[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int jr0 = max(j0 - 1, 0), jr1 = min(j1 + 1, nt);   // ext rows present in the grid
    const int roff = jr0 - (j0 - 1);                         // 0, or 1 on the tile at the lower pole
    const int ttrows = min(h + 1, nt - j0);                  // T_theta: tile rows + the row above
    // thread 0: bulk copies of every input of plane k into stage q (kernel-parameter pointers are
    // copied to registers first: no reference to the parameter space inside the helper)
    const double *const gTr = a.Tr, *const gTt = a.Tt, *const gTp = a.Tp, *const gD = a.D;
    const double *const fr = f.r, *const frlo = f.r_lo, *const frhi = f.r_hi;
    const double *const fdlo = f.d_lo, *const fdhi = f.d_hi;
    const double *const fp = f.p_old, *const fplo = f.p_lo, *const fphi = f.p_hi;
    auto issue = [=](int k, int q) {
        const TmaStage sq = tma_stage(smem + (size_t)q * stage_sz, sext, sown);
        const bool own_plane = k >= ka && k <= kb;
        const double *rp = plane_ptr(fr, frlo, frhi, k, nloc, plane);
        const double *dp = plane_ptr(gD, fdlo, fdhi, k, nloc, plane);
        const double *pp = plane_ptr(fp, fplo, fphi, k, nloc, plane);
        const uint32_t eb = (uint32_t)(8 * (size_t)(jr1 - jr0) * nr);
        const uint32_t ob = (uint32_t)(8 * (size_t)h * nr);
        const uint32_t tb = (uint32_t)(8 * (size_t)ttrows * nr);
        const bool wx = own_plane && !first;
        uint32_t bytes = eb * (first ? 2u : 3u);
        if (wx) bytes += ob;
        if (own_plane) bytes += 3u * ob + tb;
        uint64_t *bar = &bars[q];
        mbar_expect_tx(bar, bytes);
        const size_t e0 = (size_t)jr0 * nr;
        bulk_g2s(sq.r + (size_t)roff * nr, gaddr(rp, e0), eb, bar);
        bulk_g2s(sq.D + (size_t)roff * nr, gaddr(dp, e0), eb, bar);
        if (!first) bulk_g2s(sq.P + (size_t)roff * nr, gaddr(pp, e0), eb, bar);
        if (own_plane) {
            const size_t c0 = (size_t)k * plane + (size_t)j0 * nr;
            if (wx) bulk_g2s(sq.X, gaddr(x, c0), ob, bar);
            bulk_g2s(sq.Tr, gaddr(gTr, c0), ob, bar);
            bulk_g2s(sq.Tplo, gaddr(gTp, c0), ob, bar);
            bulk_g2s(sq.Tphi, gaddr(gTp, c0 + plane), ob, bar);
            bulk_g2s(sq.Tt, gaddr(gTt, c0), tb, bar);
        }
    };
    if (tid == 0) {
        issue(ka - 1, 0);
        issue(ka, 1);
    }

    Acc<EXACT> dot[1];
    const int ext_n = (h + 2) * nr, own_n = h * nr;
    const int nsteps = kb - ka + 3;   // planes ka-1 .. kb+1
    for (int kk = 0; kk < nsteps; ++kk) {
        const int k = ka - 1 + kk;
        const int q = kk % 3;
        mbar_wait(&bars[q], parity[q]);
        parity[q] ^= 1u;
        // ---- phase 1: p_new of plane k on the ext rows (shared memory only)
        const bool own_plane = k >= ka && k <= kb;
        double *slot = ring + (size_t)q * sext;
        const TmaStage S1 = tma_stage(smem + (size_t)q * stage_sz, sext, sown);
        for (int e = tid; e < ext_n; e += kTThreads) {
            const int re = (int)f.div_r.div((uint32_t)e);
            const int j = j0 - 1 + re;
            if (j < 0 || j >= nt) continue;
            const double z = __ddiv_rn(S1.r[e], S1.D[e]);
            const double po = first ? 0.0 : S1.P[e];
            const double pn = first ? z : A::axpy(beta, po, z);
            slot[e] = pn;
            if (own_plane && re >= 1 && re <= h) {
                const size_t gc = (size_t)k * plane + (size_t)(j0 - 1) * nr + e;
                f.p_new[gc] = pn;
                if (!first) x[gc] = A::axpy(alpha, po, S1.X[e - nr]);
            }
        }
        __syncthreads();
        // ---- phase 2: stencil of plane ks = k-1 (its stage is (kk-1) % 3, shared memory only)
        const int ks = k - 1;
        if (ks >= ka) {
            const double *sm_ = ring + (size_t)((kk + 1) % 3) * sext;   // plane ks-1
            const double *s0 = ring + (size_t)((kk + 2) % 3) * sext;    // plane ks
            const double *sp = slot;                                     // plane ks+1
            const TmaStage S2 = tma_stage(smem + (size_t)((kk + 2) % 3) * stage_sz, sext, sown);
            const size_t pbase = (size_t)ks * plane + (size_t)j0 * nr;
            for (int o = tid; o < own_n; o += kTThreads) {
                const int jj = (int)f.div_r.div((uint32_t)o);
                const int i = o - jj * nr;
                const int j = j0 + jj;
                const int l = nr + o;
                const double pc = s0[l];
                double s = 0.0;
                if (i > 0) s = A::acc(s, S2.Tr[o], s0[l - 1]);
                if (i < nr - 1) s = A::acc(s, S2.Tr[o + 1], s0[l + 1]);
                if (j > 0) s = A::acc(s, S2.Tt[o], s0[l - nr]);
                if (j < nt - 1) s = A::acc(s, S2.Tt[o + nr], s0[l + nr]);
                s = A::acc(s, S2.Tplo[o], sm_[l]);
                s = A::acc(s, S2.Tphi[o], sp[l]);
                const double qv = A::diag_minus(S2.D[l], pc, s);
                a.q[pbase + o] = qv;
                dot[0].add(pc, qv);
            }
        }
        __syncthreads();
        // ---- refill the stage of plane k-1 (fully consumed) with plane k+2
        if (tid == 0 && kk + 2 < nsteps) {
            fence_proxy_async();
            issue(k + 2, (kk + 2) % 3);
        }
    }
    pass_a_epilogue<EXACT, kTThreads>(a, S, dot);
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

static int sm_count(int device) {
    static int cached_dev = -1, sms = 148;
    if (cached_dev != device) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        cached_dev = device;
    }
    return sms;
}

int fused_blocks(int nr, int nt, int nloc, int bj, int device) {
    const int sms = sm_count(device);
    const size_t smem = fused_smem_bytes(nr, bj);
    cudaFuncSetAttribute(k_pass_a<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_pass_a<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long tiles = (long long)((nt + bj - 1) / bj) * nloc;
    long long b = sms;
    if (b > tiles) b = tiles;
    if (b > kRedBlocks) b = kRedBlocks;
    return (int)b;
}


bool fused_tma_geometry(int nr, int nt, int nloc, int device, int *njt, int *nch, int *hmax) {
    if (nr % 2 != 0) return false;                          // 16-byte aligned rows for the bulk copies
    const size_t limit = 224 * 1024;
    const int sms = sm_count(device);
    double best = -1.0;
    for (int c = 1; c <= nloc && c <= sms; ++c) {
        int t = sms / c;
        if (t > nt) t = nt;
        if (t < 1) break;
        const int h = (nt + t - 1) / t;
        if (tma_smem_bytes(nr, h) > limit) continue;
        const double util = (double)t * c / sms;
        // prefer full occupancy of the SMs, then taller tiles (fewer recomputed halo rows)
        const double score = (util >= 0.97 ? 1.0 : util) * 1000.0 + h;
        if (score > best) {
            best = score;
            *njt = t;
            *nch = c;
            *hmax = h;
        }
    }
    if (best < 0) return false;
    const size_t smem = tma_smem_bytes(nr, *hmax);
    cudaFuncSetAttribute(k_pass_a_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_pass_a_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return true;
}

void launch_pass_a(const Dims &d, const DevArrays &a, const FusedArgs &f, int blocks, bool exact, cudaStream_t st) {
    if (f.tma) {
        const size_t smem = tma_smem_bytes(d.nr, f.bj);
        const int grid = f.n_jt * f.nch;
        if (exact) k_pass_a_tma<true><<<grid, kTThreads, smem, st>>>(d, a, f);
        else k_pass_a_tma<false><<<grid, kTThreads, smem, st>>>(d, a, f);
        return;
    }
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
