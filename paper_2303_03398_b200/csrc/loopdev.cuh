// loopdev.cuh -- device helpers shared by the PCG loop kernels (kernels.cu, aniso.cu): programmatic
// dependent launch, the peer-halo release/acquire, cell decomposition, launch ranges and the L2 residency
// policies of the loads and stores.  Product path only (never included by oracle/).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace maspcg {
namespace {

// Programmatic dependent launch (PDL): the loop kernels are launched with programmatic stream
// serialisation, so the next kernel's blocks are scheduled onto SMs as this kernel's blocks retire
// (hiding the launch latency and the reduction tail); griddepcontrol.wait then blocks until the
// previous grid has completed and its memory is visible, before any dependent data is read.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_release_sys64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// peer mode: after a p-update that stored its boundary planes into the neighbours' halos, release them
__device__ __forceinline__ void release_p_halo(const DevArrays &a) {
    fence_acq_rel_sys();
    const unsigned long long e = a.p2p->epoch[P2P_HALO] + 1;
    a.p2p->epoch[P2P_HALO] = e;
    st_release_sys64(a.peer_flag_hi, e);
    st_release_sys64(a.peer_flag_lo, e);
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// peer mode, loop stencil: wait until both neighbours have released this iteration's halo planes (stored
// by their p-updates); every block waits before its first load, so no halo line is cached in L1 early
__device__ __forceinline__ void acquire_p_halo(const DevArrays &a) {
    if (threadIdx.x == 0) {
        const unsigned long long e = *(volatile unsigned long long *)&a.p2p->epoch[P2P_HALO];
        while (ld_acquire_sys64(&a.p2p->flags[P2P_FROM_LEFT][0]) < e) __nanosleep(32);
        while (ld_acquire_sys64(&a.p2p->flags[P2P_FROM_RIGHT][0]) < e) __nanosleep(32);
        // the halo planes may next be read by bulk copies (the async proxy) of the TMA-staged stencils: order
        // the acquired generic-proxy writes before them
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void decompose(const Dims &d, uint32_t c, int &i, int &j, int &k) {
    uint32_t row = d.div_r.div(c);
    i = (int)(c - row * (uint32_t)d.nr);
    uint32_t kk = d.div_t.div(row);
    j = (int)(row - kk * (uint32_t)d.nt);
    k = (int)kk;
}


// ---- L2 residency (Dims::l2_mask).  On a small slab (P = 4, 8) the loop's most-reused arrays fit the
// 126 MB L2: loads and stores of a kept class carry an evict_last policy so they survive the streaming
// of the others between kernels, and their HBM bytes drop out of the iteration -- the "super" scaling
// of PAPER.md:277 (§V-C).  Policies are built per kernel entry (createpolicy, no memory access).
__device__ __forceinline__ uint64_t l2_policy(const Dims &d, int cls) {
    const uint32_t m = (d.l2_mask >> (2 * cls)) & 3u;
    uint64_t pol;
    if (m == L2_KEEP) asm("createpolicy.fractional.L2::evict_last.b64 %0, 0f3F800000;" : "=l"(pol));
    else if (m == L2_KEEP_FRAC)
        asm("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(d.l2_frac));
    else if (m == L2_FIRST) asm("createpolicy.fractional.L2::evict_first.b64 %0, 0f3F800000;" : "=l"(pol));
    else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 0f3F800000;" : "=l"(pol));
    return pol;
}
// read-only for the kernel's lifetime (non-coherent path)
__device__ __forceinline__ double2 ld2h(const double *p, uint64_t pol) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld1h(const double *p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// written by this kernel (coherent path; ordered against the stores by `volatile`)
__device__ __forceinline__ double2 ld2rwh(const double *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol)
                 : "memory");
    return v;
}
// peer-written halo planes: stored over NVLink by a neighbour while this kernel may
// already run, acquired by thread 0 + a block barrier -- read through L2 (ld.global.cg), never .nc
__device__ __forceinline__ double2 ld2coh(const double *p) {
    return __ldcg(reinterpret_cast<const double2 *>(p));
}
__device__ __forceinline__ void st2h(double *p, double a, double b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol)
                 : "memory");
}


}  // namespace
}  // namespace maspcg
