// p2p_ll.cuh -- the LL ("low latency") word protocol of the peer communicator, shared by peer.cu's
// reduction kernel and the loop kernels of kernels.cu that push / combine their Dot2 pairs themselves.
// Every 8-byte word carries 4 bytes of data and the 32-bit epoch (single-copy atomic), a double travels
// as two words; the staging is double-buffered by epoch parity (peer.cu explains why that suffices).
#pragma once

#include "arith.cuh"
#include "common.cuh"

namespace maspcg {

__device__ __forceinline__ void ll_st(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ll_ld(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ll_recv(const unsigned long long *w, unsigned int e) {
    unsigned long long lo, hi;
    while (((lo = ll_ld(w)) >> 32) != e) __nanosleep(20);
    while (((hi = ll_ld(w + 1)) >> 32) != e) __nanosleep(20);
    return __hiloint2double((int)(unsigned int)hi, (int)(unsigned int)lo);
}
// words of rank `from`'s slot in a stage array, for epoch parity `par`
__device__ __forceinline__ unsigned long long *ll_slot(double *stage, int par, int from) {
    return reinterpret_cast<unsigned long long *>(stage) + ((size_t)par * kP2PMaxRanks + from) * kP2PStage +
           kP2PLLOffset;
}

// one thread: advance the LL epoch and store npairs Dot2 pairs into slot [my rank] of every rank
__device__ __forceinline__ void ll_push_pairs(const DevArrays &a, const double *pairs, int npairs) {
    P2PArea *me = a.p2p;
    const unsigned long long e64 = me->epoch[P2P_LL] + 1;
    me->epoch[P2P_LL] = e64;
    const unsigned int e = (unsigned int)e64;
    const unsigned long long tag = (unsigned long long)e << 32;
    for (int r = 0; r < a.p2p_nranks; ++r) {
        unsigned long long *dst = ll_slot(a.peer_stage[r], (int)(e & 1u), a.p2p_rank);
        for (int t = 0; t < 2 * npairs; ++t) {
            ll_st(dst + 2 * t, tag | (unsigned int)__double2loint(pairs[t]));
            ll_st(dst + 2 * t + 1, tag | (unsigned int)__double2hiint(pairs[t]));
        }
    }
}

// whole block: the values (p + s) of the npairs (<= 2) Dot2 pairs of the current LL epoch into out[],
// combined in rank order exactly as k_dd_combine does.  The threads poll the 4 npairs nranks words in
// parallel (one round trip instead of a chain of them), thread 0 combines.
template <bool EXACT>
__device__ __forceinline__ void ll_block_values(const DevArrays &a, int npairs, double *out) {
    __shared__ unsigned int half[kP2PMaxRanks * 8];
    P2PArea *me = a.p2p;
    const unsigned int e = (unsigned int)(*(volatile unsigned long long *)&me->epoch[P2P_LL]);
    double *mine = &me->stage[0][0][0];
    const int nw = 4 * npairs;   // words per rank
    for (int w = threadIdx.x; w < a.p2p_nranks * nw; w += blockDim.x) {
        const unsigned long long *src = ll_slot(mine, (int)(e & 1u), w / nw) + (w % nw);
        unsigned long long v;
        while (((v = ll_ld(src)) >> 32) != e) __nanosleep(20);
        half[w] = (unsigned int)v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 0; t < npairs; ++t) {
            auto dbl = [&](int r, int k) {   // double k (0: p, 1: s) of pair t from rank r
                const int w = r * nw + 4 * t + 2 * k;
                return __hiloint2double((int)half[w + 1], (int)half[w]);
            };
            if (EXACT) {
                Acc<true> acc;
                for (int r = 0; r < a.p2p_nranks; ++r) {
                    Acc<true> o;
                    o.p = dbl(r, 0);
                    o.s = dbl(r, 1);
                    acc.add(o);
                }
                out[t] = __dadd_rn(acc.p, acc.s);
            } else {
                double v = 0.0;
                for (int r = 0; r < a.p2p_nranks; ++r) v = __dadd_rn(v, dbl(r, 0));
                out[t] = __dadd_rn(v, 0.0);
            }
        }
    }
    __syncthreads();
}

}  // namespace maspcg
