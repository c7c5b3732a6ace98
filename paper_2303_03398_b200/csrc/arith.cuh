// arith.cuh -- floating-point policy of the PCG kernels.
//
// EXACT = true (default, MASPCG_OPT_ARITH = 0): every vector operation is one IEEE operation per
// source operation, in the order of the formulas of SURVEY.md 8(c) item 7 (no FMA contraction:
// __dmul_rn / __dadd_rn / __dsub_rn), and every dot product is Dot2 (Ogita, Rump & Oishi 2005:
// error-free TwoProduct + TwoSum, i.e. as accurate as if computed in twice the working precision
// and rounded once) -- reading R24 of DESIGN.md.  The oracle evaluates the same expressions in the
// same order and its dot products with the same Dot2, so both sides compute the same CG iterates:
// the summation order of a Dot2 sum changes its result only when the exact value lies within
// ~n^2 u^2 of a rounding boundary.
//
// EXACT = false (MASPCG_OPT_ARITH = 1): FMA-contracted updates and plain (fixed-tree) sums; cheaper
// in FP64 issue slots, parity only to the tolerance contract.
#pragma once

#include "common.cuh"

namespace maspcg {

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void two_sum(double a, double b, double &x, double &y) {
    x = __dadd_rn(a, b);
    const double z = __dsub_rn(x, a);
    y = __dadd_rn(__dsub_rn(a, __dsub_rn(x, z)), __dsub_rn(b, z));
}

// A Dot2 accumulator: value = p + s, p the running sum of the products' leading parts, s the sum
// of every rounding error (TwoProduct and TwoSum residuals).
template <bool EXACT>
struct Acc {
    double p = 0.0, s = 0.0;
    __device__ __forceinline__ void add(double a, double b) {
        if (EXACT) {
            const double h = __dmul_rn(a, b);
            const double r = fma(a, b, -h);          // exact: a*b = h + r
            double x, q;
            two_sum(p, h, x, q);
            p = x;
            s = __dadd_rn(s, __dadd_rn(q, r));
        } else {
            p = fma(a, b, p);
        }
    }
    __device__ __forceinline__ void add(const Acc &o) {
        if (EXACT) {
            double x, q;
            two_sum(p, o.p, x, q);
            p = x;
            s = __dadd_rn(__dadd_rn(s, o.s), q);
        } else {
            p = __dadd_rn(p, o.p);
        }
    }
    __device__ __forceinline__ double value() const { return EXACT ? __dadd_rn(p, s) : p; }
};

template <bool EXACT>
struct Ar {
    // y + a x
    static __device__ __forceinline__ double axpy(double a, double x, double y) {
        return EXACT ? __dadd_rn(y, __dmul_rn(a, x)) : fma(a, x, y);
    }
    // y - a x
    static __device__ __forceinline__ double ymax(double y, double a, double x) {
        return EXACT ? __dsub_rn(y, __dmul_rn(a, x)) : fma(-a, x, y);
    }
    // s + t u (stencil sum)
    static __device__ __forceinline__ double acc(double s, double t, double u) {
        return EXACT ? __dadd_rn(s, __dmul_rn(t, u)) : fma(t, u, s);
    }
    // d u - s
    static __device__ __forceinline__ double diag_minus(double d, double u, double s) {
        return EXACT ? __dsub_rn(__dmul_rn(d, u), s) : fma(d, u, -s);
    }
};

// Warp-level Dot2 combine (fixed butterfly => deterministic).
template <bool EXACT>
__device__ __forceinline__ void warp_combine(Acc<EXACT> &a) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Acc<EXACT> o;
        o.p = __shfl_xor_sync(0xffffffffu, a.p, off);
        o.s = EXACT ? __shfl_xor_sync(0xffffffffu, a.s, off) : 0.0;
        // combine in a lane-independent order so both partners get identical bits
        const int lane = threadIdx.x & 31;
        if (lane & off) {
            Acc<EXACT> t = o;
            t.add(a);
            a = t;
        } else {
            a.add(o);
        }
    }
}

// Block reduction of N accumulators (fixed tree); thread 0 ends with the totals.
template <bool EXACT, int NT, int N>
__device__ __forceinline__ void block_combine(Acc<EXACT> (&v)[N]) {
    __shared__ double sp[N][NT / 32], ss[N][NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k) warp_combine<EXACT>(v[k]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            sp[k][warp] = v[k].p;
            ss[k][warp] = v[k].s;
        }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            Acc<EXACT> a;
            if (lane < NT / 32) {
                a.p = sp[k][lane];
                a.s = ss[k][lane];
            }
            warp_combine<EXACT>(a);
            v[k] = a;
        }
    }
    __syncthreads();
}

// Per-block partials -> partials[(2k + {0,1}) * kPartialSlots + slot]; the last-arriving block (atomic
// ticket) combines all `total` partials in a fixed order and returns true (thread 0 holds out[]).
template <bool EXACT, int NT, int N>
__device__ __forceinline__ bool reduce_last(Acc<EXACT> (&v)[N], double *partials, unsigned *ticket, unsigned slot,
                                            unsigned total, Acc<EXACT> (&out)[N]) {
    __shared__ bool am_last;
    block_combine<EXACT, NT, N>(v);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            partials[(2 * k) * kPartialSlots + slot] = v[k].p;
            partials[(2 * k + 1) * kPartialSlots + slot] = v[k].s;
        }
        // release (this thread's partial stores) + acquire (every earlier block's, through the RMW chain
        // of the ticket) in one atomic; the block barrier then orders the last block's loads after it
        am_last = atom_add_acq_rel_gpu(ticket, 1u) == total - 1;
    }
    __syncthreads();
    if (!am_last) return false;
    Acc<EXACT> acc[N];
#pragma unroll
    for (int k = 0; k < N; ++k)
        for (unsigned b = threadIdx.x; b < total; b += NT) {
            Acc<EXACT> o;
            o.p = __ldcg(partials + (2 * k) * kPartialSlots + b);
            o.s = __ldcg(partials + (2 * k + 1) * kPartialSlots + b);
            acc[k].add(o);
        }
    block_combine<EXACT, NT, N>(acc);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) out[k] = acc[k];
        *ticket = 0u;
    }
    return true;
}

}  // namespace maspcg
