// peer.cu -- the peer-memory communicator (SURVEY.md 8(e) lever 4: in-kernel exchanges instead of NCCL
// calls): every exchange is a kernel that STORES into the receiving rank's memory over NVLink / NVSwitch
// (CUDA IPC mappings of the peers' workspaces, one process and one CUDA context per rank) and
// signals it with a system-scope release flag; the receiver's 1-block wait kernel spins on its flags
// with system-scope acquires.  No host round trip, no NCCL launch: the whole iteration, exchanges
// included, is device work and is captured into the CUDA graphs.
//
//   halo (the phi-slab planes of SURVEY 8(e)):  my first plane -> the left rank's upper halo plane,
//       my last plane -> the right rank's lower halo plane (one push kernel, coalesced 16-byte stores),
//       then wait for the two planes pushed into my halos;
//   all-reduce of the Dot2 pairs of the dot products: a 1-block kernel stores my pairs into slot [rank]
//       of every rank's staging area, signals, waits for all and combines them in rank order (one graph
//       node on the critical path of each PCG reduction); the plain all-gather is the same without the
//       combination;
//   all-reduce(max) of the validation flags: the same with ints, combined in rank order.
//
// Ordering.  Every exchange has a device-side epoch counter (the same sequence of exchanges runs on every
// rank, so the epochs agree); a receiver waits until each sender's flag reaches the epoch.  Staging
// areas are double-buffered by epoch parity: a fast rank can be one gather ahead of a slow one, never
// two (it would first need the slow rank's flag of the gather in between, which that rank sets only
// after it consumed the previous one).  Halo planes are written in place; two exchanges of the same
// buffer are always separated by an all-gather (PCG) or use rotating buffers (super-time-stepping), so
// a plane is never overwritten while its reader still needs it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "arith.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "p2p_ll.cuh"

namespace maspcg {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct Peers {
    unsigned long long *flag[kP2PMaxRanks];   // &peer[r].area->flags[kind][my rank]
    double *dst[kP2PMaxRanks];                // peer data destinations
    int *idst[kP2PMaxRanks];
};

// my first plane -> left's upper halo, my last plane -> right's lower halo; the last block signals
__global__ void k_p2p_push(const double *__restrict__ first, const double *__restrict__ last, double *left_hi,
                           double *right_lo, size_t count, P2PArea *me, unsigned long long *left_flag,
                           unsigned long long *right_flag, int kind, unsigned total) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const bool vec = ((count & 1) == 0) && ((((uintptr_t)first | (uintptr_t)last | (uintptr_t)left_hi |
                                               (uintptr_t)right_lo) & 15) == 0);
    if (vec) {
        for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * t < count; t += stride) {
            if (left_hi) reinterpret_cast<double2 *>(left_hi)[t] = __ldg(reinterpret_cast<const double2 *>(first) + t);
            if (right_lo) reinterpret_cast<double2 *>(right_lo)[t] = __ldg(reinterpret_cast<const double2 *>(last) + t);
        }
    } else {
        for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
            if (left_hi) left_hi[t] = __ldg(first + t);
            if (right_lo) right_lo[t] = __ldg(last + t);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();   // this block's peer stores before its ticket
        if (atomicAdd(&me->ticket[kind], 1u) == total - 1) {
            __threadfence_system();
            const unsigned long long e = me->epoch[kind] + 1;
            me->epoch[kind] = e;
            me->ticket[kind] = 0u;
            if (left_flag) st_release_sys(left_flag, e);
            if (right_flag) st_release_sys(right_flag, e);
        }
    }
}

// wait until my flags f0 (and f1) reach the epoch of `kind`
__global__ void k_p2p_wait(P2PArea *me, const unsigned long long *f0, const unsigned long long *f1, int kind) {
    if (threadIdx.x != 0) return;
    const unsigned long long e = *(volatile unsigned long long *)&me->epoch[kind];
    if (f0)
        while (ld_acquire_sys(f0) < e) __nanosleep(64);
    if (f1)
        while (ld_acquire_sys(f1) < e) __nanosleep(64);
}

// as k_p2p_wait for the halo planes of the PCG loop: returns at once when the solve is done (the p-update
// of the final iteration stores no planes, on every rank alike)
__global__ void k_p2p_wait_loop(P2PArea *me, const int *done, int kind) {
    if (threadIdx.x != 0) return;
    if (*(volatile const int *)done) return;
    const unsigned long long e = *(volatile unsigned long long *)&me->epoch[kind];
    while (ld_acquire_sys(&me->flags[P2P_FROM_LEFT][0]) < e) __nanosleep(64);
    while (ld_acquire_sys(&me->flags[P2P_FROM_RIGHT][0]) < e) __nanosleep(64);
}

// all-gather of `count` doubles (<= kP2PStage): push to every rank's staging slot [rank], signal, wait, copy
__global__ void k_p2p_gather(const double *__restrict__ send, double *__restrict__ recv, int count, P2PArea *me,
                             Peers pe, int rank, int nranks) {
    __shared__ unsigned long long e_s;
    if (threadIdx.x == 0) e_s = me->epoch[P2P_GATHER] + 1;
    __syncthreads();
    const unsigned long long e = e_s;
    const int par = (int)(e & 1);
    for (int r = 0; r < nranks; ++r)
        for (int t = threadIdx.x; t < count; t += blockDim.x)
            pe.dst[r][((size_t)par * kP2PMaxRanks + rank) * kP2PStage + t] = send[t];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        me->epoch[P2P_GATHER] = e;
        for (int r = 0; r < nranks; ++r) st_release_sys(pe.flag[r], e);
        for (int r = 0; r < nranks; ++r)
            while (ld_acquire_sys(&me->flags[P2P_GATHER][r]) < e) __nanosleep(32);
    }
    __syncthreads();
    for (int r = 0; r < nranks; ++r)
        for (int t = threadIdx.x; t < count; t += blockDim.x)
            recv[(size_t)r * count + t] = __ldcg(&me->stage[par][r][t]);
}

// all-reduce of npairs Dot2 (p, s) pairs in place, with the LL ("low latency") protocol of NCCL: every
// 8-byte store carries 4 bytes of data and the 4-byte epoch, so it is single-copy atomic and the receiver
// polls the data itself -- no system-scope fence and no separate flag on the critical path of each PCG
// reduction.  A double travels as two such words.  Staging (reinterpreted as 64-bit words, double-
// buffered by epoch parity as above); then the rank-ordered error-free combination of k_dd_combine.
template <bool EXACT>
__global__ void k_p2p_pairs(double *pairs, int npairs, P2PArea *me, Peers pe, int rank, int nranks) {
    __shared__ unsigned int e_s;
    if (threadIdx.x == 0) {
        e_s = (unsigned int)(me->epoch[P2P_LL] + 1);
        me->epoch[P2P_LL] = me->epoch[P2P_LL] + 1;
    }
    __syncthreads();
    const unsigned int e = e_s;
    const int par = (int)(e & 1u);
    const int count = 2 * npairs;   // doubles
    const size_t slot_words = kP2PStage;   // words per rank slot (the double staging reinterpreted)
    for (int r = 0; r < nranks; ++r) {
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(pe.dst[r]) +
                                  ((size_t)par * kP2PMaxRanks + rank) * slot_words + kP2PLLOffset;
        for (int t = threadIdx.x; t < count; t += blockDim.x) {
            const double v = pairs[t];
            const unsigned long long tag = (unsigned long long)e << 32;
            ll_st(dst + 2 * t, tag | (unsigned int)__double2loint(v));
            ll_st(dst + 2 * t + 1, tag | (unsigned int)__double2hiint(v));
        }
    }
    __syncthreads();
    const unsigned long long *mine = reinterpret_cast<const unsigned long long *>(&me->stage[0][0][0]);
    for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
        if (EXACT) {
            Acc<true> acc;
            for (int r = 0; r < nranks; ++r) {   // rank order: identical bits on every rank
                const unsigned long long *w = mine + ((size_t)par * kP2PMaxRanks + r) * slot_words + kP2PLLOffset + 4 * t;
                Acc<true> o;
                o.p = ll_recv(w, e);
                o.s = ll_recv(w + 2, e);
                acc.add(o);
            }
            pairs[2 * t] = acc.p;
            pairs[2 * t + 1] = acc.s;
        } else {
            double v = 0.0;
            for (int r = 0; r < nranks; ++r)
                v = __dadd_rn(v, ll_recv(mine + ((size_t)par * kP2PMaxRanks + r) * slot_words + kP2PLLOffset + 4 * t, e));
            pairs[2 * t] = v;
            pairs[2 * t + 1] = 0.0;
        }
    }
}

// all-reduce(max) of `count` ints (<= kP2PIStage), in place, rank order
__global__ void k_p2p_max(int *dev, int count, P2PArea *me, Peers pe, int rank, int nranks) {
    __shared__ unsigned long long e_s;
    if (threadIdx.x == 0) e_s = me->epoch[P2P_MAX] + 1;
    __syncthreads();
    const unsigned long long e = e_s;
    const int par = (int)(e & 1);
    for (int r = 0; r < nranks; ++r)
        for (int t = threadIdx.x; t < count; t += blockDim.x)
            pe.idst[r][((size_t)par * kP2PMaxRanks + rank) * kP2PIStage + t] = dev[t];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        me->epoch[P2P_MAX] = e;
        for (int r = 0; r < nranks; ++r) st_release_sys(pe.flag[r], e);
        for (int r = 0; r < nranks; ++r)
            while (ld_acquire_sys(&me->flags[P2P_MAX][r]) < e) __nanosleep(32);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < count; t += blockDim.x) {
        int v = __ldcg(&me->istage[par][0][t]);
        for (int r = 1; r < nranks; ++r) v = max(v, __ldcg(&me->istage[par][r][t]));
        dev[t] = v;
    }
}

}  // namespace

class PeerComm final : public Comm {
   public:
    PeerTable *tab = nullptr;   // owned by the context: regions of every rank (set as workspaces arrive)
    bool capturable() const override { return true; }

    int fail(const char *what, std::string &err, int code = ST_E_INVALID) {
        err = std::string("peer communicator: ") + what;
        return code;
    }
    // the address on rank r of my local address p (both inside one registered region)
    template <typename T>
    T *at(const T *p, int r) const {
        const char *c = reinterpret_cast<const char *>(p);
        for (int g = 0; g < kP2PRegions; ++g) {
            const char *b = tab->base[g][rank];
            if (b && c >= b && c < b + tab->bytes[g] && tab->base[g][r])
                return reinterpret_cast<T *>(tab->base[g][r] + (c - b));
        }
        return nullptr;
    }
    P2PArea *area() const { return tab->area; }
    static int ck(cudaError_t e, std::string &err) {
        if (e == cudaSuccess) return ST_OK;
        err = std::string("peer communicator: ") + cudaGetErrorString(e);
        return ST_E_CUDA;
    }

    int halo_planes(const double *first, const double *last, double *lo_recv, double *hi_recv, size_t count,
                    cudaStream_t st, std::string &err) override {
        double *left_hi = at(hi_recv, left()), *right_lo = at(lo_recv, right());
        unsigned long long *lf = at(&area()->flags[P2P_FROM_RIGHT][0], left());
        unsigned long long *rf = at(&area()->flags[P2P_FROM_LEFT][0], right());
        if (!left_hi || !right_lo || !lf || !rf) return fail("halo buffer outside the registered workspaces", err);
        unsigned g = (unsigned)((count / 2 + 255) / 256);
        if (g < 1) g = 1;
        if (g > 296) g = 296;
        k_p2p_push<<<g, 256, 0, st>>>(first, last, left_hi, right_lo, count, area(), lf, rf, P2P_HALO, g);
        k_p2p_wait<<<1, 32, 0, st>>>(area(), &area()->flags[P2P_FROM_LEFT][0], &area()->flags[P2P_FROM_RIGHT][0],
                                     P2P_HALO);
        return ck(cudaGetLastError(), err);
    }
    int halo_padded(double *buf, size_t pl, int nloc, cudaStream_t st, std::string &err) override {
        return halo_planes(buf + pl, buf + (size_t)nloc * pl, buf, buf + (size_t)(nloc + 1) * pl, pl, st, err);
    }
    int shift_right(const double *send, double *recv, size_t count, cudaStream_t st, std::string &err) override {
        double *right_dst = at(recv, right());
        unsigned long long *rf = at(&area()->flags[P2P_SHIFT][0], right());
        if (!right_dst || !rf) return fail("shift buffer outside the registered workspaces", err);
        unsigned g = (unsigned)((count + 255) / 256);
        if (g < 1) g = 1;
        if (g > 296) g = 296;
        k_p2p_push<<<g, 256, 0, st>>>(send, send, nullptr, right_dst, count, area(), nullptr, rf, P2P_SHIFT, g);
        k_p2p_wait<<<1, 32, 0, st>>>(area(), &area()->flags[P2P_SHIFT][0], nullptr, P2P_SHIFT);
        return ck(cudaGetLastError(), err);
    }
    int allgather(const double *send, double *recv, int count, cudaStream_t st, std::string &err) override {
        if (count > kP2PLLOffset) return fail("all-gather count too large", err);
        Peers pe{};
        for (int r = 0; r < nranks; ++r) {
            pe.dst[r] = at(&area()->stage[0][0][0], r);
            pe.flag[r] = at(&area()->flags[P2P_GATHER][rank], r);
            if (!pe.dst[r] || !pe.flag[r]) return fail("peer area not mapped", err);
        }
        k_p2p_gather<<<1, 256, 0, st>>>(send, recv, count, area(), pe, rank, nranks);
        return ck(cudaGetLastError(), err);
    }
    bool fusable_halo() const override { return true; }
    int halo_targets(double *buf, size_t pl, int nloc, double **hi_dst, double **lo_dst, unsigned long long **flag_hi,
                     unsigned long long **flag_lo, std::string &err) override {
        *hi_dst = at(buf + (size_t)(nloc + 1) * pl, left());   // my first plane -> left's upper halo
        *lo_dst = at(buf, right());                            // my last plane -> right's lower halo
        *flag_hi = at(&area()->flags[P2P_FROM_RIGHT][0], left());
        *flag_lo = at(&area()->flags[P2P_FROM_LEFT][0], right());
        if (!*hi_dst || !*lo_dst || !*flag_hi || !*flag_lo) return fail("halo buffer outside the registered workspaces", err);
        return ST_OK;
    }
    int halo_push(double *buf, size_t pl, int nloc, cudaStream_t st, std::string &err) override {
        double *hi, *lo;
        unsigned long long *fh, *fl;
        if (int s = halo_targets(buf, pl, nloc, &hi, &lo, &fh, &fl, err)) return s;
        unsigned g = (unsigned)((pl / 2 + 255) / 256);
        if (g < 1) g = 1;
        if (g > 296) g = 296;
        k_p2p_push<<<g, 256, 0, st>>>(buf + pl, buf + (size_t)nloc * pl, hi, lo, pl, area(), fh, fl, P2P_HALO, g);
        return ck(cudaGetLastError(), err);
    }
    int halo_wait(const int *done, cudaStream_t st, std::string &err) override {
        k_p2p_wait_loop<<<1, 32, 0, st>>>(area(), done, P2P_HALO);
        return ck(cudaGetLastError(), err);
    }
    bool has_pair_allreduce() const override { return true; }
    int ll_targets(double **stage, std::string &err) override {
        for (int r = 0; r < nranks; ++r) {
            stage[r] = at(&area()->stage[0][0][0], r);
            if (!stage[r]) return fail("peer area not mapped", err);
        }
        return ST_OK;
    }
    int allreduce_pairs(double *pairs, int npairs, bool exact, cudaStream_t st, std::string &err) override {
        if (4 * npairs > kP2PStage - kP2PLLOffset) return fail("pair all-reduce count too large", err);
        Peers pe{};
        for (int r = 0; r < nranks; ++r) {
            pe.dst[r] = at(&area()->stage[0][0][0], r);
            pe.flag[r] = at(&area()->flags[P2P_GATHER][rank], r);
            if (!pe.dst[r] || !pe.flag[r]) return fail("peer area not mapped", err);
        }
        if (exact) k_p2p_pairs<true><<<1, 128, 0, st>>>(pairs, npairs, area(), pe, rank, nranks);
        else k_p2p_pairs<false><<<1, 128, 0, st>>>(pairs, npairs, area(), pe, rank, nranks);
        return ck(cudaGetLastError(), err);
    }
    int allreduce_sum(double *, int, cudaStream_t, std::string &err) override {
        return fail("allreduce_sum is not used by the library", err);
    }
    int allreduce_max(int *dev, int count, cudaStream_t st, std::string &err) override {
        if (count > kP2PIStage) return fail("all-reduce count too large", err);
        Peers pe{};
        for (int r = 0; r < nranks; ++r) {
            pe.idst[r] = at(&area()->istage[0][0][0], r);
            pe.flag[r] = at(&area()->flags[P2P_MAX][rank], r);
            if (!pe.idst[r] || !pe.flag[r]) return fail("peer area not mapped", err);
        }
        k_p2p_max<<<1, 64, 0, st>>>(dev, count, area(), pe, rank, nranks);
        return ck(cudaGetLastError(), err);
    }
};

Comm *make_peer_comm(PeerTable *tab, int rank, int nranks, int *status, std::string &err) {
    if (!tab || nranks < 1 || nranks > kP2PMaxRanks || rank < 0 || rank >= nranks) {
        err = "peer communicator: bad rank / nranks (at most 16 ranks)";
        *status = ST_E_INVALID;
        return nullptr;
    }
    auto *c = new PeerComm();
    c->tab = tab;
    c->rank = rank;
    c->nranks = nranks;
    *status = ST_OK;
    return c;
}

// ---- CUDA IPC plumbing for ranks in different processes ----------------------------------------------
int peer_export(const void *base, size_t bytes, void *out, std::string &err) {
    // the handle names the whole cudaMalloc allocation; the region's offset inside it travels along
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        err = "cuMemGetAddressRange is unavailable";
        return ST_E_CUDA;
    }
    using Fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    CUdeviceptr alloc_base = 0;
    size_t alloc_size = 0;
    if (((Fn)fn)(&alloc_base, &alloc_size, (CUdeviceptr)base) != CUDA_SUCCESS) {
        err = "cuMemGetAddressRange failed on the workspace";
        return ST_E_CUDA;
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)alloc_base);
    if (e != cudaSuccess) {
        err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
        return ST_E_CUDA;
    }
    unsigned long long off = (unsigned long long)((CUdeviceptr)base - alloc_base), sz = bytes;
    memcpy(out, &h, sizeof(h));
    memcpy((char *)out + sizeof(h), &off, 8);
    memcpy((char *)out + sizeof(h) + 8, &sz, 8);
    return ST_OK;
}

int peer_import(const void *in, char **base, size_t *bytes, void **mapping, std::string &err) {
    cudaIpcMemHandle_t h;
    unsigned long long off = 0, sz = 0;
    memcpy(&h, in, sizeof(h));
    memcpy(&off, (const char *)in + sizeof(h), 8);
    memcpy(&sz, (const char *)in + sizeof(h) + 8, 8);
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
        return ST_E_CUDA;
    }
    *mapping = p;
    *base = (char *)p + off;
    *bytes = (size_t)sz;
    return ST_OK;
}

void peer_close(void *mapping) {
    if (mapping) cudaIpcCloseMemHandle(mapping);
}

}  // namespace maspcg
