// maspcg.cu -- host driver and C ABI of libmaspcg (include/maspcg.h).
//
// Layers (new-build table): L1 grid/metric precompute on
// the host, L3 NCCL communication (phi-slab halos + scalar all-reduces), L4
// the PCG driver (device-resident scalars, CUDA-graph chunks of iterations,
// host polls a device flag once per chunk), L5 this C ABI.  The kernels are in
// kernels.cu.  Nothing here computes on the host what the hot path computes:
// the host only precomputes O(nr + nt + np) 1-D metric factors (SURVEY 8(a)
// a1, "negligible (setup)").
#include <cuda_runtime.h>
#include <nccl.h>   // ncclGetUniqueId only; the communicator lives in comm.cu

#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/maspcg.h"
#include "cg1.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "fused.cuh"
#include "kernels.cuh"
#include "aniso.cuh"
#include "persist.cuh"
#include "vv.cuh"
#include "wave.cuh"

using namespace maspcg;

namespace {

// Period of phi (R9).  Same literal value as the definition of 2*pi.
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kPi = 3.14159265358979323846;

thread_local std::string g_create_error;

}  // namespace

struct maspcg_ctx {
    int nr = 0, nt = 0, np = 0, rank = 0, nranks = 1, device = 0;
    int k0 = 0, nloc = 0;
    Comm *comm = nullptr;            // nullptr: one rank, periodic wrap done locally
    PeerTable *ptab = nullptr;       // peer-memory communicator: the ranks' workspace regions
    std::string err;

    // grid (host copies of the 1-D metric)
    bool grid_set = false;
    std::vector<double> rf2, hr, dr, R3, C, sinf, ht, dt, sinc, dp_loc, hp_loc;
    bool metric_dirty = true;

    // workspace
    void *ws = nullptr;
    size_t ws_bytes = 0;
    DevArrays a{};
    Dims d{};

    // operator state
    bool coef_set = false, bc_set = false, D_dirty = true;
    int any_shift = 0;
    int bc_in = BC_DIRICHLET, bc_out = BC_NEUMANN0;
    int has_gin = 0, has_gout = 0;

    // streams, events, host snapshots
    cudaStream_t comm_stream = nullptr;
    cudaStream_t cap_stream = nullptr;   // graphs are captured here (the caller's may be the legacy stream)
    cudaEvent_t ev_p = nullptr, ev_halo = nullptr, ev_chunk[2] = {nullptr, nullptr};
    Scalars *snap[2] = {nullptr, nullptr};
    int *vflags_host = nullptr;      // [0..1] synchronous checks; [2..3] set_coefficients (deferred, ev_valid)
    cudaEvent_t ev_valid = nullptr;  // recorded after set_coefficients copied its validation flags
    bool valid_pending = false;      // those flags are not read yet (settle_validation)

    // graph cache (one captured chunk of `chunk` iterations)
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};   // one captured chunk per timing-event set
    const void *g_x = nullptr;
    int g_chunk = 0, g_variant = -1;
    // the device loop (MASPCG_OPT_DEVICE_LOOP): one graph whose conditional WHILE node repeats a chunk until done
    int device_loop = 1;   // MASPCG_OPT_DEVICE_LOOP (used whenever eligible: graphs on, timing off, ...)
    cudaGraphExec_t lexec = nullptr;
    const void *l_x = nullptr;
    int l_chunk = 0, l_variant = -1;
    uint32_t l_l2mask = 0;
    float l_l2frac = 1.f;
    double *hist_host = nullptr;     // pinned [kDevHist]: the device history of a device-loop solve

    // options
    int chunk = 16, use_graphs = 1, timing = 0, path_opt = 0, arith = 0;
    int fuse_halo = 2;   // peer communicator: halo stores fused into the p-update, acquired by the stencil
                         // (MASPCG_OPT_FUSE_HALO)
    int l2_keep = 1;            // MASPCG_OPT_L2_KEEP: L2 residency plan of the three-kernel loop (plan_l2)
    size_t l2_bytes = 0;        // L2 capacity of the device
    size_t l2_persist_max = 0;  // cudaDevAttrMaxPersistingL2CacheSize
    size_t l2_persist_set = 0;  // the persisting set-aside this context requested (0: none)
    size_t l2_plan_bytes = 0;   // bytes the current plan keeps
    uint32_t g_l2mask = 0;      // the plan the cached graphs were captured with
    float g_l2frac = 1.f;
    unsigned persist_grid = 0;   // path 5: co-resident grid of the persistent kernel
    // fused two-pass path geometry (fused.cu)
    int fused_bj = 1, fused_njt = 1, fused_blocks = 1;
    int tma_ok = 0, tma_njt = 1, tma_nch = 1, tma_hmax = 1, use_tma = 0;
    int wave_grid = 1;   // path 3: co-resident grid of k_wave
    cudaEvent_t ev_a = nullptr, ev_ph = nullptr;
    maspcg_stats stats{};
    std::vector<cudaEvent_t> tev;   // timing events [2 sets][6 kinds][2][chunk]: matvec, update, p-update,
                                    // all-reduce #1, all-reduce #2, halo (P > 1)
    int tset = 0;                   // event set of the chunk being enqueued

    // staggered vector viscosity (NEXT-2, vv.cu): its own workspace, 1-D metric and state; the PCG
    // driver runs on it with d / a swapped for the vector Dims dv and arrays (vmode = 1)
    std::vector<double> vv_rf, vv_rce, vv_rhor, vv_dR2, vv_rc2, vv_Cs, vv_dpp, vv_hmp;
    double vv_cap[2] = {0.0, 0.0};
    int vv_grid_ok = 0;              // both poles in t_faces and np >= 2
    void *vv_ws = nullptr;
    size_t vv_ws_bytes = 0;
    VVArrays va{};
    VVDims vd{};
    Dims dv{};
    bool vv_coef_set = false, vv_bc_set = false, vv_dirty = true;
    int vmode = 0;

    // field-aligned anisotropic conduction (NEXT-4, R33, aniso.cu): its own workspace and 1-D edge metric
    std::vector<double> an_gr, an_qr, an_gt, an_cs, an_gts;
    void *an_ws = nullptr;
    size_t an_ws_bytes = 0;
    AnisoArrays xa{};
    bool an_on = false;              // the cross terms are set: solve / apply use the 19-point operator
    bool an_metric_dirty = true;
};

#define SET_ERR(ctx, code, ...)                                              \
    do {                                                                     \
        char _b[512];                                                        \
        snprintf(_b, sizeof(_b), __VA_ARGS__);                               \
        (ctx)->err = _b;                                                     \
        return (maspcg_status)(code);                                        \
    } while (0)

#define CK(ctx, call)                                                                                \
    do {                                                                                             \
        cudaError_t _e = (call);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            SET_ERR(ctx, MASPCG_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, \
                    __LINE__);                                                                       \
    } while (0)

#define RET_IF(st)                       \
    do {                                 \
        maspcg_status _s = (st);         \
        if (_s != MASPCG_OK) return _s;  \
    } while (0)

namespace {

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Workspace layout.  base == nullptr: only computes the size.
size_t layout(const maspcg_ctx *c, char *base, DevArrays *a) {
    const size_t n = (size_t)c->nloc * c->nt * c->nr, plane = (size_t)c->nt * c->nr;
    const size_t rows = (size_t)c->nloc * c->nt;
    size_t off = 0;
    auto take = [&](size_t bytes) -> char * {
        char *p = base ? base + off : nullptr;
        off = align_up(off + bytes, 256);
        return p;
    };
    DevArrays t{};
    t.sc = (Scalars *)take(sizeof(Scalars));
    t.partials = (double *)take(sizeof(double) * 8 * kPartialSlots);
    t.p2p = (P2PArea *)take(sizeof(P2PArea));
    t.gather = (double *)take(sizeof(double) * 8 * kMaxRanks);
    t.hist_dev = (double *)take(sizeof(double) * kDevHist);
    t.P[0] = (double *)take(8 * n);
    t.P[1] = (double *)take(8 * n);
    t.rh = (double *)take(8 * 2 * plane);
    t.dh = (double *)take(8 * 2 * plane);
    t.ph = (double *)take(8 * 2 * plane);
    t.fh = (double *)take(8 * 2 * plane);
    for (int b = 0; b < 4; ++b) t.sy[b] = (double *)take(8 * (n + 2 * plane));   // STS: Y0 and 3 rotating stages
    t.sl0 = (double *)take(8 * n);
    t.cgr = (double *)take(8 * (n + 2 * plane));
    t.cgw = (double *)take(8 * n);
    t.cgs = (double *)take(8 * n);
    const size_t tpp = (size_t)wave_tiles_per_plane((uint32_t)plane);
    t.wave_counter = (unsigned *)take(256);
    t.wave_flags = (unsigned *)take(4 * (size_t)c->nloc);
    t.wave_partials = (double *)take(8 * 2 * tpp * c->nloc);
    t.Tr = (double *)take(8 * n);
    t.TrB = (double *)take(8 * rows);
    t.Tt = (double *)take(8 * n);
    t.Tp = (double *)take(8 * (n + plane));
    t.D = (double *)take(8 * n);
    t.sV = (double *)take(8 * n);
    t.gin = (double *)take(8 * rows);
    t.gout = (double *)take(8 * rows);
    t.p = (double *)take(8 * (n + 2 * plane));
    t.q = (double *)take(8 * n);
    t.r = (double *)take(8 * n);
    t.xs = (double *)take(8 * n);
    t.fs = (double *)take(8 * n);
    t.skr = (double *)take(8 * (rows * (c->nr + 1)));
    t.skt = (double *)take(8 * ((size_t)c->nloc * (c->nt + 1) * c->nr));
    t.skp = (double *)take(8 * n);
    t.ss = (double *)take(8 * n);
    t.rf2 = (double *)take(8 * (c->nr + 1));
    t.hr = (double *)take(8 * (c->nr + 1));
    t.dr = (double *)take(8 * c->nr);
    t.R3 = (double *)take(8 * c->nr);
    t.C = (double *)take(8 * c->nt);
    t.sinf = (double *)take(8 * (c->nt + 1));
    t.ht = (double *)take(8 * (c->nt + 1));
    t.dt = (double *)take(8 * c->nt);
    t.sinc = (double *)take(8 * c->nt);
    t.dp = (double *)take(8 * c->nloc);
    t.hp = (double *)take(8 * c->nloc);
    if (a) *a = t;
    return off;
}

maspcg_status bind_device(maspcg_ctx *c) {
    CK(c, cudaSetDevice(c->device));
    return MASPCG_OK;
}

maspcg_status ensure_metric(maspcg_ctx *c, cudaStream_t st) {
    if (!c->metric_dirty) return MASPCG_OK;
    auto up = [&](double *dst, const std::vector<double> &v) {
        return cudaMemcpyAsync(dst, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, st);
    };
    CK(c, up(c->a.rf2, c->rf2));
    CK(c, up(c->a.hr, c->hr));
    CK(c, up(c->a.dr, c->dr));
    CK(c, up(c->a.R3, c->R3));
    CK(c, up(c->a.C, c->C));
    CK(c, up(c->a.sinf, c->sinf));
    CK(c, up(c->a.ht, c->ht));
    CK(c, up(c->a.dt, c->dt));
    CK(c, up(c->a.sinc, c->sinc));
    CK(c, up(c->a.dp, c->dp_loc));
    CK(c, up(c->a.hp, c->hp_loc));
    CK(c, cudaStreamSynchronize(st));   // host vectors may change with the next set_grid
    c->metric_dirty = false;
    return MASPCG_OK;
}

#define COMM(ctx, call)                                        \
    do {                                                       \
        int _s = (call);                                       \
        if (_s != ST_OK) return (maspcg_status)_s;             \
    } while (0)

maspcg_status halo_padded(maspcg_ctx *c, double *buf, cudaStream_t st) {
    COMM(c, c->comm->halo_padded(buf, c->d.plane, c->nloc, st, c->err));
    return MASPCG_OK;
}

// lo/hi halo planes of a [nloc][nt][nr] array: halo[0] <- left's last plane, halo[1] <- right's first
maspcg_status halo_planes(maspcg_ctx *c, const double *arr, double *halo, cudaStream_t st) {
    const size_t pl = (size_t)c->nt * c->nr;
    COMM(c, c->comm->halo_planes(arr, arr + (size_t)(c->nloc - 1) * pl, halo, halo + pl, pl, st, c->err));
    return MASPCG_OK;
}

bool use_fused(const maspcg_ctx *c) { return !c->vmode && c->path_opt == 2 && c->fused_bj > 0; }
bool use_wave(const maspcg_ctx *c) { return !c->vmode && c->path_opt == 3 && !c->comm; }
bool exact_arith(const maspcg_ctx *c) { return c->arith == 0; }
bool use_cg1(const maspcg_ctx *c) { return !c->vmode && c->path_opt == 4; }
// persistent iteration kernel (persist.cu): single rank, 16-byte pairs
bool use_persist(const maspcg_ctx *c, const void *x) {
    return !c->vmode && c->path_opt == 5 && !c->comm && c->d.vec_ok && (c->nr % 2 == 0) && (((uintptr_t)x & 15) == 0);
}
int graph_key(const maspcg_ctx *c) {
    return (use_fused(c) ? 1 : 0) | (exact_arith(c) ? 2 : 0) | (c->use_tma ? 4 : 0) | (c->d.vec_ok ? 8 : 0) |
           (use_wave(c) ? 32 : 0) | (c->d.pdl ? 64 : 0) | (c->vmode ? 128 : 0) | (use_cg1(c) ? 256 : 0) |
           (c->a.peer_p_lo ? 512 : 0) | (c->a.gather_ranks ? 1024 : 0) | (c->a.p2p_ll ? 2048 : 0) |
           (c->an_on ? (1 << 14) : 0);
}

// Global value of `npairs` Dot2 (p, s) pairs: all-gather the ranks' pairs and combine them in rank
// order with the same error-free arithmetic (identical bits on every rank).
// consumer_combines: the loop kernel that reads the pairs combines the gathered ones itself (gather_ranks).
maspcg_status allreduce_dot2(maspcg_ctx *c, double *pairs, int npairs, cudaStream_t st,
                             bool consumer_combines = false) {
    if (!c->comm) return MASPCG_OK;
    if (c->comm->has_pair_allreduce()) {   // peer communicator: push, wait and combine in one kernel
        COMM(c, c->comm->allreduce_pairs(pairs, npairs, exact_arith(c), st, c->err));
        return MASPCG_OK;
    }
    COMM(c, c->comm->allgather(pairs, c->a.gather, 2 * npairs, st, c->err));
    if (!consumer_combines) launch_dd_combine(c->a.gather, c->nranks, npairs, pairs, exact_arith(c), st);
    return MASPCG_OK;
}

// ------------------------------------------------------------ vector viscosity (NEXT-2, vv.cu)
// Workspace of the field-aligned operator (NEXT-4).  base == nullptr: only computes the size.
size_t aniso_layout(const maspcg_ctx *c, char *base, AnisoArrays *out) {
    const size_t n = (size_t)c->nloc * c->nt * c->nr, plane = (size_t)c->nt * c->nr;
    size_t off = 0;
    auto take = [&](size_t count) -> double * {
        double *p = base ? (double *)(base + off) : nullptr;
        off = align_up(off + 8 * count, 256);
        return p;
    };
    AnisoArrays t{};
    t.Xrt = take(n);
    t.Xrp = take(n + plane);
    t.Xtp = take(n + plane);
    t.D7 = take(n);
    t.gr = take(c->nr);
    t.qr = take(c->nr);
    t.gt = take(c->nt);
    t.cs = take(c->nt);
    t.gts = take(c->nt);
    if (out) *out = t;
    return off;
}

size_t vv_layout(const maspcg_ctx *c, char *base, VVArrays *out) {
    const size_t nr = c->nr, nt = c->nt, nloc = c->nloc, pl1 = nt * nr;
    size_t off = 0;
    auto take = [&](size_t doubles) -> double * {
        double *p = base ? (double *)(base + off) : nullptr;
        off = align_up(off + 8 * doubles, 256);
        return p;
    };
    VVArrays t{};
    t.rf = take(nr + 1); t.rf2 = take(nr + 1); t.hr = take(nr + 1); t.dr = take(nr); t.R3 = take(nr);
    t.rce = take(nr + 2); t.rhor = take(nr + 1); t.dR2 = take(nr); t.rc2 = take(nr);
    t.C = take(nt); t.dt = take(nt); t.ht = take(nt + 1); t.Cs = take(nt + 1); t.sinc = take(nt); t.sinf = take(nt + 1);
    t.dpp = take(nloc + 2); t.hmp = take(nloc + 2); t.cap = take(2);
    t.wc = take((nloc + 2) * pl1); t.Wr = take((nloc + 2) * pl1); t.Wt = take((nloc + 2) * pl1);
    t.WtO = take((nloc + 2) * nt); t.Wp = take(nloc * pl1); t.WpO = take(nloc * nt);
    t.WN = take(nr); t.WS = take(nr);
    t.sM = take(3 * nloc * pl1); t.D = take(3 * nloc * pl1); t.bw = take(3 * nloc * pl1);
    t.E = take((nloc + 2) * pl1); t.TR = take((nloc + 2) * pl1); t.TT = take((nloc + 2) * pl1);
    t.TP = take((nloc + 2) * pl1); t.TTO = take((nloc + 2) * nt); t.TPO = take((nloc + 2) * nt);
    t.nu = take(nloc * pl1); t.s = take(nloc * pl1); t.nulo = take(2 * pl1); t.slo = take(2 * pl1);
    t.gin = take((nloc + 2) * 3 * nt); t.gout = take((nloc + 2) * 3 * nt);
    t.p = take((nloc + 2) * 3 * pl1); t.q = take(3 * nloc * pl1); t.r = take(3 * nloc * pl1);
    t.ring = take(4 * nr); t.nuring = take(4 * nr); t.gather = take((size_t)kMaxRanks * 4 * nr);
    if (out) *out = t;
    return off;
}

// halo planes of a padded [nloc+2][plane] array: received from the neighbours, or the periodic copies
maspcg_status pad_planes(maspcg_ctx *c, double *buf, size_t plane, cudaStream_t st) {
    if (c->comm) {
        COMM(c, c->comm->halo_padded(buf, plane, c->nloc, st, c->err));
        return MASPCG_OK;
    }
    CK(c, cudaMemcpyAsync(buf, buf + (size_t)c->nloc * plane, 8 * plane, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaMemcpyAsync(buf + (size_t)(c->nloc + 1) * plane, buf + plane, 8 * plane, cudaMemcpyDeviceToDevice, st));
    return MASPCG_OK;
}

// global ring pairs: all-gather the ranks' Dot2 pairs [2 nr] and combine them in rank order
maspcg_status vv_ring_allreduce(maspcg_ctx *c, double *ring, cudaStream_t st) {
    if (!c->comm) return MASPCG_OK;
    if (c->comm->has_pair_allreduce()) {
        COMM(c, c->comm->allreduce_pairs(ring, 2 * c->nr, exact_arith(c), st, c->err));
        return MASPCG_OK;
    }
    COMM(c, c->comm->allgather(ring, c->va.gather, 4 * c->nr, st, c->err));
    launch_dd_combine(c->va.gather, c->nranks, 2 * c->nr, ring, exact_arith(c), st);
    return MASPCG_OK;
}

// Lazy assembly after vv_set_coefficients / vv_set_bc_r: metric, coefficients and their halo planes,
// the axis weights (pole-ring means of nu), the Jacobi diagonal and the wall part of the rhs.
maspcg_status ensure_vv(maspcg_ctx *c, cudaStream_t st) {
    if (!c->vv_ws) SET_ERR(c, MASPCG_E_STATE, "vv_set_workspace must precede the vector-viscosity calls");
    if (!c->vv_coef_set || !c->vv_bc_set)
        SET_ERR(c, MASPCG_E_STATE, "vv_set_coefficients and vv_set_bc_r must precede vv_solve / vv_apply");
    if (!c->vv_dirty) return MASPCG_OK;
    VVArrays &a = c->va;
    auto up = [&](double *dst, const double *src, size_t n) {
        return cudaMemcpyAsync(dst, src, 8 * n, cudaMemcpyHostToDevice, st);
    };
    CK(c, up(a.rf, c->vv_rf.data(), c->nr + 1));
    CK(c, up(a.rf2, c->rf2.data(), c->nr + 1));
    CK(c, up(a.hr, c->hr.data(), c->nr + 1));
    CK(c, up(a.dr, c->dr.data(), c->nr));
    CK(c, up(a.R3, c->R3.data(), c->nr));
    CK(c, up(a.rce, c->vv_rce.data(), c->nr + 2));
    CK(c, up(a.rhor, c->vv_rhor.data(), c->nr + 1));
    CK(c, up(a.dR2, c->vv_dR2.data(), c->nr));
    CK(c, up(a.rc2, c->vv_rc2.data(), c->nr));
    CK(c, up(a.C, c->C.data(), c->nt));
    CK(c, up(a.dt, c->dt.data(), c->nt));
    CK(c, up(a.ht, c->ht.data(), c->nt + 1));
    CK(c, up(a.Cs, c->vv_Cs.data(), c->nt + 1));
    CK(c, up(a.sinc, c->sinc.data(), c->nt));
    CK(c, up(a.sinf, c->sinf.data(), c->nt + 1));
    CK(c, up(a.dpp, c->vv_dpp.data(), c->nloc + 2));
    CK(c, up(a.hmp, c->vv_hmp.data(), c->nloc + 2));
    CK(c, up(a.cap, c->vv_cap, 2));
    const size_t pl1 = (size_t)c->nt * c->nr;
    if (c->comm) {   // plane k0 - 1 of nu and s (the cells below the first phi-faces of the slab)
        COMM(c, c->comm->halo_planes(a.nu, a.nu + (size_t)(c->nloc - 1) * pl1, a.nulo, a.nulo + pl1, pl1, st, c->err));
        COMM(c, c->comm->halo_planes(a.s, a.s + (size_t)(c->nloc - 1) * pl1, a.slo, a.slo + pl1, pl1, st, c->err));
    } else {
        CK(c, cudaMemcpyAsync(a.nulo, a.nu + (size_t)(c->nloc - 1) * pl1, 8 * pl1, cudaMemcpyDeviceToDevice, st));
        CK(c, cudaMemcpyAsync(a.slo, a.s + (size_t)(c->nloc - 1) * pl1, 8 * pl1, cudaMemcpyDeviceToDevice, st));
    }
    launch_vv_coef(c->vd, a, st);
    CK(c, cudaGetLastError());
    RET_IF(pad_planes(c, a.wc, pl1, st));
    RET_IF(pad_planes(c, a.Wr, pl1, st));
    RET_IF(pad_planes(c, a.Wt, pl1, st));
    RET_IF(pad_planes(c, a.WtO, c->nt, st));
    launch_vv_ring(c->vd, a, 0, exact_arith(c), st);
    RET_IF(vv_ring_allreduce(c, a.nuring, st));
    launch_vv_axis_weights(c->vd, a, c->np, st);
    launch_vv_diag(c->vd, a, st);
    // bw = A(0; g): the operator on p = 0 with the wall data
    CK(c, cudaMemsetAsync(a.p, 0, 8 * (size_t)(c->nloc + 2) * 3 * pl1, st));
    CK(c, cudaMemsetAsync(a.ring, 0, 8 * 4 * (size_t)c->nr, st));
    launch_vv_matvec(c->vd, a, c->a, a.bw, false, false, true, true, st);
    CK(c, cudaGetLastError());
    if (c->comm) {
        // p (halo planes included) was zeroed above; no rank may push its next planes into our halos before
        // that: one more collective orders every rank's zeroing before any rank's next exchange
        CK(c, cudaMemsetAsync(&c->a.sc->vinvalid, 0, sizeof(int), st));
        COMM(c, c->comm->allreduce_max(&c->a.sc->vinvalid, 1, st, c->err));
    }
    CK(c, cudaStreamSynchronize(st));   // host metric vectors may change with the next set_grid
    c->stats.kernel_launches += 6;
    c->vv_dirty = false;
    return MASPCG_OK;
}

// q = A p of the vector operator: the pole-ring sums (Listing 3's per-radius reduction, all-gathered
// across the phi-slabs) on the caller's stream while the p halo planes travel on the comm stream.
maspcg_status vv_stencil(maspcg_ctx *c, double *y, bool with_dot, bool loop, cudaStream_t st) {
    if (c->comm) {
        CK(c, cudaEventRecord(c->ev_p, st));
        CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_p, 0));
        COMM(c, c->comm->halo_padded(c->va.p, c->d.plane, c->nloc, c->comm_stream, c->err));
        CK(c, cudaEventRecord(c->ev_halo, c->comm_stream));
    }
    launch_vv_ring(c->vd, c->va, 1, exact_arith(c), st);
    // NCCL: the halo send/recv (split communicator, comm stream) and the ring all-gather must not run
    // concurrently -- NCCL does not guarantee progress of two communicators' kernels at once unless both
    // are co-resident; join the halo first.  The peer communicator's exchanges are independent kernels.
    const bool serial = c->comm && !c->comm->has_pair_allreduce();
    if (serial) CK(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    RET_IF(vv_ring_allreduce(c, c->va.ring, st));
    if (c->comm && !serial) CK(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    launch_vv_matvec(c->vd, c->va, c->a, y, with_dot, loop, false, exact_arith(c), st);
    return MASPCG_OK;
}

// Halo exchange of p (P > 1) overlapped with the interior of the stencil on
// the caller's stream; joins before the boundary planes.
cudaError_t record_timing(maspcg_ctx *c, int kern, int which, int it, cudaStream_t st);

// The operator's stencil over `part`: the 7-point kernels, or the 19-point field-aligned one (NEXT-4).
unsigned op_blocks(const maspcg_ctx *c, StencilPart part, const double *y) {
    return c->an_on ? aniso_stencil_blocks(c->d, part, y) : stencil_blocks(c->d, part, y);
}
void op_matvec(const maspcg_ctx *c, const Dims &d, double *y, StencilPart part, bool with_dot, bool loop,
               unsigned slot0, unsigned total, cudaStream_t st) {
    if (c->an_on) launch_aniso_matvec(d, c->a, c->xa, y, part, with_dot, loop, slot0, total, exact_arith(c), st);
    else launch_matvec(d, c->a, y, part, with_dot, loop, slot0, total, exact_arith(c), st);
}

maspcg_status stencil_with_halo(maspcg_ctx *c, double *y, bool with_dot, bool loop, cudaStream_t st, int tslot = -1) {
    if (c->vmode) return vv_stencil(c, y, with_dot, loop, st);
    if (!c->comm) {
        op_matvec(c, c->d, y, StencilPart::Full, with_dot, loop, 0, op_blocks(c, StencilPart::Full, y), st);
        return MASPCG_OK;
    }
    if (loop && c->a.peer_wait) {   // the stencil acquires the pushed halo planes itself
        op_matvec(c, c->d, y, StencilPart::Full, with_dot, loop, 0, op_blocks(c, StencilPart::Full, y), st);
        return MASPCG_OK;
    }
    CK(c, cudaEventRecord(c->ev_p, st));
    CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_p, 0));
    if (tslot >= 0) CK(c, record_timing(c, 5, 0, tslot, c->comm_stream));
    if (loop && c->a.peer_p_lo)   // the p-update already stored its planes into the neighbours' halos
        COMM(c, c->comm->halo_wait(&c->a.sc->done, c->comm_stream, c->err));
    else
        RET_IF(halo_padded(c, c->a.p, c->comm_stream));
    if (tslot >= 0) CK(c, record_timing(c, 5, 1, tslot, c->comm_stream));
    CK(c, cudaEventRecord(c->ev_halo, c->comm_stream));
    const unsigned gi = op_blocks(c, StencilPart::Interior, y);
    const unsigned gb = op_blocks(c, StencilPart::Boundary, y);
    // MASPCG_INTERIOR_PDL=0 launches the interior planes without programmatic dependent launch (its blocks
    // then do not occupy the SMs while the p-update still runs, leaving room for the exchange kernel):
    // measured slower on the P = 8 slab of c3 with the one-rank NCCL communicator (92.6 vs 91.4 us), so
    // PDL stays on.
    static const int ipdl = getenv("MASPCG_INTERIOR_PDL") ? atoi(getenv("MASPCG_INTERIOR_PDL")) : 1;
    Dims di = c->d;
    if (!ipdl) di.pdl = 0;
    op_matvec(c, di, y, StencilPart::Interior, with_dot, loop, 0, gi + gb, st);
    CK(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    op_matvec(c, c->d, y, StencilPart::Boundary, with_dot, loop, gi, gi + gb, st);
    return MASPCG_OK;
}

// The deferred result of the last set_coefficients: E_INVALID (reported by the first call that uses the
// operator) for a negative or non-finite coefficient; the shift-present flag for the singularity check.
maspcg_status settle_validation(maspcg_ctx *c) {
    if (!c->valid_pending) return MASPCG_OK;
    CK(c, cudaEventSynchronize(c->ev_valid));
    c->valid_pending = false;
    if (c->vflags_host[2]) {
        c->coef_set = false;
        SET_ERR(c, MASPCG_E_INVALID, "a diffusion coefficient or the shift is negative or non-finite");
    }
    c->any_shift = c->vflags_host[3];
    return MASPCG_OK;
}

maspcg_status ensure_D(maspcg_ctx *c, cudaStream_t st) {
    RET_IF(settle_validation(c));
    if (!c->coef_set || !c->bc_set)
        SET_ERR(c, MASPCG_E_STATE, "set_coefficients and set_bc_r must precede solve/apply");
    if (!c->D_dirty) return MASPCG_OK;
    if (!c->any_shift && c->bc_in != BC_DIRICHLET && c->bc_out != BC_DIRICHLET)
        SET_ERR(c, MASPCG_E_SINGULAR, "shift is zero everywhere and no r boundary is Dirichlet: A is singular");
    launch_finalize_D(c->d, c->a, c->bc_in, c->bc_out, st);
    CK(c, cudaGetLastError());
    if (c->an_on) launch_aniso_diag(c->d, c->a, c->xa, st);   // D7 kept for the stencil, D = Jacobi diagonal
    if (c->comm) RET_IF(halo_planes(c, c->a.D, c->a.dh, st));   // D of the neighbours' boundary planes
    c->D_dirty = false;
    return MASPCG_OK;
}

int timing_ev_index(int kern, int which, int it, int chunk) { return (kern * 2 + which) * chunk + it; }

// Timing mode 1: events around every hot kernel of every iteration.  Timing mode 2 (sampled): only in
// the middle slot of each chunk -- every chunk-th iteration, in the steady state of the graph's kernel
// pipeline -- so the event records (which serialise the kernels they separate) cost ~1/chunk of their
// full-timing overhead; mode 3: the same in slot 0 (the first kernels of each graph launch).
bool timed_slot(const maspcg_ctx *c, int slot) {
    return c->timing == 1 || (c->timing == 2 && slot == c->chunk / 2) || (c->timing == 3 && slot == 0);
}

// Record timing event (kern, which) of iteration slot `it` of the current set.  External records so
// that, inside a stream capture, the graph node records the event at every replay.
cudaError_t record_timing(maspcg_ctx *c, int kern, int which, int it, cudaStream_t st) {
    const size_t idx = (size_t)c->tset * 12 * c->chunk + timing_ev_index(kern, which, it, c->chunk);
    return cudaEventRecordWithFlags(c->tev[idx], st, cudaEventRecordExternal);
}

// One PCG iteration.  it: index within the chunk (timing).
maspcg_status enqueue_iteration(maspcg_ctx *c, double *x, cudaStream_t st, int it) {
    const bool tm = timed_slot(c, it);
    const bool tc = tm && c->comm;
    if (tm) CK(c, record_timing(c, 0, 0, it, st));
    RET_IF(stencil_with_halo(c, c->a.q, true, true, st, tc ? it : -1));
    if (tm) CK(c, record_timing(c, 0, 1, it, st));
    if (tc) CK(c, record_timing(c, 3, 0, it, st));
    if (!c->a.p2p_ll) RET_IF(allreduce_dot2(c, c->a.sc->red1, 1, st, c->a.gather_ranks > 0));
    if (tc) CK(c, record_timing(c, 3, 1, it, st));
    if (tm) CK(c, record_timing(c, 1, 0, it, st));
    launch_update(c->d, c->a, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 1, 1, it, st));
    if (tc) CK(c, record_timing(c, 4, 0, it, st));
    if (!c->a.p2p_ll) RET_IF(allreduce_dot2(c, c->a.sc->red2, 2, st, c->a.gather_ranks > 0));
    if (tc) CK(c, record_timing(c, 4, 1, it, st));
    if (tm) CK(c, record_timing(c, 2, 0, it, st));
    launch_pupdate(c->d, c->a, x, c->chunk, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 2, 1, it, st));
    return MASPCG_OK;
}

// One PCG iteration of the fused two-pass path (fused.cu).  slot: index within the chunk; the
// chunk length is even so the p buffer parity of a slot is the same in every chunk.
maspcg_status enqueue_iteration_fused(maspcg_ctx *c, double *x, cudaStream_t st, int slot) {
    const bool tm = timed_slot(c, slot);
    const int par = (slot + 1) & 1;
    const size_t pl = c->d.plane;
    FusedArgs f{};
    f.p_old = c->a.P[par ^ 1];
    f.p_new = c->a.P[par];
    f.x = x;
    f.r = c->a.r;
    if (!c->comm) {   // periodic wrap planes of the slab itself (R9)
        const size_t last = (size_t)(c->nloc - 1) * pl;
        f.r_lo = c->a.r + last, f.r_hi = c->a.r;
        f.d_lo = c->a.D + last, f.d_hi = c->a.D;
        f.p_lo = f.p_old + last, f.p_hi = f.p_old;
    } else {
        f.r_lo = c->a.rh, f.r_hi = c->a.rh + pl;
        f.d_lo = c->a.dh, f.d_hi = c->a.dh + pl;
        f.p_lo = c->a.ph, f.p_hi = c->a.ph + pl;
    }
    f.div_r = c->d.div_r;
    if (c->tma_ok && c->use_tma && ((uintptr_t)x & 15) == 0) {   // bulk copies need 16-byte aligned x
        f.tma = 1;
        f.bj = c->tma_hmax;
        f.n_jt = c->tma_njt;
        f.nch = c->tma_nch;
    } else {
        f.tma = 0;
        f.bj = c->fused_bj;
        f.n_jt = c->fused_njt;
        f.nch = 1;
    }
    if (c->comm && slot > 0) CK(c, cudaStreamWaitEvent(st, c->ev_ph, 0));   // p_old halo of slot-1
    if (tm) CK(c, record_timing(c, 0, 0, slot, st));
    launch_pass_a(c->d, c->a, f, c->fused_blocks, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 0, 1, slot, st));
    if (c->comm) {
        // p_it halo for the next pass A, on the communication stream, overlapped with pass B
        CK(c, cudaEventRecord(c->ev_a, st));
        CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_a, 0));
        RET_IF(halo_planes(c, f.p_new, c->a.ph, c->comm_stream));
        CK(c, cudaEventRecord(c->ev_ph, c->comm_stream));
    }
    RET_IF(allreduce_dot2(c, c->a.sc->red1, 1, st));
    if (tm) CK(c, record_timing(c, 1, 0, slot, st));
    launch_pass_b(c->d, c->a, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 1, 1, slot, st));
    RET_IF(allreduce_dot2(c, c->a.sc->red2, 2, st));
    if (c->comm) {
        RET_IF(halo_planes(c, c->a.r, c->a.rh, st));            // r_it halo (critical path, one plane each way)
        if (slot == c->chunk - 1) CK(c, cudaStreamWaitEvent(st, c->ev_ph, 0));   // join before the chunk ends
    }
    if (tm) {   // keep the 3-slot event layout: no third kernel on this path
        CK(c, record_timing(c, 2, 0, slot, st));
        CK(c, record_timing(c, 2, 1, slot, st));
    }
    return MASPCG_OK;
}

// One PCG iteration of the wave path (wave.cu): the r-update of iteration k, then the p-update of
// iteration k and the stencil of iteration k+1 in one flag-ordered kernel (single rank).
maspcg_status enqueue_iteration_wave(maspcg_ctx *c, double *x, cudaStream_t st, int it) {
    const bool tm = timed_slot(c, it);
    if (tm) CK(c, record_timing(c, 1, 0, it, st));
    launch_update(c->d, c->a, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 1, 1, it, st));
    WaveArgs w{};
    w.counter = c->a.wave_counter;
    w.flags = c->a.wave_flags;
    w.tile_partials = c->a.wave_partials;
    w.tpp = wave_tiles_per_plane(c->d.plane);
    w.lag = 3;   // measured best on c3 (4096-cell tiles): a longer lag costs more in L2 misses than it saves in waits
    if (tm) CK(c, record_timing(c, 0, 0, it, st));
    launch_wave(c->d, c->a, w, x, c->chunk, c->wave_grid, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 0, 1, it, st));
    if (tm) {
        CK(c, record_timing(c, 2, 0, it, st));
        CK(c, record_timing(c, 2, 1, it, st));
    }
    return MASPCG_OK;
}

// One iteration of the single-reduction path (cg1.cu): update (with the convergence test of the
// previous iterate), r halo planes overlapped with the interior of the matvec, one all-reduce.
static_assert(offsetof(Scalars, red2) == offsetof(Scalars, red1) + 2 * sizeof(double),
              "the single-reduction path all-reduces red1 and red2 as one block of 3 Dot2 pairs");

maspcg_status cg1_matvec(maspcg_ctx *c, bool loop, cudaStream_t st) {
    DevArrays au = c->a;   // the stencil of the three-kernel path applied to u (padded cgr), writing w
    au.p = c->a.cgr;
    double *w = c->a.cgw;
    if (!c->comm) {
        launch_matvec(c->d, au, w, StencilPart::Full, true, loop, 0, stencil_blocks(c->d, StencilPart::Full, w),
                      exact_arith(c), st);
        return MASPCG_OK;
    }
    CK(c, cudaEventRecord(c->ev_p, st));
    CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_p, 0));
    RET_IF(halo_padded(c, c->a.cgr, c->comm_stream));
    CK(c, cudaEventRecord(c->ev_halo, c->comm_stream));
    const unsigned gi = stencil_blocks(c->d, StencilPart::Interior, w);
    const unsigned gb = stencil_blocks(c->d, StencilPart::Boundary, w);
    launch_matvec(c->d, au, w, StencilPart::Interior, true, loop, 0, gi + gb, exact_arith(c), st);
    CK(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    launch_matvec(c->d, au, w, StencilPart::Boundary, true, loop, gi, gi + gb, exact_arith(c), st);
    return MASPCG_OK;
}

maspcg_status enqueue_iteration_cg1(maspcg_ctx *c, double *x, cudaStream_t st, int it) {
    const bool tm = timed_slot(c, it);
    if (tm) CK(c, record_timing(c, 1, 0, it, st));
    launch_cg1_update(c->d, c->a, x, exact_arith(c), st);
    if (tm) CK(c, record_timing(c, 1, 1, it, st));
    if (tm) CK(c, record_timing(c, 0, 0, it, st));
    RET_IF(cg1_matvec(c, true, st));
    if (tm) CK(c, record_timing(c, 0, 1, it, st));
    RET_IF(allreduce_dot2(c, c->a.sc->red1, 3, st));   // red1 (w.u) and red2 (r.u, r.r) together
    if (tm) {
        CK(c, record_timing(c, 2, 0, it, st));
        CK(c, record_timing(c, 2, 1, it, st));
    }
    return MASPCG_OK;
}

maspcg_status enqueue_any(maspcg_ctx *c, double *x, cudaStream_t st, int slot) {
    if (use_cg1(c)) return enqueue_iteration_cg1(c, x, st, slot);
    if (use_wave(c)) return enqueue_iteration_wave(c, x, st, slot);
    return use_fused(c) ? enqueue_iteration_fused(c, x, st, slot) : enqueue_iteration(c, x, st, slot);
}

maspcg_status enqueue_chunk(maspcg_ctx *c, double *x, cudaStream_t st, int set) {
    c->tset = set;
    if (use_persist(c, x)) {   // one cooperative launch runs the whole chunk
        if (!c->persist_grid) c->persist_grid = persist_grid(c->device);
        CK(c, launch_persist(c->d, c->a, x, c->chunk, c->chunk, c->persist_grid, exact_arith(c), st));
        return MASPCG_OK;
    }
    if (!c->use_graphs) {
        for (int it = 0; it < c->chunk; ++it) RET_IF(enqueue_any(c, x, st, it));
        CK(c, cudaGetLastError());
        return MASPCG_OK;
    }
    const int key = graph_key(c) | (c->timing ? 16 : 0) | (c->timing << 12);
    if (!c->gexec[0] || c->g_x != x || c->g_chunk != c->chunk || c->g_variant != key ||
        c->g_l2mask != c->d.l2_mask || c->g_l2frac != c->d.l2_frac) {
        for (int b = 0; b < 2; ++b) {
            if (c->gexec[b]) {
                cudaGraphExecDestroy(c->gexec[b]);
                c->gexec[b] = nullptr;
            }
        }
        for (int b = 0; b < 2; ++b) {   // identical graphs except for the timing-event set
            c->tset = b;
            cudaGraph_t g = nullptr;
            cudaStream_t cs = c->cap_stream;
            CK(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            maspcg_status s = MASPCG_OK;
            for (int it = 0; it < c->chunk && s == MASPCG_OK; ++it) s = enqueue_any(c, x, cs, it);
            cudaError_t e = cudaStreamEndCapture(cs, &g);
            if (s != MASPCG_OK) {
                if (g) cudaGraphDestroy(g);
                return s;
            }
            CK(c, e);
            cudaError_t ei = cudaGraphInstantiate(&c->gexec[b], g, 0);
            cudaGraphDestroy(g);
            CK(c, ei);
        }
        c->g_x = x;
        c->g_chunk = c->chunk;
        c->g_variant = key;
        c->g_l2mask = c->d.l2_mask;
        c->g_l2frac = c->d.l2_frac;
        c->tset = set;
    }
    CK(c, cudaGraphLaunch(c->gexec[set], st));
    return MASPCG_OK;
}

// The whole PCG loop as ONE graph launch (MASPCG_OPT_DEVICE_LOOP; SURVEY 8(f) NEXT-3 "conditional-graph
// device loop"): a conditional WHILE node whose body is a chunk of iterations followed by k_loop_cond,
// which sets the condition to "not done".  No host round trip until the solve ends.
bool device_loop_ok(const maspcg_ctx *c, const void *x, int maxit) {
    if (!c->device_loop || !c->use_graphs || c->timing || maxit > kDevHist) return false;
    if (use_fused(c) || use_cg1(c) || use_wave(c) || use_persist(c, x)) return false;
    if (!c->comm) return true;
    // exchanges that are kernels only: the peer communicator with the halo acquired by the stencil
    return !c->vmode && c->comm->has_pair_allreduce() && c->fuse_halo == 2;
}

maspcg_status enqueue_device_loop(maspcg_ctx *c, double *x, cudaStream_t st) {
    const int key = graph_key(c);
    if (!c->lexec || c->l_x != x || c->l_chunk != c->chunk || c->l_variant != key || c->l_l2mask != c->d.l2_mask ||
        c->l_l2frac != c->d.l2_frac) {
        if (c->lexec) {
            cudaGraphExecDestroy(c->lexec);
            c->lexec = nullptr;
        }
        cudaGraph_t g = nullptr;
        CK(c, cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
        cudaGraphNode_t node;
        cudaGraphNodeParams cp{};
        if (e == cudaSuccess) {
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
        }
        if (e != cudaSuccess) {
            cudaGraphDestroy(g);
            CK(c, e);
        }
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaStream_t cs = c->cap_stream;
        e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            cudaGraphDestroy(g);
            CK(c, e);
        }
        maspcg_status s = MASPCG_OK;
        for (int it = 0; it < c->chunk && s == MASPCG_OK; ++it) s = enqueue_any(c, x, cs, it);
        if (s == MASPCG_OK) launch_loop_cond(h, c->a.sc, cs);
        cudaGraph_t out = nullptr;
        e = cudaStreamEndCapture(cs, &out);
        if (s != MASPCG_OK || e != cudaSuccess) {
            cudaGraphDestroy(g);
            RET_IF(s);
            CK(c, e);
        }
        e = cudaGraphInstantiate(&c->lexec, g, 0);
        cudaGraphDestroy(g);
        CK(c, e);
        c->l_x = x;
        c->l_chunk = c->chunk;
        c->l_variant = key;
        c->l_l2mask = c->d.l2_mask;
        c->l_l2frac = c->d.l2_frac;
    }
    CK(c, cudaGraphLaunch(c->lexec, st));
    return MASPCG_OK;
}

void accumulate_timing(maspcg_ctx *c, int set, int iters_in_chunk) {
    const size_t base = (size_t)set * 12 * c->chunk;
    const bool comm = c->comm && !use_fused(c) && !use_cg1(c) && !use_wave(c);   // events of enqueue_iteration
    for (int it = 0; it < iters_in_chunk; ++it) {
        if (!timed_slot(c, it)) continue;
        float ms[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < (comm ? 6 : 3); ++k)
            cudaEventElapsedTime(&ms[k], c->tev[base + timing_ev_index(k, 0, it, c->chunk)],
                                 c->tev[base + timing_ev_index(k, 1, it, c->chunk)]);
        c->stats.matvec_ms += ms[0];
        c->stats.matvec_launches += 1;
        c->stats.update_ms += ms[1];
        c->stats.update_launches += 1;
        c->stats.pupdate_ms += ms[2];
        c->stats.pupdate_launches += 1;
        if (comm) {   // the Fig. 3 analogue (MPI time): the two reductions and the halo
            c->stats.comm_ms += ms[3] + ms[4];
            c->stats.halo_ms += ms[5];
            c->stats.comm_launches += 1;
        }
    }
    cudaGetLastError();   // elapsed-time queries of events that were not recorded on this path
}

long long kernels_per_iteration(const maspcg_ctx *c) {
    if (c->vmode) return 5 + (c->comm ? 1 : 0);   // ring sums (+ combine), terms, rows, update, p-update
    if (use_cg1(c)) return 2 + (c->comm ? 2 : 0);   // update, matvec (+ boundary part, combine on P > 1)
    if (use_fused(c) || use_wave(c)) return 2;
    if (!c->comm) return 3;
    // peer communicator, fused: update, p-update, one stencil (halo stores, halo acquire and the Dot2
    // pair exchanges all inside these three kernels)
    if (c->a.peer_wait) return 3;
    // update, p-update, stencil interior + boundary
    long long k = 2 + (stencil_blocks(c->d, StencilPart::Interior, c->a.q) ? 1 : 0) + 1;
    if (c->a.p2p_ll) return k + 1;                   // + the halo wait kernel (pairs inside the kernels)
    if (c->comm->has_pair_allreduce()) return k + 4;   // + halo push and wait, two pair all-reduces
    return k;                                          // NCCL / loopback: their own launches only
}

bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
    const char *pa = (const char *)a, *pb = (const char *)b;
    return pa < pb + nb && pb < pa + na;
}

// L2 residency plan of the three-kernel loop (MASPCG_OPT_L2_KEEP; "super" scaling).  The
// classes in order of HBM bytes saved per resident byte and iteration: D (read by all three kernels),
// p (stencil read, p-update read and write), r (update read and write, p-update read) -- 3 accesses
// each --, then x and q (2), then the face coefficients T_r, T_theta, T_phi (1).  Greedy up to
// `budget` of the L2; the first class that does not fit is kept by the fraction that does.
// MASPCG_L2_MASK / MASPCG_L2_FRAC (explicit plan) and MASPCG_L2_BUDGET override it for A/B runs.
struct L2Range {
    const void *p;
    size_t bytes;
};
int l2_ranges(const maspcg_ctx *c, const double *x, L2Range out[8]) {
    const size_t n8 = 8 * (size_t)c->d.n, pl8 = 8 * (size_t)c->d.plane;
    int m = 0;
    auto add = [&](int cls, const void *p, size_t b) {
        if (((c->d.l2_mask >> (2 * cls)) & 3u) == L2_KEEP || ((c->d.l2_mask >> (2 * cls)) & 3u) == L2_KEEP_FRAC)
            out[m++] = L2Range{p, b};
    };
    add(L2A_D, c->a.D, n8);
    add(L2A_P, c->a.p, n8 + 2 * pl8);
    add(L2A_R, c->a.r, n8);
    add(L2A_X, x, n8);
    add(L2A_Q, c->a.q, n8);
    add(L2A_T, c->a.Tr, n8);
    add(L2A_T, c->a.Tt, n8);
    add(L2A_T, c->a.Tp, n8 + pl8);
    return m;
}

void plan_l2(maspcg_ctx *c, const double *x) {
    c->d.l2_mask = 0u;
    c->d.l2_frac = 1.f;
    c->l2_plan_bytes = 0;
    if (c->vmode) {   // the vector operator: the term rings of its chunked matvec (set at vv_set_workspace)
        c->l2_plan_bytes = (c->l2_keep && c->vd.ring) ? vv_ring_bytes(c->vd, c->vd.ring) : 0;
        return;
    }
    if (!c->l2_keep || c->an_on || use_fused(c) || use_cg1(c) || use_wave(c) || use_persist(c, x)) return;
    if (!c->d.vec_ok || (c->nr % 2) || ((uintptr_t)x & 15)) return;   // the 16-byte kernels carry the hints
    const double n8 = 8.0 * c->d.n, pl8 = 8.0 * c->d.plane;
    if (const char *e = getenv("MASPCG_L2_MASK")) {   // explicit plan (A/B runs)
        c->d.l2_mask = (uint32_t)strtoul(e, nullptr, 0);
        if (const char *f = getenv("MASPCG_L2_FRAC")) c->d.l2_frac = (float)atof(f);
        c->l2_plan_bytes = c->l2_persist_max;
        return;
    }
    // 0.45 of the L2: on the P = 8 slab of c3 keeping D and p (54.7 MB) measured 74.3 us per iteration,
    // D, p and r (81.7 MB, the whole persisting maximum of 82.9 MB) 78.7 and no plan 81.9; on the P = 4
    // slab D alone (54 MB) 143.0 against 150.6 (profiles/r02/l2_residency_plans.txt)
    double budget = 0.45;
    if (const char *e = getenv("MASPCG_L2_BUDGET")) budget = atof(e);
    double cap = budget * (double)c->l2_bytes;
    // evict_last lines are retained only inside the persisting set-aside of the L2
    // (cudaLimitPersistingL2CacheSize); the plan cannot keep more than the device allows there
    if (c->l2_persist_max && cap > (double)c->l2_persist_max) cap = (double)c->l2_persist_max;
    // Whole classes only, greedily: a partly kept class (fractional policy) and a set-aside larger than the
    // kept bytes both measured slower than no plan (the set-aside shrinks the L2 left to the streams).
    const struct {
        int cls;
        double bytes;
    } order[] = {{L2A_D, n8}, {L2A_P, n8 + 2 * pl8}, {L2A_R, n8}, {L2A_X, n8}, {L2A_Q, n8}};
    double kept = 0.0;
    for (const auto &o : order) {
        if (kept + o.bytes > cap) break;
        c->d.l2_mask |= L2_KEEP << (2 * o.cls);
        kept += o.bytes;
    }
    c->l2_plan_bytes = (size_t)kept;
    if (getenv("MASPCG_L2_VERBOSE"))
        fprintf(stderr, "maspcg l2 plan: mask 0x%x kept %.1f MB (L2 %.1f MB, persisting max %.1f MB)\n",
                c->d.l2_mask, kept / 1e6, c->l2_bytes / 1e6, c->l2_persist_max / 1e6);
}

// The persisting set-aside for a plan: exactly its kept bytes (device-wide limit; released at destroy).
void l2_setaside(maspcg_ctx *c) {
    if (!c->d.l2_mask && !c->l2_plan_bytes) return;
    const char *e = getenv("MASPCG_L2_PERSIST");
    if (e && !atoi(e)) return;
    size_t want = c->l2_plan_bytes;
    if (c->l2_persist_max && want > c->l2_persist_max) want = c->l2_persist_max;
    if (!want || c->l2_persist_set == want) return;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) c->l2_persist_set = want;
    else cudaGetLastError();
}

maspcg_status solve_impl(maspcg_ctx *c, const double *rhs, double *x, double tol, int maxit, double *hist,
                         maspcg_info *info, cudaStream_t st) {
    const size_t n = c->d.n;
    if (!rhs || !x) SET_ERR(c, MASPCG_E_INVALID, "rhs and x must be non-NULL");
    if (overlaps(rhs, 8 * n, x, 8 * n)) SET_ERR(c, MASPCG_E_INVALID, "x must not alias rhs");
    if (!(tol >= 0.0) || !std::isfinite(tol)) SET_ERR(c, MASPCG_E_INVALID, "tol must be finite and >= 0");
    if (maxit < 0) SET_ERR(c, MASPCG_E_INVALID, "maxit must be >= 0");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "no workspace");
    RET_IF(c->vmode ? ensure_vv(c, st) : ensure_D(c, st));
    if (c->an_on && !c->vmode && (use_fused(c) || use_cg1(c) || use_wave(c) || use_persist(c, x)))
        SET_ERR(c, MASPCG_E_INVALID, "the field-aligned operator runs on the three-kernel path (MASPCG_OPT_PATH 0 or 1)");
    const bool fused = use_fused(c);
    if (fused && c->ptab)
        SET_ERR(c, MASPCG_E_INVALID, "the fused path (2) is not available with the peer-memory communicator");
    if (fused && (c->chunk & 1)) c->chunk += 1;   // even chunks: fixed p-buffer parity per slot
    if (c->timing) RET_IF(maspcg_set_option(c, MASPCG_OPT_TIMING, c->timing));   // events for this chunk size

    // a3: r0 = b - A x0, z0 = r0/D, p0 = z0, dots; then PCG start scalars
    if (c->vmode) launch_vv_mask(c->vd, x, st);   // the non-unknown slots of x are 0
    launch_fill_p(c->d, c->a, x, st);
    RET_IF(stencil_with_halo(c, c->a.q, false, false, st));
    if (c->vmode)
        launch_vv_setup_residual(c->vd, c->va, c->a, c->d, rhs, exact_arith(c), st);
    else
        launch_setup_residual(c->d, c->a, rhs, c->bc_in == BC_DIRICHLET && c->has_gin,
                              c->bc_out == BC_DIRICHLET && c->has_gout, exact_arith(c), st);
    if (use_cg1(c))   // the local r0.u0 and r0.r0 travel with the first w.u (one all-reduce)
        CK(c, cudaMemcpyAsync(c->a.sc->red2, c->a.sc->red3, 32, cudaMemcpyDeviceToDevice, st));
    RET_IF(allreduce_dot2(c, c->a.sc->red3, 3, st));
    if (fused && c->comm) RET_IF(halo_planes(c, c->a.r, c->a.rh, st));   // r0 halo for pass A
    launch_setup_scalars(c->a, tol, maxit, st);
    const bool cg1 = use_cg1(c);
    // peer communicator, three-kernel path: the p-update stores its boundary planes into the neighbours'
    // halos itself (fused); the loop's stencils only wait.  p0 (from the setup) is pushed once here.
    c->a.peer_p_lo = c->a.peer_p_hi = nullptr;
    c->a.peer_flag_lo = c->a.peer_flag_hi = nullptr;
    c->a.p2p_ll = 0;
    c->a.peer_wait = 0;
    // NCCL / loopback all-gathers in the three-kernel loop: the update and p-update kernels combine the
    // gathered Dot2 pairs themselves (no combine kernel between the all-gather and its consumer)
    c->a.gather_ranks = (c->comm && !c->comm->has_pair_allreduce() && !fused && !cg1 && !use_wave(c)) ? c->nranks : 0;
    if (c->comm && c->comm->fusable_halo() && !fused && !cg1 && !use_wave(c) && !c->vmode && c->fuse_halo) {
        COMM(c, c->comm->halo_targets(c->a.p, c->d.plane, c->nloc, &c->a.peer_p_hi, &c->a.peer_p_lo,
                                      &c->a.peer_flag_hi, &c->a.peer_flag_lo, c->err));
        COMM(c, c->comm->halo_push(c->a.p, c->d.plane, c->nloc, st, c->err));
        // and the two reductions of every iteration: pushed by the producing kernels, combined by the
        // consuming ones (no reduction kernel)
        COMM(c, c->comm->ll_targets(c->a.peer_stage, c->err));
        c->a.p2p_ll = 1;
        c->a.p2p_rank = c->rank;
        c->a.p2p_nranks = c->nranks;
        c->a.gather_ranks = 0;
        c->a.peer_wait = c->fuse_halo == 2 ? 1 : 0;
    }
    if (cg1) {
        // single-reduction start: u0 = z0 (the padded p of the setup, periodic copies included), p = s = 0,
        // then w0 = A u0 and delta0 = w0.u0
        // (halo planes only on a single rank: with a communicator they arrive by the exchange -- a peer may
        // already have pushed them, so they must not be overwritten locally)
        if (c->comm)
            CK(c, cudaMemcpyAsync(c->a.cgr + c->d.plane, c->a.p + c->d.plane, 8 * n, cudaMemcpyDeviceToDevice, st));
        else
            CK(c, cudaMemcpyAsync(c->a.cgr, c->a.p, 8 * (n + 2 * (size_t)c->d.plane), cudaMemcpyDeviceToDevice, st));
        CK(c, cudaMemsetAsync(c->a.q, 0, 8 * n, st));
        CK(c, cudaMemsetAsync(c->a.cgs, 0, 8 * n, st));
        RET_IF(cg1_matvec(c, true, st));
        RET_IF(allreduce_dot2(c, c->a.sc->red1, 3, st));
    }
    if (use_wave(c)) {
        // the wave kernel fuses the stencil of iteration k+1 into the p-update of iteration k, so the
        // first stencil (q = A p0, p0.q) runs here; the dispatch counter and flags start from zero
        CK(c, cudaMemsetAsync(c->a.wave_counter, 0, sizeof(unsigned), st));
        CK(c, cudaMemsetAsync(c->a.wave_flags, 0, sizeof(unsigned) * c->nloc, st));
        launch_matvec(c->d, c->a, c->a.q, StencilPart::Full, true, true, 0,
                      stencil_blocks(c->d, StencilPart::Full, c->a.q), exact_arith(c), st);
    }
    CK(c, cudaGetLastError());
    long long launched = 4 + (c->comm ? 1 : 0);
    plan_l2(c, x);
    l2_setaside(c);

    // PCG loop: chunks of `chunk` iterations, one speculative chunk in flight.
    CK(c, cudaMemcpyAsync(c->snap[0], c->a.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
    CK(c, cudaEventRecord(c->ev_chunk[0], st));
    CK(c, cudaEventSynchronize(c->ev_chunk[0]));   // start scalars (also orders the pinned writes above)
    Scalars s0 = *c->snap[0];
    if (hist) hist[0] = s0.hist0;
    int status = s0.status, iters = 0, hdone = 0;
    const int ring = (fused || cg1) ? 2 * kMaxChunk : c->chunk;
    double rn = s0.rn, bn = s0.bn;
    bool done = s0.done != 0;
    const bool pipelined = true;   // timing events alternate between two sets, like the snapshots
    int issued = 0, cur = 0;
    auto issue = [&](int b) -> maspcg_status {
        RET_IF(enqueue_chunk(c, x, st, b));
        CK(c, cudaMemcpyAsync(c->snap[b], c->a.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
        CK(c, cudaEventRecord(c->ev_chunk[b], st));
        issued += c->chunk;
        launched += use_persist(c, x) ? 1 : (long long)c->chunk * kernels_per_iteration(c);
        return MASPCG_OK;
    };
    if (!done && device_loop_ok(c, x, maxit)) {   // the whole loop in one graph launch
        if (!c->hist_host) CK(c, cudaMallocHost((void **)&c->hist_host, sizeof(double) * kDevHist));
        c->a.hist_dev_on = 1;
        maspcg_status ls = enqueue_device_loop(c, x, st);
        c->a.hist_dev_on = 0;
        RET_IF(ls);
        CK(c, cudaMemcpyAsync(c->snap[0], c->a.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
        CK(c, cudaMemcpyAsync(c->hist_host, c->a.hist_dev, sizeof(double) * (size_t)maxit, cudaMemcpyDeviceToHost, st));
        CK(c, cudaEventRecord(c->ev_chunk[0], st));
        CK(c, cudaEventSynchronize(c->ev_chunk[0]));
        const Scalars &s = *c->snap[0];
        if (hist)
            for (int k = 1; k <= s.iter; ++k) hist[k] = c->hist_host[k - 1];
        iters = s.iter;
        status = s.status;
        rn = s.rn;
        done = true;
        const long long bodies = (iters + c->chunk - 1) / c->chunk > 0 ? (iters + c->chunk - 1) / c->chunk : 1;
        launched += bodies * (c->chunk * kernels_per_iteration(c) + 1);
    }
    if (!done) {
        RET_IF(issue(cur));
        while (true) {
            bool next_issued = false;
            if (pipelined && issued < maxit) {
                RET_IF(issue(cur ^ 1));
                next_issued = true;
            }
            CK(c, cudaEventSynchronize(c->ev_chunk[cur]));
            const Scalars &s = *c->snap[cur];
            if (c->timing) accumulate_timing(c, cur, s.iter - iters);
            const int hnew = (fused || cg1) ? s.hist_count : s.iter;
            if (hist)
                for (int k = hdone + 1; k <= hnew; ++k) hist[k] = s.hist_ring[(k - 1) % ring];
            hdone = hnew;
            iters = s.iter;
            status = s.status;
            rn = s.rn;
            if (s.done) {
                if (next_issued) CK(c, cudaEventSynchronize(c->ev_chunk[cur ^ 1]));
                break;
            }
            if (!next_issued) {
                if (issued >= maxit + 2 * c->chunk + 2) SET_ERR(c, MASPCG_E_CUDA, "PCG loop did not terminate");
                RET_IF(issue(cur ^ 1));
            }
            cur ^= 1;
        }
    }
    launch_zero_x_if(c->d, c->a, x, st);
    launched += 1;
    if (c->d.l2_mask) {   // the kept lines go back to the normal eviction priority
        L2Range rs[8];
        const int m = l2_ranges(c, x, rs);
        for (int i = 0; i < m; ++i) launch_l2_demote(rs[i].p, rs[i].bytes, st);
        launched += m;
        c->d.l2_mask = 0u;
        c->d.l2_frac = 1.f;
    }
    if (c->vmode && c->l2_plan_bytes) {   // the vector operator's term rings
        const size_t rb = vv_ring_bytes(c->vd, c->vd.ring) / 4;
        for (double *t : {c->va.E, c->va.TR, c->va.TT, c->va.TP}) launch_l2_demote(t, rb, st);
        launched += 4;
    }
    c->a.peer_p_lo = c->a.peer_p_hi = nullptr;   // only the loop's p-updates store into the neighbours
    c->a.peer_flag_lo = c->a.peer_flag_hi = nullptr;
    c->a.gather_ranks = 0;
    c->a.p2p_ll = 0;
    CK(c, cudaGetLastError());
    CK(c, cudaStreamSynchronize(st));
    if (status < 0 && status != MASPCG_E_BREAKDOWN) status = MASPCG_E_CUDA;
    c->stats.kernel_launches += launched;
    c->stats.path = c->vmode ? 5 : (cg1 ? 4 : (use_wave(c) ? 3 : (fused ? 2 : (use_persist(c, x) ? 6 : 1))));
    c->stats.solves += 1;
    c->stats.iterations += iters;
    if (info) {
        info->iters = iters;
        info->bnorm = bn;
        info->rnorm = (bn == 0.0) ? 0.0 : rn;
        info->rel_resid = (bn == 0.0 || !std::isfinite(bn)) ? 0.0 : rn / bn;
    }
    if (status == MASPCG_E_BREAKDOWN) c->err = "PCG breakdown: p.Ap <= 0 or a non-finite residual";
    return (maspcg_status)status;
}

// Runs the PCG driver on the vector operator: the flat kernels see n = nloc * 3 nt * nr values with
// 3 nt * nr per phi-plane, and p, q, r, D are the vector arrays.
struct VModeGuard {
    maspcg_ctx *c;
    Dims d;
    DevArrays a;
    explicit VModeGuard(maspcg_ctx *cc) : c(cc), d(cc->d), a(cc->a) {
        Dims v = cc->d;
        v.nt = 3 * cc->nt;
        v.plane = (uint32_t)(3 * (size_t)cc->nt * cc->nr);
        v.n = (uint32_t)((size_t)cc->nloc * v.plane);
        v.div_t = make_fastdiv((uint32_t)v.nt);
        cc->dv = v;
        cc->d = v;
        cc->a.p = cc->va.p;
        cc->a.q = cc->va.q;
        cc->a.r = cc->va.r;
        cc->a.D = cc->va.D;
        cc->vmode = 1;
    }
    ~VModeGuard() {
        c->d = d;
        c->a = a;
        c->vmode = 0;
    }
};

}  // namespace

// ================================================================ C ABI
extern "C" {

const char *maspcg_version(void) { return "maspcg 0.1 sm_100a fp64"; }

maspcg_status maspcg_get_unique_id(void *out) {
    if (!out) return MASPCG_E_INVALID;
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_create_error = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
        return MASPCG_E_NCCL;
    }
    static_assert(sizeof(ncclUniqueId) == MASPCG_NCCL_UNIQUE_ID_BYTES, "unique id size");
    memcpy(out, &id, sizeof(id));
    return MASPCG_OK;
}

static maspcg_status create_impl(int nr, int nt, int np, int rank, int nranks, const void *nccl_unique_id,
                                 void *group, int cuda_device, maspcg_ctx **out, bool peer = false) {
    if (!out) return MASPCG_E_INVALID;
    *out = nullptr;
    auto fail = [](maspcg_status s, const char *m) {
        g_create_error = m;
        return s;
    };
    if (nr < 1 || nt < 1 || np < 1) return fail(MASPCG_E_INVALID, "nr, nt, np must be >= 1");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(MASPCG_E_INVALID, "bad rank / nranks");
    if (np % nranks != 0) return fail(MASPCG_E_INVALID, "np must be divisible by nranks");
    if (!peer && !group && nranks > 1 && !nccl_unique_id)
        return fail(MASPCG_E_INVALID, "nccl_unique_id must be given when nranks > 1");
    if (peer && nranks > kP2PMaxRanks) return fail(MASPCG_E_INVALID, "the peer communicator supports at most 16 ranks");
    // the all-gather scratch of the Dot2 all-reduces (a.gather, va.gather) holds kMaxRanks rank slots
    if (nranks > kMaxRanks) return fail(MASPCG_E_INVALID, "at most 16 ranks (all-gather scratch of the reductions)");
    if (peer && group)
        return fail(MASPCG_E_INVALID, "peer mode needs one CUDA context per rank (processes, CUDA IPC): ranks sharing "
                                      "a context could spin on each other inside one device");
    const long long nloc = np / nranks;
    if ((nloc + 2) * (long long)nt * nr >= (1ll << 31))
        return fail(MASPCG_E_INVALID, "local slab too large (>= 2^31 cells with halos)");
    maspcg_ctx *c = new maspcg_ctx();
    c->nr = nr;
    c->nt = nt;
    c->np = np;
    c->rank = rank;
    c->nranks = nranks;
    c->device = cuda_device;
    c->nloc = (int)nloc;
    c->k0 = rank * (int)nloc;
    cudaError_t e = cudaSetDevice(cuda_device);
    // the communication stream at the highest priority: its exchange kernels (NCCL send/recv, peer pushes)
    // are dispatched ahead of pending stencil blocks
    int prio_lo = 0, prio_hi = 0;
    if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_p, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ph, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_chunk[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_chunk[1], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocHost((void **)&c->snap[0], sizeof(Scalars));
    if (e == cudaSuccess) e = cudaMallocHost((void **)&c->snap[1], sizeof(Scalars));
    if (e == cudaSuccess) e = cudaMallocHost((void **)&c->vflags_host, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_valid, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        g_create_error = std::string("CUDA initialisation failed: ") + cudaGetErrorString(e);
        maspcg_destroy(c);
        return MASPCG_E_CUDA;
    }
    if (peer) {   // peer-memory communicator (peer.cu), also at nranks == 1 (pushes to itself)
        int st = ST_OK;
        c->ptab = new PeerTable();
        c->comm = make_peer_comm(c->ptab, rank, nranks, &st, g_create_error);
        if (!c->comm) {
            maspcg_destroy(c);
            return (maspcg_status)st;
        }
    } else if (nranks > 1 || group || nccl_unique_id) {   // a communicator (also at nranks == 1 when one is given)
        int st = ST_OK;
        c->comm = group ? make_loopback_comm((LoopbackGroup *)group, rank, nranks, &st, g_create_error)
                        : make_nccl_comm(nccl_unique_id, rank, nranks, &st, g_create_error);
        if (!c->comm) {
            maspcg_destroy(c);
            return (maspcg_status)st;
        }
        if (!c->comm->capturable()) c->use_graphs = 0;
    }
    c->d.nr = nr;
    c->d.nt = nt;
    c->d.nloc = c->nloc;
    c->d.k0 = c->k0;
    c->d.plane = (uint32_t)((size_t)nt * nr);
    c->d.n = (uint32_t)((size_t)c->nloc * nt * nr);
    c->d.div_r = make_fastdiv((uint32_t)nr);
    c->d.div_t = make_fastdiv((uint32_t)nt);
    c->d.periodic_local = c->comm ? 0 : 1;
    c->d.vec_ok = 1;
    c->d.pdl = 1;
    {
        int l2 = 0, pmax = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, cuda_device);
        cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, cuda_device);
        c->l2_bytes = (size_t)(l2 > 0 ? l2 : 0);
        c->l2_persist_max = (size_t)(pmax > 0 ? pmax : 0);
    }
    c->fused_bj = fused_bj(nr, nt);   // 0: nr too large for one register batch per thread -> three kernels
    if (c->fused_bj > 0) {
        c->fused_njt = (nt + c->fused_bj - 1) / c->fused_bj;
        c->fused_blocks = fused_blocks(nr, nt, c->nloc, c->fused_bj, cuda_device);
    }
    c->wave_grid = wave_grid(cuda_device);
    c->tma_ok = fused_tma_geometry(nr, nt, c->nloc, cuda_device, &c->tma_njt, &c->tma_nch, &c->tma_hmax) ? 1 : 0;
    *out = c;
    return MASPCG_OK;
}

maspcg_status maspcg_create(int nr, int nt, int np, int rank, int nranks, const void *nccl_unique_id,
                            int cuda_device, maspcg_ctx **out) {
    return create_impl(nr, nt, np, rank, nranks, nccl_unique_id, nullptr, cuda_device, out);
}

maspcg_status maspcg_create_peer(int nr, int nt, int np, int rank, int nranks, void *group, int cuda_device,
                                 maspcg_ctx **out) {
    return create_impl(nr, nt, np, rank, nranks, nullptr, group, cuda_device, out, true);
}

maspcg_status maspcg_loopback_group_create(int nranks, void **group) {
    if (!group) return MASPCG_E_INVALID;
    *group = loopback_group_create(nranks);
    if (!*group) {
        g_create_error = "loopback group size must be in [1, 16]";
        return MASPCG_E_INVALID;
    }
    return MASPCG_OK;
}

maspcg_status maspcg_loopback_group_destroy(void *group) {
    loopback_group_destroy((LoopbackGroup *)group);
    return MASPCG_OK;
}

maspcg_status maspcg_create_loopback(int nr, int nt, int np, int rank, int nranks, void *group, int cuda_device,
                                     maspcg_ctx **out) {
    if (!group) {
        g_create_error = "loopback group must be non-NULL";
        return MASPCG_E_INVALID;
    }
    return create_impl(nr, nt, np, rank, nranks, nullptr, group, cuda_device, out);
}

maspcg_status maspcg_destroy(maspcg_ctx *c) {
    if (!c) return MASPCG_OK;
    cudaSetDevice(c->device);
    // captured graphs hold NCCL work of the communicator: release them (after the device is idle)
    // before the communicator is finalised, or ncclCommDestroy waits on them forever
    cudaDeviceSynchronize();
    for (int b = 0; b < 2; ++b)
        if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
    c->gexec[0] = c->gexec[1] = nullptr;
    if (c->lexec) cudaGraphExecDestroy(c->lexec);
    c->lexec = nullptr;
    if (c->hist_host) cudaFreeHost(c->hist_host);
    delete c->comm;
    if (c->ptab) {
        for (int g = 0; g < kP2PRegions; ++g)
            for (int r = 0; r < kP2PMaxRanks; ++r) peer_close(c->ptab->mapping[g][r]);
        delete c->ptab;
        c->ptab = nullptr;
    }
    for (cudaEvent_t e : c->tev) cudaEventDestroy(e);
    if (c->ev_p) cudaEventDestroy(c->ev_p);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->ev_a) cudaEventDestroy(c->ev_a);
    if (c->ev_ph) cudaEventDestroy(c->ev_ph);
    for (int b = 0; b < 2; ++b) {
        if (c->ev_chunk[b]) cudaEventDestroy(c->ev_chunk[b]);
        if (c->snap[b]) cudaFreeHost(c->snap[b]);
    }
    if (c->vflags_host) cudaFreeHost(c->vflags_host);
    if (c->ev_valid) cudaEventDestroy(c->ev_valid);
    if (c->l2_persist_set) {   // release the persisting L2 set-aside this context requested
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    }
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    delete c;
    return MASPCG_OK;
}

const char *maspcg_last_error(const maspcg_ctx *c) { return c ? c->err.c_str() : g_create_error.c_str(); }

maspcg_status maspcg_set_grid(maspcg_ctx *c, const double *rf, const double *tf, const double *pf) {
    if (!c) return MASPCG_E_INVALID;
    if (!rf || !tf || !pf) SET_ERR(c, MASPCG_E_INVALID, "face arrays must be non-NULL");
    const int nr = c->nr, nt = c->nt, np = c->np;
    // R1, R9: validity of the grid
    if (!(rf[0] > 0.0)) SET_ERR(c, MASPCG_E_INVALID, "r_faces[0] must be > 0");
    for (int i = 0; i < nr; ++i)
        if (!(rf[i + 1] > rf[i])) SET_ERR(c, MASPCG_E_INVALID, "r_faces must increase strictly");
    for (int j = 0; j < nt; ++j)
        if (!(tf[j + 1] > tf[j])) SET_ERR(c, MASPCG_E_INVALID, "t_faces must increase strictly");
    for (int k = 0; k < np; ++k)
        if (!(pf[k + 1] > pf[k])) SET_ERR(c, MASPCG_E_INVALID, "p_faces must increase strictly");
    if (!(tf[0] >= 0.0) || !(tf[nt] <= kPi)) SET_ERR(c, MASPCG_E_INVALID, "t_faces must lie in [0, pi]");
    if (!(std::fabs((pf[np] - pf[0]) - kTwoPi) <= 1e-12 * kTwoPi))
        SET_ERR(c, MASPCG_E_INVALID, "p_faces must span exactly 2*pi (periodic phi)");

    // a1: 1-D metric (R2, R3).  Centres are face midpoints; distances between
    // centres (half cells at the r walls, periodic wrap in phi).
    std::vector<double> rc(nr), tc(nt), pc(np), dpg(np), hpg(np);
    c->rf2.assign(nr + 1, 0.0);
    c->hr.assign(nr + 1, 0.0);
    c->dr.assign(nr, 0.0);
    c->R3.assign(nr, 0.0);
    for (int i = 0; i <= nr; ++i) c->rf2[i] = rf[i] * rf[i];
    for (int i = 0; i < nr; ++i) {
        rc[i] = 0.5 * (rf[i] + rf[i + 1]);
        c->dr[i] = rf[i + 1] - rf[i];
        // (r1^3 - r0^3)/3 = dr (r1^2 + r1 r0 + r0^2)/3
        c->R3[i] = c->dr[i] * (rf[i + 1] * rf[i + 1] + rf[i + 1] * rf[i] + rf[i] * rf[i]) / 3.0;
    }
    c->hr[0] = rc[0] - rf[0];
    for (int i = 1; i < nr; ++i) c->hr[i] = rc[i] - rc[i - 1];
    c->hr[nr] = rf[nr] - rc[nr - 1];

    c->C.assign(nt, 0.0);
    c->dt.assign(nt, 0.0);
    c->sinc.assign(nt, 0.0);
    c->sinf.assign(nt + 1, 0.0);
    c->ht.assign(nt + 1, 0.0);
    for (int j = 0; j < nt; ++j) {
        tc[j] = 0.5 * (tf[j] + tf[j + 1]);
        c->dt[j] = tf[j + 1] - tf[j];
        // C_j = cos t_j - cos t_{j+1} = 2 sin(tc_j) sin(dt_j / 2)
        c->C[j] = 2.0 * std::sin(tc[j]) * std::sin(0.5 * c->dt[j]);
        c->sinc[j] = std::sin(tc[j]);
    }
    for (int j = 1; j < nt; ++j) c->ht[j] = tc[j] - tc[j - 1];
    for (int j = 0; j <= nt; ++j) c->sinf[j] = std::sin(tf[j]);

    for (int k = 0; k < np; ++k) {
        pc[k] = 0.5 * (pf[k] + pf[k + 1]);
        dpg[k] = pf[k + 1] - pf[k];
    }
    for (int k = 0; k + 1 < np; ++k) hpg[k] = pc[k + 1] - pc[k];
    hpg[np - 1] = (pc[0] + kTwoPi) - pc[np - 1];
    c->dp_loc.assign(dpg.begin() + c->k0, dpg.begin() + c->k0 + c->nloc);
    c->hp_loc.assign(hpg.begin() + c->k0, hpg.begin() + c->k0 + c->nloc);

    // field-aligned conduction edge metric (NEXT-4, R33): the expressions of reading R33
    c->an_gr.assign(nr, 0.0);
    c->an_qr.assign(nr, 0.0);
    c->an_gt.assign(nt, 0.0);
    c->an_cs.assign(nt, 0.0);
    c->an_gts.assign(nt, 0.0);
    for (int i = 1; i < nr; ++i) c->an_gr[i] = (rc[i] * rc[i] + rc[i] * rc[i - 1] + rc[i - 1] * rc[i - 1]) / (3.0 * rf[i]);
    for (int i = 0; i < nr; ++i) c->an_qr[i] = c->R3[i] / (rc[i] * rc[i]);
    for (int j = 1; j < nt; ++j) {
        c->an_gt[j] = 2.0 * std::sin(0.5 * (tc[j - 1] + tc[j])) * std::sin(0.5 * c->ht[j]) / c->ht[j];
        c->an_gts[j] = c->an_gt[j] / c->sinf[j];
    }
    for (int j = 0; j < nt; ++j) c->an_cs[j] = 2.0 * std::sin(0.5 * c->dt[j]);
    c->an_metric_dirty = true;

    // vector-viscosity metric (NEXT-2, R27): the expressions of the vector oracle's grid
    c->vv_grid_ok = (tf[0] == 0.0 && std::fabs(tf[nt] - kPi) <= 1e-12 && np >= 2) ? 1 : 0;
    c->vv_rf.assign(rf, rf + nr + 1);
    c->vv_rce.assign(nr + 2, 0.0);
    c->vv_rce[0] = rf[0];
    for (int i = 0; i < nr; ++i) c->vv_rce[i + 1] = rc[i];
    c->vv_rce[nr + 1] = rf[nr];
    c->vv_rhor.assign(nr + 1, 0.0);
    for (int e = 0; e <= nr; ++e) c->vv_rhor[e] = c->hr[e] * (0.5 * (c->vv_rce[e] + c->vv_rce[e + 1]));
    c->vv_dR2.assign(nr, 0.0);
    c->vv_rc2.assign(nr, 0.0);
    for (int i = 0; i < nr; ++i) {
        c->vv_dR2[i] = rc[i] * c->dr[i];
        c->vv_rc2[i] = rc[i] * rc[i];
    }
    c->vv_Cs.assign(nt + 1, 0.0);
    for (int j = 1; j < nt; ++j) c->vv_Cs[j] = 2.0 * std::sin(0.5 * (tc[j - 1] + tc[j])) * std::sin(0.5 * c->ht[j]);
    {
        const double sN = std::sin(0.5 * tc[0]), cS = std::cos(0.5 * tc[nt - 1]);
        c->vv_cap[0] = (2.0 * kTwoPi) * (sN * sN);
        c->vv_cap[1] = (2.0 * kTwoPi) * (cS * cS);
    }
    c->vv_dpp.assign(c->nloc + 2, 0.0);
    c->vv_hmp.assign(c->nloc + 2, 0.0);
    for (int kk = 0; kk < c->nloc + 2; ++kk) {
        const int kg = ((c->k0 + kk - 1) % np + np) % np;   // global plane k0 - 1 + kk (periodic)
        c->vv_dpp[kk] = dpg[kg];
        c->vv_hmp[kk] = hpg[(kg + np - 1) % np];           // centre distance across the lower phi-face of kg
    }
    c->vv_dirty = true;
    c->vv_coef_set = false;

    c->grid_set = true;
    c->metric_dirty = true;
    c->coef_set = false;
    c->D_dirty = true;
    return MASPCG_OK;
}

maspcg_status maspcg_local_extent(const maspcg_ctx *c, int *k0, int *nloc) {
    if (!c) return MASPCG_E_INVALID;
    if (k0) *k0 = c->k0;
    if (nloc) *nloc = c->nloc;
    return MASPCG_OK;
}

// Peer mode: this rank's region `g` (workspace base, size); the peers' regions arrive by maspcg_peer_import.
static maspcg_status peer_register(maspcg_ctx *c, int g, char *base, size_t bytes) {
    if (!c->ptab) return MASPCG_OK;
    PeerTable *t = c->ptab;
    if (g == 0) {
        t->area = c->a.p2p;
        CK(c, cudaMemset(t->area, 0, sizeof(P2PArea)));
        CK(c, cudaDeviceSynchronize());
    }
    t->bytes[g] = bytes;
    for (int r = 0; r < kP2PMaxRanks; ++r) {
        if (r != c->rank && t->mapping[g][r]) {
            peer_close(t->mapping[g][r]);
            t->mapping[g][r] = nullptr;
        }
        t->base[g][r] = nullptr;
    }
    t->base[g][c->rank] = base;
    return MASPCG_OK;
}

size_t maspcg_workspace_bytes(const maspcg_ctx *c) { return c ? layout(c, nullptr, nullptr) : 0; }

maspcg_status maspcg_set_workspace(maspcg_ctx *c, void *dev_ptr, size_t bytes) {
    if (!c) return MASPCG_E_INVALID;
    if (!dev_ptr || ((uintptr_t)dev_ptr & 255)) SET_ERR(c, MASPCG_E_INVALID, "workspace must be 256-byte aligned");
    const size_t need = layout(c, nullptr, nullptr);
    if (bytes < need) SET_ERR(c, MASPCG_E_NOMEM, "workspace too small: %zu < %zu bytes", bytes, need);
    RET_IF(bind_device(c));
    c->ws = dev_ptr;
    c->ws_bytes = bytes;
    layout(c, (char *)dev_ptr, &c->a);
    CK(c, cudaMemset(c->a.sc, 0, sizeof(Scalars)));
    CK(c, cudaMemset(c->a.partials, 0, sizeof(double) * 8 * kPartialSlots));
    CK(c, cudaDeviceSynchronize());
    RET_IF(peer_register(c, 0, (char *)dev_ptr, need));
    c->metric_dirty = true;
    c->coef_set = false;
    c->bc_set = false;
    c->D_dirty = true;
    for (int b = 0; b < 2; ++b) {
        if (c->gexec[b]) {
            cudaGraphExecDestroy(c->gexec[b]);
            c->gexec[b] = nullptr;
        }
    }
    if (c->lexec) {
        cudaGraphExecDestroy(c->lexec);
        c->lexec = nullptr;
    }
    return MASPCG_OK;
}

maspcg_status maspcg_set_coefficients(maspcg_ctx *c, const double *kr, const double *kt, const double *kp,
                                      const double *shift, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!kr || !kt || !kp || !shift) SET_ERR(c, MASPCG_E_INVALID, "coefficient arrays must be non-NULL");
    if (!c->grid_set || !c->ws) SET_ERR(c, MASPCG_E_STATE, "set_grid and set_workspace must precede set_coefficients");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_metric(c, st));
    CK(c, cudaMemsetAsync(&c->a.sc->vinvalid, 0, 2 * sizeof(int), st));
    launch_assemble(c->d, c->a, kr, kt, kp, shift, st);
    CK(c, cudaGetLastError());
    const size_t pl = c->d.plane;
    if (!c->comm) {
        // face (np-1)+1/2 is the lower phi face of plane 0 (periodic, R9)
        CK(c, cudaMemcpyAsync(c->a.Tp, c->a.Tp + (size_t)c->nloc * pl, 8 * pl, cudaMemcpyDeviceToDevice, st));
    } else {
        // the face below plane 0 is the last face of the left neighbour's slab
        COMM(c, c->comm->shift_right(c->a.Tp + (size_t)c->nloc * pl, c->a.Tp, pl, st, c->err));
        COMM(c, c->comm->allreduce_max(&c->a.sc->vinvalid, 2, st, c->err));
    }
    // The validation flags (agreed across ranks above) travel to pinned host memory behind the assembly; they
    // are read by the next call that uses the operator (settle_validation), so the host does not wait here
    // for the assembly -- no host synchronisation per coefficient change (e.g. every time step).
    CK(c, cudaMemcpyAsync(c->vflags_host + 2, &c->a.sc->vinvalid, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(c, cudaEventRecord(c->ev_valid, st));
    c->valid_pending = true;
    c->stats.kernel_launches += 1;
    c->D_dirty = true;
    c->coef_set = true;
    return MASPCG_OK;
}

maspcg_status maspcg_set_coefficients_from_fields(maspcg_ctx *c, const double *field, double kappa0, int half_power,
                                                  maspcg_face_mean mean, const double *rho, double inv_dt,
                                                  void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!field) SET_ERR(c, MASPCG_E_INVALID, "field must be non-NULL");
    if (half_power < 0 || half_power > 16) SET_ERR(c, MASPCG_E_INVALID, "half_power must be in [0, 16]");
    if (mean != MASPCG_MEAN_ARITHMETIC && mean != MASPCG_MEAN_HARMONIC)
        SET_ERR(c, MASPCG_E_INVALID, "mean must be ARITHMETIC or HARMONIC");
    if (!std::isfinite(kappa0) || !std::isfinite(inv_dt)) SET_ERR(c, MASPCG_E_INVALID, "kappa0 and inv_dt must be finite");
    if (!c->grid_set || !c->ws) SET_ERR(c, MASPCG_E_STATE, "set_grid and set_workspace must precede set_coefficients");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t pl = c->d.plane;
    const double *f_hi = field;   // single rank: the plane after the slab is plane 0 (periodic)
    if (c->comm) {
        // the right neighbour's first plane of the field -> fh[1]
        COMM(c, c->comm->halo_planes(field, field + (size_t)(c->nloc - 1) * pl, c->a.fh, c->a.fh + pl, pl, st,
                                     c->err));
        f_hi = c->a.fh + pl;
    }
    launch_face_coeffs(c->d, field, f_hi, rho, kappa0, half_power, (int)mean, inv_dt, c->a.skr, c->a.skt, c->a.skp,
                       c->a.ss, st);
    CK(c, cudaGetLastError());
    c->stats.kernel_launches += 1;
    return maspcg_set_coefficients(c, c->a.skr, c->a.skt, c->a.skp, c->a.ss, stream);
}

maspcg_status maspcg_set_coefficients_host(maspcg_ctx *c, const double *kr, const double *kt, const double *kp,
                                           const double *shift, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!kr || !kt || !kp || !shift) SET_ERR(c, MASPCG_E_INVALID, "coefficient arrays must be non-NULL");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "set_workspace must precede set_coefficients_host");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)c->nloc * c->nt * c->nr;
    CK(c, cudaMemcpyAsync(c->a.skr, kr, 8 * (size_t)c->nloc * c->nt * (c->nr + 1), cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->a.skt, kt, 8 * (size_t)c->nloc * (c->nt + 1) * c->nr, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->a.skp, kp, 8 * n, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->a.ss, shift, 8 * n, cudaMemcpyHostToDevice, st));
    RET_IF(maspcg_set_coefficients(c, c->a.skr, c->a.skt, c->a.skp, c->a.ss, stream));
    return settle_validation(c);   // host buffers: returns after the copies, with the validation result
}

static maspcg_status set_bc_common(maspcg_ctx *c, maspcg_bc inner, const double *gi, maspcg_bc outer,
                                   const double *go, void *stream, cudaMemcpyKind kind) {
    if (!c) return MASPCG_E_INVALID;
    if ((inner != MASPCG_BC_DIRICHLET && inner != MASPCG_BC_NEUMANN0) ||
        (outer != MASPCG_BC_DIRICHLET && outer != MASPCG_BC_NEUMANN0))
        SET_ERR(c, MASPCG_E_INVALID, "boundary type must be DIRICHLET or NEUMANN0");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "set_workspace must precede set_bc_r");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rows = (size_t)c->nloc * c->nt;
    c->has_gin = (inner == MASPCG_BC_DIRICHLET && gi) ? 1 : 0;
    c->has_gout = (outer == MASPCG_BC_DIRICHLET && go) ? 1 : 0;
    if (c->has_gin) CK(c, cudaMemcpyAsync(c->a.gin, gi, 8 * rows, kind, st));
    if (c->has_gout) CK(c, cudaMemcpyAsync(c->a.gout, go, 8 * rows, kind, st));
    if (kind == cudaMemcpyHostToDevice) CK(c, cudaStreamSynchronize(st));
    c->bc_in = inner;
    c->bc_out = outer;
    c->bc_set = true;
    c->D_dirty = true;
    return MASPCG_OK;
}

maspcg_status maspcg_set_bc_r(maspcg_ctx *c, maspcg_bc inner, const double *gi, maspcg_bc outer,
                              const double *go, void *stream) {
    return set_bc_common(c, inner, gi, outer, go, stream, cudaMemcpyDeviceToDevice);
}

maspcg_status maspcg_set_bc_r_host(maspcg_ctx *c, maspcg_bc inner, const double *gi, maspcg_bc outer,
                                   const double *go, void *stream) {
    return set_bc_common(c, inner, gi, outer, go, stream, cudaMemcpyHostToDevice);
}

maspcg_status maspcg_solve(maspcg_ctx *c, const double *rhs, double *x, double tol, int maxit, double *hist,
                           maspcg_info *info, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    RET_IF(bind_device(c));
    return solve_impl(c, rhs, x, tol, maxit, hist, info, (cudaStream_t)stream);
}

maspcg_status maspcg_solve_host(maspcg_ctx *c, const double *rhs, double *x, double tol, int maxit, double *hist,
                                maspcg_info *info, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!rhs || !x) SET_ERR(c, MASPCG_E_INVALID, "rhs and x must be non-NULL");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "no workspace");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)c->nloc * c->nt * c->nr;
    CK(c, cudaMemcpyAsync(c->a.fs, rhs, 8 * n, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(c->a.xs, x, 8 * n, cudaMemcpyHostToDevice, st));
    maspcg_status s = solve_impl(c, c->a.fs, c->a.xs, tol, maxit, hist, info, st);
    if (s < 0) return s;
    CK(c, cudaMemcpyAsync(x, c->a.xs, 8 * n, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    return s;
}

maspcg_status maspcg_apply(maspcg_ctx *c, const double *x, double *y, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!x || !y) SET_ERR(c, MASPCG_E_INVALID, "x and y must be non-NULL");
    const size_t n = (size_t)c->nloc * c->nt * c->nr;
    if (overlaps(x, 8 * n, y, 8 * n)) SET_ERR(c, MASPCG_E_INVALID, "x and y must not alias");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_D(c, st));
    launch_fill_p(c->d, c->a, x, st);
    RET_IF(stencil_with_halo(c, y, false, false, st));
    CK(c, cudaGetLastError());
    c->stats.kernel_launches += 2 + (c->comm ? 1 : 0);
    return MASPCG_OK;
}

// RKL2 coefficients (Meyer, Balsara & Aslam 2014; R26), the same formulas in the same order as the
// oracle's: b_j = (j^2 + j - 2) / (2 j (j + 1)) (b_0 = b_1 = b_2), w1 = 4 / (s^2 + s - 2), ...
static double rkl2_b(int j) {
    if (j < 2) j = 2;
    return ((double)j * j + j - 2.0) / (2.0 * j * (j + 1.0));
}
static void rkl2_coefficients(int s, int j, double *mu, double *nu, double *mut, double *gat) {
    const double w1 = 4.0 / ((double)s * s + s - 2.0);
    if (j == 1) {
        *mu = 1.0;
        *nu = 0.0;
        *mut = rkl2_b(1) * w1;
        *gat = 0.0;
        return;
    }
    const double bj = rkl2_b(j), bj1 = rkl2_b(j - 1), bj2 = rkl2_b(j - 2);
    *mu = (2.0 * j - 1.0) / j * bj / bj1;
    *nu = -((double)j - 1.0) / j * bj / bj2;
    *mut = *mu * w1;
    *gat = -(1.0 - bj1) * *mut;
}

maspcg_status maspcg_sts_step(maspcg_ctx *c, double *u, double tau, int stages, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!u) SET_ERR(c, MASPCG_E_INVALID, "u must be non-NULL");
    if (stages < 2 || stages > 4096) SET_ERR(c, MASPCG_E_INVALID, "stages must be in [2, 4096]");
    if (c->an_on) SET_ERR(c, MASPCG_E_INVALID, "super-time-stepping uses the 7-point operator (aniso set)");
    if (!(tau > 0.0) || !std::isfinite(tau)) SET_ERR(c, MASPCG_E_INVALID, "tau must be finite and > 0");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "no workspace");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_D(c, st));
    const bool ex = exact_arith(c);
    const int din = c->bc_in == BC_DIRICHLET && c->has_gin, dout = c->bc_out == BC_DIRICHLET && c->has_gout;
    DevArrays y0 = c->a;
    y0.p = c->a.sy[3];
    launch_fill_p(c->d, y0, u, st);                     // Y0 (padded, periodic copies on one rank)
    if (c->comm) RET_IF(halo_padded(c, c->a.sy[3], st));
    double mu, nu, mut, gat;
    rkl2_coefficients(stages, 1, &mu, &nu, &mut, &gat);
    launch_sts_first(c->d, c->a, c->a.sy[3], c->a.sl0, c->a.sy[0], mut * tau, din, dout, ex, st);
    if (c->comm) RET_IF(halo_padded(c, c->a.sy[0], st));
    const double *yj2 = c->a.sy[3], *yj1 = c->a.sy[0];
    int next = 1;
    for (int j = 2; j <= stages; ++j) {
        rkl2_coefficients(stages, j, &mu, &nu, &mut, &gat);
        const double w0 = 1.0 - mu - nu;
        double *out = c->a.sy[next];
        launch_sts_stage(c->d, c->a, yj1, yj2, c->a.sy[3], c->a.sl0, out, mu, nu, w0, mut * tau, gat * tau, din, dout,
                         ex, st);
        if (c->comm) RET_IF(halo_padded(c, out, st));
        yj2 = yj1;
        yj1 = out;
        next = (next + 1) % 3;
    }
    CK(c, cudaGetLastError());
    const size_t n = (size_t)c->nloc * c->nt * c->nr;
    CK(c, cudaMemcpyAsync(u, yj1 + c->d.plane, 8 * n, cudaMemcpyDeviceToDevice, st));
    c->stats.kernel_launches += 1 + stages;
    return MASPCG_OK;
}

maspcg_status maspcg_sts_dt_limit(maspcg_ctx *c, double *dt_fe, void *stream) {
    if (!c || !dt_fe) return MASPCG_E_INVALID;
    if (c->an_on) SET_ERR(c, MASPCG_E_INVALID, "super-time-stepping uses the 7-point operator (aniso set)");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "no workspace");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_D(c, st));
    const unsigned g = launch_sts_gershgorin(c->d, c->a, c->a.partials, st);
    CK(c, cudaGetLastError());
    std::vector<double> h(g);
    CK(c, cudaMemcpyAsync(h.data(), c->a.partials, 8 * g, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    double m = 0.0;
    for (double v : h) m = std::fmax(m, v);
    if (c->comm) {
        CK(c, cudaMemcpyAsync(c->a.partials, &m, 8, cudaMemcpyHostToDevice, st));
        COMM(c, c->comm->allgather(c->a.partials, c->a.gather, 1, st, c->err));
        std::vector<double> all(c->nranks);
        CK(c, cudaMemcpyAsync(all.data(), c->a.gather, 8 * c->nranks, cudaMemcpyDeviceToHost, st));
        CK(c, cudaStreamSynchronize(st));
        for (double v : all) m = std::fmax(m, v);
    }
    if (!(m > 0.0)) SET_ERR(c, MASPCG_E_INVALID, "no diffusion coupling: the explicit step is unbounded");
    *dt_fe = 2.0 / m;
    return MASPCG_OK;
}

maspcg_status maspcg_get_operator(maspcg_ctx *c, double *Tr, double *Tt, double *Tp, double *D, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_D(c, st));
    const int nr = c->nr, nt = c->nt, nloc = c->nloc;
    const size_t n = (size_t)nloc * nt * nr, pl = (size_t)nt * nr, rows = (size_t)nloc * nt;
    std::vector<double> tr(n), trb(rows), tt(n), tp(n + pl), dd(n);
    CK(c, cudaMemcpyAsync(tr.data(), c->a.Tr, 8 * n, cudaMemcpyDeviceToHost, st));
    CK(c, cudaMemcpyAsync(trb.data(), c->a.TrB, 8 * rows, cudaMemcpyDeviceToHost, st));
    CK(c, cudaMemcpyAsync(tt.data(), c->a.Tt, 8 * n, cudaMemcpyDeviceToHost, st));
    CK(c, cudaMemcpyAsync(tp.data(), c->a.Tp, 8 * (n + pl), cudaMemcpyDeviceToHost, st));
    CK(c, cudaMemcpyAsync(dd.data(), c->a.D, 8 * n, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    for (size_t row = 0; row < rows; ++row) {
        if (Tr) {
            for (int i = 0; i < nr; ++i) Tr[row * (nr + 1) + i] = tr[row * nr + i];
            Tr[row * (nr + 1) + nr] = trb[row];
        }
    }
    if (Tt)
        for (int k = 0; k < nloc; ++k) {
            for (int j = 0; j < nt; ++j)
                for (int i = 0; i < nr; ++i)
                    Tt[((size_t)k * (nt + 1) + j) * nr + i] = tt[((size_t)k * nt + j) * nr + i];
            for (int i = 0; i < nr; ++i) Tt[((size_t)k * (nt + 1) + nt) * nr + i] = 0.0;
        }
    if (Tp) memcpy(Tp, tp.data() + pl, 8 * n);
    if (D) memcpy(D, dd.data(), 8 * n);
    return MASPCG_OK;
}

// ------------------------------------------------------------ vector viscosity (NEXT-2)
size_t maspcg_vv_workspace_bytes(const maspcg_ctx *c) { return c ? vv_layout(c, nullptr, nullptr) : 0; }

maspcg_status maspcg_vv_set_workspace(maspcg_ctx *c, void *dev_ptr, size_t bytes) {
    if (!c) return MASPCG_E_INVALID;
    if (!dev_ptr || ((uintptr_t)dev_ptr & 255)) SET_ERR(c, MASPCG_E_INVALID, "workspace must be 256-byte aligned");
    if ((size_t)(c->nloc + 2) * 3 * c->nt * c->nr >= (1ull << 31))
        SET_ERR(c, MASPCG_E_INVALID, "local slab too large for the vector operator (>= 2^31 face values)");
    const size_t need = vv_layout(c, nullptr, nullptr);
    if (bytes < need) SET_ERR(c, MASPCG_E_NOMEM, "vv workspace too small: %zu < %zu bytes", bytes, need);
    RET_IF(bind_device(c));
    c->vv_ws = dev_ptr;
    c->vv_ws_bytes = bytes;
    vv_layout(c, (char *)dev_ptr, &c->va);
    VVDims &v = c->vd;
    v.nr = c->nr;
    v.nt = c->nt;
    v.nloc = c->nloc;
    v.plane1 = (uint32_t)((size_t)c->nt * c->nr);
    v.plane3 = 3 * v.plane1;
    v.ncell = (uint32_t)((size_t)c->nloc * v.plane1);
    v.div_r = make_fastdiv((uint32_t)c->nr);
    v.div_t = make_fastdiv((uint32_t)c->nt);
    v.kb = 0;
    v.ke = c->nloc;
    v.chunk = 0;
    v.nchunks = 1;
    // chunked matvec with L2-resident term rings (vv.cu): 0.45 of the L2, within the persisting maximum
    {
        double cap = c->l2_keep ? 0.45 * (double)c->l2_bytes : 0.0;
        if (c->l2_persist_max && cap > (double)c->l2_persist_max) cap = (double)c->l2_persist_max;
        v.ring = vv_ring_planes(v, (size_t)cap);
    }
    c->vv_coef_set = c->vv_bc_set = false;
    c->vv_dirty = true;
    RET_IF(peer_register(c, 1, (char *)dev_ptr, need));
    for (int b = 0; b < 2; ++b) {
        if (c->gexec[b]) {
            cudaGraphExecDestroy(c->gexec[b]);
            c->gexec[b] = nullptr;
        }
    }
    return MASPCG_OK;
}

maspcg_status maspcg_vv_set_coefficients(maspcg_ctx *c, const double *nu, const double *shift, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!nu || !shift) SET_ERR(c, MASPCG_E_INVALID, "nu and shift must be non-NULL");
    if (!c->grid_set || !c->ws || !c->vv_ws)
        SET_ERR(c, MASPCG_E_STATE, "set_grid, set_workspace and vv_set_workspace must precede vv_set_coefficients");
    if (!c->vv_grid_ok)
        SET_ERR(c, MASPCG_E_INVALID, "the vector operator needs both poles (t_faces[0] = 0, t_faces[nt] = pi) and np >= 2");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)c->nloc * c->nt * c->nr;
    CK(c, cudaMemcpyAsync(c->va.nu, nu, 8 * n, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaMemcpyAsync(c->va.s, shift, 8 * n, cudaMemcpyDeviceToDevice, st));
    CK(c, cudaMemsetAsync(&c->a.sc->vinvalid, 0, sizeof(int), st));
    launch_vv_validate(c->vd, c->va.nu, c->va.s, &c->a.sc->vinvalid, st);
    CK(c, cudaGetLastError());
    if (c->comm) COMM(c, c->comm->allreduce_max(&c->a.sc->vinvalid, 1, st, c->err));
    CK(c, cudaMemcpyAsync(c->vflags_host, &c->a.sc->vinvalid, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    c->stats.kernel_launches += 1;
    c->vv_dirty = true;
    if (c->vflags_host[0]) {
        c->vv_coef_set = false;
        SET_ERR(c, MASPCG_E_INVALID, "the viscosity or the shift is negative or non-finite");
    }
    c->vv_coef_set = true;
    return MASPCG_OK;
}

maspcg_status maspcg_vv_set_bc_r(maspcg_ctx *c, maspcg_wall inner, const double *g_inner, maspcg_wall outer,
                                 const double *g_outer, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if ((inner != MASPCG_WALL_NO_SLIP && inner != MASPCG_WALL_FREE_SLIP) ||
        (outer != MASPCG_WALL_NO_SLIP && outer != MASPCG_WALL_FREE_SLIP))
        SET_ERR(c, MASPCG_E_INVALID, "wall type must be NO_SLIP or FREE_SLIP");
    if (!c->vv_ws) SET_ERR(c, MASPCG_E_STATE, "vv_set_workspace must precede vv_set_bc_r");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    // local planes only: the halo planes arrive by the exchange (with the peer communicator a neighbour may
    // already have stored them, so they are never written locally)
    const size_t wplane = 3 * (size_t)c->nt, wloc = (size_t)c->nloc * wplane;
    if (g_inner) CK(c, cudaMemcpyAsync(c->va.gin + wplane, g_inner, 8 * wloc, cudaMemcpyDeviceToDevice, st));
    else CK(c, cudaMemsetAsync(c->va.gin + wplane, 0, 8 * wloc, st));
    if (g_outer) CK(c, cudaMemcpyAsync(c->va.gout + wplane, g_outer, 8 * wloc, cudaMemcpyDeviceToDevice, st));
    else CK(c, cudaMemsetAsync(c->va.gout + wplane, 0, 8 * wloc, st));
    RET_IF(pad_planes(c, c->va.gin, wplane, st));
    RET_IF(pad_planes(c, c->va.gout, wplane, st));
    c->vd.wall_in = (int)inner;
    c->vd.wall_out = (int)outer;
    c->vv_bc_set = true;
    c->vv_dirty = true;
    return MASPCG_OK;
}

maspcg_status maspcg_vv_apply(maspcg_ctx *c, const double *x, double *y, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!x || !y) SET_ERR(c, MASPCG_E_INVALID, "x and y must be non-NULL");
    const size_t n = 3 * (size_t)c->nloc * c->nt * c->nr;
    if (overlaps(x, 8 * n, y, 8 * n)) SET_ERR(c, MASPCG_E_INVALID, "x and y must not alias");
    if (!c->ws) SET_ERR(c, MASPCG_E_STATE, "no workspace");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_vv(c, st));
    VModeGuard g(c);
    launch_fill_p(c->d, c->a, x, st);
    RET_IF(stencil_with_halo(c, y, false, false, st));
    CK(c, cudaGetLastError());
    c->stats.kernel_launches += 3 + (c->comm ? 1 : 0);
    return MASPCG_OK;
}

maspcg_status maspcg_vv_solve(maspcg_ctx *c, const double *f, double *x, double tol, int maxit, double *hist,
                              maspcg_info *info, void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!c->vv_ws) SET_ERR(c, MASPCG_E_STATE, "vv_set_workspace must precede vv_solve");
    RET_IF(bind_device(c));
    VModeGuard g(c);
    return solve_impl(c, f, x, tol, maxit, hist, info, (cudaStream_t)stream);
}

maspcg_status maspcg_vv_get_diag(maspcg_ctx *c, double *D, void *stream) {
    if (!c || !D) return MASPCG_E_INVALID;
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_vv(c, st));
    CK(c, cudaMemcpyAsync(D, c->va.D, 8 * 3 * (size_t)c->nloc * c->nt * c->nr, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    return MASPCG_OK;
}

maspcg_status maspcg_peer_export(maspcg_ctx *c, int region, void *out) {
    if (!c || !out) return MASPCG_E_INVALID;
    if (!c->ptab) SET_ERR(c, MASPCG_E_STATE, "not a peer-memory context (maspcg_create_peer)");
    if (region < 0 || region >= kP2PRegions || !c->ptab->base[region][c->rank])
        SET_ERR(c, MASPCG_E_STATE, "region %d has no workspace yet", region);
    RET_IF(bind_device(c));
    int st = peer_export(c->ptab->base[region][c->rank], c->ptab->bytes[region], out, c->err);
    return (maspcg_status)st;
}

maspcg_status maspcg_peer_import(maspcg_ctx *c, int region, int rank, const void *in) {
    if (!c || !in) return MASPCG_E_INVALID;
    if (!c->ptab) SET_ERR(c, MASPCG_E_STATE, "not a peer-memory context (maspcg_create_peer)");
    if (region < 0 || region >= kP2PRegions || rank < 0 || rank >= c->nranks)
        SET_ERR(c, MASPCG_E_INVALID, "bad region or rank");
    if (rank == c->rank) return MASPCG_OK;
    RET_IF(bind_device(c));
    char *base = nullptr;
    size_t bytes = 0;
    void *map = nullptr;
    int st = peer_import(in, &base, &bytes, &map, c->err);
    if (st != ST_OK) return (maspcg_status)st;
    if (bytes != c->ptab->bytes[region]) {
        peer_close(map);
        SET_ERR(c, MASPCG_E_INVALID, "peer region size %zu differs from ours (%zu)", bytes, c->ptab->bytes[region]);
    }
    if (c->ptab->mapping[region][rank]) peer_close(c->ptab->mapping[region][rank]);
    c->ptab->mapping[region][rank] = map;
    c->ptab->base[region][rank] = base;
    return MASPCG_OK;
}

// ---------------------------------------------------------------- field-aligned conduction (NEXT-4)
size_t maspcg_aniso_workspace_bytes(const maspcg_ctx *c) { return c ? aniso_layout(c, nullptr, nullptr) : 0; }

maspcg_status maspcg_aniso_set_workspace(maspcg_ctx *c, void *dev_ptr, size_t bytes) {
    if (!c) return MASPCG_E_INVALID;
    if (!dev_ptr || ((uintptr_t)dev_ptr & 255)) SET_ERR(c, MASPCG_E_INVALID, "workspace must be 256-byte aligned");
    const size_t need = aniso_layout(c, nullptr, nullptr);
    if (bytes < need) SET_ERR(c, MASPCG_E_NOMEM, "aniso workspace too small: %zu < %zu bytes", bytes, need);
    RET_IF(bind_device(c));
    c->an_ws = dev_ptr;
    c->an_ws_bytes = bytes;
    aniso_layout(c, (char *)dev_ptr, &c->xa);
    c->an_on = false;
    c->an_metric_dirty = true;
    c->D_dirty = true;
    return MASPCG_OK;
}

maspcg_status maspcg_set_aniso_coefficients(maspcg_ctx *c, const double *krt, const double *krp, const double *ktp,
                                            void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!krt && !krp && !ktp) {   // back to the 7-point operator
        c->an_on = false;
        c->D_dirty = true;
        return MASPCG_OK;
    }
    if (!krt || !krp || !ktp) SET_ERR(c, MASPCG_E_INVALID, "krt, krp, ktp must all be given (or all NULL)");
    if (!c->grid_set || !c->ws || !c->an_ws)
        SET_ERR(c, MASPCG_E_STATE, "set_grid, set_workspace and aniso_set_workspace must precede set_aniso_coefficients");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_metric(c, st));
    if (c->an_metric_dirty) {
        auto up = [&](double *dst, const std::vector<double> &v) {
            return cudaMemcpyAsync(dst, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, st);
        };
        CK(c, up(c->xa.gr, c->an_gr));
        CK(c, up(c->xa.qr, c->an_qr));
        CK(c, up(c->xa.gt, c->an_gt));
        CK(c, up(c->xa.cs, c->an_cs));
        CK(c, up(c->xa.gts, c->an_gts));
    }
    CK(c, cudaMemsetAsync(&c->a.sc->vinvalid, 0, sizeof(int), st));
    launch_aniso_edges(c->d, c->a, c->xa, krt, krp, ktp, st);
    CK(c, cudaGetLastError());
    const size_t pl = c->d.plane, last = (size_t)c->nloc * pl;
    if (!c->comm) {   // face (np-1)+1/2 is the lower phi face of plane 0 (periodic, R9)
        CK(c, cudaMemcpyAsync(c->xa.Xrp, c->xa.Xrp + last, 8 * pl, cudaMemcpyDeviceToDevice, st));
        CK(c, cudaMemcpyAsync(c->xa.Xtp, c->xa.Xtp + last, 8 * pl, cudaMemcpyDeviceToDevice, st));
    } else {   // the face below plane 0 is the last face of the left neighbour's slab
        // staged through halo scratch of the main workspace (rh, dh: [2][plane] each, rebuilt before any use
        // that needs them), the region every communicator -- also the peer one, whose exchanges store into
        // registered workspaces only -- can address; two buffers, so the second exchange cannot overwrite
        // the first one's received plane before it is copied out
        double *scratch[2] = {c->a.rh, c->a.dh};
        double *edges[2] = {c->xa.Xrp, c->xa.Xtp};
        for (int q = 0; q < 2; ++q)
            CK(c, cudaMemcpyAsync(scratch[q], edges[q] + last, 8 * pl, cudaMemcpyDeviceToDevice, st));
        for (int q = 0; q < 2; ++q) COMM(c, c->comm->shift_right(scratch[q], scratch[q] + pl, pl, st, c->err));
        for (int q = 0; q < 2; ++q)
            CK(c, cudaMemcpyAsync(edges[q], scratch[q] + pl, 8 * pl, cudaMemcpyDeviceToDevice, st));
        COMM(c, c->comm->allreduce_max(&c->a.sc->vinvalid, 1, st, c->err));
    }
    CK(c, cudaMemcpyAsync(c->vflags_host, &c->a.sc->vinvalid, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));   // host metric vectors may change with the next set_grid
    c->an_metric_dirty = false;
    c->stats.kernel_launches += 1;
    c->D_dirty = true;
    if (c->vflags_host[0]) {
        c->an_on = false;
        SET_ERR(c, MASPCG_E_INVALID, "an edge coefficient is non-finite");
    }
    c->an_on = true;
    return MASPCG_OK;
}

maspcg_status maspcg_aniso_get_operator(maspcg_ctx *c, double *Xrt, double *Xrp, double *Xtp, double *D7,
                                        void *stream) {
    if (!c) return MASPCG_E_INVALID;
    if (!c->an_on) SET_ERR(c, MASPCG_E_STATE, "no field-aligned coefficients set");
    RET_IF(bind_device(c));
    cudaStream_t st = (cudaStream_t)stream;
    RET_IF(ensure_D(c, st));
    const size_t n = (size_t)c->nloc * c->nt * c->nr, pl = (size_t)c->nt * c->nr;
    if (Xrt) CK(c, cudaMemcpyAsync(Xrt, c->xa.Xrt, 8 * n, cudaMemcpyDefault, st));
    if (Xrp) CK(c, cudaMemcpyAsync(Xrp, c->xa.Xrp + pl, 8 * n, cudaMemcpyDefault, st));
    if (Xtp) CK(c, cudaMemcpyAsync(Xtp, c->xa.Xtp + pl, 8 * n, cudaMemcpyDefault, st));
    if (D7) CK(c, cudaMemcpyAsync(D7, c->xa.D7, 8 * n, cudaMemcpyDefault, st));
    CK(c, cudaStreamSynchronize(st));
    return MASPCG_OK;
}

maspcg_status maspcg_set_option(maspcg_ctx *c, maspcg_option opt, long long v) {
    if (!c) return MASPCG_E_INVALID;
    switch (opt) {
        case MASPCG_OPT_CHUNK:
            if (v < 1 || v > kMaxChunk) SET_ERR(c, MASPCG_E_INVALID, "chunk must be in [1, %d]", kMaxChunk);
            c->chunk = (int)v;
            break;
        case MASPCG_OPT_USE_GRAPHS: c->use_graphs = v ? 1 : 0; break;
        case MASPCG_OPT_TIMING:
            if (v < 0 || v > 3)
                SET_ERR(c, MASPCG_E_INVALID, "timing must be 0, 1 (every iteration), 2 (sampled, middle slot) or 3 "
                                             "(sampled, slot 0)");
            c->timing = (int)v;
            break;
        case MASPCG_OPT_PDL:
            c->d.pdl = v ? 1 : 0;
            break;
        case MASPCG_OPT_VEC:
            c->d.vec_ok = v ? 1 : 0;
            break;
        case MASPCG_OPT_TMA:
            c->use_tma = v ? 1 : 0;
            break;
        case MASPCG_OPT_ARITH:
            if (v < 0 || v > 1) SET_ERR(c, MASPCG_E_INVALID, "arith must be 0 (oracle-exact) or 1 (fast)");
            c->arith = (int)v;
            break;
        case MASPCG_OPT_FUSE_HALO: c->fuse_halo = v < 0 ? 0 : (v > 2 ? 2 : v); break;
        case MASPCG_OPT_L2_KEEP: c->l2_keep = v ? 1 : 0; break;
        case MASPCG_OPT_DEVICE_LOOP: c->device_loop = v ? 1 : 0; break;
        case MASPCG_OPT_PATH:
            if (v < 0 || v > 5)
                SET_ERR(c, MASPCG_E_INVALID, "path must be 0 (auto), 1 (three kernels), 2 (fused), 3 (wave), 4 (single "
                                             "reduction) or 5 (persistent)");
            c->path_opt = (int)v;
            break;
        default: SET_ERR(c, MASPCG_E_INVALID, "unknown option %d", (int)opt);
    }
    if (c->timing) {
        const size_t need = (size_t)2 * 6 * 2 * c->chunk;
        RET_IF(bind_device(c));
        while (c->tev.size() < need) {
            cudaEvent_t e;
            CK(c, cudaEventCreate(&e));
            c->tev.push_back(e);
        }
    }
    return MASPCG_OK;
}

maspcg_status maspcg_get_stats(const maspcg_ctx *c, maspcg_stats *out) {
    if (!c || !out) return MASPCG_E_INVALID;
    *out = c->stats;
    return MASPCG_OK;
}

maspcg_status maspcg_reset_stats(maspcg_ctx *c) {
    if (!c) return MASPCG_E_INVALID;
    c->stats = maspcg_stats{};
    return MASPCG_OK;
}

}  // extern "C"
