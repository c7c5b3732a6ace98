// common.cuh -- shared definitions of libmaspcg (product path only; never
// included by oracle/).  See include/maspcg.h for the model and DESIGN.md for
// the data layout in HBM.
#pragma once

#include <cstddef>
#include <cstdint>

namespace maspcg {

// Status codes mirrored from include/maspcg.h for device code.
enum : int {
    ST_OK = 0,
    ST_NOT_CONVERGED = 1,
    ST_E_INVALID = -1,
    ST_E_STATE = -2,
    ST_E_SINGULAR = -3,
    ST_E_BREAKDOWN = -4,
    ST_E_CUDA = -5,
    ST_E_NCCL = -6,
    ST_E_NOMEM = -7,
};

enum : int { BC_DIRICHLET = 0, BC_NEUMANN0 = 1 };

constexpr int kMaxChunk = 256;          // PCG iterations per graph launch (upper bound)
constexpr int kRedBlocks = 1184;        // fixed grid of the streaming kernels (8 x 148)
constexpr int kPartialSlots = 2560;     // per-block Dot2 partial slots of one reduction: >= the interior +
                                        // boundary stencil grids together (2 x kRedBlocks for the scalar kernels)
constexpr int kThreads = 256;           // threads per block of the streaming kernels
constexpr int kMaxRanks = 16;           // all-gather scratch of the Dot2 all-reduce
constexpr int kDevHist = 65536;         // device residual history of the conditional-graph solve loop

// Division by a runtime constant for 0 <= n < 2^31 (round-up multiplier
// method): q = (n * m) >> p with p = 31 + ceil(log2 d), m = ceil(2^p / d).
struct FastDiv {
    uint32_t d;
    uint32_t p;
    uint64_t m;
#ifdef __CUDACC__
    __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return d == 1 ? n : static_cast<uint32_t>((static_cast<uint64_t>(n) * m) >> p);
    }
#endif
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{};
    f.d = d;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    f.p = 31 + l;
    f.m = ((1ull << f.p) + d - 1) / d;
    return f;
}

// Device-resident solver scalars (one struct in the workspace).  Written only
// by single threads (a kernel's last-arriving block or a 1-thread kernel);
// read by every block at kernel entry.  A snapshot is copied to pinned host
// memory once per graph chunk.
struct Scalars {
    // Dot2 results as (p, s) pairs, value = p + s (arith.cuh): local, then global after the all-reduce
    double red1[2];          // p.Ap
    double red2[4];          // r.z, r.r
    double red3[6];          // setup: r.z, r.r, b.b
    double rho;              // r.z of the current iterate
    double bn;               // ||b||
    double tolbn;            // tol * ||b||
    double tol;
    double hist0;            // ||r_0||
    double rn;               // ||r_iter||
    double alpha;            // alpha of the last completed iteration (fused path: deferred x update)
    double cg_gamma_old;     // single-reduction path: gamma and alpha of the previous iteration
    double cg_alpha_old;
    int iter;                // completed PCG iterations
    int maxit;
    int done;                // 1: every loop kernel returns at entry
    int status;              // provisional / final status
    int zero_x;              // b == 0: x := 0 at the end
    int vinvalid;            // set_coefficients: 1 if any input is negative or non-finite
    int vshift;              // set_coefficients: 1 if any s > 0
    int hist_count;          // fused path: history entries 1..hist_count are final
    unsigned int ticket[8];  // last-block tickets (reset by the last block)
    double hist_ring[2 * kMaxChunk];   // ||r_k|| at slot (k-1) % chunk (3-kernel) or % (2 kMaxChunk) (fused)
};

// Peer-memory communicator (peer.cu): flags, epochs and double-buffered staging of one rank, in its
// workspace; peers store into it over NVLink.
constexpr int kP2PMaxRanks = 16;
constexpr int kP2PRegions = 2;
constexpr int kP2PStage = 16384;     // doubles per rank slot of an all-gather
constexpr int kP2PIStage = 64;       // ints per rank slot of an all-reduce(max)
constexpr int kP2PHandleBytes = 64 + 16;
enum : int { P2P_FROM_LEFT = 0, P2P_FROM_RIGHT, P2P_SHIFT, P2P_GATHER, P2P_MAX, P2P_HALO, P2P_LL, kP2PKinds };
constexpr int kP2PLLOffset = kP2PStage / 2;   // a rank slot: plain all-gather doubles, then LL words
struct P2PArea {
    unsigned long long flags[kP2PKinds][kP2PMaxRanks];   // written by the senders (epoch of their last exchange)
    unsigned long long epoch[kP2PKinds];                  // this rank's exchange counters
    unsigned int ticket[kP2PKinds];
    int istage[2][kP2PMaxRanks][kP2PIStage];
    double stage[2][kP2PMaxRanks][kP2PStage];
};

// Geometry handed to kernels by value.
struct Dims {
    int nr, nt, nloc;       // local slab shape
    int k0;                 // global index of local plane 0
    uint32_t n;             // nloc * nt * nr
    uint32_t plane;         // nt * nr
    FastDiv div_r;          // / nr
    FastDiv div_t;          // / nt
    int periodic_local;     // 1: single rank, halo planes are written by the kernels
    int vec_ok;             // 1: the 16-byte vector kernels may be used (MASPCG_OPT_VEC)
    int pdl;                // 1: launch the vector loop kernels with programmatic dependent launch
    // L2 residency of the loop's arrays (vector kernels of path 1): 2 bits per array class L2A_* --
    // L2_NORMAL, L2_KEEP (every line evict_last), L2_KEEP_FRAC (the fraction l2_frac of the lines
    // evict_last), L2_FIRST (evict_first).  0 everywhere: plain loads and stores.
    uint32_t l2_mask;
    float l2_frac;
};

// A launch range over local cells: v in [0, vend), cell c = v + off0 (+ off1 once v >= split), so one
// kernel covers the interior planes or the two boundary planes of a slab.
struct Range {
    uint32_t vend, off0, split, off1;
};

// Array classes of Dims::l2_mask and their residency codes.
enum : int { L2A_D = 0, L2A_P, L2A_R, L2A_X, L2A_Q, L2A_T, kL2Arrays };
enum : uint32_t { L2_NORMAL = 0u, L2_KEEP = 1u, L2_KEEP_FRAC = 2u, L2_FIRST = 3u };

// Device pointers into the workspace.
struct DevArrays {
    // operator
    double *Tr;     // [nloc][nt][nr]  lower r-face of each cell; slot i = 0 holds the inner-boundary face
    double *TrB;    // [nloc][nt]      outer-boundary r-face (i = nr)
    double *Tt;     // [nloc][nt][nr]  lower theta-face; slot j = 0 is 0 (pole / boundary: no flux)
    double *Tp;     // [nloc+1][nt][nr] plane kk = phi face (k0 + kk - 1) + 1/2
    double *D;      // [nloc][nt][nr]
    double *sV;     // [nloc][nt][nr]  s * V
    double *gin;    // [nloc][nt]
    double *gout;   // [nloc][nt]
    // PCG vectors
    double *p;      // [nloc+2][nt][nr] plane 0 / nloc+1 are halos
    double *q;      // [nloc][nt][nr]
    double *r;      // [nloc][nt][nr]
    double *xs;     // [nloc][nt][nr]  x staging (host entry points)
    double *fs;     // [nloc][nt][nr]  rhs staging (host entry points)
    // staging for host coefficients
    double *skr, *skt, *skp, *ss;
    // 1-D metric (local where noted)
    double *rf2;    // [nr+1]  r_f^2
    double *hr;     // [nr+1]
    double *dr;     // [nr]
    double *R3;     // [nr]
    double *C;      // [nt]
    double *sinf;   // [nt+1]
    double *ht;     // [nt+1]
    double *dt;     // [nt]
    double *sinc;   // [nt]
    double *dp;     // [nloc]  local
    double *hp;     // [nloc]  local: h^phi of face (k0 + k) + 1/2
    // fused two-pass path
    double *P[2];       // [nloc][nt][nr] search directions of even / odd iterations
    double *rh, *dh, *ph;   // [2][nt][nr] received halo planes (lo, hi) of r, D, p_old (nranks > 1)
    double *fh;             // [2][nt][nr] received halo planes of a physical field (from_fields, nranks > 1)
    // single-reduction (Chronopoulos-Gear) path, MASPCG_OPT_PATH = 4 (cg1.cu); p lives in q
    double *cgr;            // [nloc+2][nt][nr] r with halo planes
    double *cgw;            // [nloc][nt][nr]   w = A u, u = r / D
    double *cgs;            // [nloc][nt][nr]   s (= A p in exact arithmetic)
    // super-time-stepping (NEXT-4)
    double *sy[4];          // [nloc+2][nt][nr] x4: three rotating RKL2 stages and Y0
    double *sl0;            // [nloc][nt][nr]   L(Y0)
    // wave path (wave.cu)
    unsigned *wave_counter; // work-item counter
    unsigned *wave_flags;   // [nloc] completed A-tiles per plane
    double *wave_partials;  // [nloc * tiles per plane][2]
    // reductions
    P2PArea *p2p;       // peer-memory communicator area
    // peer mode, three-kernel path: the p-update stores its first plane into the left rank's upper halo
    // and its last plane into the right rank's lower halo (NVLink stores fused into the update) and
    // releases their flags; nullptr otherwise
    double *peer_p_hi;                  // left rank's p + (nloc+1) plane
    double *peer_p_lo;                  // right rank's p
    unsigned long long *peer_flag_hi;   // left rank's flags[FROM_RIGHT][0]
    unsigned long long *peer_flag_lo;   // right rank's flags[FROM_LEFT][0]
    // peer communicator, path 1: the loop's Dot2 pairs are pushed to every rank by the last block of the
    // producing kernel (LL words) and combined by the consuming kernel -- no reduction kernel at all
    int p2p_ll, p2p_rank, p2p_nranks;
    // peer communicator, path 1: the loop's stencil acquires the neighbours' halo flags itself (thread 0
    // of every block, before any load) instead of a separate wait kernel and an interior/boundary split
    int peer_wait;
    double *peer_stage[kP2PMaxRanks];   // rank r's P2PArea::stage, mapped into this process
    int gather_ranks;   // > 0: the loop's dot products arrive all-gathered (gather[rank][pairs]) and the
                        // consuming kernel combines them in rank order itself (no combine kernel)
    double *hist_dev;   // [kDevHist] ||r_k|| at slot k - 1 (device loop, MASPCG_OPT_DEVICE_LOOP), written when
    int hist_dev_on;    // hist_dev_on is set
    double *partials;   // [8][kPartialSlots]  Dot2 (p, s) partials of up to 4 sums
    double *gather;     // [kMaxRanks][8]   all-gather scratch of the Dot2 all-reduce
    Scalars *sc;
};

}  // namespace maspcg
