/*
 * maspcg.h -- C ABI of the B200-native fp64 PCG solve of the implicit
 * parabolic (viscosity / thermal-conduction) terms of the MAS solar MHD code,
 * the hot path of arXiv 2303.03398 (Caplan, Stulajter, Linker, "Acceleration
 * of a production Solar MHD code with Fortran standard parallelism").
 *
 * What the paper fixes (PAPER.md, the only source text):
 *   PAPER.md:56  (Sec. III)   "logically rectangular non-uniform staggered
 *                              spherical grid", "finite-difference
 *                              discretizations", "explicit and implicit
 *                              time-stepping", "highly memory-bound";
 *   PAPER.md:240-246 (V-A)    36 M-cell coronal test on a stretched grid,
 *                              validated "to within solver tolerances";
 *   PAPER.md:282, 290-292 (V-C, Figs. 3-4)  "viscosity solver iterations"
 *                              with GPU peer-to-peer MPI halo exchanges.
 * Everything else -- the operator, boundary conditions, preconditioner,
 * stopping rule -- is a READING (R1..R18 of SURVEY.md section 8(c), restated
 * in DESIGN.md section 3); each entry point below names the readings it
 * implements.
 *
 * Model.  One process per GPU; every rank calls every function in the same
 * order (like MPI).  The global grid has nr x nt x np cells (r, theta, phi);
 * rank p owns the phi-slab k in [p*np/P, (p+1)*np/P)  (np % P == 0).  Cell
 * arrays are fp64, C order [k][j][i]: phi outermost, r contiguous (the
 * Fortran array(i,j,k) of PAPER.md:128-139, Listing 1).  "nloc" below is the
 * local number of phi planes.
 *
 * Operator (R1-R10).  (A u)_c = D_c u_c - sum_{interior faces f} T_f u_nb(f),
 * the volume-weighted form of (s - div kappa grad) u = f on the spherical grid:
 * exact finite-volume metric, face transmissibilities T = kappa * area /
 * centre distance, zero flux through theta-boundary (pole) faces, periodic
 * phi, Dirichlet (value on the face) or zero-flux Neumann r boundaries, and
 * D = s V + sum of the cell's face T (Dirichlet faces included).  A is
 * symmetric positive definite unless s == 0 and no r boundary is Dirichlet.
 *
 * Solver (R6, R11-R14).  Point-Jacobi preconditioned CG (M = D), Fletcher-
 * Reeves beta, stop when ||r_k||_2 <= tol * ||b||_2 (unweighted norms of the
 * volume-weighted system; r is the recurrence residual).  tol == 0 runs
 * exactly maxit iterations (benchmark mode).
 *
 * Memory and streams.  All device memory is caller-owned: the library never
 * calls cudaMalloc (NCCL may allocate internally).  The caller supplies a
 * workspace of maspcg_workspace_bytes() bytes (e.g. a torch uint8 tensor).
 * Device-pointer entry points enqueue work on the caller's stream (plus an
 * internal communication stream joined by events) and are ordered with other
 * work on that stream; maspcg_solve() returns after the solve has finished.
 * "_host" entry points take host pointers (pageable or pinned) and perform the
 * host<->device copies themselves, through workspace staging buffers.
 *
 * Errors.  Return codes >= 0 mean the output is valid (NOT_CONVERGED: x is
 * the maxit-th iterate).  Codes < 0 leave outputs unspecified.  Argument
 * errors are detected on every rank before any collective; data-dependent
 * errors (E_SINGULAR, E_BREAKDOWN, non-finite or negative coefficients) are
 * agreed across ranks, so all ranks return the same code.  A call made out of
 * order returns E_STATE.  maspcg_last_error() describes the last failure.  A
 * context is not thread-safe.  There is no CPU fallback: without an sm_100a
 * GPU every call that touches the device returns E_CUDA.
 */
#ifndef MASPCG_H
#define MASPCG_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MASPCG_API __attribute__((visibility("default")))
#define MASPCG_NCCL_UNIQUE_ID_BYTES 128

typedef struct maspcg_ctx maspcg_ctx; /* opaque, one per rank */

typedef enum {
    MASPCG_OK = 0,
    MASPCG_NOT_CONVERGED = 1,
    MASPCG_E_INVALID = -1,   /* bad argument, bad grid, negative / non-finite coefficient */
    MASPCG_E_STATE = -2,     /* call out of order (e.g. solve before set_coefficients) */
    MASPCG_E_SINGULAR = -3,  /* s == 0 everywhere and no Dirichlet r boundary */
    MASPCG_E_BREAKDOWN = -4, /* p.Ap <= 0 or a non-finite residual during PCG */
    MASPCG_E_CUDA = -5,
    MASPCG_E_NCCL = -6,
    MASPCG_E_NOMEM = -7      /* workspace too small / not set */
} maspcg_status;

typedef enum { MASPCG_BC_DIRICHLET = 0, MASPCG_BC_NEUMANN0 = 1 } maspcg_bc;

typedef struct {
    int iters;          /* PCG iterations (matvecs inside the loop; R13) */
    double bnorm;       /* ||b||_2, global */
    double rnorm;       /* ||r_iters||_2 (recurrence residual), global */
    double rel_resid;   /* rnorm / bnorm (0 when bnorm == 0) */
} maspcg_info;

/* Per-context counters, accumulated since creation or the last reset. */
typedef struct {
    long long kernel_launches;     /* kernels of this library enqueued (graph nodes count per replay) */
    long long solves;
    long long iterations;          /* PCG iterations executed (sum over solves) */
    double matvec_ms;              /* summed CUDA-event time of the stencil launches (stencil_matvec_dot, or pass A
                                      of the fused path) in timing mode */
    long long matvec_launches;     /* launches covered by matvec_ms */
    double update_ms;              /* update_jacobi_dots (or pass B of the fused path) */
    long long update_launches;
    double pupdate_ms;             /* p_update */
    long long pupdate_launches;
    double comm_ms;                /* the two all-reduces of the sampled iterations (timing mode, P > 1, path 1): the
                                      analogue of the MPI time of PAPER.md:282 (Fig. 3) on the critical path */
    double halo_ms;                /* the halo exchange of those iterations on the comm stream (overlapped with the
                                      interior planes of the stencil) */
    long long comm_launches;       /* sampled iterations covered by comm_ms / halo_ms */
    int path;                      /* iteration path of the last solve: 1 = three kernels, 2 = fused two passes,
                                      3 = wave, 4 = single reduction, 5 = vector viscosity, 6 = persistent */
} maspcg_stats;

/* Options for maspcg_set_option(). */
typedef enum {
    MASPCG_OPT_CHUNK = 1,        /* PCG iterations per CUDA-graph launch (1..256, default 16) */
    MASPCG_OPT_USE_GRAPHS = 2,   /* 1 (default): replay captured graphs; 0: eager launches */
    MASPCG_OPT_TIMING = 3,       /* 1: CUDA events around every hot kernel of every iteration; 2: the same on every
                                    chunk-th iteration only (the middle slot of each graph chunk; the records
                                    serialise the kernels they separate, so sampling keeps the timed run close to
                                    untimed speed); 3: as 2 in slot 0 (the first kernels of each graph launch).
                                    Events are recorded by event nodes inside the captured graphs; two event sets
                                    alternate with the two chunks in flight */
    MASPCG_OPT_ARITH = 5,        /* 0 (default): oracle-identical arithmetic -- no FMA contraction, Dot2 (compensated)
                                    dot products (R24); 1: FMA updates and plain tree sums (faster in FP64
                                    issue, parity to the tolerance contract only) */
    MASPCG_OPT_PDL = 8,          /* 1 (default): programmatic dependent launch of the vector loop kernels (the next
                                    kernel's blocks are resident before the previous one retires); 0: plain launches */
    MASPCG_OPT_VEC = 7,          /* three-kernel path: 1 (default) two cells per thread with 16-byte loads when nr is
                                    even; 0: one cell per thread */
    MASPCG_OPT_TMA = 6,          /* fused path: 1 (default) stage pass A's streams with TMA bulk copies when nr is
                                    even; 0: register-batched loads */
    MASPCG_OPT_FUSE_HALO = 9,    /* peer communicator, path 1: 1 the p-update kernel stores its boundary
                                    planes straight into the neighbours' halo planes over NVLink and releases their
                                    flags (compute and exchange in one kernel), the next stencil waits for the
                                    neighbours' flags in a 1-thread kernel on the communication stream and runs as an
                                    interior and a boundary launch; 2 (default): as 1, but every stencil block
                                    acquires the flags itself and the stencil is one launch (no wait kernel, no
                                    split; 92.2 vs 95.7 us per iteration on the P = 8 slab of c3, one rank);
                                    0: a separate push kernel */
    MASPCG_OPT_L2_KEEP = 10,     /* three-kernel path (nr even): L2 residency of the loop's arrays.  1 (default,
                                    auto): when the local slab is small enough (P = 4, 8 of c3), the arrays with the
                                    most accesses per iteration and byte -- D (3 reads), p and r (3 accesses each),
                                    then x and q -- are loaded and stored with an L2 evict_last policy, whole
                                    classes greedily up to 0.45 of the L2, inside a persisting set-aside of exactly
                                    their size (cudaLimitPersistingL2CacheSize, a device-wide limit this context
                                    sets and releases at destroy); their lines are returned to the normal priority
                                    after the solve.  The "super" scaling of PAPER.md:277 (§V-C).  0: plain loads
                                    and stores.  Arithmetic and results are unaffected. */
    MASPCG_OPT_DEVICE_LOOP = 11, /* 1 (default): the whole PCG loop is ONE CUDA-graph launch -- a conditional WHILE
                                    node whose body is a chunk of iterations followed by a kernel that sets the
                                    condition to "not done"; the history is kept on the device.
                                    Used when eligible: three-kernel path, graphs on, timing off, maxit <= 65536, one
                                    rank or the peer communicator with MASPCG_OPT_FUSE_HALO 2; otherwise (and with 0)
                                    the host loop, one snapshot per chunk with a speculative chunk in flight.
                                    Measured: c3 542.6 vs 543.2 us per iteration, P = 8 slab 73.1 vs 73.4 (one rank)
                                    and 84.4-84.6 vs 85.7-86.4 (one-rank peer). */
    MASPCG_OPT_PATH = 4         /* iteration path: 0 = auto (default, = 1), 1 = three streaming kernels (stencil+p.q,
                                    r-update+Jacobi+dots, deferred x-update+p-update; 128 B/cell), 2 = fused two passes
                                    (p- and x-update folded into a phi-marching tiled stencil + r update; 112 B/cell),
                                    3 = wave (single rank): r-update, then the p-update of iteration k and the stencil
                                    of iteration k+1 in one persistent kernel ordered by plane-completion flags, p and D
                                    re-read from L2 (112 B/cell of HBM traffic); 4 = single reduction (Chronopoulos-Gear
                                    PCG, R32): an update kernel and a matvec that forms u = r/D on the fly and reduces
                                    r.u, w.u and r.r together -- ONE all-reduce per iteration on P > 1 (128 B/cell);
                                    its iterates are those of the oracle's single-reduction variant; 5 = persistent
                                    (single rank, nr even): one cooperative kernel runs a chunk of iterations, the
                                    three phases of each separated by grid-wide (reduction) barriers instead of kernel
                                    boundaries (the arithmetic, traffic and iterates of path 1) */
} maspcg_option;

/* ---- lifetime ----------------------------------------------------------- */

/* Fill `out` (MASPCG_NCCL_UNIQUE_ID_BYTES bytes, host) with a fresh NCCL
 * unique id.  Rank 0 calls it and the caller broadcasts the bytes (e.g. with
 * torch.distributed) before every rank calls maspcg_create. */
MASPCG_API maspcg_status maspcg_get_unique_id(void *out);

/* Create a context for rank `rank` of `nranks` on CUDA device `cuda_device`.
 * nr, nt, np: GLOBAL cell counts (>= 1; np % nranks == 0; the local slab must
 * hold < 2^31 cells including two halo planes).  nccl_unique_id: the 128
 * bytes from maspcg_get_unique_id; required when nranks > 1.  With nranks == 1
 * it may be NULL (no communicator: the periodic phi wrap is a local copy) or an
 * id (a one-rank NCCL communicator: the multi-rank code path, halos sent to
 * itself -- used to exercise NCCL on a single GPU).  Collective over all ranks
 * when an id is given (ncclCommInitRank).  *out receives the context. */
MASPCG_API maspcg_status maspcg_create(int nr, int nt, int np, int rank, int nranks,
                                       const void *nccl_unique_id, int cuda_device,
                                       maspcg_ctx **out);

/* Release the context (and its NCCL communicator).  NULL is a no-op. */
MASPCG_API maspcg_status maspcg_destroy(maspcg_ctx *ctx);

/* Human-readable description of the last failure on this context (owned by
 * ctx; valid until the next call).  ctx == NULL: the last create failure. */
MASPCG_API const char *maspcg_last_error(const maspcg_ctx *ctx);

/* ---- grid and memory (R1-R3, R9) --------------------------- */

/* Face coordinates, HOST arrays, copied: r_faces[nr+1] (r_faces[0] > 0),
 * t_faces[nt+1] within [0, pi], p_faces[np+1] spanning exactly 2*pi (to 1e-12
 * relative); all strictly increasing.  Precomputes the 1-D metric on the
 * host (centres = face midpoints, centre distances, exact FV volume and area
 * factors).  E_INVALID on a bad grid.  May be called again (marks the
 * coefficients stale: set_coefficients must follow). */
MASPCG_API maspcg_status maspcg_set_grid(maspcg_ctx *ctx, const double *r_faces,
                                         const double *t_faces, const double *p_faces);

/* This rank's slab: global first plane *k0 and plane count *nloc. */
MASPCG_API maspcg_status maspcg_local_extent(const maspcg_ctx *ctx, int *k0, int *nloc);

/* Bytes of device workspace this rank needs (depends only on the sizes). */
MASPCG_API size_t maspcg_workspace_bytes(const maspcg_ctx *ctx);

/* Hand the library a device buffer of >= maspcg_workspace_bytes() bytes,
 * 256-byte aligned, owned by the caller and kept alive until destroy (or the
 * next set_workspace).  Operator state lives here: setting a new workspace
 * invalidates coefficients and boundary conditions. */
MASPCG_API maspcg_status maspcg_set_workspace(maspcg_ctx *ctx, void *dev_ptr, size_t bytes);

/* ---- coefficients and boundary conditions (R3-R10) -------- */

/* Face diffusion coefficients and shift of the local slab, DEVICE pointers,
 * consumed (the caller may free them afterwards):
 *   kr    [nloc][nt][nr+1]  r-faces i = 0..nr            (kappa >= 0)
 *   kt    [nloc][nt+1][nr]  theta-faces j = 0..nt        (the two boundary rows are ignored)
 *   kp    [nloc][nt][nr]    phi-face k+1/2 of each local plane k
 *   shift [nloc][nt][nr]    s >= 0 (e.g. rho/dt for backward Euler, R5)
 * Assembles the face transmissibilities T and s*V in library memory and
 * fetches the phi-face below the slab from the previous rank.  A negative or
 * non-finite value gives E_INVALID (agreed across ranks), reported by the
 * NEXT call that uses the operator (solve, apply, get_operator, sts_*): the
 * validation result travels to pinned host memory behind the assembly, so
 * this call does not wait for the device (no host synchronisation per
 * coefficient change, e.g. per time step).  Calls on one context must be
 * ordered on one stream.  The _host variant copies the caller's buffers,
 * waits for the copies and reports E_INVALID itself. */
MASPCG_API maspcg_status maspcg_set_coefficients(maspcg_ctx *ctx, const double *kr,
                                                 const double *kt, const double *kp,
                                                 const double *shift, void *cuda_stream);
/* Same, HOST pointers (copied through workspace staging; timed as e2e). */
MASPCG_API maspcg_status maspcg_set_coefficients_host(maspcg_ctx *ctx, const double *kr,
                                                      const double *kt, const double *kp,
                                                      const double *shift, void *cuda_stream);

/* Per-time-step assembly from physical fields (the implicit
 * viscosity / thermal-conduction terms of MAS's time loop; reading R25 of DESIGN.md).
 *   field  DEVICE [nloc][nt][nr], cell-centred (e.g. temperature T, or density rho)
 *   kappa_c = kappa0 * field_c^(half_power/2), evaluated as ((kappa0 f) f ...) sqrt(f):
 *            half_power 5 = Spitzer conduction kappa0 T^(5/2); 2 = viscosity nu rho (kappa0 = nu)
 *   face coefficient = ARITHMETIC (a+b)/2 or HARMONIC 2ab/(a+b) mean of the two cells of an
 *            interior face (phi periodic; across ranks the neighbour's plane is exchanged);
 *            the adjacent cell's value on an r or theta boundary face
 *   shift  s_c = inv_dt * rho_c (rho DEVICE [nloc][nt][nr], or NULL for s = inv_dt)
 * Then exactly as maspcg_set_coefficients (E_INVALID if a value is negative or non-finite, e.g.
 * a negative field with an odd half_power).  Collective for nranks > 1.  Synchronises the stream. */
typedef enum { MASPCG_MEAN_ARITHMETIC = 0, MASPCG_MEAN_HARMONIC = 1 } maspcg_face_mean;
MASPCG_API maspcg_status maspcg_set_coefficients_from_fields(maspcg_ctx *ctx, const double *field, double kappa0,
                                                             int half_power, maspcg_face_mean mean,
                                                             const double *rho, double inv_dt, void *cuda_stream);

/* Radial boundary conditions (R7): inner (r = r_faces[0]) and outer
 * (r = r_faces[nr]) each DIRICHLET (value on the face; g [nloc][nt], DEVICE,
 * copied; NULL means 0) or NEUMANN0 (zero flux; g ignored).  May precede or
 * follow set_coefficients; D is (re)assembled lazily at the next solve/apply. */
MASPCG_API maspcg_status maspcg_set_bc_r(maspcg_ctx *ctx, maspcg_bc inner, const double *g_inner,
                                         maspcg_bc outer, const double *g_outer, void *cuda_stream);
MASPCG_API maspcg_status maspcg_set_bc_r_host(maspcg_ctx *ctx, maspcg_bc inner,
                                              const double *g_inner, maspcg_bc outer,
                                              const double *g_outer, void *cuda_stream);

/* ---- the hot path -------------------------------------- */

/* Solve A x = b with b = V rhs + Dirichlet face terms (R5), by point-Jacobi
 * PCG from the initial guess in x.
 *   rhs  DEVICE [nloc][nt][nr], per-unit-volume source f (not modified)
 *   x    DEVICE [nloc][nt][nr], in: x0, out: the iterate; must not alias rhs
 *   tol  >= 0 (0: run exactly maxit iterations);  maxit >= 0
 *   resid_hist  HOST, >= maxit+1 doubles, receives ||r_k||_2 for
 *        k = 0..info->iters, or NULL
 *   info HOST, or NULL
 * Returns OK, NOT_CONVERGED, E_SINGULAR, E_BREAKDOWN (p.Ap <= 0 or non-finite
 * data), E_STATE, E_INVALID, E_CUDA or E_NCCL; the same code on all ranks.
 * Blocks the host until the result is known (the host polls a device flag
 * once per CUDA-graph chunk of MASPCG_OPT_CHUNK iterations). */
MASPCG_API maspcg_status maspcg_solve(maspcg_ctx *ctx, const double *rhs, double *x, double tol,
                                      int maxit, double *resid_hist, maspcg_info *info,
                                      void *cuda_stream);
/* Same, HOST rhs and x (copied in and out through workspace staging). */
MASPCG_API maspcg_status maspcg_solve_host(maspcg_ctx *ctx, const double *rhs, double *x,
                                           double tol, int maxit, double *resid_hist,
                                           maspcg_info *info, void *cuda_stream);

/* ---- explicit super-time-stepping of the same parabolic term (R26) ---- */

/* One RKL2 super-time-step (Meyer, Balsara & Aslam 2014) of the semi-discrete diffusion equation
 *   V du/dt = b_D - K u,   K = A - diag(s V)  (the operator of set_coefficients / set_bc_r without
 *   its shift; b_D the Dirichlet face terms),
 * over tau with `stages` (2..4096) stages, in place on u (DEVICE [nloc][nt][nr]).  Stable for
 * tau <= (stages^2 + stages - 2) / 4 * dt_fe (maspcg_sts_dt_limit).  No dot products, one halo
 * exchange per stage (P > 1).  E_INVALID for bad arguments, E_STATE before coefficients / BCs. */
MASPCG_API maspcg_status maspcg_sts_step(maspcg_ctx *ctx, double *u, double tau, int stages, void *cuda_stream);
/* dt_fe = 2 / max_c (K_cc + sum_f T_f) / V_c: the Gershgorin bound of the forward-Euler limit of
 * the explicit step (global over ranks; HOST output; synchronises the stream). */
MASPCG_API maspcg_status maspcg_sts_dt_limit(maspcg_ctx *ctx, double *dt_fe, void *cuda_stream);

/* y = A x on the local slab (DEVICE [nloc][nt][nr] each; halo exchanged
 * internally; x and y must not alias).  For tests and operator checks. */
MASPCG_API maspcg_status maspcg_apply(maspcg_ctx *ctx, const double *x, double *y,
                                      void *cuda_stream);

/* ---- staggered vector viscosity with the pole treatment (R27-R31) ---------- */

/* The "viscosity solver" of PAPER.md:290 (Sec. V-C, Fig. 4) on MAS's staggered grid:
 * velocity components on their faces (v_r on r-faces, v_theta on theta-faces, v_phi on phi-faces),
 * the implicit viscous step
 *     s v + curl(nu curl v) - grad(nu div v) = f          (= s v - nu lap v for constant nu)
 * discretised from the energy  1/2 sum_cells nu/V (net outflow)^2 + 1/2 sum_edges W (circulation)^2
 * (mimetic div-curl form, symmetric positive definite for s >= 0 with the walls below).  The polar
 * axis is one r-edge per radius whose circulation is the sum over the whole pole ring of v_phi times
 * its length -- the per-radius array reduction sum0(i) of PAPER.md:147-157 (Listing 3), a ring
 * reduction plus, across phi-slabs, an all-gather in every matvec.  Requires a full sphere in theta
 * (t_faces[0] = 0, t_faces[nt] = pi) and np >= 2.  Solved by the same point-Jacobi PCG (R11-R14).
 *
 * Layouts (DEVICE, the local slab): vectors [nloc][3][nt][nr] -- inside every phi-plane the three
 * components (0 r, 1 theta, 2 phi) of the LOWER faces of its cells; the slots v_r(i = 0) (inner
 * wall face) and v_theta(j = 0) (north-pole face) are not unknowns: ignored on input, 0 on output;
 * the outer wall face and the south-pole face are not stored.  Cell fields [nloc][nt][nr].  Wall
 * data [nloc][3][nt]: [0] the normal velocity on the wall face (j, k), [1] the tangential v_theta
 * at (t_faces[j], phi_c[k]), [2] the tangential v_phi at (theta_c[j], p_faces[k]).
 *
 * The vector operator has its own caller-owned workspace (maspcg_vv_workspace_bytes; 256-byte
 * aligned); the context's base workspace (maspcg_set_workspace) must also be set.  The PCG options
 * (chunk, graphs, timing, arith) apply; the iteration path is always the streaming kernels. */
typedef enum { MASPCG_WALL_NO_SLIP = 0, MASPCG_WALL_FREE_SLIP = 1 } maspcg_wall;

MASPCG_API size_t maspcg_vv_workspace_bytes(const maspcg_ctx *ctx);
MASPCG_API maspcg_status maspcg_vv_set_workspace(maspcg_ctx *ctx, void *dev_ptr, size_t bytes);
/* Cell viscosity nu >= 0 and cell shift s >= 0 (e.g. rho / dt), DEVICE [nloc][nt][nr], copied.
 * Edge viscosities are the arithmetic means of the cells around each edge (the pole ring for the
 * axis), face shifts the means of the two cells of the face (R28).  E_INVALID for a negative or
 * non-finite value (agreed across ranks) or a grid without both poles; E_STATE before set_grid /
 * set_workspace / vv_set_workspace.  The operator is (re)assembled lazily at the next vv call. */
MASPCG_API maspcg_status maspcg_vv_set_coefficients(maspcg_ctx *ctx, const double *nu, const double *shift,
                                                    void *cuda_stream);
/* r walls (R30): NO_SLIP -- the wall edges carry circulations closed through the tangential wall
 * velocity; FREE_SLIP -- no vorticity penalty on the wall edges (zero tangential stress).  Both
 * prescribe the normal velocity g[0].  g_inner / g_outer DEVICE [nloc][3][nt] or NULL (= 0). */
MASPCG_API maspcg_status maspcg_vv_set_bc_r(maspcg_ctx *ctx, maspcg_wall inner, const double *g_inner,
                                            maspcg_wall outer, const double *g_outer, void *cuda_stream);
/* y = A x (homogeneous walls), DEVICE [nloc][3][nt][nr]; x and y must not alias. */
MASPCG_API maspcg_status maspcg_vv_apply(maspcg_ctx *ctx, const double *x, double *y, void *cuda_stream);
/* Solve A v = b, b = M f - A(0; g) (R31: M the face masses area x centre distance, f per unit
 * volume DEVICE [nloc][3][nt][nr]), by Jacobi PCG from x (DEVICE [nloc][3][nt][nr], in: x0, out:
 * the iterate; must not alias f).  tol, maxit, resid_hist, info and the return codes as maspcg_solve. */
MASPCG_API maspcg_status maspcg_vv_solve(maspcg_ctx *ctx, const double *f, double *x, double tol, int maxit,
                                         double *resid_hist, maspcg_info *info, void *cuda_stream);
/* The Jacobi diagonal, HOST [nloc][3][nt][nr] (1 on the non-unknown slots); for tests. */
MASPCG_API maspcg_status maspcg_vv_get_diag(maspcg_ctx *ctx, double *D, void *cuda_stream);

/* ---- field-aligned anisotropic conduction (reading R33 of DESIGN.md) ------------ */

/* The thermal-conduction term of MAS's "full thermodynamic MHD model" (Sec. V-A) in its
 * usual coronal form: heat flux -K grad T along the magnetic field, K = kappa_perp I + kappa_par b b^T
 * (b a unit vector), on the cell-centred grid of the scalar operator (the paper gives no
 * formula).  Volume-weighted symmetric form (R33): the 7-point operator of the DIAGONAL face coefficients
 * K_aa = kappa_perp + kappa_par b_a^2 -- the caller passes them as kr, kt, kp to maspcg_set_coefficients
 * (with the shift s as usual) -- plus CROSS terms kappa_par b_a b_b on the edges where an a-face meets a
 * b-face, each the product of the two averaged face differences around the edge weighted by the exact
 * volume between the four cell centres over the two metric distances.  19-point stencil; symmetric;
 * constants in the kernel of the conduction part; b = r^ gives the radial 7-point operator; positive
 * definite with an isotropic floor kappa_perp > 0 or a shift (semi-definite without them on uniform
 * grids).  Only edges between two interior faces carry a cross term.  Solved by the same Jacobi PCG
 * (R11-R14) on the three-kernel path (MASPCG_OPT_PATH 0 / 1; other paths and super-time-stepping
 * return E_INVALID while cross terms are set), with the Jacobi diagonal including the cross terms.
 *
 * The cross terms live in their own caller-owned workspace (maspcg_aniso_workspace_bytes, 256-byte
 * aligned; about 4 doubles per cell). */
MASPCG_API size_t maspcg_aniso_workspace_bytes(const maspcg_ctx *ctx);
MASPCG_API maspcg_status maspcg_aniso_set_workspace(maspcg_ctx *ctx, void *dev_ptr, size_t bytes);
/* Cross coefficients kappa_par b_a b_b (any sign, finite) at the edge centres, DEVICE, consumed into the
 * library's edge weights (the caller may free them afterwards):
 *   krt [nloc][nt+1][nr+1]: edge (r-face ie, theta-face je) of plane k, at (r_f[ie], t_f[je], phi_c[k]);
 *   krp [nloc][nt][nr+1]:   edge (r-face ie, row j) on phi-face k+1/2, at (r_f[ie], theta_c[j], p_f[k+1]);
 *   ktp [nloc][nt+1][nr]:   edge (theta-face je, column i) on phi-face k+1/2, at (r_c[i], t_f[je], p_f[k+1]).
 * Entries on boundary faces are read (validated) but carry no term.  All three NULL: back to the 7-point
 * operator.  E_INVALID for a non-finite entry (agreed across ranks) or a partial set of NULLs; E_STATE
 * before set_grid / set_workspace / aniso_set_workspace.  The Jacobi diagonal is rebuilt lazily. */
MASPCG_API maspcg_status maspcg_set_aniso_coefficients(maspcg_ctx *ctx, const double *krt, const double *krp,
                                                       const double *ktp, void *cuda_stream);
/* Copy the edge weights Xq = X/4 and the 7-point diagonal D7 (host or device pointers, NULL skips) in the
 * library's layout [nloc][nt][nr]: Xrt (lower r-face i, lower theta-face j), Xrp / Xtp (the phi-face k+1/2
 * of plane k; lower r-face i / lower theta-face j); 0 where a face is a boundary face.  For tests. */
MASPCG_API maspcg_status maspcg_aniso_get_operator(maspcg_ctx *ctx, double *Xrt, double *Xrp, double *Xtp,
                                                   double *D7, void *cuda_stream);

/* ---- peer-memory communicator (SURVEY 8(e) lever 4: in-kernel exchanges) ---------------------- */

/* As maspcg_create, but the halo planes, all-gathers and flag all-reduces are kernels that store into
 * the peers' workspaces over NVLink / NVSwitch and signal with system-scope release flags (no NCCL, no
 * host round trip; captured into the CUDA graphs).  One process (one CUDA context) per rank; every rank
 * calls every function in the same order.  After maspcg_set_workspace (region 0) and
 * maspcg_vv_set_workspace (region 1) every rank exports its region (maspcg_peer_export, 80 bytes: the
 * CUDA IPC handle of the workspace's allocation, offset, size), the caller all-gathers the bytes (e.g.
 * torch.distributed) and imports every peer's (maspcg_peer_import), then barriers before the next call.
 * nranks == 1 needs no import (the rank pushes to itself).  group must be NULL (ranks sharing one context
 * could spin on each other inside one device: E_INVALID).  The fused iteration path (MASPCG_OPT_PATH 2)
 * is not available in this mode (E_INVALID at solve). */
MASPCG_API maspcg_status maspcg_create_peer(int nr, int nt, int np, int rank, int nranks, void *group,
                                            int cuda_device, maspcg_ctx **out);
MASPCG_API maspcg_status maspcg_peer_export(maspcg_ctx *ctx, int region, void *out /* 80 bytes, host */);
MASPCG_API maspcg_status maspcg_peer_import(maspcg_ctx *ctx, int region, int rank, const void *in /* 80 bytes */);

/* ---- in-process multi-rank emulation (TEST ONLY) ------------------------------ */

/* A loopback group lets `nranks` contexts live in ONE process on ONE device, one
 * host thread per rank, exchanging halos and all-reduce operands by device-to-
 * device copies and fixed-order sums instead of NCCL.  It exists so the phi-slab
 * decomposition (halo planes, split interior/boundary stencil, all-reduced
 * scalars) can be verified against the oracle on a single GPU.
 * Every rank must call every function concurrently from its own thread, as with
 * MPI (including maspcg_destroy, which is collective for loopback contexts).
 * Loopback contexts never use CUDA graphs.  The group must outlive its
 * contexts.  nranks in [1, 16]. */
MASPCG_API maspcg_status maspcg_loopback_group_create(int nranks, void **group);
MASPCG_API maspcg_status maspcg_loopback_group_destroy(void *group);
/* As maspcg_create, but joined to a loopback group instead of an NCCL communicator. */
MASPCG_API maspcg_status maspcg_create_loopback(int nr, int nt, int np, int rank, int nranks, void *group,
                                                int cuda_device, maspcg_ctx **out);

/* ---- introspection ------------------------------------------------------------ */

/* Copy the assembled local operator to HOST arrays in the oracle's face
 * layout (NULL skips an array): Tr [nloc][nt][nr+1], Tt [nloc][nt+1][nr],
 * Tp [nloc][nt][nr] (face k+1/2), D [nloc][nt][nr].  Finalises D first. */
MASPCG_API maspcg_status maspcg_get_operator(maspcg_ctx *ctx, double *Tr, double *Tt, double *Tp,
                                             double *D, void *cuda_stream);

MASPCG_API maspcg_status maspcg_set_option(maspcg_ctx *ctx, maspcg_option opt, long long value);
MASPCG_API maspcg_status maspcg_get_stats(const maspcg_ctx *ctx, maspcg_stats *out);
MASPCG_API maspcg_status maspcg_reset_stats(maspcg_ctx *ctx);

/* Library version string, e.g. "maspcg 0.1 sm_100a". */
MASPCG_API const char *maspcg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MASPCG_H */
