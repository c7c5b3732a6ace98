/*
 * masoracle.c -- plain, slow, sequential CPU ORACLE for the MAS implicit
 * parabolic PCG solve (arXiv 2303.03398).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * "--impl reference" legs may load this library.  The product path
 * (paper_2303_03398_b200/, libmaspcg.so) never includes, links or calls it,
 * and this file includes nothing from the product tree.
 *
 * What it follows.  PAPER.md gives no solver mathematics.  It fixes only:
 *   - "a logically rectangular non-uniform staggered spherical grid and
 *     finite-difference discretizations with a combination of explicit and
 *     implicit time-stepping methods"; "highly memory-bound"
 *     (Sec. III "The MAS Solar MHD Model");
 *   - a "stretched grid" test case of 36 M cells (Sec. V-A);
 *   - "viscosity solver iterations" with MPI halo exchanges
 *     (Sec. V-C, Fig. 4);
 *   - validation "to within solver tolerances".
 * BASELINE.json north_star fixes the rest: a symmetric 7-point spherical-metric
 * diffusion operator, point-Jacobi preconditioned CG, fp64.  Every formula
 * below is therefore a READING, numbered R1..R18 exactly as in SURVEY.md
 * section 8(c) and restated in DESIGN.md section 3; each function cites the
 * reading(s) it writes out.
 *
 * Style: triple loops in [k][j][i] order (phi outermost, r contiguous,
 * PAPER.md:128-139 Listing 1 with i fastest), left-to-right sums, no blocking,
 * no fusion, no reordering; dot products are evaluated accurately (Dot2, R24).  Built with -O2 -fno-fast-math -ffp-contract=off so
 * every product and sum is one IEEE fp64 rounding, in the order written.
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"): sum of V closed form; sphere
 * r-face areas; K*1 = 0 (annihilates constants); x.Ay = y.Ax; telescoping
 * flux sum; dense LU on tiny grids; manufactured solution second order;
 * spherical-capacitor closed form; Dirichlet-constant and shift-only exact
 * cases; circulant phi ring vs FFT with the CG iteration bound; a hand-worked
 * two-cell golden fixture (tests/golden/).  Parity status: every function is
 * pinned; the residual HISTORY beyond ~800-1000 iterations on high-contrast
 * inputs is "parity unpinned" (SURVEY.md 8(c) contract (iii)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MO_OK 0
#define MO_NOT_CONVERGED 1
#define MO_E_INVALID (-1)
#define MO_E_SINGULAR (-3)
#define MO_E_BREAKDOWN (-4)
#define MO_E_NOMEM (-7)

#define MO_BC_DIRICHLET 0
#define MO_BC_NEUMANN0 1

/* R9: periodic phi, full 2*pi span.  The period used in h^phi is this literal. */
static const double MO_TWO_PI = 6.283185307179586476925286766559;

#define IDX(k, j, i, nt_, nr_) ((((size_t)(k)) * (size_t)(nt_) + (size_t)(j)) * (size_t)(nr_) + (size_t)(i))

/* ---------------------------------------------------------------- grid (R1,R2,R3) */

/* Grid validity (R1, R9): r_f[0] > 0, all faces strictly increasing,
 * t_f within [0, pi], p_f span equal to 2*pi to 1e-12 relative. */
int masoracle_check_grid(int nr, int nt, int np, const double *rf, const double *tf,
                         const double *pf) {
    if (nr < 1 || nt < 1 || np < 1) return MO_E_INVALID;
    if (!(rf[0] > 0.0)) return MO_E_INVALID;
    for (int i = 0; i < nr; i++) if (!(rf[i + 1] > rf[i])) return MO_E_INVALID;
    for (int j = 0; j < nt; j++) if (!(tf[j + 1] > tf[j])) return MO_E_INVALID;
    for (int k = 0; k < np; k++) if (!(pf[k + 1] > pf[k])) return MO_E_INVALID;
    if (!(tf[0] >= 0.0) || !(tf[nt] <= 3.14159265358979323846)) return MO_E_INVALID;
    if (!(fabs((pf[np] - pf[0]) - MO_TWO_PI) <= 1e-12 * MO_TWO_PI)) return MO_E_INVALID;
    return MO_OK;
}

/* One-dimensional grid quantities (readings R1-R3):
 *   centres are arithmetic midpoints of the faces (R2);
 *   h^r_0 = rc_0 - r_f[0], h^r_i = rc_i - rc_{i-1}, h^r_nr = r_f[nr] - rc_{nr-1};
 *   h^t_j = tc_j - tc_{j-1} (j = 1..nt-1);
 *   h^p_k = pc_{k+1} - pc_k, h^p_{np-1} = pc_0 + 2pi - pc_{np-1} (R9);
 *   R3_i = (r_f[i+1]^3 - r_f[i]^3)/3 = dr_i (r_f[i+1]^2 + r_f[i+1] r_f[i] + r_f[i]^2)/3,
 *   C_j = 2 sin(tc_j) sin(dt_j/2)
 *   (= cos t_f[j] - cos t_f[j+1], the exact integral of sin, written in its
 *   product form, R3).                                                       */
typedef struct {
    double *rc, *dr, *hr, *R3;       /* nr, nr, nr+1, nr */
    double *tc, *dt, *ht, *C, *sinf_, *sinc; /* nt, nt, nt+1, nt, nt+1, nt */
    double *pc, *dp, *hp;            /* np, np, np */
} mo_grid;

static void mo_grid_free(mo_grid *g) {
    free(g->rc); free(g->dr); free(g->hr); free(g->R3);
    free(g->tc); free(g->dt); free(g->ht); free(g->C); free(g->sinf_); free(g->sinc);
    free(g->pc); free(g->dp); free(g->hp);
}

static int mo_grid_build(int nr, int nt, int np, const double *rf, const double *tf,
                         const double *pf, mo_grid *g) {
    memset(g, 0, sizeof(*g));
    g->rc = malloc(sizeof(double) * nr); g->dr = malloc(sizeof(double) * nr);
    g->hr = malloc(sizeof(double) * (nr + 1)); g->R3 = malloc(sizeof(double) * nr);
    g->tc = malloc(sizeof(double) * nt); g->dt = malloc(sizeof(double) * nt);
    g->ht = malloc(sizeof(double) * (nt + 1)); g->C = malloc(sizeof(double) * nt);
    g->sinf_ = malloc(sizeof(double) * (nt + 1)); g->sinc = malloc(sizeof(double) * nt);
    g->pc = malloc(sizeof(double) * np); g->dp = malloc(sizeof(double) * np);
    g->hp = malloc(sizeof(double) * np);
    if (!g->rc || !g->dr || !g->hr || !g->R3 || !g->tc || !g->dt || !g->ht || !g->C ||
        !g->sinf_ || !g->sinc || !g->pc || !g->dp || !g->hp) {
        mo_grid_free(g);
        return MO_E_NOMEM;
    }
    for (int i = 0; i < nr; i++) {
        g->rc[i] = 0.5 * (rf[i] + rf[i + 1]);
        g->dr[i] = rf[i + 1] - rf[i];
        /* (r1^3 - r0^3)/3 written as dr (r1^2 + r1 r0 + r0^2)/3: no cancellation */
        g->R3[i] = g->dr[i] * (rf[i + 1] * rf[i + 1] + rf[i + 1] * rf[i] + rf[i] * rf[i]) / 3.0;
    }
    g->hr[0] = g->rc[0] - rf[0];
    for (int i = 1; i < nr; i++) g->hr[i] = g->rc[i] - g->rc[i - 1];
    g->hr[nr] = rf[nr] - g->rc[nr - 1];

    for (int j = 0; j < nt; j++) {
        g->tc[j] = 0.5 * (tf[j] + tf[j + 1]);
        g->dt[j] = tf[j + 1] - tf[j];
        g->C[j] = 2.0 * sin(g->tc[j]) * sin(0.5 * g->dt[j]);
        g->sinc[j] = sin(g->tc[j]);
    }
    g->ht[0] = 0.0; g->ht[nt] = 0.0; /* boundary theta faces carry no flux (R8) */
    for (int j = 1; j < nt; j++) g->ht[j] = g->tc[j] - g->tc[j - 1];
    for (int j = 0; j <= nt; j++) g->sinf_[j] = sin(tf[j]);

    for (int k = 0; k < np; k++) {
        g->pc[k] = 0.5 * (pf[k] + pf[k + 1]);
        g->dp[k] = pf[k + 1] - pf[k];
    }
    for (int k = 0; k + 1 < np; k++) g->hp[k] = g->pc[k + 1] - g->pc[k];
    g->hp[np - 1] = (g->pc[0] + MO_TWO_PI) - g->pc[np - 1];
    return MO_OK;
}

/* Cell volumes V_kji = R3_i * C_j * dphi_k (R3: exact finite-volume integral
 * of r^2 sin(theta) dr dtheta dphi).                                        */
int masoracle_volumes(int nr, int nt, int np, const double *rf, const double *tf,
                      const double *pf, double *V) {
    int st = masoracle_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mo_grid g;
    if (mo_grid_build(nr, nt, np, rf, tf, pf, &g)) return MO_E_NOMEM;
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++)
                V[IDX(k, j, i, nt, nr)] = g.R3[i] * g.C[j] * g.dp[k];
    mo_grid_free(&g);
    return MO_OK;
}

/* ------------------------------------------------------- operator assembly (R3-R10) */

/* Face transmissibilities and diagonal:
 *   Tr[k][j][i], i = 0..nr   : kr * r_f[i]^2 * C_j * dphi_k / h^r_i
 *   Tt[k][j][i], j = 0..nt   : kt * sin(t_f[j]) * dr_i * dphi_k / h^t_j for
 *                              j = 1..nt-1; 0 on the two theta-boundary faces (R8)
 *   Tp[k][j][i], face k+1/2  : kp * dr_i * dtheta_j / (sin(tc_j) * h^p_k)
 *   D = s*V + Tr_lo + Tr_hi + Tt_lo + Tt_hi + Tp_lo + Tp_hi   (left to right)
 * where the r-boundary faces enter D only when that side is Dirichlet (R7),
 * and Tp_lo of plane k is the face (k-1 mod np)+1/2 (R9).  Input face
 * coefficients kr [np][nt][nr+1], kt [np][nt+1][nr], kp [np][nt][nr] and the
 * shift s [np][nt][nr] are taken as given (R4, R5).  Returns E_INVALID for a
 * negative or non-finite coefficient, E_SINGULAR when s == 0 everywhere and
 * neither r boundary is Dirichlet (R10 / operator definiteness).            */
int masoracle_assemble(int nr, int nt, int np, const double *rf, const double *tf,
                       const double *pf, const double *kr, const double *kt,
                       const double *kp, const double *s, int bc_in, int bc_out,
                       double *Tr, double *Tt, double *Tp, double *D) {
    int st = masoracle_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    if ((bc_in != MO_BC_DIRICHLET && bc_in != MO_BC_NEUMANN0) ||
        (bc_out != MO_BC_DIRICHLET && bc_out != MO_BC_NEUMANN0))
        return MO_E_INVALID;
    size_t ncell = (size_t)nr * nt * np;
    size_t nkr = (size_t)(nr + 1) * nt * np, nkt = (size_t)nr * (nt + 1) * np;
    for (size_t c = 0; c < nkr; c++) if (!(kr[c] >= 0.0) || !isfinite(kr[c])) return MO_E_INVALID;
    for (size_t c = 0; c < nkt; c++) if (!(kt[c] >= 0.0) || !isfinite(kt[c])) return MO_E_INVALID;
    for (size_t c = 0; c < ncell; c++) {
        if (!(kp[c] >= 0.0) || !isfinite(kp[c])) return MO_E_INVALID;
        if (!(s[c] >= 0.0) || !isfinite(s[c])) return MO_E_INVALID;
    }
    int any_shift = 0;
    for (size_t c = 0; c < ncell; c++) if (s[c] > 0.0) any_shift = 1;
    if (!any_shift && bc_in != MO_BC_DIRICHLET && bc_out != MO_BC_DIRICHLET)
        return MO_E_SINGULAR;

    mo_grid g;
    if (mo_grid_build(nr, nt, np, rf, tf, pf, &g)) return MO_E_NOMEM;

    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i <= nr; i++) {
                size_t f = IDX(k, j, i, nt, nr + 1);
                Tr[f] = kr[f] * (rf[i] * rf[i]) * g.C[j] * g.dp[k] / g.hr[i];
            }
    for (int k = 0; k < np; k++)
        for (int j = 0; j <= nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t f = IDX(k, j, i, nt + 1, nr);
                if (j == 0 || j == nt)
                    Tt[f] = 0.0;
                else
                    Tt[f] = kt[f] * g.sinf_[j] * g.dr[i] * g.dp[k] / g.ht[j];
            }
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                Tp[c] = kp[c] * g.dr[i] * g.dt[j] / (g.sinc[j] * g.hp[k]);
            }
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                double V = g.R3[i] * g.C[j] * g.dp[k];
                double trlo = Tr[IDX(k, j, i, nt, nr + 1)];
                double trhi = Tr[IDX(k, j, i + 1, nt, nr + 1)];
                if (i == 0 && bc_in != MO_BC_DIRICHLET) trlo = 0.0;
                if (i == nr - 1 && bc_out != MO_BC_DIRICHLET) trhi = 0.0;
                double ttlo = Tt[IDX(k, j, i, nt + 1, nr)];
                double tthi = Tt[IDX(k, j + 1, i, nt + 1, nr)];
                double tplo = Tp[IDX(km, j, i, nt, nr)];
                double tphi = Tp[c];
                double d = s[c] * V;
                d = d + trlo;
                d = d + trhi;
                d = d + ttlo;
                d = d + tthi;
                d = d + tplo;
                d = d + tphi;
                D[c] = d;
            }
    }
    mo_grid_free(&g);
    return MO_OK;
}

/* ------------------------------------------------- face coefficients from fields (NEXT-1) */

/* kappa of a cell from a physical field (R25): kappa = kappa0 * f^(m/2), evaluated as
 * kappa0 * f * f * ... (m/2 factors) * sqrt(f) (if m odd), left to right -- e.g. Spitzer
 * conduction kappa0 T^(5/2) = ((kappa0 T) T) sqrt(T), viscosity nu rho with m = 2. */
static double mo_kappa(double kappa0, int half_power, double f) {
    double v = kappa0;
    for (int m = 0; m < half_power / 2; m++) v = v * f;
    if (half_power % 2) v = v * sqrt(f);
    return v;
}

/* mean of the two cells of a face (R25): arithmetic (a + b)/2 or harmonic 2ab/(a + b) (0 if a + b == 0) */
static double mo_face_mean(int mode, double a, double b) {
    if (mode == 0) return 0.5 * (a + b);
    double sum = a + b;
    return sum == 0.0 ? 0.0 : ((2.0 * a) * b) / sum;
}

/* Face diffusion coefficients and shift of the global grid from cell fields (SURVEY 8(f) NEXT-1:
 * the per-time-step assembly of MAS's implicit parabolic terms):
 *   kappa_c = kappa0 field_c^(half_power/2); kr, kt: mean of the two cells of an interior face, the
 *   adjacent cell's value on a boundary face; kp (face k+1/2): mean of planes k and k+1 (mod np);
 *   s_c = inv_dt * rho_c (rho == NULL: inv_dt).  Layouts as masoracle_assemble's inputs.
 * Returns E_INVALID for half_power outside [0, 16] or mean not in {0, 1}.                       */
int masoracle_face_coefficients(int nr, int nt, int np, const double *field, double kappa0,
                                int half_power, int mean, const double *rho, double inv_dt,
                                double *kr, double *kt, double *kp, double *s) {
    if (half_power < 0 || half_power > 16 || (mean != 0 && mean != 1)) return MO_E_INVALID;
    for (int k = 0; k < np; k++) {
        int kp1 = (k + 1) % np;
        for (int j = 0; j < nt; j++) {
            for (int i = 0; i <= nr; i++) {
                double v;
                if (i == 0) v = mo_kappa(kappa0, half_power, field[IDX(k, j, 0, nt, nr)]);
                else if (i == nr) v = mo_kappa(kappa0, half_power, field[IDX(k, j, nr - 1, nt, nr)]);
                else v = mo_face_mean(mean, mo_kappa(kappa0, half_power, field[IDX(k, j, i - 1, nt, nr)]),
                                      mo_kappa(kappa0, half_power, field[IDX(k, j, i, nt, nr)]));
                kr[IDX(k, j, i, nt, nr + 1)] = v;
            }
        }
        for (int j = 0; j <= nt; j++)
            for (int i = 0; i < nr; i++) {
                double v;
                if (j == 0) v = mo_kappa(kappa0, half_power, field[IDX(k, 0, i, nt, nr)]);
                else if (j == nt) v = mo_kappa(kappa0, half_power, field[IDX(k, nt - 1, i, nt, nr)]);
                else v = mo_face_mean(mean, mo_kappa(kappa0, half_power, field[IDX(k, j - 1, i, nt, nr)]),
                                      mo_kappa(kappa0, half_power, field[IDX(k, j, i, nt, nr)]));
                kt[IDX(k, j, i, nt + 1, nr)] = v;
            }
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                kp[c] = mo_face_mean(mean, mo_kappa(kappa0, half_power, field[c]),
                                     mo_kappa(kappa0, half_power, field[IDX(kp1, j, i, nt, nr)]));
                s[c] = rho ? inv_dt * rho[c] : inv_dt;
            }
    }
    return MO_OK;
}

/* ------------------------------------------------------------------ apply (R4) */

/* y = A u with (A u)_c = D_c u_c - sum over the interior faces f of c of
 * T_f u_nb(f), summed in the reference order
 *   r_lo, r_hi, theta_lo, theta_hi, phi_lo, phi_hi.
 * r-boundary faces have no neighbour (their Dirichlet part lives in D);
 * theta-boundary faces carry no flux; phi wraps periodically (R9).          */
int masoracle_apply(int nr, int nt, int np, const double *Tr, const double *Tt,
                    const double *Tp, const double *D, const double *u, double *y) {
    /* each y[c] is computed independently; the pragma (the -fopenmp timing build of bench.py's
     * cpu_baseline only) splits the planes across threads without changing any value */
#pragma omp parallel for schedule(static)
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np, kp1 = (k + 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                double sum = 0.0;
                if (i > 0) sum = sum + Tr[IDX(k, j, i, nt, nr + 1)] * u[IDX(k, j, i - 1, nt, nr)];
                if (i < nr - 1) sum = sum + Tr[IDX(k, j, i + 1, nt, nr + 1)] * u[IDX(k, j, i + 1, nt, nr)];
                if (j > 0) sum = sum + Tt[IDX(k, j, i, nt + 1, nr)] * u[IDX(k, j - 1, i, nt, nr)];
                if (j < nt - 1) sum = sum + Tt[IDX(k, j + 1, i, nt + 1, nr)] * u[IDX(k, j + 1, i, nt, nr)];
                sum = sum + Tp[IDX(km, j, i, nt, nr)] * u[IDX(km, j, i, nt, nr)];
                sum = sum + Tp[c] * u[IDX(kp1, j, i, nt, nr)];
                y[c] = D[c] * u[c] - sum;
            }
    }
    return MO_OK;
}

/* -------------------------------------------------------------------- rhs (R5, R7) */

/* b = V f + [i = 0, Dirichlet] Tr_0 g_in + [i = nr-1, Dirichlet] Tr_nr g_out
 * (the boundary value sits on the face).  f is the
 * per-unit-volume right-hand side [np][nt][nr]; g_in, g_out are [np][nt] or
 * NULL for zero.                                                            */
int masoracle_rhs(int nr, int nt, int np, const double *rf, const double *tf,
                  const double *pf, const double *Tr, const double *f, int bc_in,
                  const double *g_in, int bc_out, const double *g_out, double *b) {
    int st = masoracle_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mo_grid g;
    if (mo_grid_build(nr, nt, np, rf, tf, pf, &g)) return MO_E_NOMEM;
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                double V = g.R3[i] * g.C[j] * g.dp[k];
                double v = V * f[c];
                if (i == 0 && bc_in == MO_BC_DIRICHLET && g_in)
                    v = v + Tr[IDX(k, j, 0, nt, nr + 1)] * g_in[(size_t)k * nt + j];
                if (i == nr - 1 && bc_out == MO_BC_DIRICHLET && g_out)
                    v = v + Tr[IDX(k, j, nr, nt, nr + 1)] * g_out[(size_t)k * nt + j];
                b[c] = v;
            }
    mo_grid_free(&g);
    return MO_OK;
}

/* --------------------------------------------------------------- PCG (R6, R11-R14) */

/* Dot products (R24): Dot2 of Ogita, Rump & Oishi (SIAM J. Sci. Comput. 26, 2005, Algorithm 5.3):
 * each product is split exactly into h + r (TwoProduct, Dekker/Veltkamp, plain IEEE operations), the
 * leading parts are summed with error-free TwoSum and every rounding error is accumulated separately;
 * the result equals the dot product computed in twice the working precision and rounded once.  It is
 * still the plain definition sum_i a_i b_i, only evaluated accurately -- so that the value does not
 * depend on the order of summation (up to the final rounding).  Requires -ffp-contract=off. */
static void mo_two_sum(double a, double b, double *x, double *y) {
    double s = a + b;
    double z = s - a;
    *x = s;
    *y = (a - (s - z)) + (b - z);
}

static void mo_split(double a, double *hi, double *lo) {
    double c = 134217729.0 * a; /* 2^27 + 1 */
    double h = c - (c - a);
    *hi = h;
    *lo = a - h;
}

static void mo_two_product(double a, double b, double *x, double *y) {
    double p = a * b, ah, al, bh, bl;
    mo_split(a, &ah, &al);
    mo_split(b, &bh, &bl);
    *x = p;
    *y = al * bl - (((p - ah * bh) - al * bh) - ah * bl);
}

static double mo_dot(size_t n, const double *a, const double *b) {
    double p = 0.0, s = 0.0;
    for (size_t c = 0; c < n; c++) {
        double h, r, q;
        mo_two_product(a[c], b[c], &h, &r);
        mo_two_sum(p, h, &p, &q);
        s = s + (q + r);
    }
    return p + s;
}

/* Point-Jacobi PCG, Hestenes-Stiefel form with Fletcher-Reeves beta
 * (R6, R11-R14):
 *   r0 = b - A x0; z0 = r0/D; p0 = z0; rho0 = r0.z0; bn = ||b||; hist[0] = ||r0||
 *   bn == 0 -> x = 0, OK, iters 0;   hist[0] <= tol*bn -> OK, iters 0
 *   for k = 1..maxit:
 *     q = A p; pi = p.q; pi <= 0 or non-finite -> E_BREAKDOWN
 *     alpha = rho/pi; x += alpha p; r -= alpha q; hist[k] = ||r||
 *     hist[k] <= tol*bn -> OK, iters k
 *     z = r/D; rho' = r.z; beta = rho'/rho; rho = rho'; p = z + beta p
 *   NOT_CONVERGED, iters = maxit.
 * Norms are unweighted Euclidean norms of the volume-weighted system; hist is
 * the recurrence residual.  Non-finite ||b|| or hist -> E_BREAKDOWN.
 * hist must hold maxit+1 doubles (or be NULL).                               */
/* The operator of a PCG solve: y = A u (the 7-point operator, or the field-aligned one of NEXT-4). */
typedef struct {
    int nr, nt, np;
    const double *Tr, *Tt, *Tp, *D;      /* 7-point part (D: its own diagonal) */
    const double *Xrt, *Xrp, *Xtp;       /* field-aligned cross terms, or NULL */
} mo_op;

static void mo_op_apply(const mo_op *op, const double *u, double *y);

static int mo_pcg(const mo_op *op, const double *D, const double *b, double *x, double tol, int maxit,
                  double *hist, int *iters, double *bnorm, double *rnorm);

int masoracle_pcg(int nr, int nt, int np, const double *Tr, const double *Tt,
                  const double *Tp, const double *D, const double *b, double *x,
                  double tol, int maxit, double *hist, int *iters, double *bnorm,
                  double *rnorm) {
    mo_op op = {nr, nt, np, Tr, Tt, Tp, D, NULL, NULL, NULL};
    return mo_pcg(&op, D, b, x, tol, maxit, hist, iters, bnorm, rnorm);
}

/* PCG on any operator `op` with the Jacobi diagonal D (the algorithm of masoracle_pcg above). */
static int mo_pcg(const mo_op *op, const double *D, const double *b, double *x, double tol, int maxit,
                  double *hist, int *iters, double *bnorm, double *rnorm) {
    size_t n = (size_t)op->nr * op->nt * op->np;
    if (maxit < 0 || !(tol >= 0.0)) return MO_E_INVALID;
    *iters = 0;
    double bn = sqrt(mo_dot(n, b, b));
    *bnorm = bn;
    if (!isfinite(bn)) { *rnorm = bn; return MO_E_BREAKDOWN; }
    if (bn == 0.0) {
        for (size_t c = 0; c < n; c++) x[c] = 0.0;
        if (hist) hist[0] = 0.0;
        *rnorm = 0.0;
        return MO_OK;
    }
    double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    double *p = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * n);
    if (!r || !z || !p || !q) { free(r); free(z); free(p); free(q); return MO_E_NOMEM; }
    int status = MO_NOT_CONVERGED;

    mo_op_apply(op, x, q);
#pragma omp parallel for schedule(static)
    for (size_t c = 0; c < n; c++) r[c] = b[c] - q[c];
#pragma omp parallel for schedule(static)
    for (size_t c = 0; c < n; c++) z[c] = r[c] / D[c];
#pragma omp parallel for schedule(static)
    for (size_t c = 0; c < n; c++) p[c] = z[c];
    double rho = mo_dot(n, r, z);
    double rn = sqrt(mo_dot(n, r, r));
    if (hist) hist[0] = rn;
    *rnorm = rn;
    if (!isfinite(rn) || !isfinite(rho)) { status = MO_E_BREAKDOWN; goto done; }
    if (rn <= tol * bn) { status = MO_OK; goto done; }

    for (int k = 1; k <= maxit; k++) {
        mo_op_apply(op, p, q);
        double pi = mo_dot(n, p, q);
        if (!(pi > 0.0) || !isfinite(pi)) { status = MO_E_BREAKDOWN; break; }
        double alpha = rho / pi;
#pragma omp parallel for schedule(static)
        for (size_t c = 0; c < n; c++) x[c] = x[c] + alpha * p[c];
#pragma omp parallel for schedule(static)
        for (size_t c = 0; c < n; c++) r[c] = r[c] - alpha * q[c];
        rn = sqrt(mo_dot(n, r, r));
        if (hist) hist[k] = rn;
        *iters = k;
        *rnorm = rn;
        if (!isfinite(rn)) { status = MO_E_BREAKDOWN; break; }
        if (rn <= tol * bn) { status = MO_OK; break; }
#pragma omp parallel for schedule(static)
        for (size_t c = 0; c < n; c++) z[c] = r[c] / D[c];
        double rho_new = mo_dot(n, r, z);
        double beta = rho_new / rho;
        rho = rho_new;
#pragma omp parallel for schedule(static)
        for (size_t c = 0; c < n; c++) p[c] = z[c] + beta * p[c];
    }
done:
    free(r); free(z); free(p); free(q);
    return status;
}

/* Single-reduction point-Jacobi PCG: the Chronopoulos-Gear variant (Chronopoulos & Gear, J. Comput.
 * Appl. Math. 25, 1989; SURVEY 8(f) NEXT-3 "single-reduction (Chronopoulos-Gear) ... CG"; reading R32).
 * All three dot products of an iteration follow ONE operator application, so a distributed solve needs
 * one all-reduce per iteration instead of two:
 *   r0 = b - A x0; u0 = r0/D; w0 = A u0; gamma0 = r0.u0; delta0 = w0.u0; hist[0] = ||r0||
 *   for k = 1..maxit:
 *     k == 1: beta = 0, den = delta;  else: beta = gamma/gamma_old, den = delta - (beta gamma)/alpha_old
 *     den <= 0 or non-finite -> E_BREAKDOWN
 *     alpha = gamma/den; p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s
 *     hist[k] = ||r||; hist[k] <= tol*bn -> OK, iters k
 *     u = r/D; w = A u; gamma_old = gamma; alpha_old = alpha; gamma = r.u; delta = w.u
 * In exact arithmetic s = A p, den = p.Ap and the iterates are those of masoracle_pcg; in floating
 * point they differ at rounding level (the recurrences replace p.Ap).  Early exits, norms and the
 * stopping test as masoracle_pcg (R12-R14). */
int masoracle_pcg_cg1(int nr, int nt, int np, const double *Tr, const double *Tt, const double *Tp, const double *D,
                      const double *b, double *x, double tol, int maxit, double *hist, int *iters, double *bnorm,
                      double *rnorm) {
    size_t n = (size_t)nr * nt * np;
    if (maxit < 0 || !(tol >= 0.0)) return MO_E_INVALID;
    *iters = 0;
    double bn = sqrt(mo_dot(n, b, b));
    *bnorm = bn;
    if (!isfinite(bn)) { *rnorm = bn; return MO_E_BREAKDOWN; }
    if (bn == 0.0) {
        for (size_t c = 0; c < n; c++) x[c] = 0.0;
        if (hist) hist[0] = 0.0;
        *rnorm = 0.0;
        return MO_OK;
    }
    double *r = malloc(sizeof(double) * n), *u = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
    double *p = calloc(n, sizeof(double)), *s = calloc(n, sizeof(double));
    if (!r || !u || !w || !p || !s) { free(r); free(u); free(w); free(p); free(s); return MO_E_NOMEM; }
    int status = MO_NOT_CONVERGED;
    masoracle_apply(nr, nt, np, Tr, Tt, Tp, D, x, w);
    for (size_t c = 0; c < n; c++) r[c] = b[c] - w[c];
    double rn = sqrt(mo_dot(n, r, r));
    if (hist) hist[0] = rn;
    *rnorm = rn;
    if (!isfinite(rn)) { status = MO_E_BREAKDOWN; goto done; }
    if (rn <= tol * bn) { status = MO_OK; goto done; }
    for (size_t c = 0; c < n; c++) u[c] = r[c] / D[c];
    masoracle_apply(nr, nt, np, Tr, Tt, Tp, D, u, w);
    double gamma = mo_dot(n, r, u), delta = mo_dot(n, w, u), gamma_old = 0.0, alpha_old = 0.0;
    for (int k = 1; k <= maxit; k++) {
        double beta = 0.0, den = delta;
        if (k > 1) {
            beta = gamma / gamma_old;
            double t = beta * gamma;
            t = t / alpha_old;
            den = delta - t;
        }
        if (!(den > 0.0) || !isfinite(den) || !isfinite(gamma)) { status = MO_E_BREAKDOWN; break; }
        double alpha = gamma / den;
        for (size_t c = 0; c < n; c++) p[c] = u[c] + beta * p[c];
        for (size_t c = 0; c < n; c++) s[c] = w[c] + beta * s[c];
        for (size_t c = 0; c < n; c++) x[c] = x[c] + alpha * p[c];
        for (size_t c = 0; c < n; c++) r[c] = r[c] - alpha * s[c];
        rn = sqrt(mo_dot(n, r, r));
        if (hist) hist[k] = rn;
        *iters = k;
        *rnorm = rn;
        if (!isfinite(rn)) { status = MO_E_BREAKDOWN; break; }
        if (rn <= tol * bn) { status = MO_OK; break; }
        for (size_t c = 0; c < n; c++) u[c] = r[c] / D[c];
        masoracle_apply(nr, nt, np, Tr, Tt, Tp, D, u, w);
        gamma_old = gamma;
        alpha_old = alpha;
        gamma = mo_dot(n, r, u);
        delta = mo_dot(n, w, u);
    }
done:
    free(r); free(u); free(w); free(p); free(s);
    return status;
}

/* ---------------------------------------------------- super-time-stepping (NEXT-4) */

/* RKL2 coefficients (Meyer, Balsara & Aslam 2014, J. Comput. Phys. 257, eq. 16-17; reading R26):
 * b_j = (j^2 + j - 2) / (2 j (j + 1)) for j >= 2, b_0 = b_1 = b_2; a_j = 1 - b_j;
 * w1 = 4 / (s^2 + s - 2); mu~_1 = b_1 w1; for j >= 2:
 * mu_j = (2j - 1)/j * b_j / b_{j-1}, nu_j = -(j - 1)/j * b_j / b_{j-2}, mu~_j = mu_j w1,
 * gamma~_j = -a_{j-1} mu~_j.  Evaluated left to right exactly as written.                   */
static double mo_rkl2_b(int j) {
    if (j < 2) j = 2;
    return ((double)j * j + j - 2.0) / (2.0 * j * (j + 1.0));
}

void masoracle_rkl2_coefficients(int s, int j, double *mu, double *nu, double *mut, double *gat) {
    double w1 = 4.0 / ((double)s * s + s - 2.0);
    if (j == 1) {
        *mu = 1.0; *nu = 0.0; *mut = mo_rkl2_b(1) * w1; *gat = 0.0;
        return;
    }
    double bj = mo_rkl2_b(j), bj1 = mo_rkl2_b(j - 1), bj2 = mo_rkl2_b(j - 2);
    *mu = (2.0 * j - 1.0) / j * bj / bj1;
    *nu = -((double)j - 1.0) / j * bj / bj2;
    *mut = *mu * w1;
    *gat = -(1.0 - bj1) * *mut;
}

/* L(u) = (b_D - K u) / V, the explicit form of the diffusion term of the operator (K = A - diag(sV),
 * b_D the Dirichlet face terms of masoracle_rhs with f = 0):  Ku = (A u) - (s V) u. */
static void mo_L(int nr, int nt, int np, const double *Tr, const double *Tt, const double *Tp,
                 const double *D, const double *sV, const double *V, const double *bD, const double *u,
                 double *y, double *L) {
    masoracle_apply(nr, nt, np, Tr, Tt, Tp, D, u, y);
    size_t n = (size_t)nr * nt * np;
    for (size_t c = 0; c < n; c++) {
        double Ku = y[c] - sV[c] * u[c];
        L[c] = (bD[c] - Ku) / V[c];
    }
}

/* One RKL2 super-time-step of  V du/dt = b_D - K u  over tau with `stages` >= 2 stages
 * (reading R26).  sV = s * V (as assembled), V the cell volumes, bD the
 * Dirichlet terms; u [np][nt][nr] in, out [np][nt][nr] out (may alias u).
 *   Y0 = u; Y1 = Y0 + (mu~_1 tau) L(Y0);
 *   Yj = mu_j Y_{j-1} + nu_j Y_{j-2} + (1 - mu_j - nu_j) Y0 + (mu~_j tau) L(Y_{j-1}) + (gamma~_j tau) L(Y0)
 * (terms added left to right); out = Y_s.                                                     */
int masoracle_rkl2_step(int nr, int nt, int np, const double *Tr, const double *Tt, const double *Tp,
                        const double *D, const double *sV, const double *V, const double *bD,
                        const double *u, double tau, int stages, double *out) {
    if (stages < 2) return MO_E_INVALID;
    size_t n = (size_t)nr * nt * np;
    double *Y0 = malloc(8 * n), *Ya = malloc(8 * n), *Yb = malloc(8 * n), *Yc = malloc(8 * n);
    double *L0 = malloc(8 * n), *Lj = malloc(8 * n), *y = malloc(8 * n);
    if (!Y0 || !Ya || !Yb || !Yc || !L0 || !Lj || !y) {
        free(Y0); free(Ya); free(Yb); free(Yc); free(L0); free(Lj); free(y);
        return MO_E_NOMEM;
    }
    memcpy(Y0, u, 8 * n);
    mo_L(nr, nt, np, Tr, Tt, Tp, D, sV, V, bD, Y0, y, L0);
    double mu, nu, mut, gat;
    masoracle_rkl2_coefficients(stages, 1, &mu, &nu, &mut, &gat);
    double m1 = mut * tau;
    for (size_t c = 0; c < n; c++) Ya[c] = Y0[c] + m1 * L0[c];   /* Ya = Y1, Yb = Y0 (= Y_{j-2} at j = 2) */
    memcpy(Yb, Y0, 8 * n);
    for (int j = 2; j <= stages; j++) {
        masoracle_rkl2_coefficients(stages, j, &mu, &nu, &mut, &gat);
        double w0 = 1.0 - mu - nu, mt = mut * tau, gt = gat * tau;
        mo_L(nr, nt, np, Tr, Tt, Tp, D, sV, V, bD, Ya, y, Lj);
        for (size_t c = 0; c < n; c++) {
            double t = mu * Ya[c];
            t = t + nu * Yb[c];
            t = t + w0 * Y0[c];
            t = t + mt * Lj[c];
            t = t + gt * L0[c];
            Yc[c] = t;
        }
        double *tmp = Yb; Yb = Ya; Ya = Yc; Yc = tmp;   /* Y_{j-2} <- Y_{j-1}, Y_{j-1} <- Y_j */
    }
    memcpy(out, Ya, 8 * n);
    free(Y0); free(Ya); free(Yb); free(Yc); free(L0); free(Lj); free(y);
    return MO_OK;
}

/* Whole pipeline on the global grid: assemble (R3-R10), rhs (R5), PCG (R6,
 * R11-R14).  x holds x0 on entry and the iterate on exit.                  */
int masoracle_solve(int nr, int nt, int np, const double *rf, const double *tf,
                    const double *pf, const double *kr, const double *kt, const double *kp,
                    const double *s, int bc_in, const double *g_in, int bc_out,
                    const double *g_out, const double *f, double *x, double tol, int maxit,
                    double *hist, int *iters, double *bnorm, double *rnorm) {
    size_t n = (size_t)nr * nt * np;
    double *Tr = malloc(sizeof(double) * (size_t)(nr + 1) * nt * np);
    double *Tt = malloc(sizeof(double) * (size_t)nr * (nt + 1) * np);
    double *Tp = malloc(sizeof(double) * n), *D = malloc(sizeof(double) * n);
    double *b = malloc(sizeof(double) * n);
    int st = MO_E_NOMEM;
    *iters = 0;
    if (!Tr || !Tt || !Tp || !D || !b) goto out;
    st = masoracle_assemble(nr, nt, np, rf, tf, pf, kr, kt, kp, s, bc_in, bc_out, Tr, Tt, Tp, D);
    if (st) goto out;
    st = masoracle_rhs(nr, nt, np, rf, tf, pf, Tr, f, bc_in, g_in, bc_out, g_out, b);
    if (st) goto out;
    st = masoracle_pcg(nr, nt, np, Tr, Tt, Tp, D, b, x, tol, maxit, hist, iters, bnorm, rnorm);
out:
    free(Tr); free(Tt); free(Tp); free(D); free(b);
    return st;
}

/* ============================================ field-aligned anisotropic conduction (NEXT-4, R33)
 *
 * "field-aligned anisotropic conduction (b.b.grad T, a 19-point stencil; not
 * described in the paper)" -- the usual coronal form of the thermal-conduction term of MAS's "full
 * thermodynamic MHD model" (Sec. V-A) on its staggered spherical grid (PAPER.md:56,
 * Sec. III).  PAPER.md gives no formula; everything here is reading R33:
 *
 *   flux q = -K grad T with K = kappa_perp I + kappa_par b b^T (b a unit vector), in the volume-weighted
 *   symmetric form A = diag(sV) + Hessian of the discrete energy
 *       E(T) = 1/2 sum_faces T_f (dT_f)^2  +  sum_edges X_e (a_e.T)(b_e.T)
 *   -- the first sum is the 7-point operator with face coefficients K_aa = kappa_perp + kappa_par b_a^2
 *   (caller's kr, kt, kp: the diagonal terms of (b.grad T)^2); the second the cross terms
 *   2 b_a b_b d_a T d_b T, each on the edges where an a-face meets a b-face: a_e.T and b_e.T are the
 *   two face differences of the 2x2 cells around the edge, averaged (a_e.T = da/2, b_e.T = db/2), and
 *       X_e = k_ab(edge) * V_dual(e) / (h_a * h_b)   (k_ab = kappa_par b_a b_b at the edge centre)
 *   with V_dual the exact volume between the four cell centres and h the metric distances of the two
 *   differences at the edge.  Only edges between two interior faces carry a cross term (boundary
 *   faces: the normal term only, R7, R8).  A couples a cell to its 6 face and 12 edge neighbours
 *   (19 points); it is symmetric by construction, annihilates constants, reduces to the 7-point
 *   operator when b = r^ (kt = kp = kappa_perp, no cross terms), and for constant coefficients on a
 *   uniform grid its symbol 4 x^T (cc^T + diag(1 - c_a^2)) x, x_a = b_a sin(xi_a/2), c_a = cos(xi_a/2),
 *   is >= 0: semi-definite, definite with a floor kappa_perp > 0 or a shift.
 *
 * Edge metric (1-D factors, exact integrals of the dual volumes):
 *   r-theta edge (r face ie, theta face je, plane k):  X = k * gr_ie * gt_je * dphi_k
 *   r-phi edge (r face ie, row j, phi face k+1/2):     X = k * gr_ie * cs_j
 *   theta-phi edge (theta face je, column i, phi face k+1/2): X = k * q_i * gts_je
 *     gr_ie  = (rc_ie^2 + rc_ie rc_ie-1 + rc_ie-1^2) / (3 r_f[ie])   [(rc^3 - rc'^3)/3 / (h^r r_f)]
 *     gt_je  = (cos tc_je-1 - cos tc_je) / h^t_je = 2 sin((tc_je-1 + tc_je)/2) sin(h^t_je/2) / h^t_je
 *     cs_j   = 2 sin(dtheta_j / 2)                                  [C_j / sin tc_j]
 *     q_i    = R3_i / rc_i^2,   gts_je = gt_je / sin t_f[je]
 * stored as Xq = X / 4 (the two averages' factors 1/2 folded in), so that
 *   (A u)_c = (D7_c u_c - 7-point neighbour sum) + sum_{12 edges of c} Xq_e (s_a db + s_b da)
 * with da, db the sums of the two a- and b-differences around the edge and s_a, s_b = +1 when c is on
 * the high side of the edge's a- / b-face, -1 otherwise; diag(A)_c = D7_c + sum_e Xq_e (2 s_a s_b).
 * Edge order of a cell (i, j, k): r-theta (i,j) (i+1,j) (i,j+1) (i+1,j+1); r-phi (i,k-1/2) (i+1,k-1/2)
 * (i,k+1/2) (i+1,k+1/2); theta-phi (j,k-1/2) (j+1,k-1/2) (j,k+1/2) (j+1,k+1/2); left-to-right sums.
 *
 * Layouts: krt, Xrt [np][nt+1][nr+1] (edge (ie, je) of plane k); krp, Xrp [np][nt][nr+1] (edge (ie, j)
 * on phi face k+1/2); ktp, Xtp [np][nt+1][nr] (edge (je, i) on phi face k+1/2).  Pins:
 * tests/test_oracle_aniso_pins.py.                                                                     */

/* Edge weights Xq (= X / 4) from the cross coefficients kappa_par b_a b_b given at the edge centres;
 * 0 on edges with a boundary face.  E_INVALID for a non-finite coefficient (any sign is allowed).  */
int masoracle_aniso_edges(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                          const double *krt, const double *krp, const double *ktp,
                          double *Xrt, double *Xrp, double *Xtp) {
    int st = masoracle_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    size_t nrt = (size_t)np * (nt + 1) * (nr + 1), nrp = (size_t)np * nt * (nr + 1), ntp = (size_t)np * (nt + 1) * nr;
    for (size_t c = 0; c < nrt; c++) if (!isfinite(krt[c])) return MO_E_INVALID;
    for (size_t c = 0; c < nrp; c++) if (!isfinite(krp[c])) return MO_E_INVALID;
    for (size_t c = 0; c < ntp; c++) if (!isfinite(ktp[c])) return MO_E_INVALID;
    mo_grid g;
    if (mo_grid_build(nr, nt, np, rf, tf, pf, &g)) return MO_E_NOMEM;
    for (int k = 0; k < np; k++)
        for (int je = 0; je <= nt; je++)
            for (int ie = 0; ie <= nr; ie++) {
                size_t e = IDX(k, je, ie, nt + 1, nr + 1);
                if (ie < 1 || ie > nr - 1 || je < 1 || je > nt - 1) { Xrt[e] = 0.0; continue; }
                double gr = (g.rc[ie] * g.rc[ie] + g.rc[ie] * g.rc[ie - 1] + g.rc[ie - 1] * g.rc[ie - 1]) / (3.0 * rf[ie]);
                double gt = 2.0 * sin(0.5 * (g.tc[je - 1] + g.tc[je])) * sin(0.5 * g.ht[je]) / g.ht[je];
                Xrt[e] = krt[e] * gr * gt * g.dp[k] * 0.25;
            }
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int ie = 0; ie <= nr; ie++) {
                size_t e = IDX(k, j, ie, nt, nr + 1);
                if (ie < 1 || ie > nr - 1) { Xrp[e] = 0.0; continue; }
                double gr = (g.rc[ie] * g.rc[ie] + g.rc[ie] * g.rc[ie - 1] + g.rc[ie - 1] * g.rc[ie - 1]) / (3.0 * rf[ie]);
                double cs = 2.0 * sin(0.5 * g.dt[j]);
                Xrp[e] = krp[e] * gr * cs * 0.25;
            }
    for (int k = 0; k < np; k++)
        for (int je = 0; je <= nt; je++)
            for (int i = 0; i < nr; i++) {
                size_t e = IDX(k, je, i, nt + 1, nr);
                if (je < 1 || je > nt - 1) { Xtp[e] = 0.0; continue; }
                double q = g.R3[i] / (g.rc[i] * g.rc[i]);
                double gt = 2.0 * sin(0.5 * (g.tc[je - 1] + g.tc[je])) * sin(0.5 * g.ht[je]) / g.ht[je];
                double gts = gt / g.sinf_[je];
                Xtp[e] = ktp[e] * q * gts * 0.25;
            }
    mo_grid_free(&g);
    return MO_OK;
}

/* The cross sum of cell (k, j, i) in the edge order of R33 (diag = 0), or its diagonal
 * sum_e Xq_e (2 s_a s_b) (diag = 1). */
static double mo_aniso_cross(const mo_op *op, const double *u, int k, int j, int i, int diag) {
    const int nr = op->nr, nt = op->nt, np = op->np;
    const int km = (k + np - 1) % np, kp1 = (k + 1) % np;
    double sx = 0.0;
    /* r-theta edges of plane k */
    for (int e = 0; e < 4; e++) {
        int ie = i + (e & 1), je = j + (e >> 1);
        if (ie < 1 || ie > nr - 1 || je < 1 || je > nt - 1) continue;
        double sa = (ie == i) ? 1.0 : -1.0, sb = (je == j) ? 1.0 : -1.0;
        double X = op->Xrt[IDX(k, je, ie, nt + 1, nr + 1)];
        if (diag) { sx = sx + X * (2.0 * sa * sb); continue; }
        double u00 = u[IDX(k, je - 1, ie - 1, nt, nr)], u10 = u[IDX(k, je - 1, ie, nt, nr)];
        double u01 = u[IDX(k, je, ie - 1, nt, nr)], u11 = u[IDX(k, je, ie, nt, nr)];
        double da = (u10 - u00) + (u11 - u01);   /* the two r-differences */
        double db = (u01 - u00) + (u11 - u10);   /* the two theta-differences */
        sx = sx + X * (sa * db + sb * da);
    }
    /* r-phi edges of row j: faces k-1/2 (planes km, k) and k+1/2 (planes k, kp1) */
    for (int e = 0; e < 4; e++) {
        int ie = i + (e & 1), hi = e >> 1;
        if (ie < 1 || ie > nr - 1) continue;
        int ka = hi ? k : km, kb = hi ? kp1 : k;
        double sa = (ie == i) ? 1.0 : -1.0, sb = hi ? -1.0 : 1.0;
        double X = op->Xrp[IDX(ka, j, ie, nt, nr + 1)];
        if (diag) { sx = sx + X * (2.0 * sa * sb); continue; }
        double ua0 = u[IDX(ka, j, ie - 1, nt, nr)], ua1 = u[IDX(ka, j, ie, nt, nr)];
        double ub0 = u[IDX(kb, j, ie - 1, nt, nr)], ub1 = u[IDX(kb, j, ie, nt, nr)];
        double da = (ua1 - ua0) + (ub1 - ub0);   /* the two r-differences */
        double db = (ub0 - ua0) + (ub1 - ua1);   /* the two phi-differences */
        sx = sx + X * (sa * db + sb * da);
    }
    /* theta-phi edges of column i */
    for (int e = 0; e < 4; e++) {
        int je = j + (e & 1), hi = e >> 1;
        if (je < 1 || je > nt - 1) continue;
        int ka = hi ? k : km, kb = hi ? kp1 : k;
        double sa = (je == j) ? 1.0 : -1.0, sb = hi ? -1.0 : 1.0;
        double X = op->Xtp[IDX(ka, je, i, nt + 1, nr)];
        if (diag) { sx = sx + X * (2.0 * sa * sb); continue; }
        double ua0 = u[IDX(ka, je - 1, i, nt, nr)], ua1 = u[IDX(ka, je, i, nt, nr)];
        double ub0 = u[IDX(kb, je - 1, i, nt, nr)], ub1 = u[IDX(kb, je, i, nt, nr)];
        double da = (ua1 - ua0) + (ub1 - ub0);   /* the two theta-differences */
        double db = (ub0 - ua0) + (ub1 - ua1);   /* the two phi-differences */
        sx = sx + X * (sa * db + sb * da);
    }
    return sx;
}

static void mo_op_apply(const mo_op *op, const double *u, double *y) {
    masoracle_apply(op->nr, op->nt, op->np, op->Tr, op->Tt, op->Tp, op->D, u, y);
    if (!op->Xrt) return;
#pragma omp parallel for schedule(static)
    for (int k = 0; k < op->np; k++)
        for (int j = 0; j < op->nt; j++)
            for (int i = 0; i < op->nr; i++) {
                size_t c = IDX(k, j, i, op->nt, op->nr);
                y[c] = y[c] + mo_aniso_cross(op, u, k, j, i, 0);
            }
}

/* y = A u of the field-aligned operator: the 7-point operator (Tr, Tt, Tp, its diagonal D7 from
 * masoracle_assemble with the face coefficients K_aa) plus the cross terms. */
int masoracle_aniso_apply(int nr, int nt, int np, const double *Tr, const double *Tt, const double *Tp,
                          const double *D7, const double *Xrt, const double *Xrp, const double *Xtp,
                          const double *u, double *y) {
    mo_op op = {nr, nt, np, Tr, Tt, Tp, D7, Xrt, Xrp, Xtp};
    mo_op_apply(&op, u, y);
    return MO_OK;
}

/* Jacobi diagonal of the field-aligned operator: Dj = D7 + sum_e Xq_e (2 s_a s_b). */
int masoracle_aniso_diag(int nr, int nt, int np, const double *D7, const double *Xrt, const double *Xrp,
                         const double *Xtp, double *Dj) {
    mo_op op = {nr, nt, np, NULL, NULL, NULL, D7, Xrt, Xrp, Xtp};
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                size_t c = IDX(k, j, i, nt, nr);
                Dj[c] = D7[c] + mo_aniso_cross(&op, NULL, k, j, i, 1);
            }
    return MO_OK;
}

/* Point-Jacobi PCG (masoracle_pcg's algorithm, R6, R11-R14) on the field-aligned operator with the
 * Jacobi diagonal Dj (masoracle_aniso_diag). */
int masoracle_aniso_pcg(int nr, int nt, int np, const double *Tr, const double *Tt, const double *Tp,
                        const double *D7, const double *Xrt, const double *Xrp, const double *Xtp,
                        const double *Dj, const double *b, double *x, double tol, int maxit, double *hist,
                        int *iters, double *bnorm, double *rnorm) {
    mo_op op = {nr, nt, np, Tr, Tt, Tp, D7, Xrt, Xrp, Xtp};
    return mo_pcg(&op, Dj, b, x, tol, maxit, hist, iters, bnorm, rnorm);
}
