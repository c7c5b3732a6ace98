/*
 * masoracle_vv.c -- plain, slow, sequential CPU ORACLE for the staggered
 * VECTOR viscosity solve with pole treatment.
 * TEST INFRASTRUCTURE ONLY (same rules as masoracle.c: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
 * load it; it includes nothing from the product tree).
 *
 * What it follows.  PAPER.md fixes that MAS's unknowns live on a "staggered
 * spherical grid" (Sec. III), that the profiled solver is the
 * "viscosity solver" (Sec. V-C, Fig. 4) and that MAS contains
 * per-radius array reductions over a grid plane, "sum0(i)=sum0(i)+array(i,j)*..."
 * (Listing 3, Listing 4
 * Listing 5).  It gives no formula.  The discretisation below is therefore a
 * READING (R27-R31), the mimetic ("div-curl") form of the vector
 * diffusion operator:
 *
 *   s v + curl(nu curl v) - grad(nu div v) = f        (= s v - nu lap v for constant nu)
 *
 * from the energy E(v) = 1/2 sum_c nu_c/V_c delta_c^2 + 1/2 sum_e W_e Gamma_e^2
 * (delta_c = net outflow of cell c, Gamma_e = circulation around edge e), so
 * the matrix is symmetric by construction:
 *   - unknowns: v_r on r-faces, v_t on theta-faces, v_p on phi-faces (MAC);
 *   - the face "mass" M_f = A_f l_f (face area x centre-to-centre distance);
 *   - the polar axis is an r-edge shared by the whole pole row of cells: its
 *     circulation Gamma_N(i) = sum_k l_p v_p(i, 0, k) is the per-radius sum
 *     over the pole ring -- Listing 3's array reduction sum0(i) (R29).
 *
 * Layout: vectors [np][3][nt][nr] (component c = 0: r, 1: theta, 2: phi inside
 * each phi-plane; the LOWER face of cell (i, j, k) in slot (k, c, j, i)).
 * Slots that are not unknowns: v_r on the inner wall face i = 0 (Dirichlet) and
 * v_t on the north-pole face j = 0 (zero area); they are ignored on input and
 * 0 on output.  The outer wall face (i = nr) and the south-pole face (j = nt)
 * are not stored.  Wall data g [3][np][nt]: g[0] the normal velocity on the
 * wall face (j, k); g[1] the tangential v_t at (t_f[j], phi_c[k]); g[2] the
 * tangential v_p at (theta_c[j], p_f[k]).  NULL = 0.
 *
 * Style: loops in [k][j][i] order, one IEEE rounding per operation in the
 * order written (-ffp-contract=off), Dot2 sums (R24) for the ring sums and the
 * PCG dot products.  Pins: tests/test_oracle_vv_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MV_OK 0
#define MV_NOT_CONVERGED 1
#define MV_E_INVALID (-1)
#define MV_E_BREAKDOWN (-4)
#define MV_E_NOMEM (-7)

#define MV_NO_SLIP 0
#define MV_FREE_SLIP 1

static const double MV_TWO_PI = 6.283185307179586476925286766559;
static const double MV_PI = 3.14159265358979323846;

/* cell (k, j, i) of an [np][nt][nr] array */
#define CI(k, j, i) ((((size_t)(k)) * (size_t)nt + (size_t)(j)) * (size_t)nr + (size_t)(i))
/* component c of face slot (k, j, i) of a [np][3][nt][nr] vector */
#define VI(k, c, j, i) (((((size_t)(k)) * 3 + (size_t)(c)) * (size_t)nt + (size_t)(j)) * (size_t)nr + (size_t)(i))
/* wall datum c at (j, k) of a [3][np][nt] array */
#define GI(c, k, j) ((((size_t)(c)) * (size_t)np + (size_t)(k)) * (size_t)nt + (size_t)(j))

/* ------------------------------------------------------------------ Dot2 (R24) */
static void mv_two_sum(double a, double b, double *x, double *y) {
    double s = a + b;
    double z = s - a;
    *x = s;
    *y = (a - (s - z)) + (b - z);
}
static void mv_split(double a, double *hi, double *lo) {
    double c = 134217729.0 * a;
    double h = c - (c - a);
    *hi = h;
    *lo = a - h;
}
static void mv_two_product(double a, double b, double *x, double *y) {
    double p = a * b, ah, al, bh, bl;
    mv_split(a, &ah, &al);
    mv_split(b, &bh, &bl);
    *x = p;
    *y = al * bl - (((p - ah * bh) - al * bh) - ah * bl);
}
/* sum_c a[c*sa] b[c*sb], Dot2 of Ogita, Rump & Oishi (2005), sequential */
static double mv_dot(size_t n, const double *a, size_t sa, const double *b, size_t sb) {
    double p = 0.0, s = 0.0;
    for (size_t c = 0; c < n; c++) {
        double h, r, q;
        mv_two_product(a[c * sa], b[c * sb], &h, &r);
        mv_two_sum(p, h, &p, &q);
        s = s + (q + r);
    }
    return p + s;
}

/* ------------------------------------------------------------ grid (R27) */
/* 1-D metric of the staggered vector grid.  Besides the scalar grid (R2, R3, R19, R20):
 *   rce[e], e = 0..nr+1 : r_f[0], rc_0 .. rc_{nr-1}, r_f[nr]  (centres extended by the walls)
 *   rhor[e], e = 0..nr  : hr[e] ((rce[e] + rce[e+1]) / 2) = (rce[e+1]^2 - rce[e]^2)/2, the radial
 *                         factor of the dual area of an edge on r-face e
 *   dR2[i] = rc_i dr_i  : (r_f[i+1]^2 - r_f[i]^2)/2
 *   Cs[j], j = 1..nt-1  : 2 sin((tc_{j-1} + tc_j)/2) sin(ht_j / 2) = cos tc_{j-1} - cos tc_j
 *   capN = 2 (2 pi) sin^2(tc_0 / 2), capS = 2 (2 pi) cos^2(tc_{nt-1} / 2): the polar caps
 *                         (1 - cos tc_0) 2 pi and (1 + cos tc_{nt-1}) 2 pi
 *   hm[k] = hp[k-1 mod np]: centre distance across the lower phi-face of plane k. */
typedef struct {
    double *rc, *dr, *hr, *rce, *rhor, *dR2, *R3, *rf2, *rc2;
    double *tc, *dt, *ht, *C, *Cs, *sinc, *sinf_;
    double *pc, *dp, *hp, *hm;
    double capN, capS;
} mv_grid;

static void mv_grid_free(mv_grid *g) {
    free(g->rc); free(g->dr); free(g->hr); free(g->rce); free(g->rhor); free(g->dR2); free(g->R3);
    free(g->rf2); free(g->rc2);
    free(g->tc); free(g->dt); free(g->ht); free(g->C); free(g->Cs); free(g->sinc); free(g->sinf_);
    free(g->pc); free(g->dp); free(g->hp); free(g->hm);
}

/* Grid validity for the vector operator: the scalar rules (R1, R9) plus a full sphere in theta
 * (t_f[0] = 0 and t_f[nt] = pi, both poles, R29) and np >= 2 (R27). */
int masoracle_vv_check_grid(int nr, int nt, int np, const double *rf, const double *tf, const double *pf) {
    if (nr < 1 || nt < 1 || np < 2) return MV_E_INVALID;
    if (!(rf[0] > 0.0)) return MV_E_INVALID;
    for (int i = 0; i < nr; i++) if (!(rf[i + 1] > rf[i])) return MV_E_INVALID;
    for (int j = 0; j < nt; j++) if (!(tf[j + 1] > tf[j])) return MV_E_INVALID;
    for (int k = 0; k < np; k++) if (!(pf[k + 1] > pf[k])) return MV_E_INVALID;
    if (!(tf[0] == 0.0) || !(fabs(tf[nt] - MV_PI) <= 1e-12)) return MV_E_INVALID;
    if (!(fabs((pf[np] - pf[0]) - MV_TWO_PI) <= 1e-12 * MV_TWO_PI)) return MV_E_INVALID;
    return MV_OK;
}

static int mv_grid_build(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                         mv_grid *g) {
    memset(g, 0, sizeof(*g));
#define ALLOC(f, n) g->f = malloc(sizeof(double) * (size_t)(n))
    ALLOC(rc, nr); ALLOC(dr, nr); ALLOC(hr, nr + 1); ALLOC(rce, nr + 2); ALLOC(rhor, nr + 1);
    ALLOC(dR2, nr); ALLOC(R3, nr); ALLOC(rf2, nr + 1); ALLOC(rc2, nr);
    ALLOC(tc, nt); ALLOC(dt, nt); ALLOC(ht, nt + 1); ALLOC(C, nt); ALLOC(Cs, nt + 1); ALLOC(sinc, nt);
    ALLOC(sinf_, nt + 1);
    ALLOC(pc, np); ALLOC(dp, np); ALLOC(hp, np); ALLOC(hm, np);
#undef ALLOC
    if (!g->rc || !g->dr || !g->hr || !g->rce || !g->rhor || !g->dR2 || !g->R3 || !g->rf2 || !g->rc2 ||
        !g->tc || !g->dt || !g->ht || !g->C || !g->Cs || !g->sinc || !g->sinf_ || !g->pc || !g->dp ||
        !g->hp || !g->hm) {
        mv_grid_free(g);
        return MV_E_NOMEM;
    }
    for (int i = 0; i < nr; i++) {
        g->rc[i] = 0.5 * (rf[i] + rf[i + 1]);
        g->dr[i] = rf[i + 1] - rf[i];
        g->R3[i] = g->dr[i] * (rf[i + 1] * rf[i + 1] + rf[i + 1] * rf[i] + rf[i] * rf[i]) / 3.0;
        g->dR2[i] = g->rc[i] * g->dr[i];
        g->rc2[i] = g->rc[i] * g->rc[i];
    }
    for (int i = 0; i <= nr; i++) g->rf2[i] = rf[i] * rf[i];
    g->hr[0] = g->rc[0] - rf[0];
    for (int i = 1; i < nr; i++) g->hr[i] = g->rc[i] - g->rc[i - 1];
    g->hr[nr] = rf[nr] - g->rc[nr - 1];
    g->rce[0] = rf[0];
    for (int i = 0; i < nr; i++) g->rce[i + 1] = g->rc[i];
    g->rce[nr + 1] = rf[nr];
    for (int e = 0; e <= nr; e++) g->rhor[e] = g->hr[e] * (0.5 * (g->rce[e] + g->rce[e + 1]));

    for (int j = 0; j < nt; j++) {
        g->tc[j] = 0.5 * (tf[j] + tf[j + 1]);
        g->dt[j] = tf[j + 1] - tf[j];
        g->C[j] = 2.0 * sin(g->tc[j]) * sin(0.5 * g->dt[j]);
        g->sinc[j] = sin(g->tc[j]);
    }
    g->ht[0] = 0.0; g->ht[nt] = 0.0;
    g->Cs[0] = 0.0; g->Cs[nt] = 0.0;
    for (int j = 1; j < nt; j++) {
        g->ht[j] = g->tc[j] - g->tc[j - 1];
        g->Cs[j] = 2.0 * sin(0.5 * (g->tc[j - 1] + g->tc[j])) * sin(0.5 * g->ht[j]);
    }
    for (int j = 0; j <= nt; j++) g->sinf_[j] = sin(tf[j]);
    double sN = sin(0.5 * g->tc[0]), cS = cos(0.5 * g->tc[nt - 1]);
    g->capN = (2.0 * MV_TWO_PI) * (sN * sN);
    g->capS = (2.0 * MV_TWO_PI) * (cS * cS);

    for (int k = 0; k < np; k++) {
        g->pc[k] = 0.5 * (pf[k] + pf[k + 1]);
        g->dp[k] = pf[k + 1] - pf[k];
    }
    for (int k = 0; k + 1 < np; k++) g->hp[k] = g->pc[k + 1] - g->pc[k];
    g->hp[np - 1] = (g->pc[0] + MV_TWO_PI) - g->pc[np - 1];
    for (int k = 0; k < np; k++) g->hm[k] = g->hp[(k + np - 1) % np];
    return MV_OK;
}

/* Face geometry (R27), lower faces of cell (i, j, k): area A and centre distance l.
 *   r-face i   : A = (r_f[i]^2 C_j) dphi_k,       l = hr[i]
 *   theta-face j: A = (sin t_f[j] dR2_i) dphi_k,   l = rc_i ht_j
 *   phi-face k : A = dR2_i dtheta_j,              l = (rc_i sin tc_j) hm_k
 * Distances to a wall use the wall radius in place of rc (rce[0], rce[nr+1]). */
static double A_r(const mv_grid *g, int i, int j, int k) { return (g->rf2[i] * g->C[j]) * g->dp[k]; }
static double A_t(const mv_grid *g, int i, int j, int k) { return (g->sinf_[j] * g->dR2[i]) * g->dp[k]; }
static double A_p(const mv_grid *g, int i, int j) { return g->dR2[i] * g->dt[j]; }
/* l_t and l_p at extended radial index e (e = i + 1 for cell i, 0 / nr + 1 for the walls) */
static double L_t(const mv_grid *g, int e, int j) { return g->rce[e] * g->ht[j]; }
static double L_p(const mv_grid *g, int e, int j, int k) { return (g->rce[e] * g->sinc[j]) * g->hm[k]; }

/* ------------------------------------------------------- coefficients (R28, R30) */
/* Coefficients of the vector operator from the cell viscosity nu [np][nt][nr] (>= 0) and the
 * cell shift s [np][nt][nr] (>= 0), for walls bc_in / bc_out (0 no-slip, 1 free-slip):
 *   wc [np][nt][nr]          nu_c / V_c                                  (div energy weight)
 *   Wr [np][nt][nr]          r-edge at theta-face j (1..nt-1), phi-face k: nu_e dr_i / ((rc_i^2 Cs_j) hm_k)
 *   Wt [np][nt][nr+1]        theta-edge at r-face e (0..nr), phi-face k:   nu_e (r_f[e] dt_j) / ((sin tc_j rhor_e) hm_k)
 *   Wp [np][nt][nr+1]        phi-edge at r-face e, theta-face j (1..nt-1): nu_e ((r_f[e] sin t_f[j]) dphi_k) / (rhor_e ht_j)
 *   WN [nr], WS [nr]         polar axis edges: nu_ring dr_i / (rc_i^2 cap)
 *   sM [np][3][nt][nr]       s_f M_f, s_f the mean of the two cells of the face, M_f = A_f l_f
 * nu_e is the arithmetic mean of the cells around the edge: four, two for a wall edge (both of its
 * planes / rows), the whole pole ring for the axis (Dot2 sum / np).  Wall edges carry W = 0 on a
 * free-slip wall.  Unused slots are 0.  Returns E_INVALID for negative / non-finite input. */
int masoracle_vv_coefficients(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                              const double *nu, const double *s, int bc_in, int bc_out, double *wc, double *Wr,
                              double *Wt, double *Wp, double *WN, double *WS, double *sM) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    if ((bc_in != MV_NO_SLIP && bc_in != MV_FREE_SLIP) || (bc_out != MV_NO_SLIP && bc_out != MV_FREE_SLIP))
        return MV_E_INVALID;
    size_t ncell = (size_t)nr * nt * np;
    for (size_t c = 0; c < ncell; c++) {
        if (!(nu[c] >= 0.0) || !isfinite(nu[c])) return MV_E_INVALID;
        if (!(s[c] >= 0.0) || !isfinite(s[c])) return MV_E_INVALID;
    }
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
    const size_t ne = (size_t)(nr + 1) * nt * np;
    memset(Wr, 0, sizeof(double) * ncell);
    memset(Wt, 0, sizeof(double) * ne);
    memset(Wp, 0, sizeof(double) * ne);
    memset(sM, 0, sizeof(double) * 3 * ncell);
#define EI(k, j, e) ((((size_t)(k)) * (size_t)nt + (size_t)(j)) * (size_t)(nr + 1) + (size_t)(e))
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                double V = (g.R3[i] * g.C[j]) * g.dp[k];
                wc[CI(k, j, i)] = nu[CI(k, j, i)] / V;
                if (j >= 1) {
                    double nue = ((nu[CI(km, j - 1, i)] + nu[CI(km, j, i)]) + (nu[CI(k, j - 1, i)] + nu[CI(k, j, i)])) * 0.25;
                    Wr[CI(k, j, i)] = (nue * g.dr[i]) / ((g.rc2[i] * g.Cs[j]) * g.hm[k]);
                }
            }
        for (int j = 0; j < nt; j++)
            for (int e = 0; e <= nr; e++) {
                int wall = (e == 0) ? bc_in : (e == nr ? bc_out : -1);
                if (wall == MV_FREE_SLIP) continue;
                double nue;
                if (e == 0) nue = (nu[CI(km, j, 0)] + nu[CI(k, j, 0)]) * 0.5;
                else if (e == nr) nue = (nu[CI(km, j, nr - 1)] + nu[CI(k, j, nr - 1)]) * 0.5;
                else nue = ((nu[CI(km, j, e - 1)] + nu[CI(km, j, e)]) + (nu[CI(k, j, e - 1)] + nu[CI(k, j, e)])) * 0.25;
                Wt[EI(k, j, e)] = (nue * (rf[e] * g.dt[j])) / ((g.sinc[j] * g.rhor[e]) * g.hm[k]);
            }
        for (int j = 1; j < nt; j++)
            for (int e = 0; e <= nr; e++) {
                int wall = (e == 0) ? bc_in : (e == nr ? bc_out : -1);
                if (wall == MV_FREE_SLIP) continue;
                double nue;
                if (e == 0) nue = (nu[CI(k, j - 1, 0)] + nu[CI(k, j, 0)]) * 0.5;
                else if (e == nr) nue = (nu[CI(k, j - 1, nr - 1)] + nu[CI(k, j, nr - 1)]) * 0.5;
                else nue = ((nu[CI(k, j - 1, e - 1)] + nu[CI(k, j - 1, e)]) + (nu[CI(k, j, e - 1)] + nu[CI(k, j, e)])) * 0.25;
                Wp[EI(k, j, e)] = (nue * ((rf[e] * g.sinf_[j]) * g.dp[k])) / (g.rhor[e] * g.ht[j]);
            }
        /* s_f M_f of the three lower faces */
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                if (i >= 1) {
                    double sf = (s[CI(k, j, i - 1)] + s[CI(k, j, i)]) * 0.5;
                    sM[VI(k, 0, j, i)] = sf * (A_r(&g, i, j, k) * g.hr[i]);
                }
                if (j >= 1) {
                    double sf = (s[CI(k, j - 1, i)] + s[CI(k, j, i)]) * 0.5;
                    sM[VI(k, 1, j, i)] = sf * (A_t(&g, i, j, k) * L_t(&g, i + 1, j));
                }
                double sf = (s[CI(km, j, i)] + s[CI(k, j, i)]) * 0.5;
                sM[VI(k, 2, j, i)] = sf * (A_p(&g, i, j) * L_p(&g, i + 1, j, k));
            }
    }
    /* polar axes: nu averaged over the pole rings (R29) */
    double *ones = malloc(sizeof(double) * (size_t)np);
    if (!ones) { mv_grid_free(&g); return MV_E_NOMEM; }
    for (int k = 0; k < np; k++) ones[k] = 1.0;
    const size_t kstride = (size_t)nt * nr;
    for (int i = 0; i < nr; i++) {
        double nN = mv_dot((size_t)np, nu + CI(0, 0, i), kstride, ones, 1) / (double)np;
        double nS = mv_dot((size_t)np, nu + CI(0, nt - 1, i), kstride, ones, 1) / (double)np;
        WN[i] = (nN * g.dr[i]) / (g.rc2[i] * g.capN);
        WS[i] = (nS * g.dr[i]) / (g.rc2[i] * g.capS);
    }
    free(ones);
#undef EI
    mv_grid_free(&g);
    return MV_OK;
}

/* ------------------------------------------------ discrete div and curl (R27, R29) */
/* v at slot (k, c, j, i) with the wall data substituted: v_r at i = 0 / nr and v_t at the pole
 * faces are not unknowns. */
static double vr_at(int nr, int nt, int np, const double *v, const double *gin, const double *gout, int k, int j,
                    int e) {
    if (e == 0) return gin ? gin[GI(0, k, j)] : 0.0;
    if (e == nr) return gout ? gout[GI(0, k, j)] : 0.0;
    return v[VI(k, 0, j, e)];
}

/* delta [np][nt][nr]: net outflow of every cell, sum over its faces of +-A_f v_f:
 *   delta = (fr_hi - fr_lo) + (ft_hi - ft_lo), then + (fp_hi - fp_lo)
 * with the wall normal velocities on the r-walls and zero flux through the pole faces. */
int masoracle_vv_div(int nr, int nt, int np, const double *rf, const double *tf, const double *pf, const double *v,
                     const double *gin, const double *gout, double *delta) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
    for (int k = 0; k < np; k++) {
        int kp1 = (k + 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                double fr_lo = A_r(&g, i, j, k) * vr_at(nr, nt, np, v, gin, gout, k, j, i);
                double fr_hi = A_r(&g, i + 1, j, k) * vr_at(nr, nt, np, v, gin, gout, k, j, i + 1);
                double ft_lo = (j == 0) ? 0.0 : A_t(&g, i, j, k) * v[VI(k, 1, j, i)];
                double ft_hi = (j == nt - 1) ? 0.0 : A_t(&g, i, j + 1, k) * v[VI(k, 1, j + 1, i)];
                double fp_lo = A_p(&g, i, j) * v[VI(k, 2, j, i)];
                double fp_hi = A_p(&g, i, j) * v[VI(kp1, 2, j, i)];
                double d = (fr_hi - fr_lo) + (ft_hi - ft_lo);
                d = d + (fp_hi - fp_lo);
                delta[CI(k, j, i)] = d;
            }
    }
    mv_grid_free(&g);
    return MV_OK;
}

/* Circulations (Stokes: the line integral of v around the dual loop of each edge, each dual
 * segment crossing one face f, its tangential velocity v_f over the length l_f):
 *   Gr [np][nt][nr]   r-edge (i; theta-face j = 1..nt-1; phi-face k):
 *                     (Gp(i,j,k) - Gp(i,j-1,k)) - (Gt(i,j,k) - Gt(i,j,k-1))
 *   GN [nr], GS [nr]  polar axes: GN(i) = sum_k l_p v_p(i,0,k), GS(i) = -sum_k l_p v_p(i,nt-1,k) (Dot2)
 *   Gt [np][nt][nr+1] theta-edge (r-face e = 0..nr; phi-face k):
 *                     (hr_e v_r(e,j,k) - hr_e v_r(e,j,k-1)) - (Gp_above - Gp_below)
 *   Gp [np][nt][nr+1] phi-edge (r-face e; theta-face j = 1..nt-1):
 *                     (Gt_above - Gt_below) - (hr_e v_r(e,j,k) - hr_e v_r(e,j-1,k))
 * with Gp(i,j,k) = l_p v_p, Gt(i,j,k) = l_t v_t; on a wall the cell beyond is replaced by the
 * wall: its distance uses the wall radius and its velocity the tangential wall datum. */
int masoracle_vv_curl(int nr, int nt, int np, const double *rf, const double *tf, const double *pf, const double *v,
                      const double *gin, const double *gout, double *Gr, double *GN, double *GS, double *Gt,
                      double *Gp) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
#define EI(k, j, e) ((((size_t)(k)) * (size_t)nt + (size_t)(j)) * (size_t)(nr + 1) + (size_t)(e))
    memset(Gr, 0, sizeof(double) * (size_t)nr * nt * np);
    memset(Gp, 0, sizeof(double) * (size_t)(nr + 1) * nt * np);
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np;
        for (int j = 1; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                double gp_a = L_p(&g, i + 1, j, k) * v[VI(k, 2, j, i)];
                double gp_b = L_p(&g, i + 1, j - 1, k) * v[VI(k, 2, j - 1, i)];
                double gt_a = L_t(&g, i + 1, j) * v[VI(k, 1, j, i)];
                double gt_b = L_t(&g, i + 1, j) * v[VI(km, 1, j, i)];
                Gr[CI(k, j, i)] = (gp_a - gp_b) - (gt_a - gt_b);
            }
        for (int j = 0; j < nt; j++)
            for (int e = 0; e <= nr; e++) {
                double gr_a = g.hr[e] * vr_at(nr, nt, np, v, gin, gout, k, j, e);
                double gr_b = g.hr[e] * vr_at(nr, nt, np, v, gin, gout, km, j, e);
                double up = (e < nr) ? v[VI(k, 2, j, e)] : (gout ? gout[GI(2, k, j)] : 0.0);
                double dn = (e > 0) ? v[VI(k, 2, j, e - 1)] : (gin ? gin[GI(2, k, j)] : 0.0);
                double gp_a = L_p(&g, e + 1, j, k) * up;
                double gp_b = L_p(&g, e, j, k) * dn;
                Gt[EI(k, j, e)] = (gr_a - gr_b) - (gp_a - gp_b);
            }
        for (int j = 1; j < nt; j++)
            for (int e = 0; e <= nr; e++) {
                double up = (e < nr) ? v[VI(k, 1, j, e)] : (gout ? gout[GI(1, k, j)] : 0.0);
                double dn = (e > 0) ? v[VI(k, 1, j, e - 1)] : (gin ? gin[GI(1, k, j)] : 0.0);
                double gt_a = L_t(&g, e + 1, j) * up;
                double gt_b = L_t(&g, e, j) * dn;
                double gr_a = g.hr[e] * vr_at(nr, nt, np, v, gin, gout, k, j, e);
                double gr_b = g.hr[e] * vr_at(nr, nt, np, v, gin, gout, k, j - 1, e);
                Gp[EI(k, j, e)] = (gt_a - gt_b) - (gr_a - gr_b);
            }
    }
    /* the pole rings: Listing 3's per-radius array reduction sum0(i) */
    double *lring = malloc(sizeof(double) * (size_t)np);
    if (!lring) { mv_grid_free(&g); return MV_E_NOMEM; }
    const size_t kstride = (size_t)3 * nt * nr;
    for (int i = 0; i < nr; i++) {
        for (int k = 0; k < np; k++) lring[k] = L_p(&g, i + 1, 0, k);
        GN[i] = mv_dot((size_t)np, v + VI(0, 2, 0, i), kstride, lring, 1);
        for (int k = 0; k < np; k++) lring[k] = L_p(&g, i + 1, nt - 1, k);
        GS[i] = -mv_dot((size_t)np, v + VI(0, 2, nt - 1, i), kstride, lring, 1);
    }
    free(lring);
#undef EI
    mv_grid_free(&g);
    return MV_OK;
}

/* ------------------------------------------------------------ apply (R27-R30) */
/* y = sM v + G^T diag(wc) delta + C^T diag(W) Gamma, row by row (the gradient of the energy):
 *   r-face (i >= 1): y = sM v + A_r (e(i-1) - e(i)) + hr_i c,
 *       c = ((Wt Gt(i,k) - Wt Gt(i,k+1)) - Wp Gp(i,j)) + Wp Gp(i,j+1)
 *   theta-face (j >= 1): y = sM v + A_t (e(j-1) - e(j)) + l_t c,
 *       c = ((Wr Gr(j,k+1) - Wr Gr(j,k)) + Wp Gp(i,j)) - Wp Gp(i+1,j)
 *   phi-face: y = sM v + A_p (e(k-1) - e(k)) + l_p c,
 *       c = ((Wr Gr(j,k) - Wr Gr(j+1,k)) - Wt Gt(i,k)) + Wt Gt(i+1,k)
 * with e = wc delta, the pole edge terms of the phi-face row replaced by the axis (WN GN at j = 0,
 * WS GS at j = nt), the phi-edges at the poles (zero length) absent, and each term evaluated
 * "y = y + term" left to right.  v's non-unknown slots give y = 0.  gin / gout: wall data, NULL = 0
 * (the homogeneous operator); the rhs uses y with v = 0 (masoracle_vv_rhs). */
int masoracle_vv_apply(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                       const double *wc, const double *Wr, const double *Wt, const double *Wp, const double *WN,
                       const double *WS, const double *sM, const double *v, const double *gin, const double *gout,
                       double *y) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
    size_t ncell = (size_t)nr * nt * np, ne = (size_t)(nr + 1) * nt * np;
    double *delta = malloc(sizeof(double) * ncell), *e = malloc(sizeof(double) * ncell);
    double *Gr = malloc(sizeof(double) * ncell), *Gt = malloc(sizeof(double) * ne);
    double *Gp = malloc(sizeof(double) * ne), *GN = malloc(sizeof(double) * nr), *GS = malloc(sizeof(double) * nr);
    if (!delta || !e || !Gr || !Gt || !Gp || !GN || !GS) {
        free(delta); free(e); free(Gr); free(Gt); free(Gp); free(GN); free(GS);
        mv_grid_free(&g);
        return MV_E_NOMEM;
    }
    masoracle_vv_div(nr, nt, np, rf, tf, pf, v, gin, gout, delta);
    masoracle_vv_curl(nr, nt, np, rf, tf, pf, v, gin, gout, Gr, GN, GS, Gt, Gp);
    for (size_t c = 0; c < ncell; c++) e[c] = wc[c] * delta[c];
#define EI(k, j, e_) ((((size_t)(k)) * (size_t)nt + (size_t)(j)) * (size_t)(nr + 1) + (size_t)(e_))
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np, kp1 = (k + 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                /* r-face i */
                double yr = 0.0;
                if (i >= 1) {
                    yr = sM[VI(k, 0, j, i)] * v[VI(k, 0, j, i)];
                    yr = yr + A_r(&g, i, j, k) * (e[CI(k, j, i - 1)] - e[CI(k, j, i)]);
                    double c = Wt[EI(k, j, i)] * Gt[EI(k, j, i)];
                    c = c - Wt[EI(kp1, j, i)] * Gt[EI(kp1, j, i)];
                    if (j >= 1) c = c - Wp[EI(k, j, i)] * Gp[EI(k, j, i)];
                    if (j + 1 <= nt - 1) c = c + Wp[EI(k, j + 1, i)] * Gp[EI(k, j + 1, i)];
                    yr = yr + g.hr[i] * c;
                }
                y[VI(k, 0, j, i)] = yr;
                /* theta-face j */
                double yt = 0.0;
                if (j >= 1) {
                    yt = sM[VI(k, 1, j, i)] * v[VI(k, 1, j, i)];
                    yt = yt + A_t(&g, i, j, k) * (e[CI(k, j - 1, i)] - e[CI(k, j, i)]);
                    double c = Wr[CI(kp1, j, i)] * Gr[CI(kp1, j, i)] - Wr[CI(k, j, i)] * Gr[CI(k, j, i)];
                    c = c + Wp[EI(k, j, i)] * Gp[EI(k, j, i)];
                    c = c - Wp[EI(k, j, i + 1)] * Gp[EI(k, j, i + 1)];
                    yt = yt + L_t(&g, i + 1, j) * c;
                }
                y[VI(k, 1, j, i)] = yt;
                /* phi-face k */
                double yp = sM[VI(k, 2, j, i)] * v[VI(k, 2, j, i)];
                yp = yp + A_p(&g, i, j) * (e[CI(km, j, i)] - e[CI(k, j, i)]);
                double lo = (j == 0) ? WN[i] * GN[i] : Wr[CI(k, j, i)] * Gr[CI(k, j, i)];
                double hi = (j == nt - 1) ? WS[i] * GS[i] : Wr[CI(k, j + 1, i)] * Gr[CI(k, j + 1, i)];
                double c = lo - hi;
                c = c - Wt[EI(k, j, i)] * Gt[EI(k, j, i)];
                c = c + Wt[EI(k, j, i + 1)] * Gt[EI(k, j, i + 1)];
                yp = yp + L_p(&g, i + 1, j, k) * c;
                y[VI(k, 2, j, i)] = yp;
            }
    }
#undef EI
    free(delta); free(e); free(Gr); free(Gt); free(Gp); free(GN); free(GS);
    mv_grid_free(&g);
    return MV_OK;
}

/* Jacobi diagonal D = diag(A) (R30), same term order as the rows:
 *   r-face: (sM + (A A)(wc(i-1) + wc(i))) + (hr hr) w, w = ((Wt(i,k) + Wt(i,k+1)) + Wp(i,j)) + Wp(i,j+1)
 *   theta-face: (sM + (A A)(wc(j-1) + wc(j))) + (l l) w, w = ((Wr(j,k) + Wr(j,k+1)) + Wp(i,j)) + Wp(i+1,j)
 *   phi-face: (sM + (A A)(wc(k-1) + wc(k))) + (l l) w, w = ((Wr_lo + Wr_hi) + Wt(i,k)) + Wt(i+1,k)
 * (absent pole phi-edges contribute 0, the axis W at the pole rows); 1 on non-unknown slots.
 * Exact diag(A) for np >= 2: each face enters each circulation and each outflow once. */
int masoracle_vv_diag(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                      const double *wc, const double *Wr, const double *Wt, const double *Wp, const double *WN,
                      const double *WS, const double *sM, double *D) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
#define EI(k, j, e_) ((((size_t)(k)) * (size_t)nt + (size_t)(j)) * (size_t)(nr + 1) + (size_t)(e_))
    for (int k = 0; k < np; k++) {
        int km = (k + np - 1) % np, kp1 = (k + 1) % np;
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                double d = 1.0;
                if (i >= 1) {
                    double A = A_r(&g, i, j, k), l = g.hr[i];
                    double w = Wt[EI(k, j, i)] + Wt[EI(kp1, j, i)];
                    if (j >= 1) w = w + Wp[EI(k, j, i)];
                    if (j + 1 <= nt - 1) w = w + Wp[EI(k, j + 1, i)];
                    d = sM[VI(k, 0, j, i)] + (A * A) * (wc[CI(k, j, i - 1)] + wc[CI(k, j, i)]);
                    d = d + (l * l) * w;
                }
                D[VI(k, 0, j, i)] = d;
                d = 1.0;
                if (j >= 1) {
                    double A = A_t(&g, i, j, k), l = L_t(&g, i + 1, j);
                    double w = Wr[CI(k, j, i)] + Wr[CI(kp1, j, i)];
                    w = w + Wp[EI(k, j, i)];
                    w = w + Wp[EI(k, j, i + 1)];
                    d = sM[VI(k, 1, j, i)] + (A * A) * (wc[CI(k, j - 1, i)] + wc[CI(k, j, i)]);
                    d = d + (l * l) * w;
                }
                D[VI(k, 1, j, i)] = d;
                {
                    double A = A_p(&g, i, j), l = L_p(&g, i + 1, j, k);
                    double lo = (j == 0) ? WN[i] : Wr[CI(k, j, i)];
                    double hi = (j == nt - 1) ? WS[i] : Wr[CI(k, j + 1, i)];
                    double w = lo + hi;
                    w = w + Wt[EI(k, j, i)];
                    w = w + Wt[EI(k, j, i + 1)];
                    d = sM[VI(k, 2, j, i)] + (A * A) * (wc[CI(km, j, i)] + wc[CI(k, j, i)]);
                    d = d + (l * l) * w;
                }
                D[VI(k, 2, j, i)] = d;
            }
    }
#undef EI
    mv_grid_free(&g);
    return MV_OK;
}

/* Face masses M_f = A_f l_f [np][3][nt][nr] (0 on non-unknown slots). */
int masoracle_vv_mass(int nr, int nt, int np, const double *rf, const double *tf, const double *pf, double *M) {
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    mv_grid g;
    if (mv_grid_build(nr, nt, np, rf, tf, pf, &g)) return MV_E_NOMEM;
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                M[VI(k, 0, j, i)] = (i >= 1) ? A_r(&g, i, j, k) * g.hr[i] : 0.0;
                M[VI(k, 1, j, i)] = (j >= 1) ? A_t(&g, i, j, k) * L_t(&g, i + 1, j) : 0.0;
                M[VI(k, 2, j, i)] = A_p(&g, i, j) * L_p(&g, i + 1, j, k);
            }
    mv_grid_free(&g);
    return MV_OK;
}

/* ------------------------------------------------------------------ rhs (R31) */
/* b = M f - A(0; g): the per-unit-volume forcing f [np][3][nt][nr] times the face masses, minus the
 * operator applied to the wall data alone.  0 on non-unknown slots.  `y` is scratch (3 ncell). */
int masoracle_vv_rhs(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                     const double *wc, const double *Wr, const double *Wt, const double *Wp, const double *WN,
                     const double *WS, const double *sM, const double *f, const double *gin, const double *gout,
                     double *b) {
    size_t n3 = (size_t)3 * nr * nt * np;
    double *zero = calloc(n3, sizeof(double)), *y = malloc(sizeof(double) * n3), *M = malloc(sizeof(double) * n3);
    if (!zero || !y || !M) { free(zero); free(y); free(M); return MV_E_NOMEM; }
    int st = masoracle_vv_apply(nr, nt, np, rf, tf, pf, wc, Wr, Wt, Wp, WN, WS, sM, zero, gin, gout, y);
    if (!st) st = masoracle_vv_mass(nr, nt, np, rf, tf, pf, M);
    if (!st)
        for (int k = 0; k < np; k++)
            for (int c = 0; c < 3; c++)
                for (int j = 0; j < nt; j++)
                    for (int i = 0; i < nr; i++) {
                        size_t q = VI(k, c, j, i);
                        int unknown = !((c == 0 && i == 0) || (c == 1 && j == 0));
                        b[q] = unknown ? (M[q] * f[q]) - y[q] : 0.0;
                    }
    free(zero); free(y); free(M);
    return st;
}

/* ------------------------------------------------------------------- PCG (R11-R14) */
/* Jacobi PCG on the stacked face vector, exactly the algorithm of masoracle_pcg (SURVEY 8(c)
 * item 7): r0 = b - A x0, z = r/D, p = z, Fletcher-Reeves beta, stop on ||r|| <= tol ||b||,
 * Dot2 dot products.  x's non-unknown slots are set to 0 first.  hist: maxit + 1 doubles or NULL. */
int masoracle_vv_pcg(int nr, int nt, int np, const double *rf, const double *tf, const double *pf,
                     const double *wc, const double *Wr, const double *Wt, const double *Wp, const double *WN,
                     const double *WS, const double *sM, const double *D, const double *b, double *x, double tol,
                     int maxit, double *hist, int *iters, double *bnorm, double *rnorm) {
    size_t n = (size_t)3 * nr * nt * np;
    if (maxit < 0 || !(tol >= 0.0)) return MV_E_INVALID;
    int st = masoracle_vv_check_grid(nr, nt, np, rf, tf, pf);
    if (st) return st;
    *iters = 0;
    for (int k = 0; k < np; k++)
        for (int j = 0; j < nt; j++)
            for (int i = 0; i < nr; i++) {
                if (i == 0) x[VI(k, 0, j, i)] = 0.0;
                if (j == 0) x[VI(k, 1, j, i)] = 0.0;
            }
    double bn = sqrt(mv_dot(n, b, 1, b, 1));
    *bnorm = bn;
    if (!isfinite(bn)) { *rnorm = bn; return MV_E_BREAKDOWN; }
    if (bn == 0.0) {
        for (size_t c = 0; c < n; c++) x[c] = 0.0;
        if (hist) hist[0] = 0.0;
        *rnorm = 0.0;
        return MV_OK;
    }
    double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
    double *p = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * n);
    if (!r || !z || !p || !q) { free(r); free(z); free(p); free(q); return MV_E_NOMEM; }
    int status = MV_NOT_CONVERGED;
    masoracle_vv_apply(nr, nt, np, rf, tf, pf, wc, Wr, Wt, Wp, WN, WS, sM, x, NULL, NULL, q);
    for (size_t c = 0; c < n; c++) r[c] = b[c] - q[c];
    for (size_t c = 0; c < n; c++) z[c] = r[c] / D[c];
    for (size_t c = 0; c < n; c++) p[c] = z[c];
    double rho = mv_dot(n, r, 1, z, 1);
    double rn = sqrt(mv_dot(n, r, 1, r, 1));
    if (hist) hist[0] = rn;
    *rnorm = rn;
    if (!isfinite(rn) || !isfinite(rho)) { status = MV_E_BREAKDOWN; goto done; }
    if (rn <= tol * bn) { status = MV_OK; goto done; }
    for (int k = 1; k <= maxit; k++) {
        masoracle_vv_apply(nr, nt, np, rf, tf, pf, wc, Wr, Wt, Wp, WN, WS, sM, p, NULL, NULL, q);
        double pi = mv_dot(n, p, 1, q, 1);
        if (!(pi > 0.0) || !isfinite(pi)) { status = MV_E_BREAKDOWN; break; }
        double alpha = rho / pi;
        for (size_t c = 0; c < n; c++) x[c] = x[c] + alpha * p[c];
        for (size_t c = 0; c < n; c++) r[c] = r[c] - alpha * q[c];
        rn = sqrt(mv_dot(n, r, 1, r, 1));
        if (hist) hist[k] = rn;
        *iters = k;
        *rnorm = rn;
        if (!isfinite(rn)) { status = MV_E_BREAKDOWN; break; }
        if (rn <= tol * bn) { status = MV_OK; break; }
        for (size_t c = 0; c < n; c++) z[c] = r[c] / D[c];
        double rho_new = mv_dot(n, r, 1, z, 1);
        double beta = rho_new / rho;
        rho = rho_new;
        for (size_t c = 0; c < n; c++) p[c] = z[c] + beta * p[c];
    }
done:
    free(r); free(z); free(p); free(q);
    return status;
}
