"""Pins of the vector-viscosity oracle (oracle/masoracle_vv.c) against things
other than itself (-m "not gpu").

The operator is the reading R27-R31 of DESIGN.md: the mimetic (div-curl) form of the vector
diffusion operator s v + curl(nu curl v) - grad(nu div v) on MAS's staggered spherical grid
(Sec. III), v_r / v_theta / v_phi on their faces, the polar axis handled as one
r-edge per radius whose circulation is the per-radius sum over the pole ring -- the array
reduction sum0(i) of PAPER.md:147-157 (Listing 3).  The pins: exactness of the discrete complex
(curl grad = 0 with the axis and the walls, div curl = 0), closed-form outflows and circulations
(Gauss and Stokes on fields the exact integrals reproduce), symmetry, diag(A), positive
definiteness and a dense solve on tiny grids, the nu = 0 special case, and second-order
convergence to a manufactured solution v = grad phi + r x grad chi of s v - nu lap v = f with
no-slip walls.  The test side computes its own geometry from the exact integrals.
"""
import math

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

PI = math.pi


def grid(nr, nt, np_, a=1.5, eps=0.2, phi_warp=0.15, r0=1.0, r1=2.0):
    rf = inputs.rfaces(nr, r0, r1, a)
    tf = inputs.tfaces(nt, eps)
    z = np.arange(np_ + 1) / np_
    pf = 2 * PI * (z + phi_warp * np.sin(2 * PI * z) / (2 * PI))
    pf[0], pf[-1] = 0.0, 2 * PI
    return rf, tf, pf


def geometry(rf, tf, pf):
    """Test-side face areas and centre distances (exact integrals, cosine differences)."""
    rc, tc, pc = inputs.midpoints(rf), inputs.midpoints(tf), inputs.midpoints(pf)
    nr, nt, np_ = rc.size, tc.size, pc.size
    dphi, dth = np.diff(pf), np.diff(tf)
    hphi_lo = pc - np.roll(pc, 1)
    hphi_lo[0] += 2 * PI                               # across the lower phi-face of plane k
    rce = np.concatenate([[rf[0]], rc, [rf[-1]]])      # centres extended by the walls
    g = dict(rc=rc, tc=tc, pc=pc, rce=rce, hphi_lo=hphi_lo)
    dcos = np.cos(tf[:-1]) - np.cos(tf[1:])
    g["A_r"] = rf[:, None, None] ** 2 * dcos[None, :, None] * dphi[None, None, :]         # [nr+1][nt][np]
    g["A_t"] = np.sin(tf)[:, None, None] * ((rf[1:] ** 2 - rf[:-1] ** 2) / 2)[None, :, None] * dphi  # [nt+1][nr][np]
    g["A_p"] = ((rf[1:] ** 2 - rf[:-1] ** 2) / 2)[None, :] * dth[:, None]               # [nt][nr]
    g["l_r"] = np.diff(rce)                                                             # [nr+1]
    g["V"] = ((rf[1:] ** 3 - rf[:-1] ** 3) / 3)[None, None, :] * dcos[None, :, None] * dphi[:, None, None]
    return g


def rand_fields(np_, nt, nr, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.5, 2.0, (np_, nt, nr)), rng.uniform(0.5, 1.5, (np_, nt, nr))


def dense(op):
    n = int(np.prod(op.shape))
    mask = op.unknown_mask().ravel()
    idx = np.flatnonzero(mask)
    A = np.empty((idx.size, idx.size))
    for col, c in enumerate(idx):
        e = np.zeros(n)
        e[c] = 1.0
        A[:, col] = op.apply(e.reshape(op.shape)).ravel()[idx]
    return A, idx


# ------------------------------------------------------------------ grid rules
def test_vv_grid_rules(oracle_mod):
    rf, tf, pf = grid(4, 6, 8)
    assert oracle_mod.vv_check_grid(rf, tf, pf) == 0
    assert oracle_mod.vv_check_grid(rf, inputs.tfaces(6, 0.0, 0.3, 2.5), pf) == oracle_mod.E_INVALID  # no poles
    assert oracle_mod.vv_check_grid(rf, tf, inputs.pfaces(1)) == oracle_mod.E_INVALID                # np = 1
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.VVOperator(rf, tf, pf, -np.ones((8, 6, 4)), np.ones((8, 6, 4)))


# ------------------------------------------------------------------ exactness of the complex
@pytest.mark.parametrize("shape,seed", [((5, 6, 8), 1), ((3, 4, 2), 2), ((1, 3, 5), 3)])
def test_vv_curl_of_gradient_vanishes(oracle_mod, shape, seed):
    """v = grad(phi) of a random cell potential (wall values of phi on the walls): every
    circulation -- interior edges, wall edges and both polar axes (the pole-ring sums) -- is 0."""
    nr, nt, np_ = shape
    rf, tf, pf = grid(nr, nt, np_)
    g = geometry(rf, tf, pf)
    rng = np.random.default_rng(seed)
    phi = rng.standard_normal((np_, nt, nr))
    w_in, w_out = rng.standard_normal((np_, nt)), rng.standard_normal((np_, nt))
    rc, tc, rce = g["rc"], g["tc"], g["rce"]
    v = np.zeros((np_, 3, nt, nr))
    v[:, 0, :, 1:] = np.diff(phi, axis=2) / np.diff(rc)[None, None, :]
    v[:, 1, 1:, :] = np.diff(phi, axis=1) / (rc[None, None, :] * np.diff(tc)[None, :, None])
    v[:, 2] = (phi - np.roll(phi, 1, axis=0)) / (rc[None, None, :] * np.sin(tc)[None, :, None]
                                                 * g["hphi_lo"][:, None, None])
    def wall(w, r, cell_phi, sign):
        gw = np.zeros((3, np_, nt))
        gw[0] = sign * (cell_phi - w) / abs(r - (rc[0] if sign > 0 else rc[-1]))
        gw[1][:, 1:] = np.diff(w, axis=1) / (r * np.diff(tc))[None, :]
        gw[2] = (w - np.roll(w, 1, axis=0)) / (r * np.sin(tc)[None, :] * g["hphi_lo"][:, None])
        return gw
    gin = wall(w_in, rf[0], phi[:, :, 0], +1)
    gout = wall(w_out, rf[-1], phi[:, :, -1], -1)
    Gr, GN, GS, Gt, Gp = oracle_mod.vv_curl(rf, tf, pf, v, gin, gout)
    scale = np.abs(v).max() * rf[-1] * 2 * PI
    assert np.abs(Gr).max() <= 1e-13 * scale
    assert np.abs(Gt).max() <= 1e-13 * scale
    assert np.abs(Gp).max() <= 1e-13 * scale
    assert np.abs(GN).max() <= 1e-13 * scale and np.abs(GS).max() <= 1e-13 * scale
    # and the gradient has an outflow: the pin is not vacuous
    assert np.abs(oracle_mod.vv_div(rf, tf, pf, v, gin, gout)).max() > 1e-3


@pytest.mark.parametrize("shape", [(3, 4, 4), (2, 3, 5)])
def test_vv_div_of_curl_vanishes(oracle_mod, shape):
    """div(curl psi) = 0: the face-edge incidence of the circulations (read off the oracle's curl
    on unit vectors), transposed, maps any potential on interior edges and axes to face fluxes
    whose net outflow from every cell is 0 -- the circulation and outflow stencils belong to one
    consistent complex (a wrong index or sign in either breaks it)."""
    nr, nt, np_ = shape
    rf, tf, pf = grid(nr, nt, np_)
    g = geometry(rf, tf, pf)
    n = np_ * 3 * nt * nr
    cols = []
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        Gr, GN, GS, Gt, Gp = oracle_mod.vv_curl(rf, tf, pf, e.reshape(np_, 3, nt, nr))
        cols.append(np.concatenate([Gr[:, 1:, :].ravel(), GN, GS, Gt[:, :, 1:nr].ravel(),
                                    Gp[:, 1:, 1:nr].ravel()]))
    C = np.sign(np.round(np.array(cols).T, 12))          # edges x faces, entries in {-1, 0, 1}
    psi = np.random.default_rng(7).standard_normal(C.shape[0])
    flux = (C.T @ psi).reshape(np_, 3, nt, nr)
    v = np.zeros_like(flux)
    v[:, 0, :, 1:] = flux[:, 0, :, 1:] / g["A_r"][1:nr].transpose(2, 1, 0)
    v[:, 1, 1:, :] = flux[:, 1, 1:, :] / g["A_t"][1:nt].transpose(2, 0, 1)
    v[:, 2] = flux[:, 2] / g["A_p"][None]
    assert np.abs(flux).max() > 0.1
    delta = oracle_mod.vv_div(rf, tf, pf, v)
    assert np.abs(delta).max() <= 1e-12 * np.abs(flux).max()


# ------------------------------------------------------------------ closed forms
def test_vv_outflow_closed_forms(oracle_mod):
    """Gauss on fields the exact face integrals reproduce: v = r r_hat (div v = 3) has outflow
    3 V per cell; v = theta_hat / r has outflow dphi dr (sin t_f[j+1] - sin t_f[j])."""
    nr, nt, np_ = 6, 7, 9
    rf, tf, pf = grid(nr, nt, np_, r0=1.0, r1=3.0)
    g = geometry(rf, tf, pf)
    v = np.zeros((np_, 3, nt, nr))
    v[:, 0, :, :] = rf[None, None, :-1]
    gin, gout = np.zeros((3, np_, nt)), np.zeros((3, np_, nt))
    gin[0], gout[0] = rf[0], rf[-1]
    np.testing.assert_allclose(oracle_mod.vv_div(rf, tf, pf, v, gin, gout), 3 * g["V"], rtol=1e-13)
    v[:] = 0.0
    v[:, 1, 1:, :] = 1.0 / g["rc"][None, None, :]
    exact = (np.diff(pf)[:, None, None] * np.diff(rf)[None, None, :]
             * (np.sin(np.concatenate([tf[1:-1], [0.0]])) - np.sin(np.concatenate([[0.0], tf[1:-1]])))[None, :, None])
    np.testing.assert_allclose(oracle_mod.vv_div(rf, tf, pf, v), exact, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("bc", [0, 1])
def test_vv_circulation_rigid_rotation(oracle_mod, bc):
    """Stokes on v = Omega x r (v_phi = Omega r sin theta), curl v = 2 Omega z_hat: the circulation of
    every dual loop equals the exact flux of 2 Omega z_hat through it -- r-edges
    Omega rc^2 hphi (sin^2 tc_j - sin^2 tc_{j-1}); the polar axes (the pole-ring sums, Listing 3)
    +-2 pi Omega rc^2 sin^2 tc; theta-edges -Omega sin^2 tc hphi (rce_{e+1}^2 - rce_e^2), walls
    included; phi-edges 0."""
    nr, nt, np_ = 5, 6, 7
    Om = 0.7
    rf, tf, pf = grid(nr, nt, np_)
    g = geometry(rf, tf, pf)
    rc, tc, rce, hl = g["rc"], g["tc"], g["rce"], g["hphi_lo"]
    v = np.zeros((np_, 3, nt, nr))
    v[:, 2] = Om * rc[None, None, :] * np.sin(tc)[None, :, None]
    gin, gout = np.zeros((3, np_, nt)), np.zeros((3, np_, nt))
    gin[2] = Om * rf[0] * np.sin(tc)[None, :]
    gout[2] = Om * rf[-1] * np.sin(tc)[None, :]
    Gr, GN, GS, Gt, Gp = oracle_mod.vv_curl(rf, tf, pf, v, gin, gout)
    s2 = np.sin(tc) ** 2
    ex_r = Om * rc[None, None, :] ** 2 * hl[:, None, None] * (s2[1:] - s2[:-1])[None, :, None]
    np.testing.assert_allclose(Gr[:, 1:, :], ex_r, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(GN, 2 * PI * Om * rc ** 2 * s2[0], rtol=1e-13)
    np.testing.assert_allclose(GS, -2 * PI * Om * rc ** 2 * s2[-1], rtol=1e-13)
    ex_t = -Om * s2[None, :, None] * hl[:, None, None] * (rce[1:] ** 2 - rce[:-1] ** 2)[None, None, :]
    np.testing.assert_allclose(Gt, ex_t, rtol=1e-12, atol=1e-14)
    assert np.abs(Gp).max() <= 1e-14


# ------------------------------------------------------------------ algebra on tiny grids
@pytest.mark.parametrize("bc_in,bc_out", [(0, 0), (0, 1), (1, 1)])
def test_vv_symmetric(oracle_mod, bc_in, bc_out):
    """x.Ay = y.Ax to 1e-12 (the energy form makes A symmetric by construction)."""
    nr, nt, np_ = 6, 5, 8
    rf, tf, pf = grid(nr, nt, np_)
    nu, s = rand_fields(np_, nt, nr, 11)
    op = oracle_mod.VVOperator(rf, tf, pf, nu, s, bc_in, bc_out)
    rng = np.random.default_rng(3)
    m = op.unknown_mask()
    x, y = rng.standard_normal(op.shape) * m, rng.standard_normal(op.shape) * m
    a, b = np.vdot(x, op.apply(y)), np.vdot(y, op.apply(x))
    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b))


@pytest.mark.parametrize("bc_in,bc_out,shift", [(0, 0, True), (1, 0, True), (0, 0, False), (1, 1, False)])
def test_vv_diag_spd_and_dense_solve(oracle_mod, bc_in, bc_out, shift):
    """The Jacobi diagonal equals diag(A) read off the apply; A is symmetric positive definite
    (also with s = 0); PCG to 1e-13 reproduces a dense LU solve of A x = b, b = M f - A(0; g)
    with random forcing and wall data."""
    nr, nt, np_ = 3, 4, 4
    rf, tf, pf = grid(nr, nt, np_)
    nu, s = rand_fields(np_, nt, nr, 5)
    if not shift:
        s = np.zeros_like(s)
    op = oracle_mod.VVOperator(rf, tf, pf, nu, s, bc_in, bc_out)
    A, idx = dense(op)
    np.testing.assert_allclose(np.diag(A), op.D.ravel()[idx], rtol=1e-14)
    assert np.all(op.D.ravel()[np.setdiff1d(np.arange(op.D.size), idx)] == 1.0)
    np.testing.assert_allclose(A, A.T, rtol=0, atol=1e-12 * np.abs(A).max())
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0
    rng = np.random.default_rng(9)
    f = rng.standard_normal(op.shape)
    gin, gout = rng.standard_normal((3, np_, nt)), rng.standard_normal((3, np_, nt))
    b = op.rhs(f, gin, gout)
    st, x, it, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-13, 5000)
    assert st == 0
    xd = np.linalg.solve(A, b.ravel()[idx])
    assert np.linalg.norm(x.ravel()[idx] - xd) <= 1e-11 * np.linalg.norm(xd)
    assert np.all(x.ravel()[np.setdiff1d(np.arange(x.size), idx)] == 0.0)
    # b = M f - A(0; g) is linear in the wall data with the homogeneous operator as the "A(0;.)" part
    np.testing.assert_allclose(op.rhs(f, gin, gout) - op.rhs(f), -op.apply(np.zeros(op.shape), gin, gout),
                               rtol=1e-13, atol=1e-13)


def test_vv_zero_viscosity_one_iteration(oracle_mod):
    """nu = 0: A = diag(s M) = D, so PCG stops after one iteration with x = f / s on every face."""
    nr, nt, np_ = 5, 6, 6
    rf, tf, pf = grid(nr, nt, np_)
    _, s = rand_fields(np_, nt, nr, 2)
    sf = np.full((np_, nt, nr), 1.25)
    op = oracle_mod.VVOperator(rf, tf, pf, np.zeros((np_, nt, nr)), sf)
    f = np.random.default_rng(1).standard_normal(op.shape)
    st, x, it, hist, bn, rn = op.pcg(op.rhs(f), np.zeros(op.shape), 1e-14, 50)
    m = op.unknown_mask()
    assert st == 0 and it == 1
    np.testing.assert_allclose(x[m], f[m] / 1.25, rtol=1e-15)


def test_vv_pole_ring_is_a_per_radius_sum(oracle_mod):
    """The axis circulation is the per-radius sum over the pole ring (Listing 3's sum0(i),
    PAPER.md:147-157): GN(i) = sum_k l_p v_p(i, 0, k) and GS(i) = -sum_k l_p v_p(i, nt-1, k),
    evaluated here with correctly rounded math.fsum."""
    nr, nt, np_ = 4, 5, 11
    rf, tf, pf = grid(nr, nt, np_)
    g = geometry(rf, tf, pf)
    v = np.random.default_rng(4).standard_normal((np_, 3, nt, nr))
    _, GN, GS, _, _ = oracle_mod.vv_curl(rf, tf, pf, v)
    for i in range(nr):
        lN = g["rc"][i] * math.sin(g["tc"][0]) * g["hphi_lo"]
        lS = g["rc"][i] * math.sin(g["tc"][-1]) * g["hphi_lo"]
        assert GN[i] == pytest.approx(math.fsum(lN * v[:, 2, 0, i]), rel=1e-13)
        assert GS[i] == pytest.approx(-math.fsum(lS * v[:, 2, nt - 1, i]), rel=1e-13)


# ------------------------------------------------------------------ manufactured solution
def mms_fields(r, t, p):
    """v = grad(phi) + r x grad(chi), phi = e^-r sin t cos t cos p (l = 2), chi = r e^-r (sin t sin p +
    cos t) (l = 1; the cos t part is a differential rotation about the polar axis, so the axis
    circulations are exercised); lap v = grad(lap phi) + r x grad(lap chi) (the Laplacian commutes with grad and with
    r x grad), lap(f Y_l) = (f'' + 2 f'/r - l(l+1) f / r^2) Y_l."""
    e = np.exp(-r)
    f1, f1p = e, -e
    g1 = e * (1 - 2 / r - 6 / r ** 2)
    g1p = -e * (1 - 2 / r - 6 / r ** 2) + e * (2 / r ** 2 + 12 / r ** 3)
    f2, g2 = r * e, e * (r - 4)
    st, ct, sp, cp = np.sin(t), np.cos(t), np.sin(p), np.cos(p)
    v = (f1p * st * ct * cp, f1 * np.cos(2 * t) * cp / r - f2 * cp, -f1 * ct * sp / r + f2 * (ct * sp - st))
    lap = (g1p * st * ct * cp, g1 * np.cos(2 * t) * cp / r - g2 * cp, -g1 * ct * sp / r + g2 * (ct * sp - st))
    return v, lap


def mms_error(oracle_mod, n, a, eps, nu=1.0, s=1.0):
    nr, nt, np_ = n, n, 2 * n
    rf, tf, pf = inputs.rfaces(nr, 1.0, 2.0, a), inputs.tfaces(nt, eps), inputs.pfaces(np_)
    rc, tc, pc = inputs.midpoints(rf), inputs.midpoints(tf), inputs.midpoints(pf)
    R, T, P = (lambda x: x[None, None, :]), (lambda x: x[None, :, None]), (lambda x: x[:, None, None])
    ex, f = np.zeros((np_, 3, nt, nr)), np.zeros((np_, 3, nt, nr))
    at = [(R(rf[:-1]), T(tc), P(pc)), (R(rc), T(tf[:-1]), P(pc)), (R(rc), T(tc), P(pf[:-1]))]
    for c in range(3):
        v, lap = mms_fields(*at[c])
        ex[:, c] = v[c]
        f[:, c] = s * v[c] - nu * lap[c]
    def wall(r):
        gw = np.zeros((3, np_, nt))
        wat = [(tc[None, :], pc[:, None]), (tf[:-1][None, :], pc[:, None]), (tc[None, :], pf[:-1][:, None])]
        for c in range(3):
            gw[c] = np.broadcast_to(mms_fields(r, *wat[c])[0][c], (np_, nt))
        return gw
    res = oracle_mod.vv_solve(rf, tf, pf, np.full((np_, nt, nr), nu), np.full((np_, nt, nr), s), f,
                              np.zeros_like(ex), 1e-13, 20000, 0, 0, wall(rf[0]), wall(rf[-1]))
    assert res["status"] == 0
    op = res["op"]
    m, M = op.unknown_mask(), op.mass()
    err = (res["x"] - ex) * m
    l2 = math.sqrt(np.sum(M * err ** 2) / np.sum(M * (ex * m) ** 2))
    linf = np.abs(err).max() / np.abs(ex * m).max()
    return l2, linf


@pytest.mark.parametrize("a,eps", [(0.0, 0.0), (2.0, 0.2)])
def test_vv_manufactured_solution_second_order(oracle_mod, a, eps):
    """s v - nu lap v = f with the exact solution on the no-slip walls: the mass-weighted L2 error
    falls x4 per refinement on uniform and stretched grids (measured orders 2.01, 2.02 and 1.96, 2.02);
    the max error (at the pole rows, the polar-cap dual areas) falls at least first order."""
    errs = [mms_error(oracle_mod, n, a, eps) for n in (8, 16, 32)]
    for (l2a, lia), (l2b, lib) in zip(errs, errs[1:]):
        assert math.log2(l2a / l2b) >= 1.9
        assert math.log2(lia / lib) >= 0.8
    assert errs[-1][0] < 5e-4
