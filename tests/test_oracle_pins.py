"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test checks the oracle (oracle/masoracle.c) against what the mathematics
or a hand derivation fixes -- closed forms, invariants, special cases that
reduce to a textbook or library routine, brute force on tiny inputs -- chosen
so that a plausible slip (a dropped metric factor, a wrong sign, a wrong face
index, a transposed operand, a missing periodic wrap) fails at least one.
Readings R1-R18 are those of SURVEY.md section 8(c) / DESIGN.md section 3;
PAPER.md:56 (Sec. III) is the passage the operator elaborates and
PAPER.md:246 (Sec. V-A) the "validated ... to within solver tolerances"
criterion.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

from paper_2303_03398_b200 import inputs

HERE = os.path.dirname(os.path.abspath(__file__))
PI = math.pi


def op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, bc_in, bc_out):
    return oracle_mod.Operator(rf, tf, pf, kr, kt, kp, s, bc_in, bc_out)


def dense(op):
    n = op.np * op.nt * op.nr
    A = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        A[:, c] = op.apply(e.reshape(op.shape)).ravel()
    return A


def const_fields(nr, nt, np_, kappa=1.0, s=1.0):
    return (np.full((np_, nt, nr + 1), kappa), np.full((np_, nt + 1, nr), kappa),
            np.full((np_, nt, nr), kappa), np.full((np_, nt, nr), s))


# ------------------------------------------------------------------ metric (R1-R3)
@pytest.mark.parametrize("nr,nt,np_,a,eps,band", [
    (8, 8, 16, 0.0, 0.0, None), (13, 7, 5, 5.33, 0.1, None), (40, 30, 12, 3.0, 0.3, None),
    (5, 6, 3, 1.0, 0.0, (0.3, 2.5)), (1, 1, 1, 0.0, 0.0, None)])
def test_sum_of_volumes_closed_form(oracle_mod, nr, nt, np_, a, eps, band):
    """sum V = (2 pi)(cos t_0 - cos t_nt)(r_nr^3 - r_0^3)/3 exactly (R3: exact FV integrals)."""
    rf = inputs.rfaces(nr, 1.0, 30.0, a)
    tf = inputs.tfaces(nt, eps) if band is None else inputs.tfaces(nt, 0.0, *band)
    pf = inputs.pfaces(np_)
    V = oracle_mod.volumes(rf, tf, pf)
    exact = 2 * PI * (math.cos(tf[0]) - math.cos(tf[-1])) * (rf[-1] ** 3 - rf[0] ** 3) / 3
    assert abs(V.sum() - exact) <= 1e-13 * exact
    assert (V > 0).all()


@pytest.mark.parametrize("nr,nt,np_", [(6, 9, 8), (3, 20, 7)])
def test_r_face_areas_tile_the_sphere(oracle_mod, nr, nt, np_):
    """With kr = 1: T^r_i h^r_i summed over a full shell = 4 pi r_f[i]^2 (area of the sphere)."""
    rf, tf, pf = inputs.rfaces(nr, 1.0, 4.0, 2.0), inputs.tfaces(nt, 0.3), inputs.pfaces(np_)
    kr, kt, kp, s = const_fields(nr, nt, np_)
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 0, 0)
    rc = inputs.midpoints(rf)
    h = np.concatenate([[rc[0] - rf[0]], np.diff(rc), [rf[-1] - rc[-1]]])
    area = (op.Tr * h[None, None, :]).sum(axis=(0, 1))
    np.testing.assert_allclose(area, 4 * PI * rf ** 2, rtol=1e-13)


# ------------------------------------------------------------------ operator (R4)
@pytest.mark.parametrize("seed,shape", [(1, (7, 6, 5)), (2, (4, 9, 1)), (3, (1, 5, 6)), (4, (10, 1, 2))])
def test_operator_annihilates_constants_away_from_dirichlet(oracle_mod, seed, shape):
    """K 1 = 0 in every row without a Dirichlet face (BJ north_star: 'annihilates constants')."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, shift=False, bc_in=0, bc_out=1)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 0, 1)
    y = op.apply(np.ones(op.shape))
    rows = y[:, :, 1:] if nr > 1 else y[:, :, :0]
    assert np.abs(rows).max(initial=0.0) <= 1e-13 * op.D.max()
    # the Dirichlet row is strictly positive: the boundary face only adds to D
    assert (y[:, :, 0] > 0).all()


@pytest.mark.parametrize("seed,shape,bc", [(5, (7, 6, 5), (0, 1)), (6, (4, 9, 3), (1, 0)),
                                          (7, (5, 5, 1), (0, 0)), (8, (6, 1, 2), (1, 1)),
                                          (9, (1, 1, 12), (1, 1))])
def test_operator_symmetric(oracle_mod, seed, shape, bc):
    """x.Ay = y.Ax to 1e-12 relative (BJ north_star; symmetry of the volume-weighted form, R6)."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, bc_in=bc[0], bc_out=bc[1])
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, *bc)
    rng = np.random.default_rng(seed)
    x, y = rng.standard_normal(op.shape), rng.standard_normal(op.shape)
    xay, yax = np.vdot(x, op.apply(y)), np.vdot(y, op.apply(x))
    scale = np.vdot(np.abs(x), np.abs(op.apply(np.abs(y))))
    assert abs(xay - yax) <= 1e-12 * scale


@pytest.mark.parametrize("seed,shape", [(11, (6, 7, 5)), (12, (3, 4, 2))])
def test_telescoping_flux_sum(oracle_mod, seed, shape):
    """Conservation: with Neumann r walls, 1^T A u = sum_c s_c V_c u_c (every face flux cancels)."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, bc_in=1, bc_out=1)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 1, 1)
    V = oracle_mod.volumes(p.rf, p.tf, p.pf)
    u = np.random.default_rng(seed).standard_normal(op.shape)
    lhs = op.apply(u).sum()
    rhs = (p.s * V * u).sum()
    assert abs(lhs - rhs) <= 1e-12 * np.abs(op.D * u).sum()


# ------------------------------------------------------------------ hand-worked golden
def _ev(e):
    return eval(e, {"pi": PI, "__builtins__": {}})


@pytest.mark.parametrize("case", json.load(open(os.path.join(HERE, "golden", "hand_worked.json")))["cases"],
                         ids=lambda c: c["name"])
def test_hand_worked_two_cell_golden(oracle_mod, case):
    """Two-cell operators derived by hand (tests/golden/hand_worked.json)."""
    rf, tf, pf = (np.array(case[k]) for k in ("rf", "tf", "pf"))
    np_, nt, nr = case["shape"]
    kr, kt, kp, _ = const_fields(nr, nt, np_)
    s = np.array(case["s"]).reshape(np_, nt, nr)
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, case["bc_in"], case["bc_out"])
    V = oracle_mod.volumes(rf, tf, pf).ravel()
    np.testing.assert_allclose(V, [_ev(e) for e in case["V"]["expr"]], rtol=1e-14)
    if "D" in case:
        np.testing.assert_allclose(op.D.ravel(), [_ev(e) for e in case["D"]["expr"]], rtol=1e-14)
    A = dense(op)
    Ax = np.array([[_ev(e) for e in row] for row in case["A"]["expr"]])
    np.testing.assert_allclose(A, Ax, rtol=1e-13, atol=1e-13 * np.abs(Ax).max())
    g_in = np.full((np_, nt), case["g_in"]) if case["bc_in"] == 0 else None
    g_out = np.full((np_, nt), case["g_out"]) if case["bc_out"] == 0 else None
    b = op.rhs(np.array(case["f"]).reshape(op.shape), g_in, g_out)
    np.testing.assert_allclose(b.ravel(), [_ev(e) for e in case["b"]["expr"]], rtol=1e-14,
                               atol=1e-14 * np.abs(b).max())
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-14, 10)
    assert st == 0 and iters <= 2
    np.testing.assert_allclose(x.ravel(), case["x"]["value"], rtol=1e-13)
    np.testing.assert_allclose(x.ravel(), [_ev(e) for e in case["x"]["expr"]], rtol=1e-13)


# ------------------------------------------------------------------ linear algebra (R6, R11-R14)
@pytest.mark.parametrize("seed,shape,bc", [(21, (4, 4, 8), (0, 1)), (22, (4, 4, 8), (0, 0)),
                                          (23, (3, 5, 4), (1, 0)), (24, (5, 3, 2), (1, 1))])
def test_pcg_matches_dense_lu(oracle_mod, seed, shape, bc):
    """Tiny grids: PCG at tol 1e-14 = numpy dense LU solve of the same operator to 1e-12;
    the operator is symmetric positive definite and hist[k] is the recurrence residual."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, bc_in=bc[0], bc_out=bc[1])
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, *bc)
    A = dense(op)
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0
    b = op.rhs(p.f, p.g_in, p.g_out)
    x_lu = np.linalg.solve(A, b.ravel())
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-14, 500)
    assert st == 0
    assert np.linalg.norm(x.ravel() - x_lu) <= 1e-12 * np.linalg.norm(x_lu)
    assert abs(bn - np.linalg.norm(b)) <= 1e-15 * bn
    assert hist[0] == pytest.approx(np.linalg.norm(b), rel=1e-15)     # x0 = 0
    assert hist[-1] <= 1e-14 * bn and hist[-2] > 1e-14 * bn
    # the recurrence residual tracks the true residual b - A x
    assert np.linalg.norm(b.ravel() - A @ x.ravel()) <= 1e-13 * bn


def test_pcg_nonzero_initial_guess_and_early_exit(oracle_mod):
    p = inputs.random_problem(5, 4, 6, 31)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    A = dense(op)
    b = op.rhs(p.f, p.g_in, p.g_out)
    x_lu = np.linalg.solve(A, b.ravel()).reshape(op.shape)
    x0 = np.random.default_rng(3).standard_normal(op.shape)
    st, x, iters, hist, bn, rn = op.pcg(b, x0, 1e-13, 500)
    assert st == 0 and hist[0] == pytest.approx(np.linalg.norm(b.ravel() - A @ x0.ravel()), rel=1e-13)
    np.testing.assert_allclose(x, x_lu, rtol=0, atol=1e-11 * np.abs(x_lu).max())
    # x0 already converged -> 0 iterations, x untouched
    st, x2, iters, hist, bn, rn = op.pcg(b, x_lu, 1e-6, 500)
    assert st == 0 and iters == 0 and np.array_equal(x2, x_lu)
    # b = 0 -> x = 0, OK, 0 iterations (R14)
    st, x3, iters, hist, bn, rn = op.pcg(np.zeros(op.shape), x0, 1e-10, 10)
    assert st == 0 and iters == 0 and not x3.any() and bn == 0
    # tol = 0 -> exactly maxit iterations, NOT_CONVERGED (R14)
    st, x4, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 0.0, 7)
    assert st == oracle_mod.NOT_CONVERGED and iters == 7 and hist.size == 8
    # maxit = 0 -> only hist[0]
    st, x5, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-10, 0)
    assert st == oracle_mod.NOT_CONVERGED and iters == 0 and hist.size == 1


def test_shift_only_is_one_iteration(oracle_mod):
    """kappa = 0: A = diag(sV) = M, so PCG stops after 1 iteration with x = f/s."""
    nr, nt, np_ = 6, 5, 4
    p = inputs.random_problem(nr, nt, np_, 41, bc_in=1, bc_out=1)
    z = lambda a: np.zeros_like(a)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, z(p.kr), z(p.kt), z(p.kp), p.s, 1, 1)
    b = op.rhs(p.f)
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-12, 10)
    assert st == 0 and iters == 1
    np.testing.assert_allclose(x, p.f / p.s, rtol=1e-15)


def test_dirichlet_constant_is_exact(oracle_mod):
    """g_in = g_out = c, s = 0, f = 0, random kappa: x == c (constants are annihilated)."""
    nr, nt, np_ = 6, 8, 12
    p = inputs.random_problem(nr, nt, np_, 51, shift=False, bc_in=0, bc_out=0)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 0, 0)
    c = 2.5
    g = np.full((np_, nt), c)
    b = op.rhs(np.zeros(op.shape), g, g)
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-14, 2000)
    assert st == 0
    assert np.abs(x - c).max() <= 1e-12 * c


def test_phi_ring_is_circulant_and_matches_fft(oracle_mod):
    """nr = nt = 1 theta band, uniform phi, Neumann r: A is circulant (periodic wrap, R9);
    the FFT solve equals PCG, which needs <= floor(np/2)+1 iterations (distinct eigenvalues)."""
    np_ = 16
    rf, tf, pf = np.array([1.0, 2.0]), np.array([PI / 3, 2 * PI / 3]), inputs.pfaces(np_)
    kr, kt, kp, s = const_fields(1, 1, np_, kappa=1.0, s=0.2)
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 1, 1)
    A = dense(op)
    col = A[:, 0]
    for k in range(np_):
        np.testing.assert_allclose(A[:, k], np.roll(col, k), rtol=0, atol=4e-15 * col[0])
    assert col[1] < 0 and col[-1] < 0 and np.count_nonzero(np.abs(col) > 1e-14 * col[0]) == 3
    b = np.random.default_rng(7).standard_normal(np_)
    x_fft = np.real(np.fft.ifft(np.fft.fft(b) / np.fft.fft(col)))
    st, x, iters, hist, bn, rn = op.pcg(b.reshape(op.shape), np.zeros(op.shape), 1e-14, 100)
    assert st == 0 and iters <= np_ // 2 + 1
    np.testing.assert_allclose(x.ravel(), x_fft, rtol=0, atol=1e-13 * np.abs(x_fft).max())


def test_radial_column_matches_banded_solver(oracle_mod):
    """np = nt = 1: a tridiagonal radial system on a stretched grid; scipy solve_banded agrees."""
    nr = 40
    rf = inputs.rfaces(nr, 1.0, 30.0, 5.33)
    tf, pf = np.array([0.0, PI]), inputs.pfaces(1)
    rng = np.random.default_rng(9)
    kr = rng.uniform(0.5, 2, (1, 1, nr + 1))
    kt, kp = np.ones((1, 2, nr)), np.ones((1, 1, nr))
    s = rng.uniform(0.1, 1, (1, 1, nr))
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 0, 1)
    A = dense(op)
    assert np.abs(np.triu(A, 2)).max() == 0 and np.abs(np.tril(A, -2)).max() == 0
    ab = np.zeros((3, nr))
    ab[0, 1:] = np.diag(A, 1)
    ab[1] = np.diag(A)
    ab[2, :-1] = np.diag(A, -1)
    b = op.rhs(rng.standard_normal((1, 1, nr)), np.ones((1, 1)), None)
    x_band = scipy.linalg.solve_banded((1, 1), ab, b.ravel())
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-15, 400)
    assert st == 0
    np.testing.assert_allclose(x.ravel(), x_band, rtol=1e-12)


# ------------------------------------------------------------------ discretisation order
def _spherical_capacitor_err(oracle_mod, nr):
    rf = inputs.rfaces(nr, 1.0, 30.0, 5.33)
    tf, pf = np.array([0.0, PI]), inputs.pfaces(1)
    kr, kt, kp, s = const_fields(nr, 1, 1, kappa=1.0, s=0.0)
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 0, 0)
    b = op.rhs(np.zeros(op.shape), np.ones((1, 1)), np.zeros((1, 1)))
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-15, 5 * nr)
    assert st == 0
    rc = inputs.midpoints(rf)
    exact = (1 / rc - 1 / 30.0) / (1 / 1.0 - 1 / 30.0)
    return np.abs(x.ravel() - exact).max()


def test_spherical_capacitor_second_order(oracle_mod):
    """kappa = 1, s = 0, f = 0, u(1) = 1, u(30) = 0 -> u = (1/r - 1/30)/(1 - 1/30);
    second order on the c3 radial stretching (a = 5.33)."""
    errs = [_spherical_capacitor_err(oracle_mod, n) for n in (20, 40, 80, 160)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert errs[0] < 5e-3
    assert all(1.9 < o < 2.1 for o in orders), (errs, orders)


def _mms(oracle_mod, nr, nt, np_, stretched):
    """u = e^{-r} sin(th) cos(th) cos(ph) (an l = 2 harmonic), kappa = 1 + r/2, s = 1 on r in [1, 3]:
    f = s u - [kappa u_rr + (2 kappa / r + kappa') u_r - 6 kappa u / r^2]."""
    if stretched:
        rf = 1 + 2 * np.expm1(3 * np.arange(nr + 1) / nr) / math.expm1(3)
        y = np.arange(nt + 1) / nt
        tf = PI * (y + 0.3 * np.sin(2 * PI * y) / (2 * PI))
        z = np.arange(np_ + 1) / np_
        pf = 2 * PI * (z + 0.2 * np.sin(2 * PI * z) / (2 * PI))
        tf[0], tf[-1], pf[0], pf[-1] = 0.0, PI, 0.0, 2 * PI
    else:
        rf, tf, pf = inputs.rfaces(nr, 1.0, 3.0, 0.0), inputs.tfaces(nt, 0.0), inputs.pfaces(np_)
    rc, tc, pc = (0.5 * (a[1:] + a[:-1]) for a in (rf, tf, pf))
    pfc = pf[1:]
    kap = lambda r: 1.0 + 0.5 * r
    Y = lambda t, p: np.sin(t) * np.cos(t) * np.cos(p)
    kr = np.broadcast_to(kap(rf)[None, None, :], (np_, nt, nr + 1)).copy()
    kt = np.broadcast_to(kap(rc)[None, None, :], (np_, nt + 1, nr)).copy()
    kp = np.broadcast_to(kap(rc)[None, None, :], (np_, nt, nr)).copy()
    s = np.ones((np_, nt, nr))
    R, T, P = rc[None, None, :], tc[None, :, None], pc[:, None, None]
    u = np.exp(-R) * Y(T, P)
    ur, urr = -np.exp(-R) * Y(T, P), np.exp(-R) * Y(T, P)
    k = kap(R)
    f = s * u - (k * urr + (2 * k / R + 0.5) * ur - 6 * k * u / R ** 2)
    g_in = (np.exp(-rf[0]) * Y(tc[None, :], pc[:, None]))
    g_out = (np.exp(-rf[-1]) * Y(tc[None, :], pc[:, None]))
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 0, 0)
    b = op.rhs(f, g_in, g_out)
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-13, 5000)
    assert st == 0
    V = oracle_mod.volumes(rf, tf, pf)
    e = x - u
    return math.sqrt((V * e * e).sum() / V.sum()), np.abs(e).max()


@pytest.mark.parametrize("stretched", [False, True])
def test_manufactured_solution_second_order(oracle_mod, stretched):
    """BJ north_star: 'a manufactured smooth solution converges at second order under grid
    refinement' -- volume-weighted L2 and L-inf errors fall ~4x per doubling, pole rows included."""
    res = [_mms(oracle_mod, n, n, 2 * n, stretched) for n in (8, 16, 32)]
    l2 = [r[0] for r in res]
    linf = [r[1] for r in res]
    o2 = [math.log2(l2[i] / l2[i + 1]) for i in range(2)]
    oi = [math.log2(linf[i] / linf[i + 1]) for i in range(2)]
    assert all(1.85 < o < 2.3 for o in o2), (l2, o2)
    assert all(1.7 < o < 2.4 for o in oi), (linf, oi)
    assert l2[0] < 2e-3


# ------------------------------------------------------------------ error paths
def test_error_paths(oracle_mod):
    nr, nt, np_ = 4, 3, 4
    p = inputs.random_problem(nr, nt, np_, 61, shift=False, bc_in=1, bc_out=1)
    with pytest.raises(oracle_mod.OracleError) as e:
        op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 1, 1)
    assert e.value.status == oracle_mod.E_SINGULAR
    kr = p.kr.copy()
    kr[1, 1, 1] = -1.0
    with pytest.raises(oracle_mod.OracleError) as e:
        op_from(oracle_mod, p.rf, p.tf, p.pf, kr, p.kt, p.kp, p.s + 1, 1, 1)
    assert e.value.status == oracle_mod.E_INVALID
    bad_pf = p.pf.copy()
    bad_pf[-1] = 6.0
    assert oracle_mod.check_grid(p.rf, p.tf, bad_pf) == oracle_mod.E_INVALID
    bad_rf = p.rf.copy()
    bad_rf[2] = bad_rf[1]
    assert oracle_mod.check_grid(bad_rf, p.tf, p.pf) == oracle_mod.E_INVALID
    bad_tf = p.tf.copy()
    bad_tf[-1] = 3.2
    assert oracle_mod.check_grid(p.rf, bad_tf, p.pf) == oracle_mod.E_INVALID
    # non-finite rhs -> breakdown
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s + 1, 1, 1)
    b = op.rhs(p.f)
    b[0, 0, 0] = np.nan
    st, *_ = op.pcg(b, np.zeros(op.shape), 1e-10, 10)
    assert st == oracle_mod.E_BREAKDOWN


# ------------------------------------------------------------------ generated configs
def test_config_c1_iteration_count(oracle_mod):
    """c1 (BASELINE.json configs[0]) converges to 1e-10 in 130 iterations (SURVEY Appendix X4,
    an independent scipy implementation of the same readings)."""
    r = oracle_mod.solve_problem(inputs.make_problem("c1"))
    assert r["status"] == 0 and r["iters"] == 130
    assert r["hist"][-1] <= 1e-10 * r["bnorm"]


# ------------------------------------------------------------------ face coefficients from fields (NEXT-1, R25)
def test_face_coefficients_closed_forms(oracle_mod):
    """Constant field c: every face kappa = kappa0 c^(m/2) (both means); m = 0 gives kappa0; the shift
    is inv_dt * rho.  Two-cell hand values: kappa = [1, 32] (T = [1, 4], m = 5) -> arithmetic 33/2,
    harmonic 2*32/33 on the shared face."""
    f = np.full((3, 4, 5), 2.0)
    rho = np.random.default_rng(1).uniform(0.5, 2.0, f.shape)
    for mean in (0, 1):
        kr, kt, kp, s = oracle_mod.face_coefficients(f, 1.5, 5, mean, rho, 10.0)
        for a in (kr, kt, kp):
            np.testing.assert_allclose(a, 1.5 * 2.0 ** 2.5, rtol=2e-16 * 8)
        np.testing.assert_array_equal(s, 10.0 * rho)
        kr, kt, kp, s = oracle_mod.face_coefficients(f, 0.7, 0, mean)
        assert (kr == 0.7).all() and (kp == 0.7).all() and (s == 1.0).all()
    T = np.array([1.0, 4.0]).reshape(1, 1, 2)
    kr, kt, kp, s = oracle_mod.face_coefficients(T, 1.0, 5, 0)
    assert kr.ravel().tolist() == [1.0, 16.5, 32.0]
    kr, kt, kp, s = oracle_mod.face_coefficients(T, 1.0, 5, 1)
    assert kr.ravel()[0] == 1.0 and kr.ravel()[2] == 32.0
    assert kr.ravel()[1] == pytest.approx(64.0 / 33.0, rel=1e-15)


def test_face_coefficients_means_and_periodic_wrap(oracle_mod):
    """Harmonic <= arithmetic with equality only for equal neighbours; the phi face of the last plane
    averages it with plane 0; boundary r / theta faces take the adjacent cell's kappa."""
    rng = np.random.default_rng(3)
    f = rng.uniform(0.2, 3.0, (6, 5, 7))
    ka = oracle_mod.face_coefficients(f, 2.0, 5, 0)
    kh = oracle_mod.face_coefficients(f, 2.0, 5, 1)
    for a, h in zip(ka[:3], kh[:3]):
        assert (h <= a * (1 + 1e-15)).all()
    kap = 2.0 * f ** 2.5
    np.testing.assert_allclose(ka[2][-1], 0.5 * (kap[-1] + kap[0]), rtol=1e-14)
    np.testing.assert_allclose(ka[0][:, :, 0], kap[:, :, 0], rtol=1e-14)
    np.testing.assert_allclose(ka[0][:, :, -1], kap[:, :, -1], rtol=1e-14)
    np.testing.assert_allclose(ka[1][:, 0, :], kap[:, 0, :], rtol=1e-14)
    # the operator assembled from these faces is still symmetric positive definite
    p = inputs.random_problem(7, 5, 6, 1)
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, *kh[:3], kh[3] * 0 + 1.0, 0, 1)
    x, y = rng.standard_normal(op.shape), rng.standard_normal(op.shape)
    assert abs(np.vdot(x, op.apply(y)) - np.vdot(y, op.apply(x))) <= 1e-12 * np.vdot(np.abs(x), np.abs(op.apply(np.abs(y))))
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.face_coefficients(f, 1.0, 17, 0)


# ------------------------------------------------------------------ super-time-stepping (NEXT-4, R26)
def _dense_K_over_V(oracle_mod, op, s):
    """M = V^{-1} K with K = A - diag(sV) (A from the oracle's apply, column by column)."""
    A = dense(op)
    V = oracle_mod.volumes(op.rf, op.tf, op.pf).ravel()
    K = A - np.diag(s.ravel() * V)
    return K / V[:, None], V


def test_rkl2_preserves_steady_states(oracle_mod):
    """u = const with Neumann walls (L u = 0), and u = c with Dirichlet g = c on both walls (K u = b_D):
    the RKL2 step returns u up to rounding."""
    p = inputs.random_problem(6, 5, 8, 71, bc_in=1, bc_out=1)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 1, 1)
    M, V = _dense_K_over_V(oracle_mod, op, p.s)
    tau = 0.9 * (7 * 7 + 7 - 2) / 4.0 * 2.0 / np.linalg.eigvals(M).real.max()   # inside the stability bound
    u = np.full(op.shape, 1.7)
    out = op.rkl2_step(u, p.s, tau, 7)
    assert np.abs(out - u).max() <= 1e-13 * 1.7
    p = inputs.random_problem(6, 5, 8, 72, shift=False, bc_in=0, bc_out=0)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 0, 0)
    M, V = _dense_K_over_V(oracle_mod, op, p.s)
    tau = 0.9 * (5 * 5 + 5 - 2) / 4.0 * 2.0 / np.linalg.eigvals(M).real.max()
    g = np.full((8, 5), 2.5)
    out = op.rkl2_step(np.full(op.shape, 2.5), p.s, tau, 5, g, g)
    assert np.abs(out - 2.5).max() <= 1e-13 * 2.5


def test_rkl2_second_order_against_matrix_exponential(oracle_mod):
    """V du/dt = -K u (Neumann walls): RKL2 with s = 6 stages converges to expm(-T V^-1 K) u0 at
    second order in tau (errors fall ~4x per halving)."""
    import scipy.linalg
    p = inputs.random_problem(4, 4, 8, 73, bc_in=1, bc_out=1)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 1, 1)
    M, V = _dense_K_over_V(oracle_mod, op, p.s)
    u0 = np.random.default_rng(4).standard_normal(op.shape)
    lam = np.abs(np.linalg.eigvals(M)).max()
    T = 4.0 / lam
    exact = (scipy.linalg.expm(-T * M) @ u0.ravel()).reshape(op.shape)
    errs = []
    for m in (8, 16, 32):
        u = u0.copy()
        for _ in range(m):
            u = op.rkl2_step(u, p.s, T / m, 6)
        errs.append(np.abs(u - exact).max())
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(1.8 < o < 2.3 for o in orders), (errs, orders)


def test_rkl2_stable_up_to_its_bound(oracle_mod):
    """tau = 0.99 (s^2 + s - 2)/4 * dt_FE (dt_FE = 2 / lambda_max of V^-1 K): 30 steps of a random
    initial state never increase the V-weighted energy (RKL2 is stable up to that bound), while a
    forward-Euler-sized step times 1.3 * (s^2+s-2)/4 blows up."""
    p = inputs.random_problem(5, 4, 6, 74, bc_in=1, bc_out=1)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 1, 1)
    M, V = _dense_K_over_V(oracle_mod, op, p.s)
    lam = np.linalg.eigvals(M).real.max()
    s = 8
    bound = (s * s + s - 2) / 4.0 * 2.0 / lam
    u = np.random.default_rng(5).standard_normal(op.shape)
    energy = lambda v: float((V * v.ravel() ** 2).sum())
    e0 = energy(u)
    for _ in range(30):
        u = op.rkl2_step(u, p.s, 0.99 * bound, s)
        assert energy(u) <= e0 * (1 + 1e-12)
        e0 = energy(u)
    v = np.random.default_rng(6).standard_normal(op.shape)
    for _ in range(30):
        v = op.rkl2_step(v, p.s, 1.3 * bound, s)
    assert energy(v) > 1e3 * energy(np.random.default_rng(6).standard_normal(op.shape))


# ------------------------------------------------------------------ single-reduction PCG (NEXT-3, R32)
@pytest.mark.parametrize("seed,shape,bc", [(21, (4, 4, 8), (0, 1)), (23, (3, 5, 4), (1, 0)), (24, (5, 3, 2), (0, 0))])
def test_cg1_matches_dense_lu(oracle_mod, seed, shape, bc):
    """Chronopoulos-Gear PCG at tol 1e-14 = dense LU to 1e-12; its recurrence residual tracks b - A x."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, bc_in=bc[0], bc_out=bc[1])
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, *bc)
    A = dense(op)
    b = op.rhs(p.f, p.g_in, p.g_out)
    x_lu = np.linalg.solve(A, b.ravel())
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-14, 500, variant="cg1")
    assert st == 0
    assert np.linalg.norm(x.ravel() - x_lu) <= 1e-12 * np.linalg.norm(x_lu)
    assert hist[-1] <= 1e-14 * bn and hist[-2] > 1e-14 * bn
    assert np.linalg.norm(b.ravel() - A @ x.ravel()) <= 1e-13 * bn


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_cg1_is_cg_in_exact_arithmetic(oracle_mod, name):
    """In exact arithmetic the Chronopoulos-Gear recurrences reproduce CG (s = A p, den = p.Ap), so on
    the configs both variants need the same iterations (c1 130, c2 406), their solutions agree
    to 1e-13 and their residual histories to 1e-8 above the rounding floor."""
    p = inputs.make_problem(name)
    a = oracle_mod.solve_problem(p)
    c = oracle_mod.solve_problem(p, variant="cg1")
    assert a["status"] == c["status"] == 0 and a["iters"] == c["iters"]
    assert np.linalg.norm(a["x"] - c["x"]) <= 1e-13 * np.linalg.norm(a["x"])
    floor = 1e-12 * a["bnorm"]
    m = a["hist"] > floor
    assert np.max(np.abs(a["hist"][m] - c["hist"][m]) / a["hist"][m]) <= 1e-8


def test_cg1_special_cases(oracle_mod):
    """kappa = 0 -> one iteration, x = f/s; the circulant phi ring within floor(np/2)+1 iterations;
    tol = 0 -> exactly maxit iterations; b = 0 -> x = 0."""
    nr, nt, np_ = 6, 5, 4
    p = inputs.random_problem(nr, nt, np_, 41, bc_in=1, bc_out=1)
    z = lambda a: np.zeros_like(a)
    op = op_from(oracle_mod, p.rf, p.tf, p.pf, z(p.kr), z(p.kt), z(p.kp), p.s, 1, 1)
    st, x, iters, *_ = op.pcg(op.rhs(p.f), np.zeros(op.shape), 1e-12, 10, variant="cg1")
    assert st == 0 and iters == 1
    np.testing.assert_allclose(x, p.f / p.s, rtol=1e-15)
    rf, tf, pf = np.array([1.0, 2.0]), np.array([PI / 3, 2 * PI / 3]), inputs.pfaces(16)
    kr, kt, kp, s = const_fields(1, 1, 16, kappa=1.0, s=0.2)
    op = op_from(oracle_mod, rf, tf, pf, kr, kt, kp, s, 1, 1)
    bb = np.random.default_rng(7).standard_normal(16).reshape(op.shape)
    st, x, iters, *_ = op.pcg(bb, np.zeros(op.shape), 1e-14, 100, variant="cg1")
    assert st == 0 and iters <= 16 // 2 + 1
    st, x, iters, hist, *_ = op.pcg(bb, np.zeros(op.shape), 0.0, 5, variant="cg1")
    assert st == oracle_mod.NOT_CONVERGED and iters == 5 and hist.size == 6
    st, x, iters, *_ = op.pcg(np.zeros(op.shape), bb, 1e-10, 5, variant="cg1")
    assert st == 0 and iters == 0 and not x.any()


# ------------------------------------------------------------------ the -fopenmp timing build (bench.py cpu_baseline)
def test_openmp_build_gives_identical_iterates(oracle_mod):
    """The -fopenmp build that bench.py times on all host cores (cpu_baseline, --impl reference) is the
    same oracle: its per-cell loops only run on several threads and the dot products stay sequential,
    so c1's solve (solution, count and history) is identical bit for bit to the plain build."""
    p = inputs.make_problem("c1")
    a = oracle_mod.solve_problem(p)
    oracle_mod.use_openmp(True)
    try:
        b = oracle_mod.solve_problem(p)
    finally:
        oracle_mod.use_openmp(False)
    assert a["iters"] == b["iters"] == 130
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["hist"], b["hist"])


def test_breakdown_from_an_isolated_singular_pair(oracle_mod):
    """a kappa = 0-isolated pair of cells with s = 0 and no Dirichlet face is a singular
    component the global check cannot see.  With the rhs on the pair only (equal values), z_0 = r_0 / D is
    constant on the pair, A z_0 = 0 exactly (the pair's row is D p - T p with D = T), so p.Ap = 0 in the
    first iteration: E_BREAKDOWN with iters 0 and a finite hist[0] (not a setup failure)."""
    p = inputs.isolated_pair_problem()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    b = op.rhs(p.f)
    z0 = b / op.D
    assert np.count_nonzero(z0) == 2 and z0[2, 2, 3] == z0[3, 2, 3]
    assert not op.apply(z0).any()
    st, x, iters, hist, bn, rn = op.pcg(b, np.zeros(op.shape), 1e-10, 50)
    assert st == oracle_mod.E_BREAKDOWN and iters == 0 and np.isfinite(hist[0]) and hist[0] > 0
