"""Pins of the field-aligned conduction oracle (oracle/masoracle.c, reading R33 of
DESIGN.md section 3) against things other than itself (-m "not gpu").

The thermal-conduction term belongs to MAS's "full thermodynamic MHD model" (Sec. V-A) on
its "non-uniform staggered spherical grid" (Sec. III); the paper gives no formula, so the
operator is reading R33: flux -K grad T with K = kappa_perp I + kappa_par b b^T, the volume-weighted
energy form with the diagonal terms on faces (the 7-point operator of K_aa) and the cross terms on
edges (19 points).  The pins: b = r^ reduces it to the radial 7-point operator; symmetry; constants in
the kernel; its 19-point sparsity; SPD with an isotropic floor; its Jacobi diagonal; PCG against a dense
LU solve; and second-order convergence to a manufactured solution whose source is derived symbolically
(sympy) from the continuous operator -- a dropped cross term, a wrong sign, a wrong metric factor or
a missing 1/4 fails it.
"""
import math

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs


def aniso_op(oracle_mod, p):
    return oracle_mod.AnisoOperator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out, p.krt, p.krp, p.ktp)


def dense(op):
    n = op.np * op.nt * op.nr
    A = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        A[:, c] = op.apply(e.reshape(op.shape)).ravel()
    return A


def with_b(p, bfun, kpar, kperp, s=None):
    """p's grid and boundary data with the coefficients of the field bfun."""
    kr, kt, kp, krt, krp, ktp = inputs.aniso_coefficients(kpar, kperp, bfun, p.rf, p.tf, p.pf, p.k0, p.nloc)
    q = inputs.AnisoProblem(**{**p.__dict__, "kr": kr, "kt": kt, "kp": kp, "krt": krt, "krp": krp, "ktp": ktp})
    if s is not None:
        q.s = s
    return q


const = lambda v: (lambda r, t, ph: np.full(np.broadcast_shapes(r.shape, t.shape, ph.shape), float(v)))


def test_radial_field_is_the_radial_7point_operator(oracle_mod):
    """b = r^ with no floor: no cross terms, kt = kp = 0, and the operator is exactly (bit for bit) the
    7-point operator of kr alone, which decouples into independent radial columns."""
    p = inputs.random_aniso_problem(9, 6, 8, 3)
    radial = lambda r, t, ph: (np.ones(np.broadcast_shapes(r.shape, t.shape, ph.shape)),
                               np.zeros(np.broadcast_shapes(r.shape, t.shape, ph.shape)),
                               np.zeros(np.broadcast_shapes(r.shape, t.shape, ph.shape)))
    kpar = lambda r, t, ph: 1.0 + 0.5 * np.broadcast_to(r, np.broadcast_shapes(r.shape, t.shape, ph.shape))
    q = with_b(p, radial, kpar, const(0.0))
    assert not q.krt.any() and not q.krp.any() and not q.ktp.any()
    assert not q.kt.any() and not q.kp.any()
    A = aniso_op(oracle_mod, q)
    B = oracle_mod.Operator(q.rf, q.tf, q.pf, q.kr, q.kt, q.kp, q.s, q.bc_in, q.bc_out)
    u = inputs.white_noise(77, q.nr, q.nt, 0, q.np)
    assert np.array_equal(A.apply(u), B.apply(u))
    M = dense(A).reshape(q.np, q.nt, q.nr, q.np, q.nt, q.nr)
    for k in range(q.np):
        for j in range(q.nt):
            blk = M[k, j, :, :, :, :].copy()
            blk[:, k, j, :] = 0.0
            assert not blk.any(), "a radial column couples to another column"


@pytest.mark.parametrize("seed,shape", [(1, (7, 6, 5)), (2, (10, 9, 8)), (3, (6, 8, 2))])
def test_symmetric(oracle_mod, seed, shape):
    """x.Ay = y.Ax to 1e-12 (BASELINE.json north_star's symmetry check) with oblique rough fields."""
    p = inputs.random_aniso_problem(*shape, seed)
    A = aniso_op(oracle_mod, p)
    x = inputs.white_noise(100 + seed, p.nr, p.nt, 0, p.np)
    y = inputs.white_noise(200 + seed, p.nr, p.nt, 0, p.np)
    a, b = float(np.dot(x.ravel(), A.apply(y).ravel())), float(np.dot(y.ravel(), A.apply(x).ravel()))
    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b))


def test_annihilates_constants(oracle_mod):
    """s = 0 and zero-flux r walls: K 1 = 0 in every row (the operator's kernel holds the constants),
    relative to the row's absolute sum."""
    p = inputs.random_aniso_problem(8, 7, 6, 4, bc_in=inputs.BC_NEUMANN0, bc_out=inputs.BC_NEUMANN0, shift=True)
    p.s = np.zeros_like(p.s)
    with pytest.raises(oracle_mod.OracleError):   # globally singular: the assembly refuses it
        aniso_op(oracle_mod, p)
    p.s = np.full_like(p.s, 1e-300)               # numerically zero shift, assembly accepted
    A = aniso_op(oracle_mod, p)
    y = A.apply(np.ones(A.shape))
    assert np.abs(y).max() <= 1e-13 * np.abs(A.Dj).max()


def test_19_point_sparsity_and_jacobi_diagonal(oracle_mod):
    """A couples a cell only to its 6 face and 12 edge neighbours (periodic in phi) and every one of the
    12 edge couplings is present in the interior; the Jacobi diagonal Dj is diag(A)."""
    p = inputs.random_aniso_problem(6, 6, 6, 5)
    A = aniso_op(oracle_mod, p)
    M = dense(A)
    nr, nt, np_ = p.nr, p.nt, p.np
    allowed = {(0, 0, 0)} | {o for o in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]}
    allowed |= {(a, b, 0) for a in (-1, 1) for b in (-1, 1)} | {(a, 0, c) for a in (-1, 1) for c in (-1, 1)}
    allowed |= {(0, b, c) for b in (-1, 1) for c in (-1, 1)}
    assert len(allowed) == 19
    idx = lambda k, j, i: (k * nt + j) * nr + i
    for k in range(np_):
        for j in range(nt):
            for i in range(nr):
                row = M[idx(k, j, i)]
                for k2 in range(np_):
                    for j2 in range(nt):
                        for i2 in range(nr):
                            dk = (k2 - k + 1) % np_ - 1
                            off = (i2 - i, j2 - j, dk)
                            v = row[idx(k2, j2, i2)]
                            if off not in allowed:
                                assert v == 0.0, (k, j, i, off)
                if 1 <= i <= nr - 2 and 1 <= j <= nt - 2:
                    for off in allowed - {(0, 0, 0)}:
                        di, dj, dk = off
                        assert row[idx((k + dk) % np_, j + dj, i + di)] != 0.0, off
    d = np.diag(M).reshape(A.shape)
    assert np.allclose(d, A.Dj, rtol=1e-14, atol=0.0)


@pytest.mark.parametrize("name", ["c1a-small", "c2a-small"])
def test_spd_with_isotropic_floor(oracle_mod, name):
    """With the floor kappa_perp > 0 the operator is symmetric positive definite (the condition for CG).
    Without floor and shift it is positive semi-definite on the uniform grid (c1a, the constant-coefficient
    symbol argument of R33); on the stretched grid with a varying field small negative eigenvalues can
    appear (R33 notes it; the floor or the implicit shift removes them), so there only their size is
    bounded."""
    shape = (6, 8, 8)
    p = inputs.make_aniso_problem(name.split("-")[0], shape=shape)
    M = dense(aniso_op(oracle_mod, p))
    assert np.allclose(M, M.T, rtol=0, atol=1e-13 * np.abs(M).max())
    w = np.linalg.eigvalsh(0.5 * (M + M.T))
    assert w.min() > 0.0
    kpar = lambda r, t, ph: np.ones(np.broadcast_shapes(r.shape, t.shape, ph.shape))
    q = with_b(p, inputs.b_field, kpar, const(0.0), s=np.full_like(p.s, 1e-300))
    q.bc_in = q.bc_out = inputs.BC_NEUMANN0
    M0 = dense(aniso_op(oracle_mod, q))
    w0 = np.linalg.eigvalsh(0.5 * (M0 + M0.T))
    if name.startswith("c1a"):
        assert w0.min() >= -1e-12 * w0.max()
    else:
        assert w0.min() >= -2e-3 * w0.max()


@pytest.mark.parametrize("seed,shape,bcs", [(6, (5, 6, 4), (0, 1)), (7, (4, 5, 6), (0, 0)), (8, (6, 4, 3), (1, 0))])
def test_pcg_matches_dense_lu(oracle_mod, seed, shape, bcs):
    """PCG to 1e-14 equals the dense LU solution of the assembled 19-point system to 1e-11."""
    p = inputs.random_aniso_problem(*shape, seed, bc_in=bcs[0], bc_out=bcs[1])
    A = aniso_op(oracle_mod, p)
    b = A.rhs(p.f, p.g_in, p.g_out)
    st, x, iters, hist, bn, rn = A.pcg(b, np.zeros(A.shape), 1e-14, 2000)
    assert st == 0
    xd = np.linalg.solve(dense(A), b.ravel()).reshape(A.shape)
    assert np.linalg.norm(x - xd) <= 1e-11 * np.linalg.norm(xd)


# ------------------------------------------------------------------ manufactured solution (second order)
TH0 = 0.4
LB = math.pi - 2 * TH0


def mms_functions():
    """Exact T, the field b (radial at both r walls, b_theta = 0 on both theta edges of the band), the
    coefficients and the source f = s T - div(K grad T) in spherical coordinates, derived with sympy."""
    sp = pytest.importorskip("sympy")
    r, t, ph = sp.symbols("r t ph", positive=True)
    T = sp.exp(-r) * (2 + sp.cos(2 * sp.pi * (t - TH0) / LB)) * (1 + sp.Rational(3, 10) * sp.cos(ph))
    al = sp.Rational(6, 10) * sp.sin(sp.pi * (r - 1)) ** 2
    be = sp.pi / 2 + sp.Rational(1, 2) * sp.sin(2 * sp.pi * (t - TH0) / LB)
    b = [sp.cos(al), sp.sin(al) * sp.cos(be), sp.sin(al) * sp.sin(be)]
    kpar = 1 + r / 2
    kperp = sp.Rational(1, 20)
    g = [sp.diff(T, r), sp.diff(T, t) / r, sp.diff(T, ph) / (r * sp.sin(t))]
    bg = sum(bi * gi for bi, gi in zip(b, g))
    F = [kperp * g[a] + kpar * b[a] * bg for a in range(3)]
    div = (sp.diff(r ** 2 * F[0], r) / r ** 2 + sp.diff(sp.sin(t) * F[1], t) / (r * sp.sin(t))
           + sp.diff(F[2], ph) / (r * sp.sin(t)))
    f = T - div   # s = 1
    lam = lambda e: sp.lambdify((r, t, ph), e, "numpy")
    bfun_c = [lam(bi) for bi in b]
    bfun = lambda R, Th, P: tuple(np.broadcast_to(fn(R, Th, P), np.broadcast_shapes(R.shape, Th.shape, P.shape))
                                  for fn in bfun_c)
    kp_f = lam(kpar)
    kpar_fn = lambda R, Th, P: np.broadcast_to(kp_f(R, Th, P), np.broadcast_shapes(R.shape, Th.shape, P.shape))
    return lam(T), lam(f), bfun, kpar_fn, float(kperp)


def mms_errors(oracle_mod, n, fns):
    Tex, fex, bfun, kpar, kperp = fns
    nr, nt, np_ = n, n, 2 * n
    rf = inputs.rfaces(nr, 1.0, 2.0, 0.0)
    tf = inputs.tfaces(nt, 0.0, TH0, math.pi - TH0)
    pf = inputs.pfaces(np_)
    rc, tc, pc = inputs.midpoints(rf), inputs.midpoints(tf), inputs.midpoints(pf)
    kr, kt, kp, krt, krp, ktp = inputs.aniso_coefficients(kpar, const(kperp), bfun, rf, tf, pf, 0, np_)
    R, Th, P = rc[None, None, :], tc[None, :, None], pc[:, None, None]
    f = np.broadcast_to(fex(R, Th, P), (np_, nt, nr)).copy()
    s = np.ones((np_, nt, nr))
    g_in = np.broadcast_to(Tex(1.0, tc[None, :], pc[:, None]), (np_, nt)).copy()
    g_out = np.broadcast_to(Tex(2.0, tc[None, :], pc[:, None]), (np_, nt)).copy()
    A = oracle_mod.AnisoOperator(rf, tf, pf, kr, kt, kp, s, 0, 0, krt, krp, ktp)
    b = A.rhs(f, g_in, g_out)
    st, x, iters, hist, bn, rn = A.pcg(b, np.zeros(A.shape), 1e-13, 20000)
    assert st == 0
    ex = np.broadcast_to(Tex(R, Th, P), (np_, nt, nr))
    V = oracle_mod.volumes(rf, tf, pf)
    e = x - ex
    return math.sqrt((V * e * e).sum() / (V * ex * ex).sum()), np.abs(e).max()


def test_manufactured_solution_second_order(oracle_mod):
    """Oblique field with all three cross terms active (b_r b_theta, b_r b_phi, b_theta b_phi != 0 inside the
    band): the volume-weighted L2 and max errors fall by about 4 per refinement (order >= 1.8)."""
    fns = mms_functions()
    errs = [mms_errors(oracle_mod, n, fns) for n in (8, 16, 32)]
    for (l2a, lia), (l2b, lib) in zip(errs, errs[1:]):
        assert math.log2(l2a / l2b) >= 1.8, errs
        assert math.log2(lia / lib) >= 1.7, errs


def test_manufactured_solution_fails_without_cross_terms(oracle_mod):
    """Sanity of the pin above: dropping the cross terms (the 7-point operator of K_aa alone) leaves an
    O(1) error that does not converge."""
    fns = mms_functions()
    Tex, fex, bfun, kpar, kperp = fns
    n = 16
    nr, nt, np_ = n, n, 2 * n
    rf, tf, pf = inputs.rfaces(nr, 1.0, 2.0, 0.0), inputs.tfaces(nt, 0.0, TH0, math.pi - TH0), inputs.pfaces(np_)
    rc, tc, pc = inputs.midpoints(rf), inputs.midpoints(tf), inputs.midpoints(pf)
    kr, kt, kp, krt, krp, ktp = inputs.aniso_coefficients(kpar, const(kperp), bfun, rf, tf, pf, 0, np_)
    R, Th, P = rc[None, None, :], tc[None, :, None], pc[:, None, None]
    f = np.broadcast_to(fex(R, Th, P), (np_, nt, nr)).copy()
    g_in = np.broadcast_to(Tex(1.0, tc[None, :], pc[:, None]), (np_, nt)).copy()
    g_out = np.broadcast_to(Tex(2.0, tc[None, :], pc[:, None]), (np_, nt)).copy()
    A = oracle_mod.Operator(rf, tf, pf, kr, kt, kp, np.ones((np_, nt, nr)), 0, 0)
    b = A.rhs(f, g_in, g_out)
    st, x, *_ = A.pcg(b, np.zeros(A.shape), 1e-13, 20000)
    ex = np.broadcast_to(Tex(R, Th, P), (np_, nt, nr))
    l2, _ = mms_errors(oracle_mod, n, fns)
    assert np.linalg.norm(x - ex) / np.linalg.norm(ex) > 20 * l2
