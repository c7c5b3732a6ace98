"""ctypes wrapper for the CPU oracle (oracle/masoracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2303_03398_b200`` never imports it.

The oracle is a plain, slow, single-threaded C implementation of the PCG solve
described in SURVEY.md section 8(c) (readings R1-R18):
global grid, host arrays, no ranks, no blocking or fusion.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "masoracle.c")
SRC_VV = os.path.join(HERE, "masoracle_vv.c")   # staggered vector viscosity
LIB = os.path.join(HERE, "libmasoracle.so")
# The same sources built with -fopenmp: the per-cell loops of apply and of the PCG vector updates run on
# all host cores (identical values; dot products stay sequential).  Used only to time the oracle as a
# CPU baseline on the GPU box (bench.py cpu_baseline, --impl reference), never as a checker.
LIB_OMP = os.path.join(HERE, "libmasoracle_omp.so")

OK, NOT_CONVERGED, E_INVALID, E_SINGULAR, E_BREAKDOWN, E_NOMEM = 0, 1, -1, -3, -4, -7
BC_DIRICHLET, BC_NEUMANN0 = 0, 1

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c99"]


def build(force: bool = False, openmp: bool = False) -> str:
    """Compile libmasoracle.so with gcc (plain C99, no contraction, no fast-math); openmp: the
    -fopenmp timing build libmasoracle_omp.so of the same sources."""
    out = LIB_OMP if openmp else LIB
    newest = max(os.path.getmtime(SRC), os.path.getmtime(SRC_VV), os.path.getmtime(__file__))
    if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
        tmp = out + f".tmp{os.getpid()}"
        extra = ["-fopenmp"] if openmp else []
        subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", tmp, SRC, SRC_VV, "-lm"])
        os.replace(tmp, out)
    return out


_libs = {}
_openmp = False


def use_openmp(on: bool) -> None:
    """Select the -fopenmp build for the following calls (bench.py's CPU timings only)."""
    global _openmp
    _openmp = bool(on)


def lib():
    key = _openmp
    if key not in _libs:
        _lib = ctypes.CDLL(build(openmp=key))
        d, i = ctypes.c_void_p, ctypes.c_int
        for name, args in {
            "masoracle_check_grid": [i, i, i, d, d, d],
            "masoracle_volumes": [i, i, i, d, d, d, d],
            "masoracle_assemble": [i, i, i, d, d, d, d, d, d, d, i, i, d, d, d, d],
            "masoracle_apply": [i, i, i, d, d, d, d, d, d],
            "masoracle_rhs": [i, i, i, d, d, d, d, d, i, d, i, d, d],
            "masoracle_pcg": [i, i, i, d, d, d, d, d, d, ctypes.c_double, i, d, d, d, d],
            "masoracle_face_coefficients": [i, i, i, d, ctypes.c_double, i, i, d, ctypes.c_double, d, d, d, d],
            "masoracle_rkl2_step": [i, i, i, d, d, d, d, d, d, d, d, ctypes.c_double, i, d],
            "masoracle_pcg_cg1": [i, i, i, d, d, d, d, d, d, ctypes.c_double, i, d, d, d, d],
            "masoracle_aniso_edges": [i, i, i, d, d, d, d, d, d, d, d, d],
            "masoracle_aniso_apply": [i, i, i, d, d, d, d, d, d, d, d, d],
            "masoracle_aniso_diag": [i, i, i, d, d, d, d, d],
            "masoracle_aniso_pcg": [i, i, i, d, d, d, d, d, d, d, d, d, d, ctypes.c_double, i, d, d, d, d],
            "masoracle_vv_check_grid": [i, i, i, d, d, d],
            "masoracle_vv_coefficients": [i, i, i, d, d, d, d, d, i, i, d, d, d, d, d, d, d],
            "masoracle_vv_div": [i, i, i, d, d, d, d, d, d, d],
            "masoracle_vv_curl": [i, i, i, d, d, d, d, d, d, d, d, d, d, d],
            "masoracle_vv_apply": [i, i, i, d, d, d, d, d, d, d, d, d, d, d, d, d, d],
            "masoracle_vv_diag": [i, i, i, d, d, d, d, d, d, d, d, d, d, d],
            "masoracle_vv_mass": [i, i, i, d, d, d, d],
            "masoracle_vv_rhs": [i, i, i, d, d, d, d, d, d, d, d, d, d, d, d, d, d],
            "masoracle_vv_pcg": [i, i, i, d, d, d, d, d, d, d, d, d, d, d, d, d, ctypes.c_double, i, d, d, d, d],
        }.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = i
        _libs[key] = _lib
    return _libs[key]


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: status {status}")
        self.status = status


def check_grid(rf, tf, pf) -> int:
    rf, tf, pf = _c(rf), _c(tf), _c(pf)
    return lib().masoracle_check_grid(rf.size - 1, tf.size - 1, pf.size - 1, _p(rf), _p(tf), _p(pf))


def volumes(rf, tf, pf) -> np.ndarray:
    rf, tf, pf = _c(rf), _c(tf), _c(pf)
    nr, nt, np_ = rf.size - 1, tf.size - 1, pf.size - 1
    V = np.empty((np_, nt, nr))
    st = lib().masoracle_volumes(nr, nt, np_, _p(rf), _p(tf), _p(pf), _p(V))
    if st:
        raise OracleError(st, "volumes")
    return V


def face_coefficients(field, kappa0, half_power, mean, rho=None, inv_dt=1.0):
    """(kr, kt, kp, s) of the global grid from a cell field (NEXT-1, reading R25)."""
    field = _c(field)
    np_, nt, nr = field.shape
    kr = np.empty((np_, nt, nr + 1))
    kt = np.empty((np_, nt + 1, nr))
    kp = np.empty((np_, nt, nr))
    s = np.empty((np_, nt, nr))
    st = lib().masoracle_face_coefficients(nr, nt, np_, _p(field), float(kappa0), int(half_power), int(mean),
                                           _p(_c(rho)), float(inv_dt), _p(kr), _p(kt), _p(kp), _p(s))
    if st:
        raise OracleError(st, "face_coefficients")
    return kr, kt, kp, s


class Operator:
    """Assembled oracle operator: Tr [np][nt][nr+1], Tt [np][nt+1][nr], Tp [np][nt][nr], D."""

    def __init__(self, rf, tf, pf, kr, kt, kp, s, bc_in, bc_out):
        self.rf, self.tf, self.pf = _c(rf), _c(tf), _c(pf)
        self.nr, self.nt, self.np = self.rf.size - 1, self.tf.size - 1, self.pf.size - 1
        nr, nt, np_ = self.nr, self.nt, self.np
        self.bc_in, self.bc_out = int(bc_in), int(bc_out)
        kr, kt, kp, s = _c(kr), _c(kt), _c(kp), _c(s)
        assert kr.shape == (np_, nt, nr + 1) and kt.shape == (np_, nt + 1, nr)
        assert kp.shape == (np_, nt, nr) and s.shape == (np_, nt, nr)
        self.Tr = np.empty((np_, nt, nr + 1))
        self.Tt = np.empty((np_, nt + 1, nr))
        self.Tp = np.empty((np_, nt, nr))
        self.D = np.empty((np_, nt, nr))
        self.status = lib().masoracle_assemble(
            nr, nt, np_, _p(self.rf), _p(self.tf), _p(self.pf), _p(kr), _p(kt), _p(kp), _p(s),
            self.bc_in, self.bc_out, _p(self.Tr), _p(self.Tt), _p(self.Tp), _p(self.D))
        if self.status:
            raise OracleError(self.status, "assemble")

    @property
    def shape(self):
        return (self.np, self.nt, self.nr)

    def apply(self, u) -> np.ndarray:
        u = _c(u)
        assert u.shape == self.shape
        y = np.empty(self.shape)
        lib().masoracle_apply(self.nr, self.nt, self.np, _p(self.Tr), _p(self.Tt), _p(self.Tp),
                              _p(self.D), _p(u), _p(y))
        return y

    def rhs(self, f, g_in=None, g_out=None) -> np.ndarray:
        f = _c(f)
        b = np.empty(self.shape)
        st = lib().masoracle_rhs(self.nr, self.nt, self.np, _p(self.rf), _p(self.tf), _p(self.pf),
                                 _p(self.Tr), _p(f), self.bc_in, _p(_c(g_in)), self.bc_out,
                                 _p(_c(g_out)), _p(b))
        if st:
            raise OracleError(st, "rhs")
        return b

    def rkl2_step(self, u, s, tau, stages, g_in=None, g_out=None):
        """One RKL2 super-time-step of V du/dt = b_D - K u (NEXT-4, reading R26); s = the shift the
        operator was assembled with (K = A - diag(s V))."""
        V = volumes(self.rf, self.tf, self.pf)
        sV = _c(s) * V
        bD = self.rhs(np.zeros(self.shape), g_in, g_out)
        u = _c(u)
        out = np.empty(self.shape)
        st = lib().masoracle_rkl2_step(self.nr, self.nt, self.np, _p(self.Tr), _p(self.Tt), _p(self.Tp),
                                       _p(self.D), _p(sV), _p(V), _p(bD), _p(u), float(tau), int(stages), _p(out))
        if st:
            raise OracleError(st, "rkl2_step")
        return out

    def pcg(self, b, x0, tol, maxit, variant="hs"):
        """Returns (status, x, iters, hist[0..iters], bnorm, rnorm).  variant "hs": the Hestenes-Stiefel
        PCG of SURVEY 8(c) item 7; "cg1": the single-reduction Chronopoulos-Gear variant (R32)."""
        b = _c(b)
        x = np.array(_c(x0), copy=True)
        hist = np.zeros(maxit + 1)
        iters = ctypes.c_int(0)
        bn, rn = ctypes.c_double(0), ctypes.c_double(0)
        fn = lib().masoracle_pcg if variant == "hs" else lib().masoracle_pcg_cg1
        st = fn(self.nr, self.nt, self.np, _p(self.Tr), _p(self.Tt), _p(self.Tp),
                                 _p(self.D), _p(b), _p(x), float(tol), int(maxit), _p(hist),
                                 ctypes.byref(iters), ctypes.byref(bn), ctypes.byref(rn))
        return st, x, iters.value, hist[: iters.value + 1].copy(), bn.value, rn.value


def solve_problem(prob, tol=None, maxit=None, x0=None, variant="hs"):
    """Solve an ``inputs.Problem`` covering the whole global grid (k0 = 0, nloc = np)."""
    assert prob.k0 == 0 and prob.nloc == prob.np, "the oracle works on the global grid"
    op = Operator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in, prob.bc_out)
    b = op.rhs(prob.f, prob.g_in, prob.g_out)
    st, x, iters, hist, bn, rn = op.pcg(b, prob.x0 if x0 is None else x0,
                                        prob.tol if tol is None else tol,
                                        prob.maxit if maxit is None else maxit, variant)
    return dict(status=st, x=x, iters=iters, hist=hist, bnorm=bn, rnorm=rn, op=op, b=b)


# ----------------------------------------------------------------------------------------------
# Field-aligned anisotropic conduction (masoracle.c, R33)
class AnisoOperator(Operator):
    """The 19-point field-aligned operator: the 7-point operator of the diagonal face coefficients
    kr, kt, kp (kappa_perp + kappa_par b_a^2) plus the cross terms of the edge coefficients
    krt [np][nt+1][nr+1], krp [np][nt][nr+1], ktp [np][nt+1][nr] (kappa_par b_a b_b at edge centres)."""

    def __init__(self, rf, tf, pf, kr, kt, kp, s, bc_in, bc_out, krt, krp, ktp):
        super().__init__(rf, tf, pf, kr, kt, kp, s, bc_in, bc_out)
        nr, nt, np_ = self.nr, self.nt, self.np
        krt, krp, ktp = _c(krt), _c(krp), _c(ktp)
        assert krt.shape == (np_, nt + 1, nr + 1) and krp.shape == (np_, nt, nr + 1)
        assert ktp.shape == (np_, nt + 1, nr)
        self.Xrt = np.empty((np_, nt + 1, nr + 1))
        self.Xrp = np.empty((np_, nt, nr + 1))
        self.Xtp = np.empty((np_, nt + 1, nr))
        st = lib().masoracle_aniso_edges(nr, nt, np_, _p(self.rf), _p(self.tf), _p(self.pf), _p(krt), _p(krp),
                                         _p(ktp), _p(self.Xrt), _p(self.Xrp), _p(self.Xtp))
        if st:
            raise OracleError(st, "aniso_edges")
        self.D7 = self.D
        self.Dj = np.empty(self.shape)
        lib().masoracle_aniso_diag(nr, nt, np_, _p(self.D7), _p(self.Xrt), _p(self.Xrp), _p(self.Xtp), _p(self.Dj))

    def _ptrs(self):
        return (_p(self.Tr), _p(self.Tt), _p(self.Tp), _p(self.D7), _p(self.Xrt), _p(self.Xrp), _p(self.Xtp))

    def apply(self, u) -> np.ndarray:
        u = _c(u)
        assert u.shape == self.shape
        y = np.empty(self.shape)
        lib().masoracle_aniso_apply(self.nr, self.nt, self.np, *self._ptrs(), _p(u), _p(y))
        return y

    def pcg(self, b, x0, tol, maxit, variant="hs"):
        assert variant == "hs"
        b = _c(b)
        x = np.array(_c(x0), copy=True)
        hist = np.zeros(maxit + 1)
        iters = ctypes.c_int(0)
        bn, rn = ctypes.c_double(0), ctypes.c_double(0)
        st = lib().masoracle_aniso_pcg(self.nr, self.nt, self.np, *self._ptrs(), _p(self.Dj), _p(b), _p(x),
                                       float(tol), int(maxit), _p(hist), ctypes.byref(iters), ctypes.byref(bn),
                                       ctypes.byref(rn))
        return st, x, iters.value, hist[: iters.value + 1].copy(), bn.value, rn.value


def solve_aniso_problem(prob, tol=None, maxit=None, x0=None):
    """Solve an ``inputs.AnisoProblem`` covering the whole global grid."""
    assert prob.k0 == 0 and prob.nloc == prob.np, "the oracle works on the global grid"
    op = AnisoOperator(prob.rf, prob.tf, prob.pf, prob.kr, prob.kt, prob.kp, prob.s, prob.bc_in, prob.bc_out,
                       prob.krt, prob.krp, prob.ktp)
    b = op.rhs(prob.f, prob.g_in, prob.g_out)
    st, x, iters, hist, bn, rn = op.pcg(b, prob.x0 if x0 is None else x0, prob.tol if tol is None else tol,
                                        prob.maxit if maxit is None else maxit)
    return dict(status=st, x=x, iters=iters, hist=hist, bnorm=bn, rnorm=rn, op=op, b=b)


# ----------------------------------------------------------------------------------------------
# Staggered vector viscosity (oracle/masoracle_vv.c, R27-R31)
NO_SLIP, FREE_SLIP = 0, 1


class VVOperator:
    """Vector viscosity operator of the global grid: s v + curl(nu curl v) - grad(nu div v) on the
    staggered (MAC) spherical grid with the polar-axis ring treatment.  Vectors are [np][3][nt][nr]
    (lower faces; component 0 r, 1 theta, 2 phi); wall data [3][np][nt] or None."""

    def __init__(self, rf, tf, pf, nu, s, bc_in=NO_SLIP, bc_out=NO_SLIP):
        self.rf, self.tf, self.pf = _c(rf), _c(tf), _c(pf)
        self.nr, self.nt, self.np = self.rf.size - 1, self.tf.size - 1, self.pf.size - 1
        nr, nt, np_ = self.nr, self.nt, self.np
        self.bc_in, self.bc_out = int(bc_in), int(bc_out)
        nu, s = _c(nu), _c(s)
        assert nu.shape == (np_, nt, nr) and s.shape == (np_, nt, nr)
        self.wc = np.empty((np_, nt, nr))
        self.Wr = np.empty((np_, nt, nr))
        self.Wt = np.empty((np_, nt, nr + 1))
        self.Wp = np.empty((np_, nt, nr + 1))
        self.WN = np.empty(nr)
        self.WS = np.empty(nr)
        self.sM = np.empty((np_, 3, nt, nr))
        st = lib().masoracle_vv_coefficients(nr, nt, np_, *self._g(), _p(nu), _p(s), self.bc_in, self.bc_out,
                                             _p(self.wc), _p(self.Wr), _p(self.Wt), _p(self.Wp), _p(self.WN),
                                             _p(self.WS), _p(self.sM))
        if st:
            raise OracleError(st, "vv_coefficients")
        self.D = np.empty((np_, 3, nt, nr))
        st = lib().masoracle_vv_diag(nr, nt, np_, *self._g(), *self._co(), _p(self.D))
        if st:
            raise OracleError(st, "vv_diag")

    def _g(self):
        return _p(self.rf), _p(self.tf), _p(self.pf)

    def _co(self):
        return (_p(self.wc), _p(self.Wr), _p(self.Wt), _p(self.Wp), _p(self.WN), _p(self.WS), _p(self.sM))

    @property
    def shape(self):
        return (self.np, 3, self.nt, self.nr)

    def unknown_mask(self):
        m = np.ones(self.shape, dtype=bool)
        m[:, 0, :, 0] = False
        m[:, 1, 0, :] = False
        return m

    def apply(self, v, g_in=None, g_out=None) -> np.ndarray:
        v = _c(v)
        assert v.shape == self.shape
        y = np.empty(self.shape)
        st = lib().masoracle_vv_apply(self.nr, self.nt, self.np, *self._g(), *self._co(), _p(v), _p(_c(g_in)),
                                      _p(_c(g_out)), _p(y))
        if st:
            raise OracleError(st, "vv_apply")
        return y

    def mass(self) -> np.ndarray:
        M = np.empty(self.shape)
        st = lib().masoracle_vv_mass(self.nr, self.nt, self.np, *self._g(), _p(M))
        if st:
            raise OracleError(st, "vv_mass")
        return M

    def rhs(self, f, g_in=None, g_out=None) -> np.ndarray:
        f = _c(f)
        b = np.empty(self.shape)
        st = lib().masoracle_vv_rhs(self.nr, self.nt, self.np, *self._g(), *self._co(), _p(f), _p(_c(g_in)),
                                    _p(_c(g_out)), _p(b))
        if st:
            raise OracleError(st, "vv_rhs")
        return b

    def pcg(self, b, x0, tol, maxit):
        """Returns (status, x, iters, hist[0..iters], bnorm, rnorm)."""
        b = _c(b)
        x = np.array(_c(x0), copy=True)
        hist = np.zeros(maxit + 1)
        iters = ctypes.c_int(0)
        bn, rn = ctypes.c_double(0), ctypes.c_double(0)
        st = lib().masoracle_vv_pcg(self.nr, self.nt, self.np, *self._g(), *self._co(), _p(self.D), _p(b), _p(x),
                                    float(tol), int(maxit), _p(hist), ctypes.byref(iters), ctypes.byref(bn),
                                    ctypes.byref(rn))
        return st, x, iters.value, hist[: iters.value + 1].copy(), bn.value, rn.value


def vv_check_grid(rf, tf, pf) -> int:
    rf, tf, pf = _c(rf), _c(tf), _c(pf)
    return lib().masoracle_vv_check_grid(rf.size - 1, tf.size - 1, pf.size - 1, _p(rf), _p(tf), _p(pf))


def vv_div(rf, tf, pf, v, g_in=None, g_out=None) -> np.ndarray:
    """Net outflow delta [np][nt][nr] of a face vector v [np][3][nt][nr]."""
    rf, tf, pf, v = _c(rf), _c(tf), _c(pf), _c(v)
    nr, nt, np_ = rf.size - 1, tf.size - 1, pf.size - 1
    out = np.empty((np_, nt, nr))
    st = lib().masoracle_vv_div(nr, nt, np_, _p(rf), _p(tf), _p(pf), _p(v), _p(_c(g_in)), _p(_c(g_out)), _p(out))
    if st:
        raise OracleError(st, "vv_div")
    return out


def vv_curl(rf, tf, pf, v, g_in=None, g_out=None):
    """Circulations (Gr [np][nt][nr], GN [nr], GS [nr], Gt [np][nt][nr+1], Gp [np][nt][nr+1])."""
    rf, tf, pf, v = _c(rf), _c(tf), _c(pf), _c(v)
    nr, nt, np_ = rf.size - 1, tf.size - 1, pf.size - 1
    Gr = np.empty((np_, nt, nr))
    GN, GS = np.empty(nr), np.empty(nr)
    Gt = np.empty((np_, nt, nr + 1))
    Gp = np.empty((np_, nt, nr + 1))
    st = lib().masoracle_vv_curl(nr, nt, np_, _p(rf), _p(tf), _p(pf), _p(v), _p(_c(g_in)), _p(_c(g_out)), _p(Gr),
                                 _p(GN), _p(GS), _p(Gt), _p(Gp))
    if st:
        raise OracleError(st, "vv_curl")
    return Gr, GN, GS, Gt, Gp


def vv_solve(rf, tf, pf, nu, s, f, x0, tol, maxit, bc_in=NO_SLIP, bc_out=NO_SLIP, g_in=None, g_out=None):
    op = VVOperator(rf, tf, pf, nu, s, bc_in, bc_out)
    b = op.rhs(f, g_in, g_out)
    st, x, iters, hist, bn, rn = op.pcg(b, x0, tol, maxit)
    return dict(status=st, x=x, iters=iters, hist=hist, bnorm=bn, rnorm=rn, op=op, b=b)


def vv_solve_problem(prob, tol=None, maxit=None, x0=None):
    """Solve an ``inputs.VVProblem`` covering the whole global grid (k0 = 0, nloc = np); the wall data
    [np][3][nt] are passed to the oracle in its [3][np][nt] layout."""
    assert prob.k0 == 0 and prob.nloc == prob.np, "the oracle works on the global grid"
    T = lambda g: None if g is None else np.ascontiguousarray(np.transpose(g, (1, 0, 2)))
    return vv_solve(prob.rf, prob.tf, prob.pf, prob.nu, prob.s, prob.f, prob.x0 if x0 is None else x0,
                    prob.tol if tol is None else tol, prob.maxit if maxit is None else maxit,
                    prob.wall_in, prob.wall_out, T(prob.g_in), T(prob.g_out))
