"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no metric, no
transmissibility, no operator, no PCG).  It only produces the caller-side
inputs the C-ABI takes -- face coordinates, face diffusion coefficients, the
shift field, boundary values and the right-hand side -- with the shapes, value
ranges and structure of the paper's coronal workloads:

* "a logically rectangular non-uniform staggered spherical grid"
  (Sec. III), "stretched grid" (Fig. 1);
* a "full thermodynamic MHD" coronal case of 36 M cells (Sec. V-A);
* the five configurations of BASELINE.json ``configs`` with the recipe of
  SURVEY.md section 8(d) ("Generators" and the configs table), restated in
  DESIGN.md section 4.

All arrays are numpy float64, C order ``[k][j][i]`` (phi outermost, r
contiguous).  Every field is a function of GLOBAL coordinates and GLOBAL cell
indices, so a rank's phi-slab ``[k0, k0+nloc)`` is bitwise the corresponding
slice of the global arrays (decomposition independent).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

BC_DIRICHLET = 0
BC_NEUMANN0 = 1

TWO_PI = 2.0 * math.pi


# --------------------------------------------------------------------------- faces
def rfaces(nr: int, r0: float, r1: float, a: float) -> np.ndarray:
    """r_f[i] = r0 + (r1-r0)(e^{a x}-1)/(e^a-1), x = i/nr (a = 0: uniform)."""
    x = np.arange(nr + 1, dtype=np.float64) / nr
    if a == 0.0:
        rf = r0 + (r1 - r0) * x
    else:
        rf = r0 + (r1 - r0) * np.expm1(a * x) / math.expm1(a)
    rf[0], rf[-1] = r0, r1
    return rf


def tfaces(nt: int, eps: float, t0: float = 0.0, t1: float = math.pi) -> np.ndarray:
    """t_f[j] = t0 + (t1-t0)(y + eps sin(2 pi y)/(2 pi)), y = j/nt; eps > 0 refines mid-band."""
    y = np.arange(nt + 1, dtype=np.float64) / nt
    tf = t0 + (t1 - t0) * (y + eps * np.sin(TWO_PI * y) / TWO_PI)
    tf[0], tf[-1] = t0, t1
    return tf


def pfaces(np_: int) -> np.ndarray:
    """Uniform periodic phi faces on [0, 2 pi] (p_f[np] - p_f[0] = 2 pi exactly)."""
    pf = TWO_PI * (np.arange(np_ + 1, dtype=np.float64) / np_)
    pf[0], pf[-1] = 0.0, TWO_PI
    return pf


def midpoints(f: np.ndarray) -> np.ndarray:
    """Coordinates at which cell-centred input fields are sampled."""
    return 0.5 * (f[:-1] + f[1:])


# --------------------------------------------------------------------------- noise
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64 finaliser on uint64 counters (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def white_noise(seed: int, nr: int, nt: int, k0: int, nloc: int) -> np.ndarray:
    """w = uniform[-1, 1) from splitmix64(seed * 2^32 + global linear cell index), top 53 bits."""
    lin = (np.arange(k0, k0 + nloc, dtype=np.uint64)[:, None, None] * np.uint64(nt * nr)
           + np.arange(nt, dtype=np.uint64)[None, :, None] * np.uint64(nr)
           + np.arange(nr, dtype=np.uint64)[None, None, :])
    with np.errstate(over="ignore"):
        ctr = np.uint64(seed) * np.uint64(1 << 32) + lin
    u53 = (splitmix64(ctr) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u53 - 1.0


def angular_field(theta: np.ndarray, phi: np.ndarray, seed: int) -> np.ndarray:
    """G(theta, phi) = sum_{l=1..6} sum_{m=0..l} (a cos m phi + b sin m phi) sin^m cos^{l-m} / l,
    normalised by sum(|a|+|b|)/l so that |G| <= 1; (a, b) drawn in (l, m) order.
    Returns an array of shape (len(phi), len(theta))."""
    rng = np.random.default_rng(seed)
    th = theta[None, :]
    ph = phi[:, None]
    G = np.zeros((phi.size, theta.size))
    norm = 0.0
    for l in range(1, 7):
        for m in range(0, l + 1):
            a, b = rng.standard_normal(2)
            G += (a * np.cos(m * ph) + b * np.sin(m * ph)) * np.sin(th) ** m * np.cos(th) ** (l - m) / l
            norm += (abs(a) + abs(b)) / l
    return G / norm


def rho_hydro(r: np.ndarray) -> np.ndarray:
    """Hydrostatic-like density rho(r) = exp(-14.5 (1 - 1/r)) (1 -> 8e-7 over [1, 30])."""
    return np.exp(-14.5 * (1.0 - 1.0 / r))


def t_profile(r: np.ndarray) -> np.ndarray:
    """Transition-region temperature T(r) = 0.0133 + 0.9867 (1 + tanh((r - 1.03)/0.01))/2."""
    return 0.0133 + 0.9867 * 0.5 * (1.0 + np.tanh((r - 1.03) / 0.01))


# --------------------------------------------------------------------------- problem
@dataclasses.dataclass
class Problem:
    """One rank's share of a generated problem (global grid, local phi-slab fields)."""
    name: str
    nr: int
    nt: int
    np: int
    k0: int
    nloc: int
    rf: np.ndarray
    tf: np.ndarray
    pf: np.ndarray
    kr: np.ndarray          # [nloc][nt][nr+1]
    kt: np.ndarray          # [nloc][nt+1][nr]
    kp: np.ndarray          # [nloc][nt][nr]   face k+1/2
    s: np.ndarray           # [nloc][nt][nr]
    f: np.ndarray           # [nloc][nt][nr]   per-unit-volume rhs
    x0: np.ndarray          # [nloc][nt][nr]
    bc_in: int
    bc_out: int
    g_in: np.ndarray | None  # [nloc][nt] or None (= 0)
    g_out: np.ndarray | None
    tol: float
    maxit: int

    @property
    def ncell_local(self) -> int:
        return self.nloc * self.nt * self.nr

    @property
    def ncell_global(self) -> int:
        return self.np * self.nt * self.nr


CONFIGS = {
    # name: (nr, nt, np) and recipe id (BASELINE.json configs[0..4])
    "c1": (16, 16, 32),
    "c2": (64, 64, 128),
    "c3": (150, 300, 600),
    "c4": (400, 400, 800),      # per GPU; global np = 800 * P
    "c5": (200, 300, 600),
}


def _fields_on_faces(func_rtp, rf, tf, pf, k0, nloc):
    """Evaluate a coefficient kappa(r, theta, phi) at the geometric centre of every face.
    func_rtp(r[None,None,:], th[None,:,None], ph[:,None,None]) -> broadcast array."""
    rc, tc, pc = midpoints(rf), midpoints(tf), midpoints(pf)
    ph_c = pc[k0:k0 + nloc]
    ph_face = pf[k0 + 1:k0 + nloc + 1]          # face k+1/2
    R = lambda r: r[None, None, :]
    T = lambda t: t[None, :, None]
    P = lambda p: p[:, None, None]
    kr = np.broadcast_to(func_rtp(R(rf), T(tc), P(ph_c)), (nloc, tc.size, rf.size)).copy()
    kt = np.broadcast_to(func_rtp(R(rc), T(tf), P(ph_c)), (nloc, tf.size, rc.size)).copy()
    kp = np.broadcast_to(func_rtp(R(rc), T(tc), P(ph_face)), (nloc, tc.size, rc.size)).copy()
    return kr, kt, kp


def make_problem(name: str, k0: int | None = None, nloc: int | None = None, *,
                 nranks: int = 1, shape: tuple[int, int, int] | None = None,
                 x0_seed: int | None = None) -> Problem:
    """Build config ``name`` (c1..c5) for the phi-slab [k0, k0+nloc).

    ``shape`` overrides (nr, nt, np) keeping the recipe (used for reduced-size
    parity cases).  For c4 the global np is 800 * nranks (weak scaling).
    ``x0_seed`` gives a non-zero initial guess 0.1 * w(x0_seed)."""
    if name not in CONFIGS:
        raise ValueError(f"unknown config {name!r}")
    nr, nt, np_ = shape if shape is not None else CONFIGS[name]
    if name == "c4" and shape is None:
        np_ = np_ * nranks
    if k0 is None:
        k0, nloc = 0, np_
    assert nloc is not None and 0 <= k0 and k0 + nloc <= np_
    tol, maxit = 1e-10, 20000
    g_in = g_out = None
    if name == "c1":
        rf, tf, pf = rfaces(nr, 1.0, 2.0, 0.0), tfaces(nt, 0.0), pfaces(np_)
        one = lambda r, t, p: np.ones(np.broadcast_shapes(r.shape, t.shape, p.shape))
        kr, kt, kp = _fields_on_faces(one, rf, tf, pf, k0, nloc)
        s = np.ones((nloc, nt, nr))
        f = 1.0 + 0.5 * white_noise(1, nr, nt, k0, nloc)
        bc_in, bc_out = BC_DIRICHLET, BC_DIRICHLET
    else:
        rf = rfaces(nr, 1.0, 30.0, 4.0 if name == "c2" else 5.33)
        tf, pf = tfaces(nt, 0.1), pfaces(np_)
        rc, tc, pc = midpoints(rf), midpoints(tf), midpoints(pf)
        bc_in, bc_out = BC_DIRICHLET, BC_NEUMANN0
        if name == "c2":
            kap = lambda r, t, p: np.broadcast_to((0.3 + 0.7 * np.exp(-(r - 1.0) / 5.0)) ** 2.5,
                                                  np.broadcast_shapes(r.shape, t.shape, p.shape))
            s = np.full((nloc, nt, nr), 1.0 / 1e-2)
        elif name in ("c3", "c5"):
            nu = 1e-3
            kap = lambda r, t, p: np.broadcast_to(nu * rho_hydro(r),
                                                  np.broadcast_shapes(r.shape, t.shape, p.shape))
            s = np.broadcast_to(rho_hydro(rc)[None, None, :] / 1e-2, (nloc, nt, nr)).copy()
        else:  # c4: high-contrast thermal conduction kappa = (T(r) 10^{0.4 G})^{5/2}
            def kap(r, t, p):
                G = angular_field(t.reshape(-1), p.reshape(-1), 101)[:, :, None]
                return (t_profile(r) * 10.0 ** (0.4 * G)) ** 2.5
            s = np.broadcast_to(rho_hydro(rc)[None, None, :] / 1.0, (nloc, nt, nr)).copy()
            tol, maxit = 0.0, 500
        kr, kt, kp = _fields_on_faces(kap, rf, tf, pf, k0, nloc)
        G1 = angular_field(tc, pc[k0:k0 + nloc], 1)[:, :, None]
        radial = np.exp(-(rc - 1.0) / 5.0)[None, None, :]
        f = s * (1.0 + 0.5 * G1 * radial) + 0.05 * s * white_noise(2, nr, nt, k0, nloc)
    x0 = np.zeros((nloc, nt, nr)) if x0_seed is None else 0.1 * white_noise(x0_seed, nr, nt, k0, nloc)
    return Problem(name, nr, nt, np_, k0, nloc, rf, tf, pf,
                   np.ascontiguousarray(kr), np.ascontiguousarray(kt), np.ascontiguousarray(kp),
                   np.ascontiguousarray(s), np.ascontiguousarray(f), np.ascontiguousarray(x0),
                   bc_in, bc_out, g_in, g_out, tol, maxit)


def slab_extent(np_: int, rank: int, nranks: int) -> tuple[int, int]:
    """phi-slab of ``rank``: [rank*np/P, (rank+1)*np/P); requires np % P == 0."""
    if nranks < 1 or np_ % nranks != 0:
        raise ValueError(f"np={np_} is not divisible by nranks={nranks}")
    nloc = np_ // nranks
    return rank * nloc, nloc


def random_problem(nr: int, nt: int, np_: int, seed: int, *, bc_in=BC_DIRICHLET,
                   bc_out=BC_NEUMANN0, stretched=True, shift=True, k0=0, nloc=None,
                   theta_band: tuple[float, float] | None = None) -> Problem:
    """Small random problem for parity tests: random kappa in [0.5, 2] on faces
    (spatially rough), random s in [0.5, 1.5] (or 0), random rhs and boundary values."""
    nloc = np_ if nloc is None else nloc
    rf = rfaces(nr, 1.0, 3.0, 2.0 if stretched else 0.0)
    tf = tfaces(nt, 0.2 if stretched else 0.0) if theta_band is None else \
        tfaces(nt, 0.0, theta_band[0], theta_band[1])
    pf = pfaces(np_)
    base = seed * 16
    u = lambda s_, shp_r, shp_t: 0.5 * (1.0 + white_noise(base + s_, shp_r, shp_t, k0, nloc))
    kr = 0.5 + 1.5 * u(1, nr + 1, nt)
    kt = 0.5 + 1.5 * u(2, nr, nt + 1)
    kp = 0.5 + 1.5 * u(3, nr, nt)
    s = (0.5 + u(4, nr, nt)) if shift else np.zeros((nloc, nt, nr))
    f = white_noise(base + 5, nr, nt, k0, nloc)
    g_in = white_noise(base + 6, 1, nt, k0, nloc)[:, :, 0].copy() if bc_in == BC_DIRICHLET else None
    g_out = white_noise(base + 7, 1, nt, k0, nloc)[:, :, 0].copy() if bc_out == BC_DIRICHLET else None
    x0 = np.zeros((nloc, nt, nr))
    return Problem(f"rand{seed}", nr, nt, np_, k0, nloc, rf, tf, pf, kr, kt, kp, s, f, x0,
                   bc_in, bc_out, g_in, g_out, 1e-10, 20000)


# --------------------------------------------------------------------------- vector viscosity (NEXT-2)
WALL_NO_SLIP, WALL_FREE_SLIP = 0, 1


@dataclasses.dataclass
class VVProblem:
    """One rank's share of a generated staggered vector-viscosity problem.
    Vectors are [nloc][3][nt][nr] (component 0 r, 1 theta, 2 phi on the LOWER faces of each cell),
    wall data [nloc][3][nt]; the oracle takes the global [np][3][nt][nr] and [3][np][nt]."""
    name: str
    nr: int
    nt: int
    np: int
    k0: int
    nloc: int
    rf: np.ndarray
    tf: np.ndarray
    pf: np.ndarray
    nu: np.ndarray          # [nloc][nt][nr] cell viscosity
    s: np.ndarray           # [nloc][nt][nr] cell shift
    f: np.ndarray           # [nloc][3][nt][nr] per-unit-volume forcing
    x0: np.ndarray          # [nloc][3][nt][nr]
    wall_in: int
    wall_out: int
    g_in: np.ndarray | None  # [nloc][3][nt]
    g_out: np.ndarray | None
    tol: float
    maxit: int

    @property
    def shape(self):
        return (self.nloc, 3, self.nt, self.nr)


VV_CONFIGS = {
    # c3 grid with the viscosity of c3 (BASELINE.json configs[2]) as a staggered vector solve
    "c3v": (150, 300, 600),
    "c2v": (64, 64, 128),
}


def make_vv_problem(name: str, k0: int | None = None, nloc: int | None = None, *,
                    shape: tuple[int, int, int] | None = None, seed: int = 1,
                    wall_in: int = WALL_NO_SLIP, wall_out: int = WALL_FREE_SLIP,
                    x0_seed: int | None = None) -> VVProblem:
    """``rand``: random nu in [0.5, 2] and s in [0.5, 1.5] per cell, white-noise forcing and wall data,
    stretched grid r in [1, 3] (needs ``shape``).  ``c3v`` / ``c2v``: the coronal grid of c3 / c2 with
    nu = 1e-3 rho(r) and s = rho(r)/dt (dt = 1e-2), forcing s (0.5 G_c(theta, phi) e^{-(r-1)/5} + 0.05 w)
    per component (G_c three seeded angular fields), v = 0 on the inner wall, free-slip outer wall."""
    if name == "rand":
        assert shape is not None
        nr, nt, np_ = shape
    else:
        nr, nt, np_ = shape if shape is not None else VV_CONFIGS[name]
    if k0 is None:
        k0, nloc = 0, np_
    assert nloc is not None
    tol, maxit = 1e-10, 20000
    if name == "rand":
        rf, tf, pf = rfaces(nr, 1.0, 3.0, 2.0), tfaces(nt, 0.2), pfaces(np_)
        base = seed * 16
        u = lambda s_: 0.5 * (1.0 + white_noise(base + s_, nr, nt, k0, nloc))
        nu = 0.5 + 1.5 * u(1)
        s = 0.5 + u(2)
        f = np.stack([white_noise(base + 3 + c, nr, nt, k0, nloc) for c in range(3)], axis=1)
        gw = lambda s_: np.stack([white_noise(base + s_ + c, 1, nt, k0, nloc)[:, :, 0] for c in range(3)], axis=1)
        g_in, g_out = gw(8), gw(12)
    else:
        rf = rfaces(nr, 1.0, 30.0, 4.0 if name == "c2v" else 5.33)
        tf, pf = tfaces(nt, 0.1), pfaces(np_)
        rc, tc, pc = midpoints(rf), midpoints(tf), midpoints(pf)
        rho_c = rho_hydro(rc)
        nu = np.broadcast_to(1e-3 * rho_c[None, None, :], (nloc, nt, nr)).copy()
        s = np.broadcast_to(rho_c[None, None, :] / 1e-2, (nloc, nt, nr)).copy()
        pos = [(rf[:-1], tc, pc), (rc, tf[:-1], pc), (rc, tc, pf[:-1])]   # lower-face centres per component
        f = np.empty((nloc, 3, nt, nr))
        for c, (r, t, p) in enumerate(pos):
            G = angular_field(t, p[k0:k0 + nloc], 3 + c)[:, :, None]
            sr = (rho_hydro(r) / 1e-2)[None, None, :]
            f[:, c] = sr * (0.5 * G * np.exp(-(r - 1.0) / 5.0)[None, None, :]
                            + 0.05 * white_noise(20 + c, nr, nt, k0, nloc))
        g_in = g_out = None
    x0 = np.zeros((nloc, 3, nt, nr)) if x0_seed is None else \
        0.1 * np.stack([white_noise(x0_seed + c, nr, nt, k0, nloc) for c in range(3)], axis=1)
    return VVProblem(name, nr, nt, np_, k0, nloc, rf, tf, pf, np.ascontiguousarray(nu), np.ascontiguousarray(s),
                     np.ascontiguousarray(f), np.ascontiguousarray(x0), wall_in, wall_out,
                     None if g_in is None else np.ascontiguousarray(g_in),
                     None if g_out is None else np.ascontiguousarray(g_out), tol, maxit)


# --------------------------------------------------------------------------- field-aligned conduction (NEXT-4)
def b_field(r: np.ndarray, th: np.ndarray, ph: np.ndarray):
    """Unit vector of a coronal-like magnetic field (dipole + open monopole flux + spiral, with a
    non-axisymmetric perturbation; B_r >= (2.5 r - 2)/r^3 > 0 on r >= 1, so no null points):
        B_r = (2 cos th + 2.5 r)/r^3, B_th = sin th (1 + 0.3 cos ph)/r^3, B_ph = -sin th (0.5 r + 0.2 sin 2ph)/r^3.
    Returns (b_r, b_th, b_ph) broadcast over the inputs."""
    r, th, ph = np.broadcast_arrays(r, th, ph)
    Br = (2.0 * np.cos(th) + 2.5 * r) / r ** 3
    Bt = np.sin(th) * (1.0 + 0.3 * np.cos(ph)) / r ** 3
    Bp = -np.sin(th) * (0.5 * r + 0.2 * np.sin(2.0 * ph)) / r ** 3
    n = np.sqrt(Br * Br + Bt * Bt + Bp * Bp)
    return Br / n, Bt / n, Bp / n


@dataclasses.dataclass
class AnisoProblem(Problem):
    """A Problem with field-aligned conduction: kr, kt, kp are the diagonal face coefficients
    kappa_perp + kappa_par b_a^2, and the edge coefficients kappa_par b_a b_b are
    krt [nloc][nt+1][nr+1] (edge r-face ie, theta-face je, plane k), krp [nloc][nt][nr+1] (r-face ie, row j,
    phi face k+1/2), ktp [nloc][nt+1][nr] (theta-face je, column i, phi face k+1/2)."""
    krt: np.ndarray = None
    krp: np.ndarray = None
    ktp: np.ndarray = None


def aniso_coefficients(kpar, kperp, bfun, rf, tf, pf, k0, nloc):
    """kr, kt, kp (kappa_perp + kappa_par b_a^2 at face centres) and krt, krp, ktp (kappa_par b_a b_b at
    edge centres) of the phi-slab [k0, k0 + nloc); kpar(r, th, ph), kperp(r, th, ph), bfun(r, th, ph) ->
    (b_r, b_th, b_ph).  Evaluation only (generator): no method arithmetic."""
    rc, tc, pc = midpoints(rf), midpoints(tf), midpoints(pf)
    phc, phf = pc[k0:k0 + nloc], pf[k0 + 1:k0 + nloc + 1]
    R = lambda r: r[None, None, :]
    T = lambda t: t[None, :, None]
    P = lambda p: p[:, None, None]

    def at(r, t, p, a, b=None):
        shp = np.broadcast_shapes(r.shape, t.shape, p.shape)
        bb = bfun(r, t, p)
        kpa = np.broadcast_to(kpar(r, t, p), shp)
        if b is None:
            return np.broadcast_to(kperp(r, t, p), shp) + kpa * bb[a] * bb[a]
        return kpa * bb[a] * bb[b]

    kr = at(R(rf), T(tc), P(phc), 0)
    kt = at(R(rc), T(tf), P(phc), 1)
    kp = at(R(rc), T(tc), P(phf), 2)
    krt = at(R(rf), T(tf), P(phc), 0, 1)
    krp = at(R(rf), T(tc), P(phf), 0, 2)
    ktp = at(R(rc), T(tf), P(phf), 1, 2)
    c = lambda x: np.ascontiguousarray(x, dtype=np.float64)
    return c(kr), c(kt), c(kp), c(krt), c(krp), c(ktp)


ANISO_CONFIGS = {
    # field-aligned thermal conduction on the grids of BASELINE.json configs[0..2]
    "c1a": (16, 16, 32),
    "c2a": (64, 64, 128),
    "c3a": (150, 300, 600),
}


def make_aniso_problem(name: str, k0: int | None = None, nloc: int | None = None, *,
                       shape: tuple[int, int, int] | None = None) -> AnisoProblem:
    """Field-aligned conduction on the grid of c1 / c2 / c3: kappa_par = (0.3 + 0.7 e^{-(r-1)/5})^{5/2}
    (the T^{5/2} profile of c2) along b_field, an isotropic floor kappa_perp = 1e-2 kappa_par, shift
    s = 1/dt (dt = 1e-2; c1a: s = 1), rhs and boundary conditions as the base config."""
    base = {"c1a": "c1", "c2a": "c2", "c3a": "c3"}[name]
    nr, nt, np_ = shape if shape is not None else ANISO_CONFIGS[name]
    if k0 is None:
        k0, nloc = 0, np_
    p = make_problem(base, k0, nloc, shape=(nr, nt, np_))
    if base == "c1":
        kpar = lambda r, t, p_: np.ones(np.broadcast_shapes(r.shape, t.shape, p_.shape))
        s = np.ones((nloc, nt, nr))
    else:
        kpar = lambda r, t, p_: np.broadcast_to((0.3 + 0.7 * np.exp(-(r - 1.0) / 5.0)) ** 2.5,
                                                np.broadcast_shapes(r.shape, t.shape, p_.shape))
        s = np.full((nloc, nt, nr), 1.0 / 1e-2)
    kperp = lambda r, t, p_: 1e-2 * kpar(r, t, p_)
    kr, kt, kp, krt, krp, ktp = aniso_coefficients(kpar, kperp, b_field, p.rf, p.tf, p.pf, k0, nloc)
    f = p.f if base == "c1" else p.f / p.s * s
    return AnisoProblem(name, nr, nt, np_, k0, nloc, p.rf, p.tf, p.pf, kr, kt, kp, np.ascontiguousarray(s),
                        np.ascontiguousarray(f), p.x0, p.bc_in, p.bc_out, p.g_in, p.g_out, p.tol, p.maxit,
                        krt, krp, ktp)


def random_aniso_problem(nr: int, nt: int, np_: int, seed: int, *, bc_in=BC_DIRICHLET, bc_out=BC_NEUMANN0,
                         k0=0, nloc=None, shift=True) -> AnisoProblem:
    """Small random field-aligned problem for parity tests: rough kappa_par in [0.5, 2] at every face and
    edge (white noise), the smooth b_field, kappa_perp = 0.2, random s in [0.5, 1.5], rhs and wall data."""
    nloc = np_ if nloc is None else nloc
    p = random_problem(nr, nt, np_, seed, bc_in=bc_in, bc_out=bc_out, k0=k0, nloc=nloc, shift=shift)
    rng_seed = seed * 16 + 9

    def rough(r, t, ph):
        shp = np.broadcast_shapes(r.shape, t.shape, ph.shape)
        n = int(np.prod(shp))
        # decomposition-independent: noise indexed by the evaluation point's global coordinates
        key = np.round((np.broadcast_to(r, shp) * 7919.0 + np.broadcast_to(t, shp) * 104729.0 +
                        np.broadcast_to(ph, shp) * 1299709.0) * 1e6).astype(np.uint64).reshape(n)
        w = (splitmix64(key ^ np.uint64(rng_seed)) >> np.uint64(11)).astype(np.float64) / float(1 << 53)
        return (0.5 + 1.5 * w).reshape(shp)

    kperp = lambda r, t, ph: np.full(np.broadcast_shapes(r.shape, t.shape, ph.shape), 0.2)
    kr, kt, kp, krt, krp, ktp = aniso_coefficients(rough, kperp, b_field, p.rf, p.tf, p.pf, k0, nloc)
    return AnisoProblem(f"arand{seed}", nr, nt, np_, k0, nloc, p.rf, p.tf, p.pf, kr, kt, kp, p.s, p.f, p.x0,
                        p.bc_in, p.bc_out, p.g_in, p.g_out, p.tol, p.maxit, krt, krp, ktp)


def isolated_pair_problem(nr: int = 8, nt: int = 6, np_: int = 8, seed: int = 31) -> Problem:
    """A singular connected component the global E_SINGULAR check cannot see: the two
    phi-neighbour cells (k = 2, 3) at (j = 2, i = 3) have kappa = 0 on their 10 outer faces and s = 0, all
    other cells s > 0; the rhs is zero except an equal value on the pair (uniform phi faces give the pair
    equal volumes).  Then p_0 is constant on the pair and A p_0 = 0 exactly: p.Ap = 0 in iteration 1."""
    p = random_problem(nr, nt, np_, seed, bc_in=BC_NEUMANN0, bc_out=BC_NEUMANN0)
    i, j, k = 3, 2, 2
    kr, kt, kp, s = p.kr.copy(), p.kt.copy(), p.kp.copy(), p.s.copy()
    for kk in (k, k + 1):
        kr[kk, j, i] = kr[kk, j, i + 1] = 0.0
        kt[kk, j, i] = kt[kk, j + 1, i] = 0.0
        s[kk, j, i] = 0.0
    kp[k - 1, j, i] = kp[k + 1, j, i] = 0.0     # the pair's outer phi faces; kp[k] (between them) stays > 0
    f = np.zeros_like(p.f)
    f[k, j, i] = f[k + 1, j, i] = 1.0
    return Problem("isolated-pair", nr, nt, np_, 0, np_, p.rf, p.tf, p.pf, kr, kt, kp, s, f, p.x0,
                   BC_NEUMANN0, BC_NEUMANN0, None, None, 1e-10, 100)
