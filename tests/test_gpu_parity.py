"""GPU parity of libmaspcg (through the C ABI) against the CPU oracle (-m gpu).

Contract (BASELINE.json north_star; SURVEY.md 8(c) "Proposed parity contract";
DESIGN.md section 6):
  * operator (face transmissibilities T and diagonal D): bit-identical -- both
    sides evaluate the same formulas with one IEEE rounding per operation;
  * y = A x: per cell |y_gpu - y_orc| <= 1e-14 * (D|x| + sum T|x_nb|) (the
    stencil is summed in a different order with FMA);
  * solve: solution relative L2 <= 1e-10, iteration count equal +-1, residual
    history max_k |h_gpu - h_orc| / h_orc <= 1e-10 (all k; every case here
    needs < 1000 iterations, the regime where the history is pinned).
Inputs are the seeded generators of paper_2303_03398_b200/inputs.py.
"""
import math

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = pytest.mark.gpu

SOL_TOL = 1e-10
HIST_TOL = 1e-10
APPLY_TOL = 1e-14


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_2303_03398_b200 import build
    build.build()
    return torch


@pytest.fixture(scope="module")
def M(torch_cuda):
    from paper_2303_03398_b200 import maspcg
    return maspcg


def dev(torch, a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_solve(torch, M, prob, tol=None, maxit=None, chunk=16, x0=None, opts=None):
    S = M.solver_for_problem(prob, chunk=chunk)
    for k, v in (opts or {}).items():
        S.set_option(k, v)
    x = dev(torch, prob.x0 if x0 is None else x0)
    st, info, hist = S.solve(dev(torch, prob.f), x, prob.tol if tol is None else tol,
                             prob.maxit if maxit is None else maxit, raise_on_error=False)
    torch.cuda.synchronize()
    return st, info, hist, x.cpu().numpy(), S


def assert_solve_parity(g, o, exact=True):
    """The tolerance contract; with exact=True (the default arithmetic, MASPCG_OPT_ARITH = 0, R24)
    also the stronger property that the iterates are the oracle's bit for bit."""
    st, info, hist, x, _ = g
    if exact:
        assert info["iters"] == o["iters"]
        assert np.array_equal(hist, o["hist"]), np.abs(hist - o["hist"]).max()
        assert np.array_equal(x, o["x"]), np.abs(x - o["x"]).max()
    assert st == o["status"], (st, o["status"])
    assert abs(info["iters"] - o["iters"]) <= 1, (info["iters"], o["iters"])
    nx = np.linalg.norm(o["x"])
    assert np.linalg.norm(x - o["x"]) <= SOL_TOL * max(nx, 1e-300), np.linalg.norm(x - o["x"]) / nx
    assert_hist(hist, o["hist"], o["bnorm"])
    assert info["bnorm"] == pytest.approx(o["bnorm"], rel=1e-13)


def assert_hist(hist, ohist, bn):
    """History parity: relative 1e-10 on every entry above the rounding floor 1e-12 ||b||;
    entries below it (a tiny system solved to machine precision) agree to 1e-12 ||b|| absolute."""
    k = min(hist.size, ohist.size)
    h, o = hist[:k], ohist[:k]
    floor = 1e-12 * bn
    big = o >= floor
    rel = np.abs(h[big] - o[big]) / o[big]
    assert rel.size == 0 or rel.max() <= HIST_TOL, (rel.max(), int(np.flatnonzero(big)[rel.argmax()]))
    assert np.all(np.abs(h[~big] - o[~big]) <= floor)


RANDOM_SHAPES = [(13, 7, 5), (33, 17, 9), (1, 5, 6), (6, 1, 4), (5, 4, 1), (1, 1, 7), (40, 3, 2), (64, 32, 8)]


@pytest.mark.parametrize("shape", RANDOM_SHAPES)
@pytest.mark.parametrize("bc", [(0, 1), (0, 0), (1, 0)])
def test_operator_bitwise_identical(torch_cuda, M, oracle_mod, shape, bc):
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, 100 + nr + nt + np_, bc_in=bc[0], bc_out=bc[1])
    S = M.solver_for_problem(p)
    Tr, Tt, Tp, D = S.get_operator()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, *bc)
    assert np.array_equal(Tr, op.Tr)
    assert np.array_equal(Tt, op.Tt)
    assert np.array_equal(Tp, op.Tp)
    assert np.array_equal(D, op.D)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_operator_bitwise_configs(torch_cuda, M, oracle_mod, name):
    p = inputs.make_problem(name)
    S = M.solver_for_problem(p)
    got = S.get_operator()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    for g, o in zip(got, (op.Tr, op.Tt, op.Tp, op.D)):
        assert np.array_equal(g, o)


def apply_err(op, x, y):
    mag = 2.0 * op.D * np.abs(x) - op.apply(np.abs(x))     # D|x| + sum T|x_nb| (T, D >= 0)
    return np.abs(y - op.apply(x)) / np.maximum(mag, 1e-300)


@pytest.mark.parametrize("shape", RANDOM_SHAPES + [(150, 30, 12)])
def test_apply_parity(torch_cuda, M, oracle_mod, shape):
    torch = torch_cuda
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, 7 + nr, bc_in=0, bc_out=1)
    S = M.solver_for_problem(p)
    x = np.random.default_rng(nr * nt).standard_normal((np_, nt, nr))
    y = S.apply(dev(torch, x)).cpu().numpy()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 0, 1)
    assert apply_err(op, x, y).max() <= APPLY_TOL


PATHS = [1, 2, 3]   # MASPCG_OPT_PATH: three kernels, fused two passes, wave (flag-ordered p-update + stencil)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_solve_parity_fast_arithmetic(torch_cuda, M, oracle_mod, name, path):
    """MASPCG_OPT_ARITH = 1 (FMA, plain tree sums): the tolerance contract only."""
    p = inputs.make_problem(name)
    o = oracle_mod.solve_problem(p)
    g = gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: path, M.OPT_ARITH: M.ARITH_FAST})
    assert_solve_parity(g, o, exact=False)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_solve_parity_configs(torch_cuda, M, oracle_mod, name, path):
    p = inputs.make_problem(name)
    o = oracle_mod.solve_problem(p)
    assert o["status"] == 0
    g = gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: path})
    assert_solve_parity(g, o)
    assert g[4].stats()["path"] == path


@pytest.mark.parametrize("seed,shape,bc", [(1, (13, 7, 5), (0, 1)), (2, (33, 17, 9), (0, 0)),
                                          (3, (8, 12, 16), (1, 0)), (4, (5, 4, 1), (0, 1)),
                                          (5, (1, 9, 6), (1, 1)), (6, (20, 1, 3), (0, 0))])
@pytest.mark.parametrize("path", PATHS)
def test_solve_parity_random(torch_cuda, M, oracle_mod, seed, shape, bc, path):
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, seed, bc_in=bc[0], bc_out=bc[1])
    o = oracle_mod.solve_problem(p)
    assert_solve_parity(gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: path}), o)


@pytest.mark.parametrize("path", PATHS)
def test_solve_parity_warm_start(torch_cuda, M, oracle_mod, path):
    p = inputs.make_problem("c2", x0_seed=9)
    o = oracle_mod.solve_problem(p)
    assert_solve_parity(gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: path}), o)


@pytest.mark.parametrize("shape", [(16, 16, 32), (40, 3, 2), (64, 32, 8), (12, 20, 9), (150, 30, 12)])
def test_fused_tma_and_register_variants_identical(torch_cuda, M, oracle_mod, shape):
    """Pass A staged by TMA bulk copies (nr even) and the register-batched pass A give the oracle's
    iterates bit for bit."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, 300 + nr, bc_in=0, bc_out=1)
    o = oracle_mod.solve_problem(p)
    for tma in (1, 0):
        g = gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: M.PATH_FUSED, M.OPT_TMA: tma})
        assert_solve_parity(g, o)


@pytest.mark.parametrize("shape", [(16, 16, 32), (40, 3, 2), (64, 32, 8), (13, 7, 5), (150, 30, 12)])
def test_vector_and_scalar_kernels_identical(torch_cuda, M, oracle_mod, shape):
    """Three-kernel path with 16-byte vector kernels (nr even) and scalar kernels: oracle iterates."""
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, 400 + nr, bc_in=0, bc_out=1)
    o = oracle_mod.solve_problem(p)
    for vec in (1, 0):
        g = gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: M.PATH_THREE_KERNELS, M.OPT_VEC: vec})
        assert_solve_parity(g, o)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("chunk,graphs,timing", [(1, 1, 0), (3, 1, 0), (16, 0, 0), (64, 1, 0), (7, 1, 1)])
def test_solve_loop_modes_identical(torch_cuda, M, oracle_mod, chunk, graphs, timing, path):
    """Chunking, graph replay and timing mode change how kernels are issued, never the bits."""
    p = inputs.make_problem("c1")
    ref = gpu_solve(torch_cuda, M, p, chunk=16, opts={M.OPT_PATH: path})
    g = gpu_solve(torch_cuda, M, p, chunk=chunk,
                  opts={M.OPT_PATH: path, M.OPT_USE_GRAPHS: graphs, M.OPT_TIMING: timing})
    assert g[0] == ref[0] and g[1]["iters"] == ref[1]["iters"]
    assert np.array_equal(g[2], ref[2]) and np.array_equal(g[3], ref[3])
    if timing:
        st = g[4].stats()
        assert st["matvec_launches"] == g[1]["iters"]
        assert st["matvec_ms"] > 0 and st["update_ms"] > 0 and st["pupdate_ms"] > 0


def test_deterministic_run_to_run(torch_cuda, M):
    p = inputs.make_problem("c2")
    a = gpu_solve(torch_cuda, M, p)
    b = gpu_solve(torch_cuda, M, p)
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("path", PATHS)
def test_edge_cases(torch_cuda, M, oracle_mod, path):
    torch = torch_cuda
    p = inputs.random_problem(9, 6, 8, 77)
    o = oracle_mod.solve_problem(p)
    S = M.solver_for_problem(p)
    S.set_option(M.OPT_PATH, path)
    f = dev(torch, p.f)
    # tol = 0: exactly maxit iterations
    x = dev(torch, p.x0)
    st, info, hist = S.solve(f, x, 0.0, 5)
    oo = oracle_mod.solve_problem(p, tol=0.0, maxit=5)
    assert st == M.NOT_CONVERGED == oo["status"] and info["iters"] == 5 and hist.size == 6
    np.testing.assert_allclose(hist, oo["hist"], rtol=1e-12)
    np.testing.assert_allclose(x.cpu().numpy(), oo["x"], rtol=0, atol=1e-12 * np.abs(oo["x"]).max())
    # maxit = 0: only hist[0]
    x = dev(torch, p.x0)
    st, info, hist = S.solve(f, x, 1e-10, 0)
    assert st == M.NOT_CONVERGED and info["iters"] == 0 and hist[0] == pytest.approx(o["hist"][0], rel=1e-13)
    # b = 0 (f = 0, g = 0): x = 0, OK, 0 iterations
    S0 = M.solver_for_problem(inputs.random_problem(9, 6, 8, 77, bc_in=1, bc_out=1))
    S0.set_option(M.OPT_PATH, path)
    x = dev(torch, np.ones((8, 6, 9)))
    st, info, hist = S0.solve(dev(torch, np.zeros((8, 6, 9))), x, 1e-10, 50)
    assert st == M.OK and info["iters"] == 0 and not x.cpu().numpy().any()
    # converged initial guess: 0 iterations, x untouched
    x = dev(torch, o["x"])
    st, info, hist = S.solve(f, x, 1e-6, 50)
    assert st == M.OK and info["iters"] == 0 and np.array_equal(x.cpu().numpy(), o["x"])
    # non-finite rhs -> breakdown
    fb = p.f.copy()
    fb[3, 2, 1] = np.nan
    x = dev(torch, p.x0)
    st, info, hist = S.solve(dev(torch, fb), x, 1e-10, 50, raise_on_error=False)
    assert st == M.E_BREAKDOWN
    # aliasing and bad arguments
    with pytest.raises(M.MaspcgError) as e:
        S.solve(f, f, 1e-10, 5)
    assert e.value.status == M.E_INVALID
    with pytest.raises(M.MaspcgError):
        S.solve(f, dev(torch, p.x0), -1.0, 5)


def test_error_paths(torch_cuda, M):
    torch = torch_cuda
    p = inputs.random_problem(6, 5, 4, 5, shift=False, bc_in=1, bc_out=1)
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf)
    x = dev(torch, p.x0)
    with pytest.raises(M.MaspcgError) as e:       # solve before coefficients
        S.solve(dev(torch, p.f), x, 1e-10, 5)
    assert e.value.status == M.E_STATE
    S.set_coefficients(dev(torch, p.kr), dev(torch, p.kt), dev(torch, p.kp), dev(torch, p.s))
    S.set_bc_r(1, None, 1, None)
    with pytest.raises(M.MaspcgError) as e:       # s == 0 and Neumann on both sides
        S.solve(dev(torch, p.f), x, 1e-10, 5)
    assert e.value.status == M.E_SINGULAR
    S.set_bc_r(0, None, 1, None)                   # a Dirichlet side makes it definite
    st, info, hist = S.solve(dev(torch, p.f), x, 1e-10, 500)
    assert st == M.OK
    kr = p.kr.copy()
    kr[1, 2, 3] = -1.0
    with pytest.raises(M.MaspcgError) as e:   # reported by the next call that uses the operator (deferred)
        S.set_coefficients(dev(torch, kr), dev(torch, p.kt), dev(torch, p.kp), dev(torch, p.s))
        S.solve(dev(torch, p.f), x, 1e-10, 5)
    assert e.value.status == M.E_INVALID
    with pytest.raises(M.MaspcgError) as e:   # host entry point: reported by the call itself
        S.set_coefficients(kr, p.kt, p.kp, p.s)
    assert e.value.status == M.E_INVALID
    bad = p.pf.copy()
    bad[-1] = 6.0
    with pytest.raises(M.MaspcgError) as e:
        S.set_grid(p.rf, p.tf, bad)
    assert e.value.status == M.E_INVALID


def test_host_entry_points(torch_cuda, M, oracle_mod):
    """maspcg_set_coefficients_host / maspcg_solve_host: identical bits to the device entry points."""
    p = inputs.make_problem("c1")
    ref = gpu_solve(torch_cuda, M, p)
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf)
    S.set_coefficients(p.kr, p.kt, p.kp, p.s)
    S.set_bc_r(p.bc_in, None, p.bc_out, None)
    x = p.x0.copy()
    st, info, hist = S.solve(p.f, x, p.tol, p.maxit)
    assert st == ref[0] and info["iters"] == ref[1]["iters"]
    assert np.array_equal(x, ref[3]) and np.array_equal(hist, ref[2])


@pytest.mark.slow
def test_solve_parity_c3_half_resolution(torch_cuda, M, oracle_mod):
    """c3 recipe (coronal viscosity, stretched grid) at 75 x 150 x 300 = 3.4 M cells, both paths."""
    p = inputs.make_problem("c3", shape=(75, 150, 300))
    o = oracle_mod.solve_problem(p)
    assert o["status"] == 0 and o["iters"] < 1000
    for path in PATHS:
        assert_solve_parity(gpu_solve(torch_cuda, M, p, opts={M.OPT_PATH: path}), o)


@pytest.mark.slow
def test_c3_full_size(torch_cuda, M, oracle_mod):
    """The bench workload (c3, 150 x 300 x 600 = 27 M cells) in the bench's launch configuration:
    20 fixed iterations against the oracle, then the full solve checked by its true residual."""
    torch = torch_cuda
    p = inputs.make_problem("c3")
    S = M.solver_for_problem(p)
    f = dev(torch, p.f)
    # (1) 20 iterations, tol = 0
    x = dev(torch, p.x0)
    st, info, hist = S.solve(f, x, 0.0, 20)
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    b = op.rhs(p.f, p.g_in, p.g_out)
    ost, ox, oit, ohist, obn, orn = op.pcg(b, p.x0, 0.0, 20)
    xg = x.cpu().numpy()
    assert info["iters"] == oit == 20
    assert np.array_equal(xg, ox) and np.array_equal(hist, ohist)     # R24: identical iterates
    assert np.linalg.norm(xg - ox) <= SOL_TOL * np.linalg.norm(ox)
    assert_hist(hist, ohist, obn)
    # (2) apply at full size, sampled cells vs the oracle's full apply
    y = S.apply(x).cpu().numpy()
    assert apply_err(op, xg, y).max() <= APPLY_TOL
    # (3) full solve to 1e-10: converged, and the true residual b - A x agrees with the recurrence
    x = dev(torch, p.x0)
    st, info, hist = S.solve(f, x, p.tol, p.maxit)
    assert st == M.OK and hist[-1] <= p.tol * info["bnorm"]
    true_r = np.linalg.norm(b - op.apply(x.cpu().numpy())) / np.linalg.norm(b)
    assert true_r <= 2 * p.tol


@pytest.mark.slow
@pytest.mark.parametrize("shape,min_iters", [((40, 40, 80), 1000), ((80, 80, 160), 2400)])
def test_c4_recipe_long_high_contrast_solve_exact(torch_cuda, M, oracle_mod, shape, min_iters):
    """c4 physics (kappa = (T 10^{0.4 G})^{5/2}, contrast ~4e5) solved to 1e-10 (1,060 and 2,504
    iterations): long CG runs where rounding differences grow past 1e-10 in the history after ~1,000
    iterations.  With the default arithmetic (R24) the GPU reproduces the
    oracle's iterates exactly over the whole solve."""
    p = inputs.make_problem("c4", shape=shape)
    o = oracle_mod.solve_problem(p, tol=1e-10, maxit=20000)
    assert o["status"] == 0 and o["iters"] >= min_iters
    for path in PATHS:
        g = gpu_solve(torch_cuda, M, p, tol=1e-10, maxit=20000, opts={M.OPT_PATH: path})
        assert_solve_parity(g, o)


@pytest.mark.slow
def test_c5_warm_started_time_loop_exact(torch_cuda, M, oracle_mod):
    """c5: repeated implicit solves of a backward-Euler time loop (f = s u^{n-1}, x0 = u^{n-1}) at
    50 x 75 x 150; every step matches the oracle's iterates exactly."""
    torch = torch_cuda
    p = inputs.make_problem("c5", shape=(50, 75, 150))
    S = M.solver_for_problem(p)
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    f = p.f.copy()
    u_o = p.x0.copy()
    x = dev(torch, p.x0)
    iters = []
    for step in range(3):
        b = op.rhs(f, p.g_in, p.g_out)
        ost, ox, oit, ohist, obn, orn = op.pcg(b, u_o, p.tol, p.maxit)
        st, info, hist = S.solve(dev(torch, f), x, p.tol, p.maxit)
        xg = x.cpu().numpy()
        assert st == ost == 0 and info["iters"] == oit
        assert np.array_equal(xg, ox) and np.array_equal(hist, ohist)
        iters.append(oit)
        u_o = ox
        f = p.s * ox          # caller's time loop: b = s V u^{n-1}
    assert iters[1] < iters[0]  # warm starts converge faster (R12: tolerance relative to ||b||)


@pytest.mark.parametrize("mean,half_power,with_rho", [(0, 5, True), (1, 5, False), (1, 2, True), (0, 0, False)])
def test_coefficients_from_fields_bitwise(torch_cuda, M, oracle_mod, mean, half_power, with_rho):
    """maspcg_set_coefficients_from_fields (NEXT-1): face kappa from a cell field and the shift from
    rho, assembled on the device -- the operator equals the oracle's bit for bit."""
    torch = torch_cuda
    p = inputs.random_problem(14, 9, 10, 500 + half_power)
    rng = np.random.default_rng(half_power + 10 * mean)
    T = rng.uniform(0.3, 2.0, (p.np, p.nt, p.nr))
    rho = rng.uniform(0.5, 1.5, T.shape) if with_rho else None
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf)
    S.set_coefficients_from_fields(dev(torch, T), 0.8, half_power, mean, dev(torch, rho), 25.0)
    S.set_bc_r(p.bc_in, dev(torch, p.g_in), p.bc_out, None)
    kr, kt, kp, s = oracle_mod.face_coefficients(T, 0.8, half_power, mean, rho, 25.0)
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, kr, kt, kp, s, p.bc_in, p.bc_out)
    for g, o in zip(S.get_operator(), (op.Tr, op.Tt, op.Tp, op.D)):
        assert np.array_equal(g, o)
    with pytest.raises(M.MaspcgError) as e:          # T^(5/2) of a negative temperature -> NaN
        S.set_coefficients_from_fields(dev(torch, -T), 1.0, 5, mean, None, 1.0)
        S.get_operator()                              # (reported by the next use of the operator)
    assert e.value.status == M.E_INVALID


@pytest.mark.slow
def test_nonlinear_conduction_time_loop_exact(torch_cuda, M, oracle_mod):
    """Backward-Euler thermal conduction with lagged kappa(T) = kappa0 T^(5/2) (the per-step
    assembly of NEXT-1 feeding the PCG of every step): 4 steps of (rho/dt - div kappa(T^n) grad) T^{n+1}
    = rho/dt T^n on the c2 grid, identical to the oracle step by step."""
    torch = torch_cuda
    p = inputs.make_problem("c2", shape=(32, 32, 64))
    rc = inputs.midpoints(p.rf)
    T = np.broadcast_to(inputs.t_profile(1.0 + 0.02 * (rc - 1.0))[None, None, :], (p.np, p.nt, p.nr)).copy()
    T *= 1.0 + 0.1 * inputs.white_noise(9, p.nr, p.nt, 0, p.np)
    rho = np.broadcast_to(inputs.rho_hydro(rc)[None, None, :], T.shape).copy()
    dt = 0.05
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf)
    S.set_bc_r(M.BC_DIRICHLET, dev(torch, T[:, :, 0].copy()), M.BC_NEUMANN0, None)
    Tg, To = dev(torch, T), T.copy()
    for step in range(4):
        S.set_coefficients_from_fields(Tg.clone(), 1.0, 5, M.MEAN_HARMONIC, dev(torch, rho), 1.0 / dt)
        f = (rho / dt) * To                           # per-unit-volume source s T^n
        kr, kt, kp, s = oracle_mod.face_coefficients(To, 1.0, 5, 1, rho, 1.0 / dt)
        op = oracle_mod.Operator(p.rf, p.tf, p.pf, kr, kt, kp, s, 0, 1)
        b = op.rhs(f, T[:, :, 0].copy(), None)
        ost, ox, oit, ohist, obn, orn = op.pcg(b, To, 1e-10, 5000)
        st, info, hist = S.solve(dev(torch, f), Tg, 1e-10, 5000)
        assert st == ost == 0 and info["iters"] == oit
        assert np.array_equal(Tg.cpu().numpy(), ox) and np.array_equal(hist, ohist)
        To = ox


@pytest.mark.parametrize("bc,stages,nr", [((1, 1), 6, 12), ((0, 1), 10, 12), ((0, 0), 3, 12), ((1, 0), 5, 11)])
def test_sts_step_bitwise(torch_cuda, M, oracle_mod, bc, stages, nr):
    """maspcg_sts_step (NEXT-4): RKL2 super-time-steps of V du/dt = b_D - K u equal the oracle's bit for
    bit (even nr: the two-cells-per-thread stage kernel; odd nr: one cell per thread);
    maspcg_sts_dt_limit is a valid forward-Euler bound (dt * lambda_max(V^-1 K) <= 2)."""
    torch = torch_cuda
    p = inputs.random_problem(nr, 7, 8, 600 + stages, bc_in=bc[0], bc_out=bc[1])
    S = M.solver_for_problem(p)
    dt = S.sts_dt_limit()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, *bc)
    n = p.np * p.nt * p.nr
    A = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        A[:, c] = op.apply(e.reshape(op.shape)).ravel()
    V = oracle_mod.volumes(p.rf, p.tf, p.pf).ravel()
    lam = np.linalg.eigvals((A - np.diag(p.s.ravel() * V)) / V[:, None]).real.max()
    assert dt * lam <= 2.0 * (1 + 1e-12) and dt * lam > 0.2
    tau = 0.9 * (stages * stages + stages - 2) / 4.0 * dt
    u0 = np.random.default_rng(stages).standard_normal(op.shape)
    ug = dev(torch, u0)
    uo = u0.copy()
    for _ in range(3):
        S.sts_step(ug, tau, stages)
        uo = op.rkl2_step(uo, p.s, tau, stages, p.g_in, p.g_out)
    torch.cuda.synchronize()
    assert np.array_equal(ug.cpu().numpy(), uo)


@pytest.mark.timeout(600, method="thread")
def test_sts_c3_full_size_bitwise(torch_cuda, M, oracle_mod):
    """`bench.py --sts-stages` workload: one 10-stage RKL2 step on the full c3 grid (27 M cells, the
    two-plane halo copies and the Dirichlet inner boundary included) equals the oracle's bit for bit."""
    torch = torch_cuda
    p = inputs.make_problem("c3")
    S = M.solver_for_problem(p)
    dt = S.sts_dt_limit()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    tau = 0.9 * (10 * 10 + 10 - 2) / 4.0 * dt
    u0 = np.random.default_rng(10).standard_normal(op.shape)
    ug = dev(torch, u0)
    S.sts_step(ug, tau, 10)
    torch.cuda.synchronize()
    uo = op.rkl2_step(u0, p.s, tau, 10, p.g_in, p.g_out)
    assert np.array_equal(ug.cpu().numpy(), uo)
    S.close()


@pytest.mark.parametrize("name", ["c1", "c2", "rand"])
@pytest.mark.parametrize("chunk", [16, 5])
def test_device_loop_bitwise(torch_cuda, M, oracle_mod, name, chunk):
    """MASPCG_OPT_DEVICE_LOOP: the whole PCG loop as one CUDA-graph launch (a conditional WHILE node over a
    chunk of iterations) gives the oracle's iterates, count and history bit for bit."""
    p = inputs.random_problem(14, 9, 10, 17) if name == "rand" else inputs.make_problem(name)
    o = oracle_mod.solve_problem(p)
    g = gpu_solve(torch_cuda, M, p, chunk=chunk, opts={M.OPT_DEVICE_LOOP: 1})
    assert_solve_parity(g, o)
    g[4].close()


def test_device_loop_edge_cases(torch_cuda, M, oracle_mod):
    """Device loop: tol = 0 runs exactly maxit iterations (also when maxit is not a multiple of the chunk);
    a converged x0 returns at once."""
    torch = torch_cuda
    p = inputs.make_problem("c1")
    for maxit in (7, 33):
        o = oracle_mod.solve_problem(p, tol=0.0, maxit=maxit)
        g = gpu_solve(torch, M, p, tol=0.0, maxit=maxit, opts={M.OPT_DEVICE_LOOP: 1})
        assert g[0] == M.NOT_CONVERGED and g[1]["iters"] == maxit
        assert_solve_parity(g, o)
        g[4].close()
    o = oracle_mod.solve_problem(p)
    g = gpu_solve(torch, M, p, x0=o["x"], tol=1e-6, opts={M.OPT_DEVICE_LOOP: 1})
    assert g[0] == M.OK and g[1]["iters"] == 0
    g[4].close()
