"""GPU parity of the field-aligned anisotropic conduction operator (reading R33;
csrc/aniso.cu) against the CPU oracle (oracle/masoracle.c, pinned in tests/test_oracle_aniso_pins.py),
through the C ABI (-m gpu).

Both sides evaluate the same R33 formulas with one IEEE rounding per operation in the same order, so
the contract is bitwise: edge weights, the 7-point diagonal D7 and the Jacobi diagonal, y = A x, and the
whole PCG solve (solution, iteration count, residual history) -- on ragged shapes (odd nr, nt = 1 and
np = 1 degenerate cases, pole rows), all r-boundary combinations, the c1a / c2a configurations, 2-4
loopback ranks, and the full c3a grid in the bench's launch configuration for a fixed number of
iterations.
"""
import threading

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_2303_03398_b200 import build, maspcg
    build.build()
    return maspcg


def dev(a):
    import torch
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def oracle_op(oracle_mod, p):
    return oracle_mod.AnisoOperator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out, p.krt, p.krp, p.ktp)


def lib_layout(o):
    """The oracle's edge arrays in the library's [np][nt][nr] layout (lower faces; boundary rows dropped)."""
    nt, nr = o.nt, o.nr
    return o.Xrt[:, :nt, :nr], o.Xrp[:, :, :nr], o.Xtp[:, :nt, :]


SHAPES = [(13, 7, 5), (10, 9, 8), (1, 5, 6), (6, 1, 4), (5, 4, 1), (12, 6, 2), (33, 17, 9), (64, 16, 8)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bc", [(0, 1), (0, 0), (1, 0)])
def test_operator_bitwise(M, oracle_mod, shape, bc):
    """Edge weights, D7, the Jacobi diagonal and y = A x are bit-identical to the oracle."""
    p = inputs.random_aniso_problem(*shape, sum(shape) + 3 * bc[0] + bc[1], bc_in=bc[0], bc_out=bc[1])
    o = oracle_op(oracle_mod, p)
    S = M.solver_for_problem(p)
    Xrt, Xrp, Xtp, D7 = S.aniso_get_operator()
    ort, orp, otp = lib_layout(o)
    assert np.array_equal(Xrt, ort) and np.array_equal(Xrp, orp) and np.array_equal(Xtp, otp)
    assert np.array_equal(D7, o.D7)
    Tr, Tt, Tp, D = S.get_operator()
    assert np.array_equal(D, o.Dj)
    assert np.array_equal(Tr, o.Tr) and np.array_equal(Tt, o.Tt) and np.array_equal(Tp, o.Tp)
    x = inputs.white_noise(91, p.nr, p.nt, 0, p.np)
    y = S.apply(dev(x)).cpu().numpy()
    assert np.array_equal(y, o.apply(x)), np.abs(y - o.apply(x)).max()
    S.close()


def gpu_solve(M, p, tol=None, maxit=None, chunk=16, opts=None):
    import torch
    S = M.solver_for_problem(p, chunk=chunk)
    for k, v in (opts or {}).items():
        S.set_option(k, v)
    x = dev(p.x0)
    st, info, hist = S.solve(dev(p.f), x, p.tol if tol is None else tol, p.maxit if maxit is None else maxit,
                             raise_on_error=False)
    torch.cuda.synchronize()
    out = (st, info, hist, x.cpu().numpy())
    S.close()
    return out


def assert_bitwise(g, o):
    st, info, hist, x = g
    assert st == o["status"], (st, o["status"])
    assert info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]), np.abs(hist - o["hist"]).max()
    assert np.array_equal(x, o["x"]), np.abs(x - o["x"]).max()


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bc", [(0, 1), (0, 0), (1, 0)])
def test_solve_bitwise_random(M, oracle_mod, shape, bc):
    p = inputs.random_aniso_problem(*shape, 2 * sum(shape) + bc[0], bc_in=bc[0], bc_out=bc[1])
    assert_bitwise(gpu_solve(M, p), oracle_mod.solve_aniso_problem(p))


@pytest.mark.parametrize("name", ["c1a", "c2a"])
@pytest.mark.parametrize("chunk", [16, 5])
def test_solve_bitwise_configs(M, oracle_mod, name, chunk):
    """c1a (uniform shell) and c2a (stretched, pole rows, the coronal field): the oracle's iterates bit for
    bit, also with another graph chunk size."""
    p = inputs.make_aniso_problem(name)
    o = oracle_mod.solve_aniso_problem(p)
    assert o["status"] == 0
    assert_bitwise(gpu_solve(M, p, chunk=chunk), o)


def test_cross_terms_off_is_the_7point_operator(M, oracle_mod):
    """Passing NULL cross coefficients returns to the 7-point operator of the same kr, kt, kp, s (bitwise
    the oracle's masoracle_pcg), and setting them again restores the 19-point solve."""
    import torch
    p = inputs.make_aniso_problem("c1a")
    S = M.solver_for_problem(p)
    S.set_aniso_coefficients(None, None, None)
    x = dev(p.x0)
    st, info, hist = S.solve(dev(p.f), x, p.tol, p.maxit)
    o7 = oracle_mod.solve_problem(p)
    assert info["iters"] == o7["iters"] and np.array_equal(x.cpu().numpy(), o7["x"])
    S.set_aniso_coefficients(dev(p.krt), dev(p.krp), dev(p.ktp))
    x = dev(p.x0)
    st, info, hist = S.solve(dev(p.f), x, p.tol, p.maxit)
    torch.cuda.synchronize()
    oa = oracle_mod.solve_aniso_problem(p)
    assert info["iters"] == oa["iters"] and np.array_equal(x.cpu().numpy(), oa["x"])
    S.close()


def test_errors(M):
    """Non-finite edge coefficient -> E_INVALID; a partial set of NULLs -> E_INVALID; the other iteration
    paths and super-time-stepping refuse the 19-point operator."""
    p = inputs.random_aniso_problem(8, 6, 4, 3)
    S = M.solver_for_problem(p)
    bad = p.krp.copy()
    bad[1, 2, 3] = np.nan
    with pytest.raises(M.MaspcgError) as e:
        S.set_aniso_coefficients(dev(p.krt), dev(bad), dev(p.ktp))
    assert e.value.status == M.E_INVALID
    with pytest.raises(M.MaspcgError):
        S.set_aniso_coefficients(dev(p.krt), None, dev(p.ktp))
    S.set_aniso_coefficients(dev(p.krt), dev(p.krp), dev(p.ktp))
    S.set_option(M.OPT_PATH, 4)
    st, info, hist = S.solve(dev(p.f), dev(p.x0), 1e-10, 100, raise_on_error=False)
    assert st == M.E_INVALID
    S.set_option(M.OPT_PATH, 0)
    with pytest.raises(M.MaspcgError):
        S.sts_dt_limit()
    S.close()


# ------------------------------------------------------------------ multi-rank (loopback)
def run_ranks(M, P, fn):
    import torch
    group = M.LoopbackGroup(P)
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, group)
            s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=500)
    assert not any(t.is_alive() for t in th), "a rank hung"
    group.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("name,P,fn", [
    ("c1a", 2, lambda k0, n: inputs.make_aniso_problem("c1a", k0, n)),
    ("c1a", 4, lambda k0, n: inputs.make_aniso_problem("c1a", k0, n)),
    ("rand", 3, lambda k0, n: inputs.random_aniso_problem(9, 7, 6, 11, bc_in=0, bc_out=0, k0=k0 or 0, nloc=n)),
    ("rand-np2", 2, lambda k0, n: inputs.random_aniso_problem(8, 5, 2, 12, k0=k0 or 0, nloc=n)),
], ids=["c1a-P2", "c1a-P4", "rand-P3", "rand-np2-P2"])
def test_multirank_bitwise(M, oracle_mod, name, P, fn):
    """phi-slabs on 2-4 loopback ranks: the edge planes below each slab come from the left rank, the p
    halo as in the 7-point path; every rank returns the global oracle's iterates bit for bit."""
    import torch
    full = fn(None, None)
    o = oracle_mod.solve_aniso_problem(full)

    def rank(r, group):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        p = fn(k0, nloc)
        S = M.solver_for_problem(p, loopback=(group, r))
        x = dev(p.x0)
        st, info, hist = S.solve(dev(p.f), x, p.tol, p.maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        res = (st, info["iters"], hist, x.cpu().numpy(), S.aniso_get_operator())
        S.close()
        return res

    out = run_ranks(M, P, rank)
    x = np.concatenate([r[3] for r in out], axis=0)
    ort, orp, otp = lib_layout(oracle_op(oracle_mod, full))
    for r, (st, it, hist, _, ops) in enumerate(out):
        assert st == o["status"] and it == o["iters"]
        assert np.array_equal(hist, o["hist"])
        k0, nloc = inputs.slab_extent(full.np, r, P)
        assert np.array_equal(ops[0], ort[k0:k0 + nloc]) and np.array_equal(ops[1], orp[k0:k0 + nloc])
        assert np.array_equal(ops[2], otp[k0:k0 + nloc])
    assert np.array_equal(x, o["x"])


# ------------------------------------------------------------------ full size (bench launch configuration)
@pytest.mark.slow
def test_full_c3a_fixed_iterations_bitwise(M, oracle_mod):
    """The bench workload c3a (150 x 300 x 600, 27 M cells) in the bench's launch configuration (graphs,
    chunk 16): 12 PCG iterations at tol = 0, iterate and history bitwise against the oracle (its -fopenmp
    build for speed: identical values, tests/test_oracle_pins.py::test_openmp_build_gives_identical_iterates)."""
    p = inputs.make_aniso_problem("c3a")
    oracle_mod.use_openmp(True)
    try:
        o = oracle_mod.solve_aniso_problem(p, tol=0.0, maxit=12)
    finally:
        oracle_mod.use_openmp(False)
    g = gpu_solve(M, p, tol=0.0, maxit=12)
    assert g[0] == o["status"] == M.NOT_CONVERGED
    assert_bitwise(g, o)


# ------------------------------------------------------------------ the plane-marching TMA operator (default)
@pytest.mark.parametrize("tj,grid", [(None, None), (1, None), (3, 5), (2, 1)])
@pytest.mark.parametrize("shape,bc", [((12, 6, 2), (0, 1)), ((64, 16, 8), (1, 0)), ((10, 9, 8), (0, 0)),
                                      ((2, 5, 3), (0, 1)), ((20, 13, 11), (1, 0))])
def test_march_operator_and_solve_bitwise(M, oracle_mod, monkeypatch, tj, grid, shape, bc):
    """The default stencil for even nr: one plane-marching kernel whose p planes and coefficient rows arrive by
    bulk copies (k_aniso_march).  y = A x and whole solves bit-identical to the oracle; forced small tiles (ragged
    last tile) and grids (several (tile, plane) segments per block, the rings carried across segments)."""
    if tj:
        monkeypatch.setenv("MASPCG_ANISO_MARCH_TJ", str(tj))
    if grid:
        monkeypatch.setenv("MASPCG_ANISO_MARCH_GRID", str(grid))
    p = inputs.random_aniso_problem(*shape, 5 * sum(shape) + bc[0], bc_in=bc[0], bc_out=bc[1])
    o = oracle_op(oracle_mod, p)
    S = M.solver_for_problem(p)
    x = inputs.white_noise(93, p.nr, p.nt, 0, p.np)
    y = S.apply(dev(x)).cpu().numpy()
    S.close()
    assert np.array_equal(y, o.apply(x)), np.abs(y - o.apply(x)).max()
    assert_bitwise(gpu_solve(M, p), oracle_mod.solve_aniso_problem(p))


@pytest.mark.parametrize("march", ["0", "1"])
def test_march_and_pair_kernels_c2a(M, oracle_mod, monkeypatch, march):
    """c2a with the marching kernel and with the previous TMA pair kernel (MASPCG_ANISO_MARCH=0): both the
    oracle's iterates bit for bit."""
    monkeypatch.setenv("MASPCG_ANISO_MARCH", march)
    p = inputs.make_aniso_problem("c2a")
    assert_bitwise(gpu_solve(M, p), oracle_mod.solve_aniso_problem(p))


def test_march_multirank_bitwise(M, oracle_mod, monkeypatch):
    """The marching kernel on the interior planes of 3 loopback slabs (the boundary planes by the pair kernel),
    forced small tiles and grids: every rank returns the global oracle's iterates."""
    import torch
    monkeypatch.setenv("MASPCG_ANISO_MARCH_TJ", "3")
    monkeypatch.setenv("MASPCG_ANISO_MARCH_GRID", "4")
    P = 3
    fn = lambda k0, n: inputs.random_aniso_problem(10, 7, 12, 21, bc_in=0, bc_out=1, k0=k0 or 0, nloc=n)
    full = fn(None, None)
    o = oracle_mod.solve_aniso_problem(full)

    def rank(r, group):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        p = fn(k0, nloc)
        S = M.solver_for_problem(p, loopback=(group, r))
        xr = dev(p.x0)
        st, info, hist = S.solve(dev(p.f), xr, p.tol, p.maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        res = (st, info["iters"], hist, xr.cpu().numpy())
        S.close()
        return res

    out = run_ranks(M, P, rank)
    for st, it, hist, _ in out:
        assert st == o["status"] and it == o["iters"] and np.array_equal(hist, o["hist"])
    assert np.array_equal(np.concatenate([r[3] for r in out], axis=0), o["x"])


@pytest.mark.parametrize("name", ["c1a", "c2a"])
def test_march_fast_arithmetic_tolerance_contract(M, oracle_mod, name):
    """MASPCG_OPT_ARITH = 1 through the marching stencil: the tolerance contract (solution relative L2 <= 1e-10,
    iterations +-1)."""
    p = inputs.make_aniso_problem(name)
    o = oracle_mod.solve_aniso_problem(p)
    st, info, hist, x = gpu_solve(M, p, opts={M.OPT_ARITH: M.ARITH_FAST})
    assert st == o["status"] == 0
    assert abs(info["iters"] - o["iters"]) <= 1
    assert np.linalg.norm(x - o["x"]) <= 1e-10 * np.linalg.norm(o["x"])
