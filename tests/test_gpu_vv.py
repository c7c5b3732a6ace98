"""GPU parity of the staggered vector viscosity through the C ABI (-m gpu).

maspcg_vv_* against the vector oracle (oracle/masoracle_vv.c) on the same seeded inputs
(paper_2303_03398_b200/inputs.py make_vv_problem):
  * the Jacobi diagonal and y = A x: bit-identical (both sides evaluate the operator's formulas with
    one IEEE rounding per operation in the same order, readings R27-R31; the pole-ring sums are
    Dot2, R24);
  * the solve: x, the iteration count and every residual-history entry identical to the oracle's
    (np.array_equal), single rank and 2-4 loopback ranks (the pole-ring sums all-gathered across the
    phi-slabs, Listing 3's array reduction of PAPER.md:147-157);
  * edge cases: tol = 0, maxit = 0, non-unknown slots of x0 ignored, a grid without poles, call
    order.
"""
import threading

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300, method="thread")]


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
    return oracle_mod.VVOperator(p.rf, p.tf, p.pf, p.nu, p.s, p.wall_in, p.wall_out)


def gpu_solver(M, p, loopback=None, chunk=16):
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, chunk=chunk, loopback=loopback)
    assert (S.k0, S.nloc) == (p.k0, p.nloc)
    S.vv_set_coefficients(dev(p.nu), dev(p.s))
    S.vv_set_bc_r(p.wall_in, dev(p.g_in), p.wall_out, dev(p.g_out))
    return S


def gpu_vv_solve(M, p, tol=None, maxit=None, loopback=None, chunk=16, x0=None, opts=None):
    import torch
    S = gpu_solver(M, p, loopback, chunk)
    try:
        for k, v in (opts or {}).items():
            S.set_option(k, v)
        x = dev(p.x0 if x0 is None else x0)
        st, info, hist = S.vv_solve(dev(p.f), x, p.tol if tol is None else tol,
                                    p.maxit if maxit is None else maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        return st, info, hist, x.cpu().numpy(), S.vv_get_diag(), S.stats()
    finally:
        S.close()   # collective for loopback contexts: every rank closes, also on failure


SHAPES = [(5, 6, 8), (13, 7, 6), (8, 4, 2), (1, 3, 5), (16, 16, 32), (33, 17, 9)]
WALLS = [(0, 0), (0, 1), (1, 1), (1, 0)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("walls", WALLS)
def test_vv_diag_and_apply_bitwise(M, oracle_mod, shape, walls):
    import torch
    p = inputs.make_vv_problem("rand", shape=shape, seed=sum(shape), wall_in=walls[0], wall_out=walls[1])
    op = oracle_op(oracle_mod, p)
    S = gpu_solver(M, p)
    assert np.array_equal(S.vv_get_diag(), op.D)
    x = np.stack([inputs.white_noise(77 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1)
    y = S.vv_apply(dev(x))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), op.apply(x))
    S.close()


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("walls", [(0, 0), (0, 1), (1, 1)])
def test_vv_solve_exact(M, oracle_mod, shape, walls):
    p = inputs.make_vv_problem("rand", shape=shape, seed=3 + sum(shape), wall_in=walls[0], wall_out=walls[1])
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, x, D, stats = gpu_vv_solve(M, p)
    assert st == o["status"] == 0
    assert info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"])
    assert np.array_equal(x, o["x"])
    assert stats["path"] == 5


@pytest.mark.parametrize("name,shape", [("c2v", None), ("c2v", (40, 60, 96))])
def test_vv_coronal_solve_exact(M, oracle_mod, name, shape):
    """The coronal recipe (nu = 1e-3 rho, s = rho/dt, no-slip inner / free-slip outer wall), with a
    warm start, in the bench's launch configuration (graphs, chunk 16)."""
    p = inputs.make_vv_problem(name, shape=shape, x0_seed=5)
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, x, D, stats = gpu_vv_solve(M, p)
    assert st == o["status"] == 0 and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(x, o["x"])


@pytest.mark.timeout(600, method="thread")
def test_vv_c3v_full_size_operator_bitwise(M, oracle_mod):
    """The bench workload of `bench.py --operator vv` (c3v: 150 x 300 x 600 cells, 81 M unknowns): the
    Jacobi diagonal and y = A x of the device operator equal the oracle's on every entry."""
    import torch
    p = inputs.make_vv_problem("c3v")
    op = oracle_op(oracle_mod, p)
    S = gpu_solver(M, p)
    try:
        assert np.array_equal(S.vv_get_diag(), op.D)
        x = np.stack([inputs.white_noise(7 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1)
        y = S.vv_apply(dev(x))
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), op.apply(x))
    finally:
        S.close()


@pytest.mark.parametrize("chunk,graphs", [(1, 1), (7, 1), (16, 0)])
def test_vv_loop_modes_identical(M, oracle_mod, chunk, graphs):
    p = inputs.make_vv_problem("rand", shape=(9, 8, 10), seed=4)
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, x, D, _ = gpu_vv_solve(M, p, chunk=chunk, opts={M.OPT_USE_GRAPHS: graphs})
    assert st == 0 and info["iters"] == o["iters"]
    assert np.array_equal(x, o["x"]) and np.array_equal(hist, o["hist"])


def test_vv_edge_cases(M, oracle_mod):
    import torch
    p = inputs.make_vv_problem("rand", shape=(6, 5, 4), seed=9, x0_seed=3)
    # tol = 0: exactly maxit iterations; non-unknown slots of x0 are ignored (set to 0)
    o = oracle_mod.vv_solve_problem(p, tol=0.0, maxit=7)
    st, info, hist, x, _, _ = gpu_vv_solve(M, p, tol=0.0, maxit=7)
    assert st == o["status"] == 1 and info["iters"] == 7
    assert np.array_equal(x, o["x"]) and np.array_equal(hist, o["hist"])
    assert np.all(x[:, 0, :, 0] == 0.0) and np.all(x[:, 1, 0, :] == 0.0)
    # maxit = 0
    st, info, hist, x, _, _ = gpu_vv_solve(M, p, maxit=0)
    assert st == 1 and info["iters"] == 0 and hist.size == 1
    # zero forcing and zero wall data: x = 0, OK, 0 iterations
    q = inputs.make_vv_problem("rand", shape=(6, 5, 4), seed=9, x0_seed=3)
    q.f[:] = 0.0
    q.g_in = q.g_out = None
    st, info, hist, x, _, _ = gpu_vv_solve(M, q)
    assert st == 0 and info["iters"] == 0 and np.all(x == 0.0)
    # a theta band without poles is rejected; call order
    S = M.Solver(4, 5, 6, inputs.rfaces(4, 1, 2, 0), inputs.tfaces(5, 0.0, 0.3, 2.5), inputs.pfaces(6))
    S.vv_enable()
    with pytest.raises(M.MaspcgError) as e:
        S.vv_set_coefficients(dev(np.ones((6, 5, 4))), dev(np.ones((6, 5, 4))))
    assert e.value.status == M.E_INVALID
    x = dev(np.zeros((6, 3, 5, 4)))
    st, _, _ = S.vv_solve(x.clone(), x, 1e-10, 10, raise_on_error=False)
    assert st == M.E_STATE
    S.close()
    # negative viscosity
    S = gpu_solver(M, p)
    with pytest.raises(M.MaspcgError) as e:
        S.vv_set_coefficients(dev(-p.nu), dev(p.s))
    assert e.value.status == M.E_INVALID
    S.close()
    torch.cuda.synchronize()


def test_vv_scalar_solves_unaffected(M, oracle_mod):
    """A vector solve on a context leaves its scalar operator and solve intact (the driver's state
    is swapped back), and vice versa."""
    import torch
    p = inputs.make_problem("c1")
    S = M.solver_for_problem(p)
    v = inputs.make_vv_problem("rand", shape=(16, 16, 32), seed=2)
    v.rf, v.tf, v.pf = p.rf, p.tf, p.pf      # the context's grid
    S.vv_set_coefficients(dev(v.nu), dev(v.s))
    S.vv_set_bc_r(v.wall_in, dev(v.g_in), v.wall_out, dev(v.g_out))
    ov = oracle_mod.vv_solve_problem(v)
    os_ = oracle_mod.solve_problem(p)
    for _ in range(2):
        x = dev(p.x0)
        st, info, hist = S.solve(dev(p.f), x, p.tol, p.maxit)
        assert st == 0 and np.array_equal(x.cpu().numpy(), os_["x"])
        xv = dev(v.x0)
        st, info, hist = S.vv_solve(dev(v.f), xv, v.tol, v.maxit)
        assert st == 0 and np.array_equal(xv.cpu().numpy(), ov["x"]) and np.array_equal(hist, ov["hist"])
    S.close()
    torch.cuda.synchronize()


# ------------------------------------------------------------------ multi-rank (loopback, one GPU)
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
        t.join(timeout=250)
    assert not any(t.is_alive() for t in th), "a rank hung"
    group.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("P,shape,walls", [(2, (7, 6, 8), (0, 1)), (3, (5, 9, 6), (0, 0)), (4, (8, 5, 8), (1, 1)),
                                           (4, (16, 16, 4), (0, 1)), (3, (8, 6, 9), (0, 1))])
def test_vv_multirank_exact(M, oracle_mod, monkeypatch, P, shape, walls):
    """phi-slabs on P loopback ranks: the diagonal of each slab, the iterates and the history equal the
    global oracle's bit for bit (nloc = 1 included), identical on every rank (even nr: the marching operator)."""
    full = inputs.make_vv_problem("rand", shape=shape, seed=P, wall_in=walls[0], wall_out=walls[1])
    o = oracle_mod.vv_solve_problem(full)
    op = o["op"]

    def fn(r, group):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        p = inputs.make_vv_problem("rand", k0, nloc, shape=shape, seed=P, wall_in=walls[0], wall_out=walls[1])
        return gpu_vv_solve(M, p, loopback=(group, r))

    res = run_ranks(M, P, fn)
    xs = np.concatenate([r[3] for r in res], axis=0)
    Ds = np.concatenate([r[4] for r in res], axis=0)
    assert np.array_equal(Ds, op.D)
    for st, info, hist, *_ in res:
        assert st == o["status"] == 0 and info["iters"] == o["iters"]
        assert np.array_equal(hist, o["hist"])
    assert np.array_equal(xs, o["x"])


@pytest.mark.parametrize("ring", [3, 4, 7])
@pytest.mark.parametrize("shape,walls", [((8, 4, 9), (0, 1)), ((16, 16, 32), (1, 0)), ((20, 30, 48), (0, 1))])
def test_vv_chunked_operator_exact(M, oracle_mod, monkeypatch, ring, shape, walls):
    """The chunked matvec (the default on large slabs: the phase-1 terms of ring - 2 planes at a time in
    L2-resident rings, then that chunk's rows; the rows' Dot2 pairs combined per chunk, then in chunk
    order): apply and whole solves identical to the oracle.  MASPCG_VV_CHUNK forces a ring size on these
    small grids (ring 3: one plane per chunk)."""
    import torch
    monkeypatch.setenv("MASPCG_VV_CHUNK", str(ring))
    p = inputs.make_vv_problem("rand", shape=shape, seed=21 + ring, wall_in=walls[0], wall_out=walls[1])
    op = oracle_op(oracle_mod, p)
    S = gpu_solver(M, p)
    x = np.stack([inputs.white_noise(81 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1)
    y = S.vv_apply(dev(x))
    torch.cuda.synchronize()
    S.close()
    assert np.array_equal(y.cpu().numpy(), op.apply(x))
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, xs, _, _ = gpu_vv_solve(M, p)
    assert st == o["status"] == 0 and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(xs, o["x"])


def test_vv_chunked_multirank_exact(M, oracle_mod, monkeypatch):
    """Chunked matvec on 2 loopback ranks (4 chunks per slab)."""
    monkeypatch.setenv("MASPCG_VV_CHUNK", "4")
    shape = (10, 8, 16)
    full = inputs.make_vv_problem("rand", shape=shape, seed=31)
    o = oracle_mod.vv_solve_problem(full)

    def fn(r, group):
        k0, nloc = inputs.slab_extent(full.np, r, 2)
        p = inputs.make_vv_problem("rand", k0, nloc, shape=shape, seed=31)
        return gpu_vv_solve(M, p, loopback=(group, r))

    res = run_ranks(M, 2, fn)
    for st, info, hist, *_ in res:
        assert st == o["status"] == 0 and info["iters"] == o["iters"] and np.array_equal(hist, o["hist"])
    assert np.array_equal(np.concatenate([r[3] for r in res], axis=0), o["x"])


# ------------------------------------------------------------------ the plane-marching TMA operator (vv_march.cu)
@pytest.mark.parametrize("tj,grid", [(None, None), (1, None), (3, 5), (2, 1)])
@pytest.mark.parametrize("shape,walls", [((8, 4, 2), (0, 1)), ((16, 16, 32), (1, 0)), ((20, 30, 48), (0, 1)),
                                         ((2, 5, 3), (0, 0)), ((6, 9, 7), (1, 1))])
def test_vv_march_operator_exact(M, oracle_mod, monkeypatch, tj, grid, shape, walls):
    """The default operator for even nr: one plane-marching kernel per matvec whose p planes and coefficient
    rows arrive by bulk copies (vv_march.cu).  Apply and whole solves identical to the oracle; forced small
    tiles (ragged last tile, halo rows at both ends) and forced small grids (several tile/plane segments per
    block, the rings carried across segments)."""
    import torch
    if tj:
        monkeypatch.setenv("MASPCG_VV_MARCH_TJ", str(tj))
    if grid:
        monkeypatch.setenv("MASPCG_VV_MARCH_GRID", str(grid))
    p = inputs.make_vv_problem("rand", shape=shape, seed=41 + sum(shape), wall_in=walls[0], wall_out=walls[1])
    op = oracle_op(oracle_mod, p)
    S = gpu_solver(M, p)
    x = np.stack([inputs.white_noise(61 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1)
    y = S.vv_apply(dev(x))
    torch.cuda.synchronize()
    S.close()
    assert np.array_equal(y.cpu().numpy(), op.apply(x))
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, xs, _, _ = gpu_vv_solve(M, p)
    assert st == o["status"] == 0 and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(xs, o["x"])


@pytest.mark.parametrize("shape", [(16, 16, 32), (20, 30, 48)])
def test_vv_two_phase_operator_exact(M, oracle_mod, monkeypatch, shape):
    """MASPCG_VV_MARCH=0: the two-phase kernels (terms, then rows) stay bit-identical too."""
    import torch
    monkeypatch.setenv("MASPCG_VV_MARCH", "0")
    p = inputs.make_vv_problem("rand", shape=shape, seed=5 + sum(shape), wall_in=0, wall_out=1)
    op = oracle_op(oracle_mod, p)
    S = gpu_solver(M, p)
    x = np.stack([inputs.white_noise(71 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1)
    y = S.vv_apply(dev(x))
    torch.cuda.synchronize()
    S.close()
    assert np.array_equal(y.cpu().numpy(), op.apply(x))
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, xs, _, _ = gpu_vv_solve(M, p)
    assert st == o["status"] == 0 and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(xs, o["x"])


@pytest.mark.parametrize("P,shape", [(2, (10, 8, 16)), (4, (8, 13, 8)), (3, (4, 7, 9))])
def test_vv_march_multirank_exact(M, oracle_mod, monkeypatch, P, shape):
    """The marching operator on phi-slabs (halo planes of p from the loopback exchange), forced small tiles
    and grids: iterates and history equal the global oracle's on every rank."""
    monkeypatch.setenv("MASPCG_VV_MARCH_TJ", "3")
    monkeypatch.setenv("MASPCG_VV_MARCH_GRID", "4")
    full = inputs.make_vv_problem("rand", shape=shape, seed=50 + P, wall_in=0, wall_out=1)
    o = oracle_mod.vv_solve_problem(full)

    def fn(r, group):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        p = inputs.make_vv_problem("rand", k0, nloc, shape=shape, seed=50 + P, wall_in=0, wall_out=1)
        return gpu_vv_solve(M, p, loopback=(group, r))

    res = run_ranks(M, P, fn)
    for st, info, hist, *_ in res:
        assert st == o["status"] == 0 and info["iters"] == o["iters"] and np.array_equal(hist, o["hist"])
    assert np.array_equal(np.concatenate([r[3] for r in res], axis=0), o["x"])


@pytest.mark.parametrize("name,shape", [("c2v", None), ("rand", (16, 16, 32))])
def test_vv_fast_arithmetic_tolerance_contract(M, oracle_mod, name, shape):
    """MASPCG_OPT_ARITH = 1 (FMA-contracted updates, plain dot sums) through the marching operator: the tolerance
    contract of BASELINE.json (solution relative L2 <= 1e-10 against the oracle, iterations +-1)."""
    p = inputs.make_vv_problem(name, shape=shape, seed=3) if shape else inputs.make_vv_problem(name)
    o = oracle_mod.vv_solve_problem(p)
    st, info, hist, x, _, _ = gpu_vv_solve(M, p, opts={M.OPT_ARITH: M.ARITH_FAST})
    assert st == o["status"] == 0
    assert abs(info["iters"] - o["iters"]) <= 1
    assert np.linalg.norm(x - o["x"]) <= 1e-10 * np.linalg.norm(o["x"])
