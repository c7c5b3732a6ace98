"""GPU parity of the single-reduction (Chronopoulos-Gear) PCG path, MASPCG_OPT_PATH = 4 (-m gpu).

SURVEY 8(f) NEXT-3 / reading R32: one operator application and one fused reduction (r.u, w.u, r.r) per
iteration -- one all-reduce instead of two across phi-slabs.  Compared through the C ABI with the
oracle's own single-reduction variant (oracle masoracle_pcg_cg1, pinned in test_oracle_pins.py against
dense LU and against CG in exact arithmetic): x, the iteration count and every residual-history entry
are identical (np.array_equal) -- single rank (16-byte pair kernels and, for odd nr, one cell per
thread), every CUDA-graph chunking, and 2-8 loopback ranks with the r halo overlapped with the interior
of the matvec.
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


def gpu_cg1(M, prob, tol=None, maxit=None, chunk=16, loopback=None, opts=None, x0=None):
    import torch
    S = M.solver_for_problem(prob, chunk=chunk, loopback=loopback)
    try:
        S.set_option(M.OPT_PATH, 4)
        for k, v in (opts or {}).items():
            S.set_option(k, v)
        x = dev(prob.x0 if x0 is None else x0)
        st, info, hist = S.solve(dev(prob.f), x, prob.tol if tol is None else tol,
                                 prob.maxit if maxit is None else maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        return st, info, hist, x.cpu().numpy(), S.stats()
    finally:
        S.close()


def assert_same(g, o):
    st, info, hist, x, stats = g
    assert st == o["status"], (st, o["status"], info)
    assert info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]), np.abs(hist - o["hist"]).max()
    assert np.array_equal(x, o["x"]), np.abs(x - o["x"]).max()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_cg1_configs_exact(M, oracle_mod, name):
    p = inputs.make_problem(name)
    o = oracle_mod.solve_problem(p, variant="cg1")
    g = gpu_cg1(M, p)
    assert_same(g, o)
    assert g[4]["path"] == 4


SHAPES = [(13, 7, 5), (33, 17, 9), (1, 5, 6), (6, 1, 4), (5, 4, 1), (40, 3, 2), (64, 32, 8)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bc", [(0, 1), (0, 0), (1, 0)])
def test_cg1_random_exact(M, oracle_mod, shape, bc):
    nr, nt, np_ = shape
    p = inputs.random_problem(nr, nt, np_, 300 + nr + nt + np_, bc_in=bc[0], bc_out=bc[1])
    assert_same(gpu_cg1(M, p), oracle_mod.solve_problem(p, variant="cg1"))


@pytest.mark.parametrize("chunk,graphs,vec", [(1, 1, 1), (7, 1, 1), (16, 0, 1), (16, 1, 0)])
def test_cg1_loop_modes(M, oracle_mod, chunk, graphs, vec):
    p = inputs.make_problem("c2", shape=(32, 32, 64), x0_seed=3)
    o = oracle_mod.solve_problem(p, variant="cg1")
    assert_same(gpu_cg1(M, p, chunk=chunk, opts={M.OPT_USE_GRAPHS: graphs, M.OPT_VEC: vec}), o)


def test_cg1_edge_cases(M, oracle_mod):
    p = inputs.random_problem(9, 6, 8, 17)
    for tol, maxit in [(0.0, 7), (1e-10, 0), (1e-10, 1), (1e-3, 500)]:
        o = oracle_mod.solve_problem(p, tol=tol, maxit=maxit, variant="cg1")
        assert_same(gpu_cg1(M, p, tol=tol, maxit=maxit), o)
    q = inputs.random_problem(9, 6, 8, 17, bc_in=1, bc_out=1)
    q.f[:] = 0.0
    st, info, hist, x, _ = gpu_cg1(M, q)
    assert st == 0 and info["iters"] == 0 and not x.any()


def test_cg1_c3_half_resolution_exact(M, oracle_mod):
    """The c3 recipe at half resolution (3.4 M cells, ~225 iterations), the bench's launch configuration."""
    p = inputs.make_problem("c3", shape=(75, 150, 300))
    assert_same(gpu_cg1(M, p), oracle_mod.solve_problem(p, variant="cg1"))


def test_cg1_c3_full_size_exact(M, oracle_mod):
    """The full c3 grid (27 M cells) in the bench's launch configuration (graphs, chunk 16): 12 fixed
    iterations of the single-reduction path identical to the oracle's variant."""
    p = inputs.make_problem("c3")
    o = oracle_mod.solve_problem(p, tol=0.0, maxit=12, variant="cg1")
    assert_same(gpu_cg1(M, p, tol=0.0, maxit=12), o)


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


CASES = [
    ("c1", 2, lambda k0, n: inputs.make_problem("c1", k0, n)),
    ("c1", 4, lambda k0, n: inputs.make_problem("c1", k0, n)),
    ("c2", 2, lambda k0, n: inputs.make_problem("c2", k0, n)),
    ("rand-np6", 3, lambda k0, n: inputs.random_problem(12, 5, 6, 6, bc_in=0, bc_out=0, k0=k0 or 0, nloc=n)),
    ("rand-np8", 8, lambda k0, n: inputs.random_problem(7, 6, 8, 7, bc_in=1, bc_out=0, k0=k0 or 0, nloc=n)),
]


@pytest.mark.parametrize("name,P,fn", CASES, ids=[f"{c[0]}-P{c[1]}" for c in CASES])
def test_cg1_multirank_exact(M, oracle_mod, name, P, fn):
    full = fn(None, None)
    o = oracle_mod.solve_problem(full, variant="cg1")

    def rank(r, g):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        return gpu_cg1(M, fn(k0, nloc), loopback=(g, r))

    res = run_ranks(M, P, rank)
    for st, info, hist, _, _ in res:
        assert st == o["status"] and info["iters"] == o["iters"] and np.array_equal(hist, o["hist"])
    assert np.array_equal(np.concatenate([r[3] for r in res], axis=0), o["x"])
