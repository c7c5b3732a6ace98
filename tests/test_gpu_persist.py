"""GPU parity of the persistent iteration kernel, MASPCG_OPT_PATH = 5 (-m gpu): one cooperative launch per
chunk of iterations, grid-wide barriers between the stencil, update and p-update phases.  Same
arithmetic and the same Dot2 partial combination as the three-kernel path, so the iterates are the
oracle's bit for bit (R24)."""
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


def run(M, p, tol=None, maxit=None, chunk=16):
    import torch
    S = M.solver_for_problem(p, chunk=chunk)
    try:
        S.set_option(M.OPT_PATH, 5)
        x = torch.from_numpy(p.x0.copy()).cuda()
        st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, p.tol if tol is None else tol,
                                 p.maxit if maxit is None else maxit, raise_on_error=False)
        torch.cuda.synchronize()
        return st, info, hist, x.cpu().numpy(), S.stats()
    finally:
        S.close()


def same(g, o):
    st, info, hist, x, stats = g
    assert st == o["status"] and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(x, o["x"])


@pytest.mark.parametrize("name,shape", [("c1", None), ("c2", None), ("c3", (76, 150, 300))])
def test_persist_configs_exact(M, oracle_mod, name, shape):
    p = inputs.make_problem(name, shape=shape)
    g = run(M, p)
    same(g, oracle_mod.solve_problem(p))
    assert g[4]["path"] == 6


@pytest.mark.parametrize("shape", [(14, 7, 5), (32, 17, 9), (40, 3, 2), (2, 5, 6)])
@pytest.mark.parametrize("bc", [(0, 1), (1, 0)])
def test_persist_random_exact(M, oracle_mod, shape, bc):
    p = inputs.random_problem(*shape, 500 + sum(shape), bc_in=bc[0], bc_out=bc[1])
    same(run(M, p), oracle_mod.solve_problem(p))


@pytest.mark.parametrize("chunk", [1, 7, 64])
def test_persist_chunks_and_edges(M, oracle_mod, chunk):
    p = inputs.make_problem("c2", shape=(32, 32, 64), x0_seed=3)
    same(run(M, p, chunk=chunk), oracle_mod.solve_problem(p))
    for tol, maxit in [(0.0, 9), (1e-10, 0), (1e-3, 500)]:
        same(run(M, p, tol=tol, maxit=maxit, chunk=chunk), oracle_mod.solve_problem(p, tol=tol, maxit=maxit))
