"""Breakdown and non-finite edge cases, GPU against the oracle (-m gpu; the oracle side alone is pinned in
tests/test_oracle_pins.py::test_breakdown_from_an_isolated_singular_pair).

SURVEY 8(c) item 4: a connected component of the face graph with no shift and no Dirichlet face makes A
singular there; the global check (E_SINGULAR) cannot see it, and PCG surfaces it as E_BREAKDOWN (p.Ap = 0).
The case below isolates two phi-neighbour cells (kappa = 0 on their 10 outer faces, s = 0 on them) and puts
the whole rhs on them with equal values: p_0 is constant on the pair, A p_0 = 0 exactly and p.Ap = 0 in
the first iteration on both sides.  A NaN in x_0 makes r_0 non-finite: E_BREAKDOWN before the loop.
"""
import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_2303_03398_b200 import build, maspcg
    build.build()
    return maspcg


def isolated_pair_problem(**kw):
    return inputs.isolated_pair_problem(**kw)


def run(M, p, x0=None):
    import torch
    S = M.solver_for_problem(p)
    x = torch.from_numpy(p.x0 if x0 is None else x0).cuda()
    st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, p.tol, p.maxit, raise_on_error=False)
    torch.cuda.synchronize()
    out = (st, info["iters"], hist, x.cpu().numpy())
    S.close()
    return out


@pytest.mark.parametrize("vec", [0, 1])
def test_breakdown_isolated_singular_pair(M, oracle_mod, vec):
    p = isolated_pair_problem(nr=8 if vec else 9)
    o = oracle_mod.solve_problem(p)
    assert o["status"] == oracle_mod.E_BREAKDOWN and o["iters"] == 0
    st, iters, hist, x = run(M, p)
    assert st == M.E_BREAKDOWN and iters == o["iters"]
    assert hist[0] == o["hist"][0]
    assert np.array_equal(x, o["x"])


def test_nan_initial_guess(M, oracle_mod):
    p = inputs.random_problem(9, 6, 4, 21)
    x0 = np.zeros_like(p.x0)
    x0[1, 2, 3] = np.nan
    o = oracle_mod.solve_problem(p, x0=x0)
    assert o["status"] == oracle_mod.E_BREAKDOWN and o["iters"] == 0
    st, iters, hist, x = run(M, p, x0=x0)
    assert st == M.E_BREAKDOWN and iters == 0
