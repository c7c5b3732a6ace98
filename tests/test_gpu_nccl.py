"""The NCCL communicator on ONE GPU (-m gpu): a one-rank NCCL communicator (maspcg_create with
nranks = 1 and a unique id) runs the multi-rank code path for real -- ncclCommInitRank +
ncclCommSplit, grouped ncclSend/ncclRecv of the halo planes (to itself: the periodic phi wrap),
ncclAllGather of the Dot2 pairs, ncclAllReduce(max) of the validation flags -- including inside the
captured CUDA graphs.  Results must be the oracle's bit for bit (R24), as for the loopback ranks.
"""
import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_2303_03398_b200 import build, maspcg
    build.build()
    return maspcg


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("graphs", [1, 0])
@pytest.mark.parametrize("name", ["c1", "rand"])
def test_nccl_single_rank_solve(M, oracle_mod, name, path, graphs):
    import torch
    p = inputs.make_problem("c1") if name == "c1" else inputs.random_problem(10, 6, 5, 31, bc_in=0, bc_out=1)
    o = oracle_mod.solve_problem(p)
    S = M.solver_for_problem(p, force_comm=True)
    S.set_option(M.OPT_PATH, path)
    S.set_option(M.OPT_USE_GRAPHS, graphs)
    x = torch.from_numpy(p.x0.copy()).cuda()
    st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, p.tol, p.maxit)
    torch.cuda.synchronize()
    assert st == o["status"] and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(x.cpu().numpy(), o["x"])
    Tr, Tt, Tp, D = S.get_operator()
    op = o["op"]
    assert np.array_equal(Tp, op.Tp) and np.array_equal(D, op.D)
    S.close()


def test_nccl_single_rank_sts_and_invalid(M, oracle_mod):
    import torch
    p = inputs.random_problem(9, 5, 6, 32, bc_in=0, bc_out=0)
    S = M.solver_for_problem(p, force_comm=True)
    dt = S.sts_dt_limit()
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, 0, 0)
    u0 = np.random.default_rng(1).standard_normal(op.shape)
    u = torch.from_numpy(u0.copy()).cuda()
    S.sts_step(u, 0.9 * 28 * dt, 8)
    torch.cuda.synchronize()
    assert np.array_equal(u.cpu().numpy(), op.rkl2_step(u0, p.s, 0.9 * 28 * dt, 8, p.g_in, p.g_out))
    # validation flags go through ncclAllReduce(max): a negative coefficient is reported
    kr = p.kr.copy()
    kr[0, 0, 1] = -1.0
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    with pytest.raises(M.MaspcgError):
        S.set_coefficients(T(kr), T(p.kt), T(p.kp), T(p.s))
        x = torch.zeros(S.local_shape, dtype=torch.float64, device="cuda")
        S.solve(T(p.f), x, 1e-8, 10)
    S.close()
