"""Multi-rank phi-slab decomposition on ONE GPU (-m gpu), through the C ABI's loopback group.

The loopback group (maspcg_loopback_group_create / maspcg_create_loopback) runs P ranks in one
process, one host thread each, replacing only the NCCL calls by device-to-device copies and
fixed-order sums.  Everything else is the production multi-rank path of SURVEY.md 8(e): local
slabs, the T_phi face fetched from the left rank, halo planes of p, the stencil split into
interior planes (overlapped with the halo on the communication stream) and boundary planes with
one combined deterministic reduction, and the all-reduced p.Ap, r.z, r.r, b.b and validation flags.
Results are compared with the global oracle (same contract as test_gpu_parity.py) and across ranks
(identical status, iteration count and residual history, bit for bit).
"""
import threading

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


def run_ranks(M, P, fn):
    """Run fn(rank, group) on P threads, each with its own CUDA stream; returns the results."""
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
        except BaseException as e:  # noqa: BLE001 -- re-raised in the main thread
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


def slab_of(prob_fn, P, r):
    """The generator evaluated on rank r's slab (decomposition-independent)."""
    full = prob_fn(None, None)
    k0, nloc = inputs.slab_extent(full.np, r, P)
    return prob_fn(k0, nloc)


def solve_rank(M, prob, r, group, tol=None, maxit=None, path=0):
    import torch
    S = M.solver_for_problem(prob, loopback=(group, r))
    S.set_option(M.OPT_PATH, path)
    x = torch.from_numpy(prob.x0.copy()).cuda()
    st, info, hist = S.solve(torch.from_numpy(prob.f).cuda(), x, prob.tol if tol is None else tol,
                             prob.maxit if maxit is None else maxit, raise_on_error=False)
    torch.cuda.current_stream().synchronize()
    res = (st, info, hist, x.cpu().numpy(), S.get_operator())
    S.close()
    return res


CASES = [
    ("c1", 1, lambda k0, n: inputs.make_problem("c1", k0, n)),   # one rank with a communicator: halo to itself
    ("c1", 2, lambda k0, n: inputs.make_problem("c1", k0, n)),
    ("c1", 4, lambda k0, n: inputs.make_problem("c1", k0, n)),
    ("c2", 2, lambda k0, n: inputs.make_problem("c2", k0, n)),
    ("rand-np2", 2, lambda k0, n: inputs.random_problem(9, 7, 2, 5, k0=k0 or 0, nloc=n)),
    ("rand-np6", 3, lambda k0, n: inputs.random_problem(12, 5, 6, 6, bc_in=0, bc_out=0, k0=k0 or 0, nloc=n)),
    ("rand-np8", 8, lambda k0, n: inputs.random_problem(7, 6, 8, 7, bc_in=1, bc_out=0, k0=k0 or 0, nloc=n)),
]


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("name,P,fn", CASES, ids=[f"{c[0]}-P{c[1]}" for c in CASES])
def test_multirank_solve_matches_oracle(M, oracle_mod, name, P, fn, path):
    full = fn(None, None)
    o = oracle_mod.solve_problem(full)
    res = run_ranks(M, P, lambda r, g: solve_rank(M, slab_of(fn, P, r), r, g, path=path))
    # every rank agrees bit for bit on the scalars of the solve
    errs = [(r[0], r[1].get("error")) for r in res]
    assert all(r[0] >= 0 for r in res), f"rank errors: {errs}"
    for st, info, hist, _, _ in res[1:]:
        assert st == res[0][0] and info == res[0][1] and np.array_equal(hist, res[0][2])
    st, info, hist = res[0][:3]
    x = np.concatenate([r[3] for r in res], axis=0)
    # R24 arithmetic: the decomposed solve reproduces the oracle's iterates bit for bit
    assert info["iters"] == o["iters"] and np.array_equal(hist, o["hist"]) and np.array_equal(x, o["x"])
    assert st == o["status"] and abs(info["iters"] - o["iters"]) <= 1
    assert np.linalg.norm(x - o["x"]) <= 1e-10 * np.linalg.norm(o["x"])
    from test_gpu_parity import assert_hist
    assert_hist(hist, o["hist"], o["bnorm"])
    # the assembled operator of every slab is the bitwise slice of the global one
    op = o["op"]
    for r, (_, _, _, _, (Tr, Tt, Tp, D)) in enumerate(res):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        sl = slice(k0, k0 + nloc)
        assert np.array_equal(Tr, op.Tr[sl]) and np.array_equal(Tt, op.Tt[sl])
        assert np.array_equal(Tp, op.Tp[sl]) and np.array_equal(D, op.D[sl])


@pytest.mark.parametrize("nr", [63, 64])
def test_multirank_large_slab_split_reduction(M, oracle_mod, nr):
    """A slab whose interior and boundary stencil launches together have more blocks than one launch may
    (odd nr, one cell per thread: 1,184 + 32 blocks; even nr: the 16-byte pair kernels): the p.q partial
    slots of both launches must not overlap.  Five iterations, bit for bit against the oracle."""
    fn = lambda k0, n: inputs.random_problem(nr, 64, 160, 41, k0=k0 or 0, nloc=n)
    full = fn(None, None)
    o = oracle_mod.solve_problem(full, tol=0.0, maxit=5)
    res = run_ranks(M, 2, lambda r, g: solve_rank(M, slab_of(fn, 2, r), r, g, tol=0.0, maxit=5, path=1))
    for st, info, hist, _, _ in res:
        assert info["iters"] == 5 and np.array_equal(hist, o["hist"])
    assert np.array_equal(np.concatenate([r[3] for r in res], axis=0), o["x"])


@pytest.mark.parametrize("P", [2, 4])
def test_multirank_apply(M, oracle_mod, P):
    import torch
    fn = lambda k0, n: inputs.random_problem(11, 6, 8, 21, k0=k0 or 0, nloc=n)
    full = fn(None, None)
    xg = np.random.default_rng(3).standard_normal((full.np, full.nt, full.nr))

    def rank(r, g):
        p = slab_of(fn, P, r)
        S = M.solver_for_problem(p, loopback=(g, r))
        y = S.apply(torch.from_numpy(xg[p.k0:p.k0 + p.nloc].copy()).cuda()).cpu().numpy()
        S.close()
        return y

    y = np.concatenate(run_ranks(M, P, rank), axis=0)
    op = oracle_mod.Operator(full.rf, full.tf, full.pf, full.kr, full.kt, full.kp, full.s, full.bc_in, full.bc_out)
    mag = 2.0 * op.D * np.abs(xg) - op.apply(np.abs(xg))
    assert (np.abs(y - op.apply(xg)) / mag).max() <= 1e-14


def test_multirank_errors_agree(M):
    """A negative coefficient on one rank only: every rank returns E_INVALID (all-reduced flags)."""
    import torch
    fn = lambda k0, n: inputs.random_problem(6, 5, 4, 9, k0=k0 or 0, nloc=n)

    def rank(r, g):
        p = slab_of(fn, 2, r)
        S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, loopback=(g, r))
        kr = p.kr.copy()
        if r == 1:
            kr[0, 1, 2] = -3.0
        T = lambda a: torch.from_numpy(a).cuda()
        try:   # the validation is reported by the first call that uses the operator (deferred, no host sync)
            S.set_coefficients(T(kr), T(p.kt), T(p.kp), T(p.s))
            S.get_operator()
            return M.OK
        except M.MaspcgError as e:
            return e.status
        finally:
            S.close()

    assert run_ranks(M, 2, rank) == [M.E_INVALID, M.E_INVALID]


@pytest.mark.parametrize("P", [2, 3])
def test_multirank_coefficients_from_fields(M, oracle_mod, P):
    """NEXT-1 across ranks: the phi face of each slab's last plane needs the right neighbour's first
    plane of the field (exchanged); every slab operator equals the oracle's slice bit for bit."""
    import torch
    fn = lambda k0, n: inputs.random_problem(10, 7, 6, 33, k0=k0 or 0, nloc=n)
    full = fn(None, None)
    T = np.random.default_rng(P).uniform(0.4, 2.0, (full.np, full.nt, full.nr))

    def rank(r, g):
        p = slab_of(fn, P, r)
        S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, loopback=(g, r))
        Tl = torch.from_numpy(T[p.k0:p.k0 + p.nloc].copy()).cuda()
        S.set_coefficients_from_fields(Tl, 1.3, 5, M.MEAN_HARMONIC, None, 4.0)
        S.set_bc_r(p.bc_in, torch.from_numpy(p.g_in).cuda(), p.bc_out, None)
        ops = S.get_operator()
        S.close()
        return ops

    res = run_ranks(M, P, rank)
    kr, kt, kp, s = oracle_mod.face_coefficients(T, 1.3, 5, 1, None, 4.0)
    op = oracle_mod.Operator(full.rf, full.tf, full.pf, kr, kt, kp, s, full.bc_in, full.bc_out)
    for r, (Tr, Tt, Tp, D) in enumerate(res):
        k0, nloc = inputs.slab_extent(full.np, r, P)
        sl = slice(k0, k0 + nloc)
        assert np.array_equal(Tr, op.Tr[sl]) and np.array_equal(Tt, op.Tt[sl])
        assert np.array_equal(Tp, op.Tp[sl]) and np.array_equal(D, op.D[sl])


@pytest.mark.parametrize("P", [2, 4])
def test_multirank_sts_step(M, oracle_mod, P):
    """RKL2 stages across ranks (one halo exchange per stage): bitwise equal to the oracle."""
    import torch
    fn = lambda k0, n: inputs.random_problem(10, 6, 8, 44, bc_in=0, bc_out=1, k0=k0 or 0, nloc=n)
    full = fn(None, None)
    u0 = np.random.default_rng(P).standard_normal((full.np, full.nt, full.nr))
    op = oracle_mod.Operator(full.rf, full.tf, full.pf, full.kr, full.kt, full.kp, full.s, full.bc_in, full.bc_out)

    def rank(r, g):
        p = slab_of(fn, P, r)
        S = M.solver_for_problem(p, loopback=(g, r))
        dt = S.sts_dt_limit()
        u = torch.from_numpy(u0[p.k0:p.k0 + p.nloc].copy()).cuda()
        for _ in range(2):
            S.sts_step(u, 0.8 * 20 * dt, 5)
        out = (dt, u.cpu().numpy())
        S.close()
        return out

    res = run_ranks(M, P, rank)
    dts = {r[0] for r in res}
    assert len(dts) == 1
    dt = dts.pop()
    uo = u0.copy()
    for _ in range(2):
        uo = op.rkl2_step(uo, full.s, 0.8 * 20 * dt, 5, full.g_in, full.g_out)
    assert np.array_equal(np.concatenate([r[1] for r in res], axis=0), uo)
