"""The peer-memory communicator (maspcg_create_peer; SURVEY 8(e) lever 4) on one B200 (-m gpu).

Exchanges are kernels that store into the receiving rank's workspace and signal with system-scope
release flags; receivers spin on acquire loads -- no NCCL, no host round trip, captured into the CUDA
graphs.  One process per rank (one CUDA context each; the workspaces are mapped with CUDA IPC handles
all-gathered over gloo) -- here several processes share the one device, which time-slices their
contexts; on an 8-GPU node the same mappings go over NVLink.  The decomposed solves must reproduce the
global oracle bit for bit (R24): three-kernel and single-reduction paths, super-time-stepping (halo
planes of rotating buffers with no all-gather between stages) and the vector viscosity (3-component
halos, pole-ring all-gathers).  One rank alone pushes to itself.
"""
import os
import socket
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


def solve(M, prob, path, graphs=1, loopback=None, fuse_halo=1):
    import torch
    S = M.solver_for_problem(prob, loopback=loopback, comm="peer")
    try:
        S.set_option(M.OPT_PATH, path)
        S.set_option(M.OPT_USE_GRAPHS, graphs)
        S.set_option(M.OPT_FUSE_HALO, fuse_halo)
        x = dev(prob.x0)
        st, info, hist = S.solve(dev(prob.f), x, prob.tol, prob.maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        return st, info, hist, x.cpu().numpy()
    finally:
        S.close()


@pytest.mark.parametrize("path,fuse_halo", [(1, 1), (1, 2), (1, 0), (4, 1)])
@pytest.mark.parametrize("graphs", [1, 0])
def test_peer_single_rank(M, oracle_mod, path, fuse_halo, graphs):
    """One rank: every halo plane and all-gather goes through the push kernels to itself (fuse_halo 2:
    the stencil blocks acquire the halo flags themselves)."""
    p = inputs.make_problem("c1")
    o = oracle_mod.solve_problem(p, variant="hs" if path == 1 else "cg1")
    st, info, hist, x = solve(M, p, path, graphs, fuse_halo=fuse_halo)
    assert st == 0 and info["iters"] == o["iters"]
    assert np.array_equal(hist, o["hist"]) and np.array_equal(x, o["x"])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, out_dir):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_03398_b200 import maspcg
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = {}
    try:
        # scalar solves, three-kernel and single-reduction paths
        for name, fn in [("c1", lambda k0, n: inputs.make_problem("c1", k0, n)),
                         ("rand", lambda k0, n: inputs.random_problem(10, 6, 8, 31, bc_in=0, bc_out=1,
                                                                      k0=k0 or 0, nloc=n))]:
            k0, nloc = inputs.slab_extent(fn(None, None).np, rank, world)
            p = fn(k0, nloc)
            for path in (1, 4, "1nofuse", "1acquire"):
                S = maspcg.solver_for_problem(p, comm="peer")   # CUDA IPC handles all-gathered over gloo
                S.set_option(maspcg.OPT_PATH, 4 if path == 4 else 1)
                if path == 1:   # halo stores in the p-update, a wait kernel before a split stencil
                    S.set_option(maspcg.OPT_FUSE_HALO, 1)
                if path == "1nofuse":   # the halo push as its own kernel instead of inside the p-update
                    S.set_option(maspcg.OPT_FUSE_HALO, 0)
                if path == "1acquire":   # the stencil blocks acquire the halo flags (one stencil launch)
                    S.set_option(maspcg.OPT_FUSE_HALO, 2)
                x = T(p.x0)
                st, info, hist = S.solve(T(p.f), x, p.tol, p.maxit)
                torch.cuda.synchronize()
                out[(name, path)] = (st, info["iters"], hist, x.cpu().numpy())
                if name == "rand" and path == 1:   # super-time-stepping on the same operator
                    dt = S.sts_dt_limit()
                    u0 = np.random.default_rng(1).standard_normal((p.np, p.nt, p.nr))
                    u = T(u0[k0:k0 + nloc])
                    S.sts_step(u, 0.9 * 28 * dt, 8)
                    torch.cuda.synchronize()
                    out["sts"] = (dt, u.cpu().numpy())
                dist.barrier()
                S.close()
        # vector viscosity
        k0, nloc = inputs.slab_extent(8, rank, world)
        pv = inputs.make_vv_problem("rand", k0, nloc, shape=(6, 5, 8), seed=5)
        S = maspcg.Solver(pv.nr, pv.nt, pv.np, pv.rf, pv.tf, pv.pf, comm="peer")
        S.vv_set_coefficients(T(pv.nu), T(pv.s))
        S.vv_set_bc_r(pv.wall_in, T(pv.g_in), pv.wall_out, T(pv.g_out))
        x = T(pv.x0)
        st, info, hist = S.vv_solve(T(pv.f), x, pv.tol, pv.maxit)
        torch.cuda.synchronize()
        out["vv"] = (st, info["iters"], hist, x.cpu().numpy())
        dist.barrier()
        S.close()
        np.save(os.path.join(out_dir, f"ipc{rank}.npy"), out, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_processes_ipc(tmp_path, oracle_mod, world):
    """world processes on the same device, workspaces mapped with CUDA IPC (the multi-process path of
    the peer communicator; on an 8-GPU node the same mapping goes over NVLink)."""
    import torch.multiprocessing as mp
    mp.spawn(_ipc_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"ipc{r}.npy", allow_pickle=True).item() for r in range(world)]
    probs = {"c1": inputs.make_problem("c1"), "rand": inputs.random_problem(10, 6, 8, 31, bc_in=0, bc_out=1)}
    for name, p in probs.items():
        for path in (1, 4, "1nofuse", "1acquire"):
            o = oracle_mod.solve_problem(p, variant="cg1" if path == 4 else "hs")
            for r in res:
                st, it, hist, _ = r[(name, path)]
                assert st == o["status"] == 0 and it == o["iters"] and np.array_equal(hist, o["hist"]), (name, path)
            assert np.array_equal(np.concatenate([r[(name, path)][3] for r in res], axis=0), o["x"]), (name, path)
    p = probs["rand"]
    op = oracle_mod.Operator(p.rf, p.tf, p.pf, p.kr, p.kt, p.kp, p.s, p.bc_in, p.bc_out)
    dt = res[0]["sts"][0]
    assert all(r["sts"][0] == dt for r in res)
    u0 = np.random.default_rng(1).standard_normal(op.shape)
    assert np.array_equal(np.concatenate([r["sts"][1] for r in res], axis=0),
                          op.rkl2_step(u0, p.s, 0.9 * 28 * dt, 8, p.g_in, p.g_out))
    ov = oracle_mod.vv_solve_problem(inputs.make_vv_problem("rand", shape=(6, 5, 8), seed=5))
    for r in res:
        st, it, hist, _ = r["vv"]
        assert st == 0 and it == ov["iters"] and np.array_equal(hist, ov["hist"])
    assert np.array_equal(np.concatenate([r["vv"][3] for r in res], axis=0), ov["x"])


def test_peer_single_rank_vv_and_group_rejected(M, oracle_mod):
    import torch
    v = inputs.make_vv_problem("rand", shape=(6, 5, 8), seed=5)
    ov = oracle_mod.vv_solve_problem(v)
    S = M.Solver(v.nr, v.nt, v.np, v.rf, v.tf, v.pf, comm="peer")
    S.vv_set_coefficients(dev(v.nu), dev(v.s))
    S.vv_set_bc_r(v.wall_in, dev(v.g_in), v.wall_out, dev(v.g_out))
    x = dev(v.x0)
    st, info, hist = S.vv_solve(dev(v.f), x, v.tol, v.maxit)
    torch.cuda.synchronize()
    assert st == 0 and np.array_equal(hist, ov["hist"]) and np.array_equal(x.cpu().numpy(), ov["x"])
    S.set_option(M.OPT_PATH, 2)     # the fused path is not available in peer mode
    p = inputs.make_problem("c1")
    S2 = M.solver_for_problem(p, comm="peer")
    S2.set_option(M.OPT_PATH, 2)
    st, _, _ = S2.solve(dev(p.f), dev(p.x0), p.tol, p.maxit, raise_on_error=False)
    assert st == M.E_INVALID
    S2.close()
    S.close()
    g = M.LoopbackGroup(2)
    with pytest.raises(M.MaspcgError):
        M.Solver(4, 4, 8, inputs.rfaces(4, 1, 2, 0), inputs.tfaces(4, 0.0), inputs.pfaces(8), loopback=(g, 0),
                 comm="peer")
    g.close()


def test_peer_single_rank_c3_full_size(M, oracle_mod):
    """The full c3 grid through the peer communicator with one rank (halo stores into its own halos by
    the p-update, the stencil acquiring them, LL pair words to itself): 20 iterations bit for bit."""
    p = inputs.make_problem("c3")
    o = oracle_mod.solve_problem(p, tol=0.0, maxit=20)
    p.tol, p.maxit = 0.0, 20
    st, info, hist, x = solve(M, p, 1, 1, fuse_halo=2)
    assert info["iters"] == 20 and np.array_equal(hist, o["hist"]) and np.array_equal(x, o["x"])


def _stress_worker(rank, world, port, out_dir):
    """Many peer-mode iterations with random per-rank delays: a host sleep and a GPU spin kernel of random
    length before every solve, so the ranks' stencils start at different times and the halo acquire / the
    coherent halo loads (DESIGN 9; ld.global.cg after ld.acquire.sys) are exercised under skew."""
    import sys
    import time
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_03398_b200 import maspcg
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    rng = np.random.default_rng(1000 + rank)
    out = {}
    try:
        for name, fn in [("rand", lambda k0, n: inputs.random_problem(12, 10, 8, 41, k0=k0 or 0, nloc=n)),
                         ("aniso", lambda k0, n: inputs.random_aniso_problem(12, 10, 8, 42, k0=k0 or 0, nloc=n))]:
            k0, nloc = inputs.slab_extent(8, rank, world)
            p = fn(k0, nloc)
            S = maspcg.solver_for_problem(p, comm="peer")
            S.set_option(maspcg.OPT_FUSE_HALO, 2)     # the stencil blocks acquire the halo flags themselves
            for rep in range(6):
                time.sleep(float(rng.uniform(0.0, 0.03)))
                torch.cuda._sleep(int(rng.integers(0, 2_000_000)))   # a GPU-side delay on this rank's stream
                x = T(p.x0)
                st, info, hist = S.solve(T(p.f), x, 0.0, 300)
                torch.cuda.synchronize()
                out[(name, rep)] = (st, info["iters"], hist, x.cpu().numpy())
            dist.barrier()
            S.close()
        np.save(os.path.join(out_dir, f"stress{rank}.npy"), out, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_stress_random_delays(tmp_path, oracle_mod, world):
    """world processes, 300 iterations x 6 solves each of the 7-point and the field-aligned operators with
    random host and GPU delays per rank before every solve: every solve equals the oracle's 300 iterates
    bit for bit on every rank."""
    import torch.multiprocessing as mp
    mp.spawn(_stress_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"stress{r}.npy", allow_pickle=True).item() for r in range(world)]
    ref = {"rand": oracle_mod.solve_problem(inputs.random_problem(12, 10, 8, 41), tol=0.0, maxit=300),
           "aniso": oracle_mod.solve_aniso_problem(inputs.random_aniso_problem(12, 10, 8, 42), tol=0.0, maxit=300)}
    for name, o in ref.items():
        for rep in range(6):
            for r in res:
                st, it, hist, _ = r[(name, rep)]
                assert st == o["status"] and it == o["iters"] == 300 and np.array_equal(hist, o["hist"]), (name, rep)
            x = np.concatenate([r[(name, rep)][3] for r in res], axis=0)
            assert np.array_equal(x, o["x"]), (name, rep)
