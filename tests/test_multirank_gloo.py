"""Host logic of the N > 1 path on CPU (-m "not gpu"): world size 2 over torch.distributed/gloo.

What runs here is the decomposition protocol of SURVEY.md 8(e) that libmaspcg implements with
NCCL: phi-slab ownership (np % P == 0), slab inputs equal to slices of the global inputs, the T_phi
face below a slab taken from the left rank, halo planes of p (lo <- left's last plane, hi <- right's
first plane; at P = 2 both neighbours are the same rank), and dot products all-reduced so every rank
holds identical scalars.  The per-rank arithmetic is the oracle's global operator sliced to the
slab (test infrastructure), driven through gloo send/recv and all_reduce; the distributed PCG must
reproduce the global oracle solve.  The bench's max-over-ranks timing reduction is checked too.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2303_03398_b200 import inputs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = {}
        full = inputs.make_problem("c1")
        k0, nloc = inputs.slab_extent(full.np, rank, world)
        slab = inputs.make_problem("c1", k0, nloc)
        sl = slice(k0, k0 + nloc)
        for name in ("kr", "kt", "kp", "s", "f", "x0"):
            assert np.array_equal(getattr(slab, name), getattr(full, name)[sl]), name
        op = oracle.Operator(full.rf, full.tf, full.pf, full.kr, full.kt, full.kp, full.s, full.bc_in, full.bc_out)
        Tr, Tt, D = op.Tr[sl], op.Tt[sl], op.D[sl]
        Tp_hi = op.Tp[sl]
        L, R = (rank - 1) % world, (rank + 1) % world
        TO_LEFT, TO_RIGHT = 1, 2

        def exchange(first_send, last_send):
            """returns (lo halo = left's last plane, hi halo = right's first plane)."""
            lo, hi = torch.empty_like(first_send), torch.empty_like(first_send)
            reqs = [dist.isend(first_send, L, tag=TO_LEFT), dist.isend(last_send, R, tag=TO_RIGHT),
                    dist.irecv(hi, R, tag=TO_LEFT), dist.irecv(lo, L, tag=TO_RIGHT)]
            for q in reqs:
                q.wait()
            return lo.numpy(), hi.numpy()

        # T_phi face below the slab = the left rank's last face
        t_last = torch.from_numpy(np.ascontiguousarray(Tp_hi[-1]))
        t_lo, _ = exchange(t_last.clone(), t_last.clone())
        Tp_lo = np.concatenate([t_lo[None], Tp_hi[:-1]], axis=0)
        assert np.array_equal(Tp_lo, op.Tp[(np.arange(k0, k0 + nloc) - 1) % full.np])

        def apply(u):
            lo, hi = exchange(torch.from_numpy(u[0].copy()), torch.from_numpy(u[-1].copy()))
            um = np.concatenate([lo[None], u[:-1]], 0)
            up = np.concatenate([u[1:], hi[None]], 0)
            s = np.zeros_like(u)
            s[:, :, 1:] += Tr[:, :, 1:full.nr] * u[:, :, :-1]
            s[:, :, :-1] += Tr[:, :, 1:full.nr] * u[:, :, 1:]
            s[:, 1:, :] += Tt[:, 1:full.nt, :] * u[:, :-1, :]
            s[:, :-1, :] += Tt[:, 1:full.nt, :] * u[:, 1:, :]
            s += Tp_lo * um
            s += Tp_hi * up
            return D * u - s

        def split(a):
            c = 134217729.0 * a
            h = c - (c - a)
            return h, a - h

        def terms(a, b):
            """exact expansion of the local part of a.b: a_i b_i = h_i + r_i (TwoProduct)"""
            a, b = a.ravel(), b.ravel()
            h = a * b
            ah, al = split(a)
            bh, bl = split(b)
            return np.concatenate([h, al * bl - (((h - ah * bh) - al * bh) - ah * bl)])

        def allsum(*pairs):
            """global dot products, correctly rounded (R24): gather every rank's exact terms, fsum"""
            import math
            loc = [terms(a, b) for a, b in pairs]
            out = [None] * world
            dist.all_gather_object(out, loc)
            return [math.fsum(np.concatenate([o[k] for o in out])) for k in range(len(pairs))]

        # distributed apply == slice of the oracle's global apply
        u = np.random.default_rng(5).standard_normal(full.x0.shape)
        y = apply(u[sl].copy())
        ref = op.apply(u)[sl]
        mag = (2 * op.D * np.abs(u) - op.apply(np.abs(u)))[sl]
        res["apply_err"] = float((np.abs(y - ref) / mag).max())

        # distributed PCG with all-reduced scalars
        b = op.rhs(full.f, full.g_in, full.g_out)[sl]
        x = slab.x0.copy()
        r = b - apply(x)
        z = r / D
        p = z.copy()
        rho, rr, bb = allsum((r, z), (r, r), (b, b))
        bn = np.sqrt(bb)
        hist = [np.sqrt(rr)]
        it = 0
        for it in range(1, full.maxit + 1):
            q = apply(p)
            (pi,) = allsum((p, q))
            alpha = rho / pi
            x = x + alpha * p
            r = r - alpha * q
            z = r / D
            rz, rr = allsum((r, z), (r, r))
            hist.append(np.sqrt(rr))
            if hist[-1] <= full.tol * bn:
                break
            beta = rz / rho
            rho = rz
            p = z + beta * p
        res["iters"] = it
        res["hist"] = np.array(hist)
        res["x"] = x
        # bench: the timed region is the max over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["tmax"] = float(t.item())
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_decomposition_reproduces_global_oracle(tmp_path, oracle_mod):
    import torch.multiprocessing as mp
    from paper_2303_03398_b200 import inputs
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"rank{r}.npy", allow_pickle=True).item() for r in range(world)]
    o = oracle_mod.solve_problem(inputs.make_problem("c1"))
    for r in res:
        assert r["apply_err"] <= 1e-14
        assert r["iters"] == res[0]["iters"] and np.array_equal(r["hist"], res[0]["hist"])
        assert r["tmax"] == 2.0
    assert abs(res[0]["iters"] - o["iters"]) <= 1
    x = np.concatenate([r["x"] for r in res], axis=0)
    assert np.linalg.norm(x - o["x"]) <= 1e-10 * np.linalg.norm(o["x"])
    # same expressions in the same order + correctly rounded dot products (R24): the decomposed
    # solve reproduces the oracle's iterates exactly, bit for bit
    assert res[0]["iters"] == o["iters"]
    assert np.array_equal(x, o["x"]) and np.array_equal(res[0]["hist"], o["hist"])


def test_slab_extent_rules():
    from paper_2303_03398_b200 import inputs
    assert inputs.slab_extent(600, 3, 8) == (225, 75)
    assert inputs.slab_extent(32, 1, 2) == (16, 16)
    with pytest.raises(ValueError):
        inputs.slab_extent(600, 0, 7)
    # slabs tile the global index range
    ext = [inputs.slab_extent(128, r, 4) for r in range(4)]
    assert [e[0] for e in ext] == [0, 32, 64, 96] and all(e[1] == 32 for e in ext)


def _vv_worker(rank, world, port, out_dir):
    """Vector viscosity (NEXT-2) host logic over gloo: phi-slabs of the [np][3][nt][nr] vector, the
    3-component halo planes, and the pole-ring reduction of Listing 3 decomposed as
    the library does it -- each rank sums its own planes of the ring, the partial sums travel in one
    all-gather and are combined in rank order -- against the global oracle's axis circulations."""
    import math
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2303_03398_b200 import inputs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        res = {}
        shape = (6, 5, 8)
        full = inputs.make_vv_problem("rand", shape=shape, seed=3)
        k0, nloc = inputs.slab_extent(full.np, rank, world)
        slab = inputs.make_vv_problem("rand", k0, nloc, shape=shape, seed=3)
        sl = slice(k0, k0 + nloc)
        for name in ("nu", "s", "f", "g_in", "g_out"):
            assert np.array_equal(getattr(slab, name), getattr(full, name)[sl]), name
        v = np.random.default_rng(11).standard_normal((full.np, 3, full.nt, full.nr))
        vloc = v[sl].copy()
        # 3-component halo planes: lo <- left's last plane, hi <- right's first plane
        L, R = (rank - 1) % world, (rank + 1) % world
        lo, hi = torch.empty(vloc[0].shape, dtype=torch.float64), torch.empty(vloc[0].shape, dtype=torch.float64)
        reqs = [dist.isend(torch.from_numpy(vloc[0].copy()), L, tag=1), dist.isend(torch.from_numpy(vloc[-1].copy()), R, tag=2),
                dist.irecv(hi, R, tag=1), dist.irecv(lo, L, tag=2)]
        for q in reqs:
            q.wait()
        res["halo_ok"] = bool(np.array_equal(lo.numpy(), v[(k0 - 1) % full.np]) and
                              np.array_equal(hi.numpy(), v[(k0 + nloc) % full.np]))
        # the ring sums: sum_k l_phi v_phi(i, pole row, k) with l_phi = (rc sin tc) h_phi across the lower face
        rc, tc, pc = inputs.midpoints(full.rf), inputs.midpoints(full.tf), inputs.midpoints(full.pf)
        hlo = pc - np.roll(pc, 1)
        hlo[0] += 2 * math.pi
        part = []
        for j in (0, full.nt - 1):
            for i in range(full.nr):
                terms = [((rc[i] * math.sin(tc[j])) * hlo[k]) * v[k, 2, j, i] for k in range(k0, k0 + nloc)]
                part.append(math.fsum(terms))
        out = [None] * world
        dist.all_gather_object(out, part)
        ring = np.array([math.fsum([o[t] for o in out]) for t in range(2 * full.nr)])
        res["ring"] = ring
        _, GN, GS, _, _ = oracle.vv_curl(full.rf, full.tf, full.pf, v)
        res["GN"], res["GS"] = GN, GS
        np.save(os.path.join(out_dir, f"vv_rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_vector_viscosity_decomposition(tmp_path, oracle_mod):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_vv_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"vv_rank{r}.npy", allow_pickle=True).item() for r in range(world)]
    for r in res:
        assert r["halo_ok"]
        nr = r["GN"].size
        assert np.array_equal(r["ring"], res[0]["ring"])     # identical on every rank
        # the rank-decomposed ring sums are the global axis circulations (Dot2 there, fsum here)
        np.testing.assert_allclose(r["ring"][:nr], r["GN"], rtol=1e-14, atol=0)
        np.testing.assert_allclose(-r["ring"][nr:], r["GS"], rtol=1e-14, atol=0)
