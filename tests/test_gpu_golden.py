"""Full-size solves against golden fixtures written by the CPU oracle alone (-m gpu).

tests/golden/{c3,c5,c4,c2v,c3v,c3a}_full_solve.json come from tools/make_golden.py, which calls only oracle/ and the
seeded generators: the complete residual history of the oracle's solve of BASELINE.json configs[2] (c3,
150 x 300 x 600, 830 iterations to 1e-10), of step 0 of configs[4] (c5, 200 x 300 x 600) and of the first
40 (tol = 0) iterations of configs[3]'s one-GPU slab (c4, 400 x 400 x 800, 128 M cells), its
iteration count, the SHA-256 of the whole solution, ||x||^2 (fsum) and x at a fixed sample of 4,096 cells.  The GPU solves the same generated
problem in the bench's launch configuration (three-kernel path, CUDA graphs, chunk 16) and must
reproduce every history entry, the count and the sampled solution bit for bit (R24).
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from paper_2303_03398_b200 import inputs

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("-m gpu tests need a CUDA device")
    from paper_2303_03398_b200 import build, maspcg
    build.build()
    return maspcg


@pytest.mark.parametrize("name", ["c3", "c5", "c4"])
def test_full_size_solve_matches_oracle_golden(M, name):
    import torch
    path = os.path.join(HERE, "golden", f"{name}_full_solve.json")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_golden.py {name}")
    g = json.load(open(path))
    p = inputs.make_problem(name)
    assert [p.nr, p.nt, p.np] == g["shape"]
    S = M.solver_for_problem(p, chunk=16)
    x = torch.from_numpy(p.x0).cuda()
    st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, p.tol, g.get("maxit", p.maxit))
    torch.cuda.synchronize()
    xs = x.cpu().numpy().ravel()
    S.close()
    assert st == g["status"] and st >= 0
    assert info["iters"] == g["iters"]
    assert info["bnorm"] == g["bnorm"]
    assert np.array_equal(hist, np.array(g["hist"])), np.abs(hist - np.array(g["hist"])).max()
    idx = np.array(g["x_sample_index"], dtype=np.int64)
    assert np.array_equal(xs[idx], np.array(g["x_sample"]))
    assert math.fsum(xs * xs) == g["x_norm2_fsum"]
    # every cell of the solution, bit for bit
    assert hashlib.sha256(np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.parametrize("name", ["c2v", "c3v"])
def test_vv_full_size_solve_matches_oracle_golden(M, name):
    """The staggered vector viscosity at full size: tests/golden/{c2v,c3v}_full_solve.json
    from tools/make_golden.py (oracle/masoracle_vv.c alone); c3v is the workload of `bench.py --operator vv`
    (150 x 300 x 600 cells, 81 M unknowns, 841 iterations to 1e-10), solved here in the bench's launch
    configuration (the plane-marching operator, CUDA graphs, chunk 16).  Every history entry, the iteration count,
    a sample and the SHA-256 of the whole solution bit for bit."""
    import torch
    path = os.path.join(HERE, "golden", f"{name}_full_solve.json")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_golden.py {name}")
    g = json.load(open(path))
    p = inputs.make_vv_problem(name)
    assert [p.nr, p.nt, p.np] == g["shape"]
    dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, chunk=16)
    try:
        S.vv_set_coefficients(dev(p.nu), dev(p.s))
        S.vv_set_bc_r(p.wall_in, dev(p.g_in), p.wall_out, dev(p.g_out))
        x = dev(p.x0)
        st, info, hist = S.vv_solve(dev(p.f), x, p.tol, g.get("maxit", p.maxit))
        torch.cuda.synchronize()
        xs = x.cpu().numpy().ravel()
    finally:
        S.close()
    assert st == g["status"] and st >= 0
    assert info["iters"] == g["iters"]
    assert info["bnorm"] == g["bnorm"]
    assert np.array_equal(hist, np.array(g["hist"])), np.abs(hist - np.array(g["hist"])).max()
    idx = np.array(g["x_sample_index"], dtype=np.int64)
    assert np.array_equal(xs[idx], np.array(g["x_sample"]))
    assert math.fsum(xs * xs) == g["x_norm2_fsum"]
    assert hashlib.sha256(np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.parametrize("name", ["c3a"])
def test_aniso_full_size_solve_matches_oracle_golden(M, name):
    """Field-aligned conduction at full size: tests/golden/c3a_full_solve.json from
    tools/make_golden.py (oracle/masoracle.c alone); the workload of `bench.py --operator aniso` (150 x 300 x 600,
    the whole solve to 1e-10) in the bench's launch configuration (the plane-marching stencil, CUDA graphs, chunk 16).
    Every history entry, the iteration count, a sample and the SHA-256 of the whole solution bit for bit."""
    import torch
    path = os.path.join(HERE, "golden", f"{name}_full_solve.json")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_golden.py {name}")
    g = json.load(open(path))
    p = inputs.make_aniso_problem(name)
    assert [p.nr, p.nt, p.np] == g["shape"]
    S = M.solver_for_problem(p, chunk=16)
    try:
        x = torch.from_numpy(p.x0).cuda()
        st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, p.tol, g.get("maxit", p.maxit))
        torch.cuda.synchronize()
        xs = x.cpu().numpy().ravel()
    finally:
        S.close()
    assert st == g["status"] and st >= 0
    assert info["iters"] == g["iters"]
    assert info["bnorm"] == g["bnorm"]
    assert np.array_equal(hist, np.array(g["hist"])), np.abs(hist - np.array(g["hist"])).max()
    idx = np.array(g["x_sample_index"], dtype=np.int64)
    assert np.array_equal(xs[idx], np.array(g["x_sample"]))
    assert math.fsum(xs * xs) == g["x_norm2_fsum"]
    assert hashlib.sha256(np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest() == g["x_sha256"]


# ------------------------------------------------------------------ the 8-GPU decomposition at full size (loopback)
def _run_loopback(M, P, fn):
    """P ranks in one process on cuda:0 (the loopback communicator: the library's halo exchanges and rank-ordered
    reductions, without NCCL), one host thread each."""
    import threading

    import torch
    group = M.LoopbackGroup(P)
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, group)
            st.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=800)
    assert not any(t.is_alive() for t in th), "a rank hung"
    group.close()
    if errs:
        raise errs[0]
    return out


def _check_slabs_against_golden(g, res):
    xs = np.concatenate([r[3].reshape(r[3].shape[0], -1) for r in res], axis=0).ravel()
    for st, iters, hist, _ in res:
        assert st == g["status"] and iters == g["iters"]
        assert np.array_equal(hist, np.array(g["hist"]))
    assert hashlib.sha256(np.ascontiguousarray(xs, dtype="<f8").tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.timeout(1500)
@pytest.mark.parametrize("name", ["c3", "c3v", "c3a"])
def test_full_size_8_slabs_match_golden(M, name):
    """The bench workloads split into the 8 phi-slabs of the 8-GPU strong-scaling run (75 planes each), on 8 loopback
    ranks: every rank's history and the concatenated solution equal the single-rank oracle golden bit for bit (c3:
    830 iterations, the scalar operator; c3v: 841, the vector operator with its pole-ring sums all-gathered; c3a:
    1,028, the field-aligned operator with the edge planes below each slab from the left rank)."""
    import torch
    g = json.load(open(os.path.join(HERE, "golden", f"{name}_full_solve.json")))
    P = 8
    vv = name.endswith("v")
    np_ = inputs.VV_CONFIGS[name][2] if vv else g["shape"][2]

    def fn(r, group):
        dev = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
        if vv:
            k0, nloc = inputs.slab_extent(np_, r, P)
            p = inputs.make_vv_problem(name, k0, nloc)
            S = M.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, chunk=16, loopback=(group, r))
            S.vv_set_coefficients(dev(p.nu), dev(p.s))
            S.vv_set_bc_r(p.wall_in, dev(p.g_in), p.wall_out, dev(p.g_out))
            x = dev(p.x0)
            st, info, hist = S.vv_solve(dev(p.f), x, p.tol, p.maxit, raise_on_error=False)
        else:
            mk = inputs.make_aniso_problem if name.endswith("a") else inputs.make_problem
            p = mk(name, *inputs.slab_extent(np_, r, P))
            S = M.solver_for_problem(p, chunk=16, loopback=(group, r))
            x = dev(p.x0)
            st, info, hist = S.solve(dev(p.f), x, p.tol, p.maxit, raise_on_error=False)
        torch.cuda.current_stream().synchronize()
        res = (st, info["iters"], hist, x.cpu().numpy())
        S.close()
        return res

    _check_slabs_against_golden(g, _run_loopback(M, P, fn))
