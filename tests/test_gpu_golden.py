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
