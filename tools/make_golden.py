#!/usr/bin/env python
"""Golden fixtures of the full-size solves, written by the CPU ORACLE ONLY (oracle/ + the seeded input
generators; nothing from the CUDA path).  Used by tests/test_gpu_golden.py to compare the GPU's full-size
solves element by element: the whole residual history, the iteration count, the SHA-256 of the whole
solution x (every cell, bit for bit, without storing 216 MB), ||x||^2 (math.fsum, deterministic) and x at a
fixed sample of cells.

    python tools/make_golden.py c3      # BASELINE.json configs[2], 150 x 300 x 600, tol 1e-10
    python tools/make_golden.py c5      # configs[4] step 0 (cold solve), 200 x 300 x 600
    python tools/make_golden.py c4      # configs[3] one-GPU slab 400 x 400 x 800, the first 40 of its
                                        # tol = 0 iterations (the bench runs 500)
    python tools/make_golden.py c3v     # the staggered vector viscosity on the c3 grid (bench.py --operator
                                        # vv), 81 M unknowns, tol 1e-10 (oracle/masoracle_vv.c, single thread)
    python tools/make_golden.py c3a     # field-aligned conduction on the c3 grid (bench.py --operator aniso),
                                        # tol 1e-10 (oracle/masoracle.c -fopenmp)

Runs the oracle's -fopenmp build (identical values to the plain build,
tests/test_oracle_pins.py::test_openmp_build_gives_identical_iterates).
"""
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2303_03398_b200 import inputs  # noqa: E402

NSAMPLE = 4096


def sample_index(n, seed=12345):
    """Fixed cell sample: splitmix64 of 0..NSAMPLE-1 modulo n (sorted, unique)."""
    idx = inputs.splitmix64(np.arange(NSAMPLE, dtype=np.uint64) + np.uint64(seed)) % np.uint64(n)
    return np.unique(idx.astype(np.int64))


def main(name):
    oracle.use_openmp(True)
    vv = name in inputs.VV_CONFIGS
    an = name in inputs.ANISO_CONFIGS
    p = inputs.make_vv_problem(name) if vv else (inputs.make_aniso_problem(name) if an else inputs.make_problem(name))
    maxit = 40 if name == "c4" else p.maxit
    t0 = time.time()
    if vv:
        o = oracle.vv_solve_problem(p, maxit=maxit)
    elif an:
        o = oracle.solve_aniso_problem(p, maxit=maxit)
    else:
        o = oracle.solve_problem(p, maxit=maxit)
    dt = time.time() - t0
    x = o["x"].ravel()
    idx = sample_index(x.size)
    out = {
        "source": (f"tools/make_golden.py {name}: oracle/masoracle_vv.c vector-viscosity PCG on "
                   f"inputs.make_vv_problem('{name}'), tol {p.tol}, maxit {maxit}") if vv else
                  (f"tools/make_golden.py {name}: oracle/masoracle.c (-fopenmp build) field-aligned PCG on "
                   f"inputs.make_aniso_problem('{name}'), tol {p.tol}, maxit {maxit}") if an else
                  (f"tools/make_golden.py {name}: oracle/masoracle.c (-fopenmp build) masoracle_pcg on "
                   f"inputs.make_problem('{name}') (BASELINE.json {name}), tol {p.tol}, maxit {maxit}"),
        "maxit": maxit,
        "config": name, "shape": [p.nr, p.nt, p.np], "status": int(o["status"]), "iters": int(o["iters"]),
        "bnorm": o["bnorm"], "hist": [float(v) for v in o["hist"]],
        "x_sha256": hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest(),
        "x_norm2_fsum": math.fsum(x * x), "x_sample_index": idx.tolist(), "x_sample": [float(v) for v in x[idx]],
        "oracle_seconds": dt,
    }
    path = os.path.join(ROOT, "tests", "golden", f"{name}_full_solve.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(path, o["status"], o["iters"], f"{dt:.0f} s")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c3")
